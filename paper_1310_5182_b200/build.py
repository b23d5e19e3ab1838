"""Build the sm_100a C-ABI library in-tree: paper_1310_5182_b200/liblagp_b200.so.

Plain nvcc (no torch extension machinery): the library has a C ABI with plain
pointers, so the Python side binds it with ctypes. Compiled for sm_100a only.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblagp_b200.so")
ROOT = os.path.dirname(PKG)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


OBJ = os.path.join(ROOT, "build", "obj")


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + [os.path.join(ROOT, "include", "lagp.h")])


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + _headers())


def _nvcc() -> str:
    nvcc = os.environ.get("NVCC", "nvcc")
    if os.path.exists("/usr/local/cuda/bin/nvcc") and nvcc == "nvcc":
        nvcc = "/usr/local/cuda/bin/nvcc"
    return nvcc


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB, obj_dir: str = OBJ) -> str:
    """One object per .cu (compiled in parallel, reused while it is newer than its
    source and every header), then one shared-library link. `defines` / `lib` /
    `obj_dir`: experiment builds (e.g. -DLAGP_V2_PROF into liblagp_b200_prof.so)."""
    if lib == LIB and not (force or _stale()):
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    nvcc = _nvcc()
    os.makedirs(obj_dir, exist_ok=True)
    th = max([os.path.getmtime(f) for f in _headers()] + [0.0])

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(th, os.path.getmtime(src)):
            return obj, "", 0
        r = subprocess.run([nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", "-o", obj + ".tmp", src], capture_output=True, text=True)
        if r.returncode == 0:
            with open(obj + ".ptxas", "w") as f:
                f.write(r.stderr)
            os.replace(obj + ".tmp", obj)
        return obj, r.stdout + r.stderr, r.returncode

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(compile_one, sources()))
    bad = [out for _, out, rc in res if rc != 0]
    if bad:
        sys.stderr.write("\n".join(bad))
        raise RuntimeError("nvcc failed building liblagp_b200.so")
    objs = [o for o, _, _ in res]
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                        "-o", lib + ".tmp", *objs], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking liblagp_b200.so")
    os.replace(lib + ".tmp", lib)
    if lib != LIB:
        return lib
    report = "".join(out for _, out, _ in res)
    if verbose:
        sys.stderr.write(report)
    with open(os.path.join(PKG, "ptxas_report.txt"), "w") as f:  # ptxas -v of every object
        for o in objs:
            if os.path.exists(o + ".ptxas"):
                f.write(open(o + ".ptxas").read())
    return LIB


if __name__ == "__main__":
    if "--prof" in sys.argv:  # clock-probe build of the incremental kernel (scripts/v2_probe.py)
        print(build(force=True, defines=["LAGP_V2_PROF", "LAGP_MLE_PROF", "LAGP_NN_PROF"], lib=os.path.join(PKG, "liblagp_b200_prof.so"),
                    obj_dir=os.path.join(ROOT, "build", "obj_prof")))
    else:
        build(force="--force" in sys.argv, verbose=True)
        print(LIB)
