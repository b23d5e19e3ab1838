"""CPU-side checks of the boundary: the library loads, exports every symbol
include/lagp.h declares, and rejects bad arguments with LAGP_EINVAL before
touching the device (no compute calls here: there is no GPU in this container)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lagp():
    from paper_1310_5182_b200 import build

    build.build()
    import paper_1310_5182_b200 as m

    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lagp.h")).read()
    return sorted(set(re.findall(r"^(?:lagp_status\s+|const char \*\s*|int\s+)(\w+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for s in ("laGP_alc_batch", "laGP_alc_scores", "lagp_last_error", "lagp_abi_version", "laGP_nn_pool",
              "laGP_pinv_update", "laGP_predict", "laGP_alc_batch_ex", "laGP_alc_batch_host", "laGP_alc_batch_theta",
              "laGP_mle", "laGP_local_fit", "laGP_exp_nonpos", "laGP_alc_batch_sep"):
        assert s in syms


def test_library_exports_every_declared_symbol(lagp):
    lib = lagp.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert lagp.abi_version() == 4


def test_library_is_sm100a_only(lagp):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", lagp._lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def _call_batch(lagp, **kw):
    a = dict(X=1, N=100, p=2, Z=1, XX=1, M=10, d=0.1, g=1e-4, n0=6, n=50, Nprime=60, idx=1, mean=1, s2=1)
    a.update(kw)
    lib = lagp.lib()
    vp = lambda v: ctypes.c_void_p(v) if v else None  # noqa: E731
    return lib.laGP_alc_batch(vp(a["X"]), a["N"], a["p"], vp(a["Z"]), vp(a["XX"]), a["M"], a["d"], a["g"], a["n0"],
                              a["n"], a["Nprime"], vp(a["idx"]), vp(a["mean"]), vp(a["s2"]), None, None, None, None)


@pytest.mark.parametrize(
    "kw,word",
    [
        (dict(d=0.0), "theta"),
        (dict(d=float("nan")), "theta"),
        (dict(g=-1e-3), "eta"),
        (dict(g=float("inf")), "eta"),
        (dict(n0=0), "n0"),
        (dict(n=5), "n must be >= n0"),
        (dict(n=129, Nprime=200), "LAGP_NMAX"),
        (dict(Nprime=40), "Nprime must be >= n"),
        (dict(Nprime=101), "Nprime must be <= N"),
        (dict(p=0), "p must be"),
        (dict(p=17), "p must be"),
        (dict(N=0), "N must be"),
        (dict(M=-1), "M must be"),
        (dict(XX=0), "non-NULL"),
        (dict(idx=0), "non-NULL"),
    ],
)
def test_batch_rejects_bad_arguments(lagp, kw, word):
    st = _call_batch(lagp, **kw)
    assert st == lagp.LAGP_EINVAL
    assert word in lagp.last_error()


def test_empty_batch_is_ok_without_device(lagp):
    # M = 0: validated, nothing launched
    assert _call_batch(lagp, M=0, XX=0, idx=0, mean=0, s2=0) == lagp.LAGP_OK


def test_diag_entry_points_validate(lagp):
    lib = lagp.lib()
    assert lib.laGP_nn_pool(None, 10, 2, None, 1, 11, None, None, None) == lagp.LAGP_EINVAL
    assert lib.laGP_alc_scores(1, 0, 2, 5, None, None, None, None, None, 0.1, 0.0, None, None, None, None) == 2
    assert lib.laGP_pinv_update(1, 128, None, None, 1.0, None, None) == 2
    assert lib.laGP_predict(1, 200, 2, None, None, None, 0.1, 0.0, None, None, None, None) == 2
    assert "n must be" in lagp.last_error()


def test_incremental_form_flag_validated(lagp):
    lib = lagp.lib()
    vp = ctypes.c_void_p
    st = lib.laGP_alc_batch_ex(vp(1), 100, 2, vp(1), vp(1), 10, 0.1, 1e-4, 6, 50, 60, vp(1), vp(1), vp(1), None,
                               None, None, 7, None, None)
    assert st == lagp.LAGP_EINVAL and "alc_form" in lagp.last_error()


def test_exp_nonpos_validates(lagp):
    lib = lagp.lib()
    assert lib.laGP_exp_nonpos(None, None, -1, None) == 2
    assert "n must be" in lagp.last_error()
    assert lib.laGP_exp_nonpos(None, None, 4, None) == 2
    assert lib.laGP_exp_nonpos(None, None, 0, None) == 0


def test_alc_batch_sep_validates(lagp):
    import ctypes

    lib = lagp.lib()
    th = (ctypes.c_double * 2)(0.1, -1.0)
    # p = 2, theta[1] <= 0 -> EINVAL before any device work (null device pointers are never touched)
    st = lib.laGP_alc_batch_sep(1, 10, 2, 1, 1, 4, th, 1e-4, 2, 4, 6, 1, 1, 1, None, None, None, 1, None, None)
    assert st == 2 and "theta[1]" in lagp.last_error()
    st = lib.laGP_alc_batch_sep(1, 10, 2, 1, 1, 4, None, 1e-4, 2, 4, 6, 1, 1, 1, None, None, None, 1, None, None)
    assert st == 2 and "theta" in lagp.last_error()


def test_timing_struct_layout_matches_header(tmp_path):
    """The ctypes lagp_timing (paper_1310_5182_b200/_lib.py) has the C struct's size and
    field offsets (include/lagp.h, ABI 4), checked with the host C compiler."""
    import subprocess

    from paper_1310_5182_b200 import _lib

    fields = [f for f, _ in _lib.Timing._fields_]
    src = tmp_path / "t.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "lagp.h"\nint main(void){printf("%zu'
                   + "".join(" %zu" for _ in fields) + '\\n", sizeof(lagp_timing)'
                   + "".join(f", offsetof(lagp_timing, {f})" for f in fields) + ");return 0;}\n")
    exe = tmp_path / "t"
    inc = os.path.join(ROOT, "include")
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["gcc", "-I", inc, "-I", cuda_inc, str(src), "-o", str(exe)], check=True)
    out = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert out[0] == ctypes.sizeof(_lib.Timing)
    for f, off in zip(fields, out[1:]):
        assert getattr(_lib.Timing, f).offset == off, f
