"""Clock-probe timeline of the incremental v2 kernel: lane 0 of every warp of CTA 0
on its first location, per greedy step, from the profiling build
liblagp_b200_prof.so (python -m paper_1310_5182_b200.build --prof; -DLAGP_V2_PROF).

    python scripts/v2_probe.py [--config C2] [--M 10000] [--steps 10,20,30,40]
Events: 0 step start, 1 keys, 2 warp argmax, 3 posted (at the barrier), 4 after the
barrier (winner known), 5 winner TMEM published (publishing warps), 6 1/rho formed,
7 K(x_c,x*) done, 9/10 before/after the TMEM-publication wait, 8 dot done,
11 downdate done. Times are cycles after the step's earliest event 0.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_5182_b200 as lagp  # noqa: E402
from lagp_data import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--M", type=int, default=10000)
ap.add_argument("--steps", default="8,20,30,40,48")
a = ap.parse_args()
lagp._LIB = lagp._lib.load(os.path.join(ROOT, "paper_1310_5182_b200", "liblagp_b200_prof.so"))
cfg = make_config(a.config, M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental", timing=True)
torch.cuda.synchronize()
print(r["timing"])
NEV = 12
buf = (ctypes.c_longlong * (128 * 32 * NEV))()
lagp._LIB.lagp_v2_prof(buf)
ev = np.frombuffer(buf, dtype=np.int64).reshape(128, 32, NEV).astype(np.float64)
n, n0 = cfg["n"], cfg["n0"]
nw = int((ev[n0, :, 0] > 0).sum())
ev = ev[:, :nw]
ev[ev == 0] = np.nan
names = ["start", "keys", "wargmax", "posted", "winner", "publ", "rrho", "kx", "dot", "wait0", "wait1", "downd"]
t0 = np.nanmin(ev[:, :, 0], axis=1)
rel = ev - t0[:, None, None]
step = np.append(np.diff(t0), np.nan)
print(f"warps {nw}; cycles per step (j = n0..n-2): mean {np.nanmean(step[n0:n-1]):.0f}")
print("mean over steps n0..n-2 of (max over warps | mean over warps) per event:")
for k in range(NEV):
    v = rel[n0:n - 1, :, k]
    if np.all(np.isnan(v)):
        continue
    print(f"  {k:2d} {names[k]:8s} max {np.nanmean(np.nanmax(v, axis=1)):7.0f}  mean {np.nanmean(v):7.0f}")
for j in [int(x) for x in a.steps.split(",")]:
    print(f"step {j}: {step[j]:.0f} cycles")
    print("  warp " + " ".join(f"{nm:>7s}" for nm in names))
    for w in range(nw):
        print(f"  {w:4d} " + " ".join("      -" if np.isnan(x) else f"{x:7.0f}" for x in rel[j, w]))
