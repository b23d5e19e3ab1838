"""Clock-probe timeline of the v2 incremental kernel (thread 0, first location of
CTA 0), from the profiling build liblagp_b200_prof.so (-DLAGP_V2_PROF).

    python scripts/v2_probe.py [--config C2] [--M 2000]
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
ap.add_argument("--M", type=int, default=2000)
a = ap.parse_args()
lagp._LIB = lagp._lib.load(os.path.join(ROOT, "paper_1310_5182_b200", "liblagp_b200_prof.so"))
cfg = make_config(a.config, M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental", timing=True)
torch.cuda.synchronize()
print(r["timing"])
buf = (ctypes.c_longlong * (160 * 8 + 160 * 32))()
lagp._LIB.lagp_v2_prof(buf)
allv = np.frombuffer(buf, dtype=np.int64)
t = allv[:160 * 8].reshape(160, 8)
arr = allv[160 * 8:].reshape(160, 32)
n = cfg["n"]
names = ["start", "keys", "warpredux", "xwarp", "record", "kx", "dot", "downdate"]
print("step " + " ".join(f"{x:>9s}" for x in names[1:]) + "      total")
for j in range(n):
    row = t[j]
    nxt = t[j + 1][0] if j + 1 < n else row[7]
    d = []
    prev = row[0]
    for k in range(1, 8):
        if row[k] == 0:
            d.append("        -")
            continue
        d.append(f"{row[k] - prev:9d}")
        prev = row[k]
    print(f"{j:4d} " + " ".join(d) + f" {nxt - row[0]:10d}")
print("barrier arrivals per step (cycles after the first warp; the last warp's id)")
for j in range(cfg["n0"], n, 4):
    a = arr[j][:16]
    if a.min() <= 0:
        continue
    rel = a - a.min()
    print(f"{j:4d} spread {rel.max():6d}  last warp {int(rel.argmax()):2d}  " + " ".join(f"{v:5d}" for v in rel))
