"""Row f2 kernel alone on C2 designs: laGP_mle over the local designs of
laGP_alc_batch (incremental), timed with CUDA events; iteration statistics.

    python scripts/mle_profile.py [--M 10000] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_5182_b200 as lagp  # noqa: E402
from lagp_data import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=10000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = make_config("C2", M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental")
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    m = lagp.mle(X, Z, XX, r["idx"], cfg["d"], 1e-3, 10.0, cfg["g"])
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
it = m["iters"].cpu().numpy() if "iters" in m else None
out = {"M": a.M, "ms": min(ts), "us_per_fit_per_sm": min(ts) * 1e3 / (a.M / 148)}
if it is not None:
    out.update({"iters_mean": float(it.mean()), "iters_max": int(it.max()),
                "iters_hist": np.bincount(it).tolist()})
print(json.dumps(out))
