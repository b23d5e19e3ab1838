"""A/B of the row f2 MLE kernel between library builds on C2 designs: min time over
reps per build, and the largest relative theta-hat difference from the first build.

    python scripts/mle_ab.py --libs liblagp_b200.so liblagp_b200_x.so [--M 10000] [--reps 5]
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
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--M", type=int, default=10000)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
cfg = make_config("C2", M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental")
ref = None
for name in a.libs:
    lagp._LIB = lagp._lib.load(os.path.join(ROOT, "paper_1310_5182_b200", name))
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m = lagp.mle(X, Z, XX, r["idx"], cfg["d"], 1e-3, 10.0, cfg["g"])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    th = m["theta"].cpu().numpy()
    if ref is None:
        ref = th
    print(json.dumps({"lib": name, "ms": round(min(ts[1:] or ts), 3), "max_rel_theta_vs_first": float(np.max(np.abs(th - ref) / np.abs(ref))),
                      "identical": int((th == ref).sum())}))
