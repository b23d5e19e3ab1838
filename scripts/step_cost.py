"""Per-step cost of the incremental local-design kernel vs design size n
(C2 inputs, N'=1000): alc_ms / (locations per SM x n) for several n.

    python scripts/step_cost.py [--M 14800] [--ns 8,16,24,32,40,50,64]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1310_5182_b200 as lagp  # noqa: E402
from lagp_data import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=14800)
ap.add_argument("--config", default="C2")
ap.add_argument("--ns", default="8,16,24,32,40,50,64")
ap.add_argument("--Nprime", type=int, default=None)
a = ap.parse_args()
cfg = make_config(a.config, M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
Np = a.Nprime or cfg["Nprime"]
sms = torch.cuda.get_device_properties(0).multi_processor_count
for n in [int(v) for v in a.ns.split(",")]:
    best = None
    for _ in range(3):
        r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], min(cfg["n0"], n), n, Np, form="incremental", timing=True)
        t = r["timing"]["alc_ms"]
        best = t if best is None else min(best, t)
    per_loc_us = best * 1e3 / (a.M / sms)
    print(json.dumps({"n": n, "alc_ms": round(best, 3), "us_per_location_per_sm": round(per_loc_us, 2),
                      "us_per_step": round(per_loc_us / n, 3), "cycles_per_step@1.965": round(per_loc_us / n * 1965)}))
