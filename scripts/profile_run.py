"""One laGP_alc_batch call on the C2 workload (optionally fewer locations), for ncu.

    python scripts/profile_run.py [--M 2000] [--form explicit] [--config C2] [--reps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1310_5182_b200 as lagp  # noqa: E402
from lagp_data import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=None)
ap.add_argument("--config", default="C2")
ap.add_argument("--form", default="explicit")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--Nprime", type=int, default=None)
ap.add_argument("--lib", default=None, help="experiment build of the library (e.g. an ablation .so)")
a = ap.parse_args()
if a.lib:
    lagp._LIB = lagp._lib.load(a.lib)
over = {k: v for k, v in (("n", a.n), ("Nprime", a.Nprime)) if v is not None}
cfg = make_config(a.config, M=a.M, **over)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
for _ in range(a.reps):
    r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form=a.form, timing=True)
torch.cuda.synchronize()
print(r["timing"], int(r["status"]))
