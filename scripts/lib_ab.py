"""A/B of library builds on one config: laGP_alc_batch with each .so (same inputs),
min over reps of the per-phase device times, and agreement of the index sequences
with the first build.

    python scripts/lib_ab.py --libs liblagp_b200.so liblagp_b200_x.so [--config C2] [--M 10000] [--reps 5]
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
ap.add_argument("--config", default="C2")
ap.add_argument("--M", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--form", default="auto")
ap.add_argument("--flush", action="store_true", help="write 256 MiB before every rep (L2 flushed, as in bench.py)")
a = ap.parse_args()
cfg = make_config(a.config, M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
ref = None
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev) if a.flush else None
for name in a.libs:
    lagp._LIB = lagp._lib.load(os.path.join(ROOT, "paper_1310_5182_b200", name))
    best = None
    for _ in range(a.reps):
        if flush is not None:
            flush.fill_(1.0)
        r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form=a.form, timing=True)
        torch.cuda.synchronize()
        t = r["timing"]
        if best is None or t["total_ms"] < best["total_ms"]:
            best = t
    idx = r["idx"].cpu().numpy()
    if ref is None:
        ref = idx
    print(json.dumps({"lib": name, "config": a.config, "nn_ms": round(best["nn_ms"], 4), "alc_ms": round(best["alc_ms"], 4),
                      "total_ms": round(best["total_ms"], 4), "form": best["alc_form"],
                      "same_idx_as_first": int((idx == ref).all(axis=1).sum()), "M": int(idx.shape[0])}))
