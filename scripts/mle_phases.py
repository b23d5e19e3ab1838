"""Clock-probe phase split of the row f2 MLE kernel (profiling build
liblagp_b200_prof.so: python -m paper_1310_5182_b200.build --prof; -DLAGP_MLE_PROF):
thread 0 of each CTA accumulates cycles per phase of every evaluation.

    python scripts/mle_phases.py [--M 10000]
"""
import argparse
import ctypes
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
a = ap.parse_args()
cfg = make_config("C2", M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental")
torch.cuda.synchronize()
plib = lagp._lib.load(os.path.join(ROOT, "paper_1310_5182_b200", "liblagp_b200_prof.so"))
lagp._LIB = plib
plib.lagp_mle_prof(None, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
m = lagp.mle(X, Z, XX, r["idx"], cfg["d"], 1e-3, 10.0, cfg["g"])
e1.record()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (1024 * 8))()
plib.lagp_mle_prof(buf, 0)
ph = np.frombuffer(buf, dtype=np.int64).reshape(1024, 8).astype(np.float64)
ph = ph[ph[:, 7] > 0]
names = ["K+chol", "inverse", "WtW", "al+psi", "v=Pa", "trAPAP", "traces"]
ev = ph[:, 7].sum()
tot = ph[:, :7].sum()
out = {"ms": e0.elapsed_time(e1), "evals": int(ev), "cycles_per_eval": tot / ev,
       "phases": {nm: round(ph[:, k].sum() / ev, 1) for k, nm in enumerate(names)}}
print(json.dumps(out))
