"""Clock-probe phase split of the NN pool kernel (profiling build liblagp_b200_prof.so:
python -m paper_1310_5182_b200.build --prof; -DLAGP_NN_PROF): thread 0 of each CTA
accumulates cycles per phase of every query group.

    python scripts/nn_phases.py [--config C2] [--M 10000]
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
ap.add_argument("--config", default="C2")
ap.add_argument("--M", type=int, default=10000)
ap.add_argument("--lib", default="liblagp_b200_prof.so")
a = ap.parse_args()
cfg = make_config(a.config, M=a.M)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
plib = lagp._lib.load(os.path.join(ROOT, "paper_1310_5182_b200", a.lib))
lagp._LIB = plib
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], timing=True)
torch.cuda.synchronize()
plib.lagp_nn_prof(None, 1)
r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], timing=True)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (1024 * 12))()
plib.lagp_nn_prof(buf, 0)
ph = np.frombuffer(buf, dtype=np.int64).reshape(1024, 12).astype(np.float64)
ph = ph[ph[:, 7] > 0]
names = ["setup+T1", "T2", "list", "filter", "exact", "rescale", "select+out"]
ng = ph[:, 7].sum()
out = {"lib": a.lib, "cr": os.environ.get("LAGP_NN_CR"), "config": a.config, "M": a.M, "nn_ms": r["timing"].get("nn_ms"), "groups": int(ng),
       "rounds_per_group": ph[:, 8].sum() / ng, "ctas": int(len(ph)),
       "cycles_per_group": {nm: round(ph[:, k].sum() / ng) for k, nm in enumerate(names)},
       "emit_in_exact_per_group": round(ph[:, 9].sum() / ng), "emits_per_group": ph[:, 10].sum() / ng}
print(json.dumps(out))
