"""Small calls of every kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_5182_b200 as lagp  # noqa: E402
from lagp_data import make_config  # noqa: E402

dev = torch.device("cuda", 0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
for name, over, M in (("C1", {}, 6), ("C2", dict(Nprime=300, n=30), 4), ("C1", dict(n0=1, n=12, Nprime=40), 3),
                      ("C1", dict(n=80, Nprime=600), 2), ("C2", dict(n=64, Nprime=1000), 2)):
    cfg = make_config(name, M=M, N=5000 if name == "C2" else None, **over)
    args = (cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    for form in ("explicit", "explicit_dfma", "incremental"):
        r = lagp.alc_batch(T(cfg["X"]), T(cfg["Z"]), T(cfg["XX"]), *args, form=form, gaps=True)
        torch.cuda.synchronize()
        print(name, over, form, "ok", r["idx"][0, :8].tolist())
cfg = make_config("C1", M=4)
lagp.nn_pool(T(cfg["X"]), T(cfg["XX"]), 300, with_d2=True)
rng = np.random.default_rng(0)
B, j, p, nc = 2, 9, 2, 50
Xj = rng.random((B, j, p))
K = np.exp(-((Xj[:, :, None] - Xj[:, None]) ** 2).sum(-1) / 0.1) + 1e-3 * np.eye(j)
Kinv = np.linalg.inv(K)
Kinv = 0.5 * (Kinv + Kinv.transpose(0, 2, 1))
lagp.alc_scores(T(Xj), T(Kinv), T(rng.random((B, nc, p))), T(np.arange(B * nc, dtype=np.int32).reshape(B, nc)),
                T(rng.random((B, p))), 0.1, 1e-3)
lagp.pinv_update(T(Kinv), T(rng.random((B, j))), 1.001)
lagp.predict(T(Xj), T(rng.random((B, j))), T(rng.random((B, p))), 0.1, 1e-3)
torch.cuda.synchronize()
print("sanitize run done")
# row f4 path (DMMA contraction), row f3 (separable), row f2 (MLE / two-stage), table exp
B, j, nc = 1, 100, 2000
Xj = rng.random((B, j, p))
K = np.exp(-((Xj[:, :, None] - Xj[:, None]) ** 2).sum(-1) / 0.1) + 1e-3 * np.eye(j)
lagp.alc_scores(T(Xj), T(np.linalg.inv(K)), T(rng.random((B, nc, p))), T(np.arange(nc, dtype=np.int32)[None]),
                T(rng.random((B, p))), 0.1, 1e-3)
cfg = make_config("C1", M=3)
lagp.alc_batch_sep(T(cfg["X"]), T(cfg["Z"]), T(cfg["XX"]), [0.02, 0.07], cfg["g"], 6, 40, 500)
lagp.local_fit(T(cfg["X"]), T(cfg["Z"]), T(cfg["XX"]), cfg["d"], 1e-3, 10.0, cfg["g"], 6, 30, 500, stages=2)
lagp.exp_nonpos(T(-rng.random(1000) * 50))
torch.cuda.synchronize()
print("sanitize run done (f2-f4)")
