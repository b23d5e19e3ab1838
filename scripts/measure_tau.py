"""Reading R18: measure tau_cfg, the oracle's own score noise, for the full-size
named configurations and store it in tests/golden/tau_cfg.json.

tau_cfg = max over 16 seeded locations of the configuration and over every greedy
step of |Delta_explicit - Delta_ref| / max Delta_ref, where Delta_explicit are the
oracle's explicit-K^{-1} scores along its own trajectory and Delta_ref a fresh
long-double solve (oracle.score_noise). Calls only oracle/ and lagp_data/.

    python scripts/measure_tau.py [C1 C2 ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from lagp_data import make_config  # noqa: E402

NAMES = ["C1", "C2", "C3", "C3j", "C4", "C5_2d", "C5_8d"]
OUT = os.path.join(ROOT, "tests", "golden", "tau_cfg.json")


def measure(name, k=16, seed=18):
    cfg = make_config(name)
    M = cfg["XX"].shape[0]
    sel = np.sort(np.random.default_rng(seed).choice(M, min(k, M), replace=False))
    XX = cfg["XX"][sel]
    o = oracle.alc_batch(cfg["X"], cfg["Z"], XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    per, gmin = [], []
    for i in range(len(sel)):
        nz, rg = oracle.score_noise(cfg["X"], XX[i], o["idx"][i], cfg["d"], cfg["g"], cfg["n0"], cfg["n"],
                                    cfg["Nprime"])
        per.append(float(np.nanmax(nz)))
        gmin.append(float(np.nanmin(rg)))
    return dict(tau_cfg=max(per), per_location=per, locations=sel.tolist(), min_ref_gap=gmin, d=cfg["d"],
                g=cfg["g"], n0=cfg["n0"], n=cfg["n"], Nprime=cfg["Nprime"], N=int(cfg["X"].shape[0]),
                M=int(M), p=int(cfg["X"].shape[1]))


def main():
    names = sys.argv[1:] or NAMES
    data = {"how": __doc__.strip().splitlines()[0], "script": "scripts/measure_tau.py", "configs": {}}
    if os.path.exists(OUT):
        data = json.load(open(OUT))
    for nm in names:
        t0 = time.time()
        data["configs"][nm] = measure(nm)
        print(nm, data["configs"][nm]["tau_cfg"], f"{time.time() - t0:.1f}s", flush=True)
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)


if __name__ == "__main__":
    main()
