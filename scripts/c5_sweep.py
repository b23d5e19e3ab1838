"""C5 — candidate-set sweep (BASELINE configs[4]): N' x n x p grid, ALC-kernel
roofline fraction per point for the explicit (paper) and incremental forms, and a
sampled parity check against the oracle at every point.

    python scripts/c5_sweep.py [--Nprimes 500,1000,2000,5000] [--ns 50,128] [--ps 2,8]
                               [--target-ms 400] [--sample 4] [--out profiles/c5_sweep_r01.jsonl]

Design N = 200,000 (uniform 2-d / LHS 8-d borehole); M is picked per
point so the local-design kernel runs for about --target-ms (power of two, >= 64).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_5182_b200 as lagp  # noqa: E402
from bench import alc_paper_flops_per_location, form_work, fp64_peak_tflops  # noqa: E402
from lagp_data import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--Nprimes", default="500,1000,2000,5000")
ap.add_argument("--ns", default="50,128")
ap.add_argument("--ps", default="2,8")
ap.add_argument("--forms", default="explicit,incremental")
ap.add_argument("--target-ms", type=float, default=400.0)
ap.add_argument("--sample", type=int, default=4)
ap.add_argument("--min-m", type=int, default=512)
ap.add_argument("--out", default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
nominal, meas = fp64_peak_tflops()
out = open(a.out, "w") if a.out else None
for p in [int(x) for x in a.ps.split(",")]:
    name = "C5_2d" if p == 2 else "C5_8d"
    base = make_config(name, M=32768)
    X, Z = (torch.from_numpy(base[k]).to(dev) for k in ("X", "Z"))
    XXall = torch.from_numpy(base["XX"]).to(dev)
    for n in [int(x) for x in a.ns.split(",")]:
        for Np in [int(x) for x in a.Nprimes.split(",")]:
            if Np < n:
                continue
            args = (base["d"], base["g"], 6, n, Np)
            for form in a.forms.split(","):
                # calibrate M
                M = 64
                try:
                    r = lagp.alc_batch(X, Z, XXall[:M], *args, form=form, timing=True)
                except lagp.LagpError as ex:  # outside this build's limits: record, continue
                    line = json.dumps(dict(p=p, n=n, Nprime=Np, form=form, unsupported=str(ex)))
                    print(line, flush=True)
                    if out:
                        out.write(line + "\n")
                    continue
                while r["timing"]["alc_ms"] < a.target_ms / 2 and M < 32768:
                    M = min(32768, M * 2 if r["timing"]["alc_ms"] > 0 else M * 4)
                    r = lagp.alc_batch(X, Z, XXall[:M], *args, form=form, timing=True)
                # at least two locations per SM in flight: a grid narrower than the GPU
                # understates the kernel (the slowest points calibrate to M = 64 otherwise)
                M = max(M, a.min_m)
                best = None
                for _ in range(2):
                    r = lagp.alc_batch(X, Z, XXall[:M], *args, form=form, timing=True, gaps=True)
                    if best is None or r["timing"]["alc_ms"] < best["timing"]["alc_ms"]:
                        best = r
                tm = best["timing"]
                work = form_work(form, 6, n, Np, p)
                ach = M * work / (tm["alc_ms"] / 1e3) / 1e12
                rec = dict(p=p, n=n, Nprime=Np, N=int(base["X"].shape[0]), M=M, form=form, alc_ms=tm["alc_ms"],
                           nn_ms=tm["nn_ms"], locations_per_s=M / (tm["total_ms"] / 1e3),
                           alc_evals_per_s=M * sum(Np - j for j in range(6, n)) / (tm["alc_ms"] / 1e3),
                           roofline={"bound": "alu", "achieved": ach, "peak": nominal, "frac": ach / nominal,
                                     "unit": "TFLOP/s",
                                     "work": "paper count" if form != "incremental" else "incremental count"},
                           paper_count_tflops=M * alc_paper_flops_per_location(6, n, Np) / (tm["alc_ms"] / 1e3) / 1e12)
                if a.sample > 0 and form == "incremental":
                    import oracle
                    from parity import check

                    sel = np.arange(a.sample)
                    g = {k: v.cpu().numpy()[sel] for k, v in best.items() if hasattr(v, "cpu")}
                    t0 = time.time()
                    o = oracle.alc_batch(base["X"], base["Z"], base["XX"][sel], *args)
                    try:
                        pr = check(g, o, dict(base, XX=base["XX"][sel], n0=6, n=n, Nprime=Np), form)
                        rec["parity"] = {"ok": True, "sampled": len(sel), "identical": pr["identical"],
                                         "explained": len(pr["explained"]), "max_rel_s2": pr["max_rel_s2"]}
                    except AssertionError as ex:
                        rec["parity"] = {"ok": False, "error": str(ex)[:300]}
                    rec["oracle_s"] = time.time() - t0
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
