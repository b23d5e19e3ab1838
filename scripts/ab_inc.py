"""A/B of the incremental local-design kernels on one config: v2 (default) vs
v1 (LAGP_INC_V1=1), same inputs; prints timings and output agreement.

    python scripts/ab_inc.py [--config C2] [--M 10000] [--reps 3]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if os.environ.get("AB_CHILD"):
    import numpy as np
    import torch

    import paper_1310_5182_b200 as lagp
    from lagp_data import make_config

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out")
    a = ap.parse_args()
    cfg = make_config(a.config, M=a.M)
    dev = torch.device("cuda", 0)
    X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
    ts = []
    for _ in range(a.reps):
        r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental",
                           timing=True, gaps=True)
        ts.append(r["timing"])
    np.savez(a.out, idx=r["idx"].cpu().numpy(), mean=r["mean"].cpu().numpy(), s2=r["s2"].cpu().numpy(),
             flags=r["flags"].cpu().numpy(), gaps=r["gaps"].cpu().numpy())
    print(json.dumps({"timing": ts[-1], "status": int(r["status"])}))
    sys.exit(0)

args = [a for a in sys.argv[1:] if not a.startswith("--variants=")]
spec = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--variants=")), "v2:;v1:LAGP_INC_V1=1")
variants = []
for item in spec.split(";"):
    name, _, envs = item.partition(":")
    variants.append((name, dict(kv.split("=") for kv in envs.split(",") if kv)))
res = {}
for name, env in variants:
    out = f"/tmp/ab_{name}.npz"
    e = dict(os.environ, AB_CHILD="1", **env)
    p = subprocess.run([sys.executable, __file__, *args, "--out", out], env=e, capture_output=True, text=True)
    print(name, p.stdout.strip(), p.stderr.strip()[-2000:])
    res[name] = out
import numpy as np  # noqa: E402

names = list(res)
a, b = np.load(res[names[0]]), np.load(res[names[-1]])
print("compare", names[0], "vs", names[-1])
same = (a["idx"] == b["idx"]).all(axis=1)
print("identical index sequences:", int(same.sum()), "/", len(same))
rel = np.abs(a["mean"] - b["mean"])[same] / np.maximum(np.abs(b["mean"][same]), np.std(b["mean"]))
print("max rel mean diff (same seq):", float(rel.max()) if rel.size else None)
rs = np.abs(a["s2"] - b["s2"])[same] / b["s2"][same]
print("max rel s2 diff (same seq):", float(rs.max()) if rs.size else None)
print("flags equal:", bool((a["flags"] == b["flags"]).all()))
if not same.all():
    i = int(np.where(~same)[0][0])
    k = int(np.where(a["idx"][i] != b["idx"][i])[0][0])
    print("first divergence loc", i, "step", k, "gap v1", b["gaps"][i][k - 6] if k >= 6 else None)
