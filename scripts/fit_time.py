import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_1310_5182_b200 as lagp
from lagp_data import make_config
cfg = make_config("C2", M=10000)
dev = torch.device("cuda", 0)
X, Z, XX = (torch.from_numpy(cfg[k]).to(dev) for k in ("X", "Z", "XX"))
d0 = cfg["d"]
for it in range(3):
    r = lagp.local_fit(X, Z, XX, d0, d0 / 1000, d0 * 10, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], stages=2, form="incremental", timing=True)
    torch.cuda.synchronize()
    print(r["timing"])
th = r["theta"].cpu().numpy()
print("theta pct", np.percentile(th[0], [0, 10, 50, 90, 100]), np.percentile(th[1], [0, 50, 100]))
fl = r["flags"].cpu().numpy()
print("bound frac", np.mean((fl & 16) > 0), "maxit", np.mean((fl & 32) > 0), "fail", np.mean((fl & 64) > 0))
a = lagp.alc_batch(X, Z, XX, d0, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental")
torch.cuda.synchronize()
t = time.time()
m = lagp.mle(X, Z, XX, a["idx"], d0, d0 / 1000, d0 * 10, cfg["g"])
torch.cuda.synchronize()
print("mle alone s", time.time() - t, "iters mean", m["iters"].float().mean().item())
