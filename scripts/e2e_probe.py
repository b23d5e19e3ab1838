import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1310_5182_b200 as lagp
from lagp_data import make_config
cfg = make_config("C2")
dev = torch.device("cuda", 0)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
Xh, Zh, XXh = pin(cfg["X"]), pin(cfg["Z"]), pin(cfg["XX"])
M, n = XXh.shape[0], cfg["n"]
hout = dict(idx=torch.empty((M, n), dtype=torch.int32).pin_memory().numpy(), mean=torch.empty(M, dtype=torch.float64).pin_memory().numpy(),
            s2=torch.empty(M, dtype=torch.float64).pin_memory().numpy(), var=torch.empty(M, dtype=torch.float64).pin_memory().numpy(),
            flags=torch.empty(M, dtype=torch.int32).pin_memory().numpy().view(np.uint32))
a = (cfg["d"], cfg["g"], cfg["n0"], n, cfg["Nprime"])
X, Z, XX = (torch.from_numpy(v).to(dev) for v in (cfg["X"], cfg["Z"], cfg["XX"]))
for _ in range(3):
    lagp.alc_batch_host(Xh, Zh, XXh, *a, out=hout); lagp.alc_batch(X, Z, XX, *a)
torch.cuda.synchronize()
def tm(f, k=5):
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    return min(ts)
print("device call", tm(lambda: lagp.alc_batch(X, Z, XX, *a)))
print("host call  ", tm(lambda: lagp.alc_batch_host(Xh, Zh, XXh, *a, out=hout)))
dX = torch.empty_like(X)
xt = torch.from_numpy(Xh)
print("H2D X 6.4MB", tm(lambda: dX.copy_(xt, non_blocking=True)))
