"""GPU parity for row f2 (local MLE + multi-stage scheme, Fig 1 steps 3-5):
laGP_mle, laGP_alc_batch_theta and laGP_local_fit through the C ABI against the
oracle (oracle.mle / oracle.local_design / oracle.local_fit) on seeded inputs.

Tolerances: theta-hat 1e-8 relative (both sides iterate Newton to a step of
1e-10 in log theta, quadratic convergence puts the final iterate at rounding
level); l(theta-hat) 1e-10 relative; predictions 1e-8 relative as tests/parity.py.
"""
import numpy as np
import pytest

import oracle
from lagp_data import make_config
from parity import compare, tau_cfg, tau_form

pytestmark = pytest.mark.gpu
REL = 1e-8


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    return torch, torch.device("cuda", 0)


@pytest.fixture(scope="module")
def lagp():
    import paper_1310_5182_b200 as m

    m.lib()
    return m


def T(torch, dev, a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def designs(seed, M, N, n, p):
    rng = np.random.default_rng(seed)
    X = rng.random((N, p))
    Z = np.sin(5 * X[:, 0]) + np.cos(3 * X[:, -1]) + 0.3 * X.sum(1) + 0.02 * rng.standard_normal(N)
    idx = np.stack([rng.choice(N, n, replace=False) for _ in range(M)]).astype(np.int32)
    XX = rng.random((M, p))
    return X, Z, idx, XX


@pytest.mark.parametrize("n,p", [(6, 2), (20, 1), (50, 8), (80, 3), (100, 2), (128, 4)])
def test_mle_vs_oracle(torch_dev, lagp, n, p):
    torch, dev = torch_dev
    M, N, g = 24, 600, 1e-4
    X, Z, idx, XX = designs(n * 31 + p, M, N, n, p)
    rng = np.random.default_rng(n)
    lo, hi = 1e-3, 10.0
    th_in = np.exp(rng.uniform(np.log(0.01), np.log(3.0), M))
    r = lagp.mle(T(torch, dev, X), T(torch, dev, Z), T(torch, dev, XX), T(torch, dev, idx), 0.5, lo, hi, g,
                 theta_in=T(torch, dev, th_in))
    r = {k: v.cpu().numpy() for k, v in r.items() if hasattr(v, "cpu")}
    for i in range(M):
        Xn, Yn = X[idx[i]], Z[idx[i]]
        th, lh, its, fl = oracle.mle(Xn, Yn, th_in[i], lo, hi, g)
        assert abs(r["theta"][i] - th) <= REL * th, (i, r["theta"][i], th, its, int(r["iters"][i]))
        assert abs(r["loglik"][i] - lh) <= 1e-10 * max(1.0, abs(lh))
        assert (int(r["flags"][i]) & 0x70) == fl
        m, s2, v = oracle.predict(Xn, Yn, XX[i], th, g)
        assert abs(r["mean"][i] - m) <= REL * max(abs(m), np.std(Z))
        assert abs(r["s2"][i] - s2) <= REL * s2
        assert abs(r["var"][i] - v) <= REL * v


def test_mle_exhausted_prefix_and_failure(torch_dev, lagp):
    torch, dev = torch_dev
    X, Z, idx, XX = designs(7, 4, 300, 30, 2)
    idx[1, 17:] = -1  # exhausted design: the valid prefix is used
    X[idx[2, 1]] = X[idx[2, 0]]  # duplicate rows with eta = 0: K singular -> MLE_FAIL
    g = 0.0
    r = lagp.mle(T(torch, dev, X), T(torch, dev, Z), T(torch, dev, XX), T(torch, dev, idx), 0.3, 1e-3, 10.0, g)
    assert r["status"] == lagp.LAGP_PARTIAL  # the failed location is flagged NONFINITE
    r = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in r.items()}
    th, lh, its, fl = oracle.mle(X[idx[1, :17]], Z[idx[1, :17]], 0.3, 1e-3, 10.0, g)
    assert abs(r["theta"][1] - th) <= REL * th
    assert r["flags"][2] & lagp.FLAG_MLE_FAIL
    assert r["theta"][2] == 0.3
    assert oracle.mle(X[idx[2]], Z[idx[2]], 0.3, 1e-3, 10.0, g)[3] & oracle.MLE_FLAG_FAIL
    # K is singular at every theta: no prediction (NaN, as oracle_predict / oracle_local_fit report it)
    assert r["flags"][2] & lagp.FLAG_NONFINITE
    assert np.isnan(r["mean"][2]) and np.isnan(r["s2"][2]) and np.isnan(r["var"][2])
    with pytest.raises(np.linalg.LinAlgError):
        oracle.predict(X[idx[2]], Z[idx[2]], XX[2], 0.3, g)
    assert np.isfinite(r["mean"][[0, 1, 3]]).all() and not (r["flags"][[0, 1, 3]] & lagp.FLAG_NONFINITE).any()


@pytest.mark.parametrize("form", ["explicit", "incremental"])
def test_alc_batch_per_location_theta(torch_dev, lagp, form):
    torch, dev = torch_dev
    cfg = make_config("C1", M=40)
    rng = np.random.default_rng(3)
    th = cfg["d"] * np.exp(rng.uniform(-1.0, 1.0, 40))
    r = lagp.alc_batch(T(torch, dev, cfg["X"]), T(torch, dev, cfg["Z"]), T(torch, dev, cfg["XX"]), cfg["d"], cfg["g"],
                       cfg["n0"], cfg["n"], cfg["Nprime"], form=form, gaps=True, theta=T(torch, dev, th))
    g = {k: v.cpu().numpy() for k, v in r.items() if hasattr(v, "cpu")}
    rows = [oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"][i:i + 1], th[i], cfg["g"], cfg["n0"], cfg["n"],
                             cfg["Nprime"]) for i in range(40)]
    o = {k: np.concatenate([rr[k] for rr in rows]) for k in ("idx", "mean", "s2", "var", "flags", "gaps")}
    # R18 with each location's own theta: the oracle's score noise on 16 of the locations
    tau = max(tau_cfg(dict(cfg, XX=cfg["XX"][i:i + 1], d=float(th[i])), {"idx": o["idx"][i:i + 1]})
              for i in range(0, 40, 3))
    compare(g, o, cfg["n0"], float(np.std(cfg["Z"])), tau, form=form, label="per-location-theta")


@pytest.mark.parametrize(
    "name,M,N,over",
    [("C1", 48, None, {}), ("C2", 16, 20000, {}), ("C3", 24, None, {}), ("C1", 4, 60, dict(n0=5, n=60, Nprime=60)),
     ("C5_2d", 3, None, dict(n=20, Nprime=9000))],  # N' > 8192: the HBM-streaming design kernel, per-location theta
)
@pytest.mark.parametrize("form", ["explicit", "incremental"])
def test_local_fit_vs_oracle(torch_dev, lagp, name, M, N, over, form):
    torch, dev = torch_dev
    cfg = make_config(name, M=M, N=N, **over)
    d0 = cfg["d"]
    lo, hi = 1e-3 * d0, 10.0 * d0
    args = (cfg["X"], cfg["Z"], cfg["XX"])
    for stages in (1, 2):
        r = lagp.local_fit(*(T(torch, dev, a) for a in args), d0, lo, hi, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"],
                           stages=stages, form=form)
        g = {k: v.cpu().numpy() for k, v in r.items() if hasattr(v, "cpu")}
        o = oracle.local_fit(*args, d0, lo, hi, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], stages=stages)
        same = (g["idx"] == o["idx"]).all(axis=1)
        for i in np.where(~same)[0]:  # a divergence must sit on an oracle near-tie (R18)
            th = d0 if stages == 1 else o["theta"][stages - 2, i]
            des = oracle.local_design(cfg["X"], cfg["Z"], cfg["XX"][i], th, cfg["g"], cfg["n0"], cfg["n"],
                                      cfg["Nprime"])
            t = int(np.argmax(g["idx"][i] != o["idx"][i]))
            tau = tau_cfg(dict(cfg, XX=cfg["XX"][i:i + 1], d=float(th)), {"idx": des["idx"][None, :]})
            assert t >= cfg["n0"] and des["gaps"][t - cfg["n0"]] < max(1e-12, tau_form(tau, form)), (i, t)
        assert (~same).sum() <= max(1, M // 50)
        dth = np.abs(g["theta"] - o["theta"])[:, same]
        assert (dth <= REL * o["theta"][:, same]).all(), np.max(dth / o["theta"][:, same])
        m_o, s_o = o["mean"][same], o["s2"][same]
        assert (np.abs(g["mean"][same] - m_o) <= REL * np.maximum(np.abs(m_o), np.std(cfg["Z"]))).all()
        assert (np.abs(g["s2"][same] - s_o) <= REL * s_o).all()
        assert np.array_equal(g["flags"][same].astype(np.uint32) & 0x76, o["flags"][same] & 0x76)


def test_local_fit_stage1_equals_batch_then_mle(torch_dev, lagp):
    # composition through the ABI: local_fit(stages=1) == alc_batch + mle
    torch, dev = torch_dev
    cfg = make_config("C1", M=32)
    X, Z, XX = (T(torch, dev, cfg[k]) for k in ("X", "Z", "XX"))
    d0 = cfg["d"]
    a = lagp.alc_batch(X, Z, XX, d0, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], form="incremental")
    m = lagp.mle(X, Z, XX, a["idx"], d0, d0 / 1000, d0 * 10, cfg["g"])
    f = lagp.local_fit(X, Z, XX, d0, d0 / 1000, d0 * 10, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], stages=1,
                       form="incremental")
    assert torch.equal(f["idx"], a["idx"])
    assert torch.equal(f["theta"][0], m["theta"])
    assert torch.equal(f["mean"], m["mean"]) and torch.equal(f["s2"], m["s2"])
