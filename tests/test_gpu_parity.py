"""GPU parity tests: the sm_100a path, called through the C ABI, against the
CPU oracle on the same seeded inputs (rules in tests/parity.py)."""
import numpy as np
import pytest

import oracle
from lagp_data import make_config
from parity import check, golden_tau

pytestmark = pytest.mark.gpu


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


# ------------------------------------------------------------------ a1: NN
@pytest.mark.parametrize(
    "name,M,N,Nprime",
    [("C1", 100, None, 500), ("C2", 48, None, 1000), ("C3", 64, None, 1000), ("C3j", 32, None, 1000),
     ("C1", 9, 600, 600), ("C1", 5, 300, 1), ("C2", 7, 5000, 4096)],
)
def test_nn_pool_bit_exact(torch_dev, lagp, name, M, N, Nprime):
    torch, dev = torch_dev
    cfg = make_config(name, M=M, N=N)
    pool, d2 = lagp.nn_pool(T(torch, dev, cfg["X"]), T(torch, dev, cfg["XX"]), Nprime, with_d2=True)
    pool = pool.cpu().numpy()
    d2 = d2.cpu().numpy()
    for i in range(M):
        ref, rd2 = oracle.nn(cfg["X"], cfg["XX"][i], Nprime)
        assert np.array_equal(pool[i], ref), (i, np.where(pool[i] != ref)[0][:5])
        assert np.array_equal(d2[i], rd2)


def _cell_cases():
    """Inputs that stress the filter's spatial cells (nn.cu nn_cell_of): a constant
    cell axis (zero-width box), half the rows in one tight cluster (one crowded cell),
    queries far outside the bounding box of X, heavy exact ties on the cell axes,
    and the 1-d grid."""
    rng = np.random.default_rng(77)
    out = []
    X = rng.random((30000, 3)); X[:, 0] = 0.25                       # constant axis 0
    out.append(("const_axis0", X, rng.random((40, 3))))
    X = rng.random((30000, 2)); X[:15000] = 0.5 + 1e-7 * rng.standard_normal((15000, 2))  # one crowded cell
    out.append(("cluster", X, np.vstack([rng.random((30, 2)), np.full((2, 2), 0.5)])))
    X = rng.random((20000, 4))
    out.append(("far_queries", X, np.vstack([rng.random((8, 4)) * 10 - 5, [[3.0, -2.0, 0.5, 0.5]]])))
    X = np.floor(rng.random((25000, 2)) * 40) / 40                     # grid: exact ties everywhere
    out.append(("ties_grid", X, np.floor(rng.random((24, 2)) * 40) / 40))
    X = rng.random((50000, 1))
    out.append(("p1", X, rng.random((20, 1))))
    X = rng.standard_normal((40000, 5)) * [1e3, 1e-3, 1, 1, 1]         # very unequal axis scales
    out.append(("scales", X, rng.standard_normal((20, 5)) * [1e3, 1e-3, 1, 1, 1]))
    return out


@pytest.mark.parametrize("case", range(6))
@pytest.mark.parametrize("Nprime", [1, 700])
def test_nn_pool_cells_bit_exact(torch_dev, lagp, case, Nprime):
    torch, dev = torch_dev
    name, X, XX = _cell_cases()[case]
    pool, d2 = lagp.nn_pool(T(torch, dev, X), T(torch, dev, XX), Nprime, with_d2=True)
    pool, d2 = pool.cpu().numpy(), d2.cpu().numpy()
    for i in range(XX.shape[0]):
        ref, rd2 = oracle.nn(X, XX[i], Nprime)
        assert np.array_equal(pool[i], ref), (name, i, np.where(pool[i] != ref)[0][:5])
        assert np.array_equal(d2[i], rd2), name


def _multi_cell_cases():
    """Inputs for the multi-axis cell grid (p >= 4, nn.cu nn_cells / build_list): zero-width
    cut axes, a tight 8-d cluster holding 40 % of the rows (a crowded cell and near-equal
    keys in one value bin of the selection), a coarse 4-d grid (exact key ties everywhere),
    a tiny box far from the origin (cell margins with |lo| >> slab width), queries far
    outside the box, and very unequal axis scales."""
    rng = np.random.default_rng(91)
    out = []
    X = rng.random((30000, 8)); X[:, 1] = 0.5; X[:, 4] = -2.0          # constant cut axes
    out.append(("const_axes_8d", X, rng.random((24, 8))))
    X = rng.random((30000, 8)); X[:12000] = 0.3 + 1e-7 * rng.standard_normal((12000, 8))
    out.append(("cluster_8d", X, np.vstack([rng.random((16, 8)), np.full((4, 8), 0.3)])))
    X = np.floor(rng.random((40000, 4)) * 5) / 5                      # ties everywhere
    out.append(("grid_4d", X, np.floor(rng.random((20, 4)) * 5) / 5))
    X = 1e6 + rng.random((30000, 6)) * 1e-3
    out.append(("offset_6d", X, 1e6 + rng.random((20, 6)) * 1e-3))
    X = rng.random((30000, 8))
    out.append(("far_8d", X, np.vstack([rng.random((8, 8)) * 20 - 10, rng.random((8, 8))])))
    X = rng.standard_normal((40000, 5)) * [1e3, 1e-3, 1, 1, 1]
    out.append(("scales_5d", X, rng.standard_normal((16, 5)) * [1e3, 1e-3, 1, 1, 1]))
    return out


@pytest.mark.parametrize("case", range(6))
@pytest.mark.parametrize("Nprime", [1, 50, 1000])
def test_nn_pool_multi_cells_bit_exact(torch_dev, lagp, case, Nprime):
    """The multi-axis cell grid (per-query cell lists) on its edge cases: the sorted pool
    and its d^2 bit-exact against the oracle."""
    torch, dev = torch_dev
    name, X, XX = _multi_cell_cases()[case]
    pool, d2 = lagp.nn_pool(T(torch, dev, X), T(torch, dev, XX), Nprime, with_d2=True)
    pool, d2 = pool.cpu().numpy(), d2.cpu().numpy()
    for i in range(XX.shape[0]):
        ref, rd2 = oracle.nn(X, XX[i], Nprime)
        assert np.array_equal(pool[i], ref), (name, i, np.where(pool[i] != ref)[0][:5])
        assert np.array_equal(d2[i], rd2), name


@pytest.mark.parametrize("p,N,Nprime", [(7, 30000, 500), (10, 40000, 1000), (16, 20000, 300), (12, 120000, 2000)])
def test_nn_pool_multi_cells_generic_p(torch_dev, lagp, p, N, Nprime):
    """The multi-axis grid on the generic-p kernel (p not in {1,2,3,4,8}; p > 8 cuts only
    the first 8 coordinates): gaussian rows with unequal axis scales, queries inside and
    outside the cloud; sorted pool and d^2 bit-exact against the oracle."""
    torch, dev = torch_dev
    rng = np.random.default_rng(100 + p)
    sc = np.exp(rng.uniform(-2.0, 2.0, p))
    X = rng.standard_normal((N, p)) * sc
    XX = np.vstack([rng.standard_normal((12, p)) * sc, rng.standard_normal((4, p)) * sc * 4.0])
    pool, d2 = lagp.nn_pool(T(torch, dev, X), T(torch, dev, XX), Nprime, with_d2=True)
    pool, d2 = pool.cpu().numpy(), d2.cpu().numpy()
    for i in range(XX.shape[0]):
        ref, rd2 = oracle.nn(X, XX[i], Nprime)
        assert np.array_equal(pool[i], ref), (p, i, np.where(pool[i] != ref)[0][:5])
        assert np.array_equal(d2[i], rd2), p


@pytest.mark.parametrize("case", range(6))
@pytest.mark.parametrize("Nprime,n0", [(50, 6), (1000, 6), (1000, 0), (3000, 128)])
def test_nn_pool_selected_bit_exact(torch_dev, lagp, case, Nprime, n0):
    """The pool as the design kernels receive it (LAGP_NN_POOL_SELECT=n0: the value-bin
    selection of select_pool, with its radix fallback on crowded bins): the n0 nearest
    first in the oracle's (d^2, index) order, the whole pool the oracle's set."""
    import os

    torch, dev = torch_dev
    name, X, XX = _multi_cell_cases()[case]
    os.environ["LAGP_NN_POOL_SELECT"] = str(n0)
    try:
        pool = lagp.nn_pool(T(torch, dev, X), T(torch, dev, XX), Nprime).cpu().numpy()
    finally:
        os.environ.pop("LAGP_NN_POOL_SELECT", None)
    for i in range(XX.shape[0]):
        ref, _ = oracle.nn(X, XX[i], Nprime)
        assert np.array_equal(pool[i, :n0], ref[:n0]), (name, i)
        assert np.array_equal(np.sort(pool[i]), np.sort(ref)), (name, i)


@pytest.mark.parametrize("env", [{}, {"LAGP_NN_CELLS": "2"}, {"LAGP_NN_CELLS": "0"}])
def test_nn_work_counters(torch_dev, lagp, env):
    """lagp_timing's NN work counters (ABI 4) obey their definitions: prefilter pairs
    fewer than the M N exhaustive pairs with the multi-axis cells and at least M N with
    one cell; sample pairs at most M N; exact keys (the filter survivors) at least N'
    per location."""
    import os

    torch, dev = torch_dev
    cfg = make_config("C2", M=200, N=20000)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        X, Z, XX = (T(torch, dev, cfg[k]) for k in ("X", "Z", "XX"))
        r = lagp.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], timing=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    t = r["timing"]
    M, N = cfg["XX"].shape[0], cfg["X"].shape[0]
    assert 0 < t["nn_filter_pairs"] <= 6 * M * N  # at most NN_MAX_ROUNDS filter rounds
    if not env:
        assert t["nn_filter_pairs"] < M * N  # the multi-axis cell lists prune
    if env.get("LAGP_NN_CELLS") == "0":
        assert t["nn_filter_pairs"] >= M * N  # one cell: every row for every active query, >= 1 round
    assert 0 <= t["nn_sample_pairs"] <= M * N
    assert t["nn_exact_keys"] >= M * cfg["Nprime"]


def test_nn_pool_massive_ties_fallback(torch_dev, lagp):
    """Every row at the same distance -> threshold filter cannot split; the exact
    radix-select fallback must return the lowest indices."""
    torch, dev = torch_dev
    X = np.zeros((20000, 2))
    XX = np.array([[0.5, 0.5], [0.0, 0.0]])
    pool = lagp.nn_pool(T(torch, dev, X), T(torch, dev, XX), 300).cpu().numpy()
    assert (pool == np.arange(300)[None, :]).all()


# ------------------------------------------------------------ a3: ALC score
@pytest.mark.parametrize("j,p,nc,B", [(1, 2, 40, 4), (6, 2, 500, 4), (23, 8, 300, 4), (49, 3, 1000, 4),
                                       (128, 8, 77, 4), (6, 2, 500, 600), (100, 3, 5000, 3), (256, 2, 3000, 2),
                                       (512, 8, 2000, 1), (16, 2, 60000, 1), (768, 4, 300, 1)])
def test_alc_scores_vs_oracle(torch_dev, lagp, j, p, nc, B):
    """a3 alone against oracle_alc_scores: the one-CTA-per-location kernel (small
    batches) and the DMMA contraction (row f4: the paper's Fig 4 scale, j <= 768,
    N' = 60,000)."""
    torch, dev = torch_dev
    rng = np.random.default_rng(j * 100 + p)
    d, g = 0.3 if p > 3 else 0.05, 1e-4
    Xj = rng.random((B, j, p))
    cands = rng.random((B, nc, p))
    x = rng.random((B, p))
    Kinv = np.stack([oracle.invert_spd(np.exp(-((Xj[b][:, None] - Xj[b][None]) ** 2).sum(-1) / d) + g * np.eye(j))
                     for b in range(B)])
    cidx = np.stack([rng.permutation(10 * nc)[:nc] for _ in range(B)]).astype(np.int32)
    delta, best, gap = lagp.alc_scores(T(torch, dev, Xj), T(torch, dev, Kinv), T(torch, dev, cands),
                                       T(torch, dev, cidx), T(torch, dev, x), d, g)
    delta = delta.cpu().numpy()
    best = best.cpu().numpy()
    for b in range(min(B, 6)):
        ref, _, minv = oracle.alc_scores(Xj[b], Kinv[b], cands[b], x[b], d, g)
        ok = minv > 1e-12
        scale = np.abs(ref[ok]).max()
        # explicit-inverse noise: eps * cond * j / min(s) (pin P1 ill-conditioned bound), or
        # per candidate the first-order forward-error bound of two FP64 evaluations of
        # s = 1 + g - k^T K^{-1} k and cov = kappa - (K^{-1} h)^T k in different orders:
        # |ds| <= 4 j eps |k|^T |K^{-1}| |k|, |dcov| <= 4 j eps (|K^{-1}| |h|)^T |k|
        eps = 2.0 ** -53
        kc = np.exp(-((cands[b][:, None, :] - Xj[b][None]) ** 2).sum(-1) / d)
        hb = np.exp(-((Xj[b] - x[b]) ** 2).sum(-1) / d)
        aK = np.abs(Kinv[b])
        ds = 4 * j * eps * np.einsum("ca,ab,cb->c", kc, aK, kc)
        dcv = 4 * j * eps * (kc @ (aK @ hb)) + 4 * eps
        sv = np.where(ok, minv, 1.0)
        cov = np.sqrt(np.maximum(ref, 0) * sv)
        bound = (np.maximum(ref, 0) * ds / sv + 2 * cov * dcv / sv + dcv ** 2 / sv)[ok]
        tol = np.maximum(max(1e-9, 1e-5 if p <= 3 else 1e-8) * scale, 4 * bound)
        assert np.all(np.abs(delta[b][ok] - ref[ok]) <= tol)
        assert np.all(np.isneginf(delta[b][~ok]))
        o = np.lexsort((cidx[b][ok], -ref[ok]))[0]
        ob = np.where(ok)[0][o]
        srt = np.sort(ref[ok])[::-1]
        if len(srt) < 2 or (srt[0] - srt[1]) / srt[0] > 1e-6:
            assert best[b] == ob


# ------------------------------------------------------------- a4: update
@pytest.mark.parametrize("j", [1, 5, 31, 64, 127])
def test_pinv_update_vs_oracle(torch_dev, lagp, j):
    torch, dev = torch_dev
    rng = np.random.default_rng(j)
    B, p, d, g = 3, 3, 0.05, 1e-3
    XS = rng.random((B, j + 1, p))
    K = np.exp(-((XS[:, :, None] - XS[:, None]) ** 2).sum(-1) / d) + g * np.eye(j + 1)
    Kinv = np.stack([np.linalg.inv(K[b, :j, :j]) for b in range(B)])
    Kinv = 0.5 * (Kinv + Kinv.transpose(0, 2, 1))  # exactly symmetric input
    k = np.ascontiguousarray(K[:, :j, j])
    out = lagp.pinv_update(T(torch, dev, Kinv), T(torch, dev, k), 1.0 + g).cpu().numpy()
    for b in range(B):
        ref, rc = oracle.pinv_update(Kinv[b], k[b], 1.0 + g)
        assert np.linalg.norm(out[b] - ref) <= 1e-10 * np.linalg.norm(ref)
        assert np.array_equal(out[b], out[b].T)


# ------------------------------------------------------------- a5: predict
@pytest.mark.parametrize("n,p", [(3, 2), (8, 1), (50, 8), (128, 3)])
def test_predict_vs_oracle(torch_dev, lagp, n, p):
    torch, dev = torch_dev
    rng = np.random.default_rng(n + p)
    B, d, g = 5, 0.2 if p > 2 else 0.02, 1e-4
    Xn = rng.random((B, n, p))
    Yn = rng.normal(size=(B, n))
    x = rng.random((B, p))
    mean, s2, var = (t.cpu().numpy() for t in lagp.predict(T(torch, dev, Xn), T(torch, dev, Yn), T(torch, dev, x),
                                                          d, g))
    for b in range(B):
        m, s, v = oracle.predict(Xn[b], Yn[b], x[b], d, g)
        assert abs(mean[b] - m) <= 1e-8 * max(1.0, abs(m))
        assert abs(s2[b] - s) <= 1e-8 * s
        if n > 2:
            assert abs(var[b] - v) <= 1e-8 * v
        else:
            assert np.isnan(var[b])


# ------------------------------------------------------- full path (a1-a5)
def run_both(torch, dev, lagp, cfg, form="explicit", threads=0):
    X, Z, XX = cfg["X"], cfg["Z"], cfg["XX"]
    r = lagp.alc_batch(T(torch, dev, X), T(torch, dev, Z), T(torch, dev, XX), cfg["d"], cfg["g"], cfg["n0"], cfg["n"],
                       cfg["Nprime"], form=form, gaps=True)
    g = {k: v.cpu().numpy() for k, v in r.items() if hasattr(v, "cpu")}
    o = oracle.alc_batch(X, Z, XX, cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"], threads=threads)
    return g, o


@pytest.mark.parametrize(
    "name,M,N,over",
    [
        ("C1", 100, None, {}),  # full C1
        ("C2", 96, None, {}),  # C2 design, 96 locations
        ("C3", 96, None, {}),  # LGBB grid (distance ties at the N'-th NN)
        ("C3j", 48, None, {}),
        ("C1", 33, 800, dict(n0=1, n=12, Nprime=40)),
        ("C1", 17, 500, dict(n0=6, n=6, Nprime=6)),  # no greedy step: NN only
        ("C2", 9, 3000, dict(n0=4, n=128, Nprime=300)),  # n = LAGP_NMAX
        ("C1", 5, 60, dict(n0=5, n=60, Nprime=60)),  # n = N' = N: full GP
    ],
)
@pytest.mark.parametrize("form", ["explicit", "explicit_dfma", "incremental"])
def test_alc_batch_vs_oracle(torch_dev, lagp, name, M, N, over, form):
    torch, dev = torch_dev
    cfg = make_config(name, M=M, N=N, **over)
    g, o = run_both(torch, dev, lagp, cfg, form=form)
    p = cfg["X"].shape[1]
    # the incremental form on the named workloads: no divergence at all
    strict = form == "incremental" and not over and N is None and name in ("C1", "C2", "C3", "C3j", "C4")
    rep = check(g, o, cfg, form, **({"max_explained": 0.0} if strict else {}))
    print(name, form, rep)


FORMS = ["explicit", "explicit_dfma", "incremental"]


@pytest.mark.parametrize("form", ["explicit", "explicit_dfma"])
def test_large_pool_explicit(torch_dev, lagp, form):
    """N' > 8192 (C5's large pools): NN selection in the global survivor buffers
    and the explicit forms with kappa/chosen in the global slab."""
    torch, dev = torch_dev
    cfg = make_config("C5_2d", M=3, Nprime=12000, n=20)
    g, o = run_both(torch, dev, lagp, cfg, form=form)
    check(g, o, cfg, form)


@pytest.mark.parametrize("form,Nprime,n,p", [("explicit", 20000, 64, 8), ("explicit_dfma", 10000, 128, 2),
                                             ("incremental", 20000, 128, 8)])
def test_large_pool_deep_design(torch_dev, lagp, form, Nprime, n, p):
    """Large pools with deep designs (C5's N' = 10^4-2*10^4 at n = 64 / 128, the shapes of
    the C5 sweep's large-pool rows): the explicit DMMA kernel at its n = 64 limit, the
    DFMA explicit kernel at n = LAGP_NMAX, and the HBM-streaming incremental kernel at
    n = 128, against the oracle on two locations each."""
    torch, dev = torch_dev
    cfg = make_config("C5_2d" if p == 2 else "C5_8d", M=2, Nprime=Nprime, n=n)
    g, o = run_both(torch, dev, lagp, cfg, form=form)
    check(g, o, cfg, form)


@pytest.mark.parametrize("Nprime,n,p", [(9000, 20, 2), (12000, 30, 2), (20000, 24, 8)])
def test_incremental_stream_large_pool(torch_dev, lagp, Nprime, n, p):
    """N' > 8192 (the paper's LGBB N' = 10,000 variant, C5's large pools): the
    incremental form on the HBM-streaming kernel (per-candidate state in HBM)."""
    torch, dev = torch_dev
    cfg = make_config("C5_2d" if p == 2 else "C5_8d", M=3, Nprime=Nprime, n=n)
    g, o = run_both(torch, dev, lagp, cfg, form="incremental")
    check(g, o, cfg, "incremental")


@pytest.mark.parametrize("form", FORMS)
def test_full_gp_special_case(torch_dev, lagp, form):
    """n = N' = N: the local design is all of X; prediction equals Eq (1)-(2)."""
    torch, dev = torch_dev
    rng = np.random.default_rng(5)
    X = rng.random((40, 2))
    Z = np.sin(3 * X[:, 0]) + X[:, 1]
    XX = rng.random((6, 2))
    d, g = 0.1, 1e-4
    r = lagp.alc_batch(T(torch, dev, X), T(torch, dev, Z), T(torch, dev, XX), d, g, 3, 40, 40, form=form)
    K = np.exp(-((X[:, None] - X[None]) ** 2).sum(-1) / d) + g * np.eye(40)
    for i in range(6):
        assert sorted(r["idx"][i].cpu().tolist()) == list(range(40))
        k = np.exp(-((X - XX[i]) ** 2).sum(-1) / d)
        mu = k @ np.linalg.solve(K, Z)
        s2 = (Z @ np.linalg.solve(K, Z)) * (1 + g - k @ np.linalg.solve(K, k)) / 40
        assert abs(r["mean"][i].item() - mu) <= 1e-8 * max(1, abs(mu))
        assert abs(r["s2"][i].item() - s2) <= 1e-7 * s2


@pytest.mark.parametrize("form", FORMS)
def test_exhausted_and_sentinel(torch_dev, lagp, form):
    torch, dev = torch_dev
    X = np.array([[0.5, 0.5]] * 3 + [[0.9, 0.9]])
    Z = np.array([1.0, 1.0, 1.0, 2.0])
    XX = np.array([[0.4, 0.5]])
    cfg = dict(X=X, Z=Z, XX=XX, d=0.1, g=0.0, n0=1, n=3, Nprime=3)
    g, o = run_both(torch, dev, lagp, cfg, form=form)
    assert g["idx"].tolist() == o["idx"].tolist() == [[0, -1, -1]]
    assert g["flags"][0] & lagp.FLAG_EXHAUSTED and g["flags"][0] & lagp.FLAG_SENTINEL
    assert abs(g["mean"][0] - o["mean"][0]) < 1e-14 and abs(g["s2"][0] - o["s2"][0]) < 1e-14
    assert np.isnan(g["var"][0])


@pytest.mark.parametrize("form", FORMS)
def test_exact_tie_lowest_index(torch_dev, lagp, form):
    torch, dev = torch_dev
    X = np.array([[0.0], [0.1], [-0.1], [0.2], [-0.2]])
    Z = X[:, 0].copy()
    cfg = dict(X=X, Z=Z, XX=np.array([[0.0]]), d=0.05, g=1e-4, n0=1, n=3, Nprime=5)
    g, o = run_both(torch, dev, lagp, cfg, form=form)
    assert g["idx"][0, :2].tolist() == [0, 1]
    assert g["flags"][0] & lagp.FLAG_NEAR_TIE
    assert g["gaps"][0, 0] == 0.0


@pytest.mark.parametrize("form", FORMS)
def test_determinism_and_chunk_composition(torch_dev, lagp, form):
    torch, dev = torch_dev
    cfg = make_config("C2", M=300, N=20000)
    X, Z, XX = (T(torch, dev, cfg[k]) for k in ("X", "Z", "XX"))
    args = (cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    a = lagp.alc_batch(X, Z, XX, *args, form=form)
    b = lagp.alc_batch(X, Z, XX, *args, form=form)
    c1 = lagp.alc_batch(X, Z, XX[:113], *args, form=form)
    c2 = lagp.alc_batch(X, Z, XX[113:], *args, form=form)
    for k in ("idx", "mean", "s2", "var", "flags"):
        assert torch.equal(a[k], b[k]), k
        assert torch.equal(a[k], torch.cat([c1[k], c2[k]])), k


def test_forms_agree(torch_dev, lagp):
    """Explicit (DMMA), explicit (DFMA) and incremental forms select the same
    designs on the C1 locations (all three within the parity rules)."""
    torch, dev = torch_dev
    cfg = make_config("C1")
    X, Z, XX = (T(torch, dev, cfg[k]) for k in ("X", "Z", "XX"))
    args = (cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    res = {f: lagp.alc_batch(X, Z, XX, *args, form=f) for f in FORMS}
    same = [(res[f]["idx"] == res["incremental"]["idx"]).all(1).float().mean().item() for f in FORMS]
    assert min(same) >= 0.97, same


def test_host_entry_point_matches_device(torch_dev, lagp):
    torch, dev = torch_dev
    cfg = make_config("C1", M=20)
    args = (cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    h = lagp.alc_batch_host(cfg["X"], cfg["Z"], cfg["XX"], *args)
    d = lagp.alc_batch(T(torch, dev, cfg["X"]), T(torch, dev, cfg["Z"]), T(torch, dev, cfg["XX"]), *args)
    assert np.array_equal(h["idx"], d["idx"].cpu().numpy())
    assert np.array_equal(h["mean"], d["mean"].cpu().numpy())


@pytest.mark.parametrize("form", FORMS)
def test_full_size_C2_sampled(torch_dev, lagp, form):
    """The bench configuration (C2: N=1e5, M=1e4) in the bench's launch
    configuration, checked on a seeded sample of 48 locations."""
    torch, dev = torch_dev
    cfg = make_config("C2")
    r = lagp.alc_batch(T(torch, dev, cfg["X"]), T(torch, dev, cfg["Z"]), T(torch, dev, cfg["XX"]), cfg["d"], cfg["g"],
                       cfg["n0"], cfg["n"], cfg["Nprime"], gaps=True, form=form)
    sel = np.sort(np.random.default_rng(7).choice(cfg["XX"].shape[0], 48, replace=False))
    g = {k: v.cpu().numpy()[sel] for k, v in r.items() if hasattr(v, "cpu")}
    o = oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"][sel], cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    check(g, o, dict(cfg, XX=cfg["XX"][sel]), form, tau=golden_tau("C2"),
          **({"max_explained": 0.0} if form == "incremental" else {}))
    # properties at every location: indices distinct and in range, s2 > 0
    idx = r["idx"].cpu().numpy()
    assert (idx >= 0).all() and (idx < cfg["X"].shape[0]).all()
    srt = np.sort(idx, axis=1)
    assert (np.diff(srt, axis=1) > 0).all()
    assert (r["s2"].cpu().numpy() > 0).all()


def test_exp_nonpos_table_ulp(torch_dev, lagp):
    """The incremental kernels' exp (laGP_exp_nonpos) against the correctly
    rounded exp of each double input (decimal arithmetic): <= 1 ulp on x in
    [-708, 0], exact at 0, 0 below -708, NaN propagated."""
    import math
    from decimal import Decimal, getcontext

    torch, dev = torch_dev
    rng = np.random.default_rng(7)
    x = np.concatenate([-rng.uniform(0, 708, 1500), -rng.uniform(0, 1, 500), -rng.uniform(0, 1e-3, 200),
                        -np.logspace(-300, 2.85, 300), [0.0, -0.0, -708.0, -707.99999, -1e-320]])
    y = lagp.exp_nonpos(torch.from_numpy(x).to(dev)).cpu().numpy()
    getcontext().prec = 40
    worst = 0.0
    for xi, yi in zip(x, y):
        ref = float(Decimal(float(xi)).exp())
        ulp = math.ulp(ref)
        worst = max(worst, abs(yi - ref) / ulp)
    assert worst <= 1.0, worst
    assert y[x == 0.0].tolist() == [1.0, 1.0]
    z = lagp.exp_nonpos(torch.tensor([-708.0001, -1e4, float("nan")], dtype=torch.float64, device=dev)).cpu().numpy()
    assert z[0] == 0.0 and z[1] == 0.0 and np.isnan(z[2])


def _synthetic(seed, N, M, p):
    rng = np.random.default_rng(seed)
    X = rng.random((N, p))
    Z = np.sin(4 * X).sum(1) + 0.5 * X[:, 0]
    XX = rng.random((M, p))
    return X, Z, XX


@pytest.mark.parametrize("stream", ["0", "1"])
@pytest.mark.parametrize("Nprime,p,n", [(1500, 2, 30), (4000, 8, 40), (8192, 2, 24), (2048, 3, 70)])
def test_incremental_large_pools(torch_dev, lagp, Nprime, p, n, stream):
    """1024 < N' <= 8192: the 1024-thread incremental kernel with several
    candidates per thread (the v2 kernel covers N' <= 1024), and the HBM-streaming
    kernel on the same shapes (LAGP_INC_STREAM=1)."""
    import os

    torch, dev = torch_dev
    X, Z, XX = _synthetic(Nprime + p, 40000, 6, p)
    cfg = dict(X=X, Z=Z, XX=XX, d=0.02 * p, g=1e-4, n0=6, n=n, Nprime=Nprime)
    old = os.environ.get("LAGP_INC_STREAM")
    os.environ["LAGP_INC_STREAM"] = stream
    try:
        g, o = run_both(torch, dev, lagp, cfg, form="incremental")
    finally:
        if old is None:
            os.environ.pop("LAGP_INC_STREAM", None)
        else:
            os.environ["LAGP_INC_STREAM"] = old
    check(g, o, cfg, "incremental")


@pytest.mark.parametrize("p", [1, 5, 7])
@pytest.mark.parametrize("form", FORMS)
def test_generic_dimension(torch_dev, lagp, p, form):
    """p outside {2, 3, 4, 8}: the generic-p instantiations of the NN and design kernels."""
    torch, dev = torch_dev
    X, Z, XX = _synthetic(100 + p, 6000, 10, p)
    cfg = dict(X=X, Z=Z, XX=XX, d=0.05 * p, g=1e-4, n0=4, n=30, Nprime=400)
    g, o = run_both(torch, dev, lagp, cfg, form=form)
    check(g, o, cfg, form)


@pytest.mark.parametrize("p", [1, 5])
def test_incremental_stream_generic_p(torch_dev, lagp, p):
    """The HBM-streaming kernel's p = 1 and generic-p (P = 0) instantiations (N' > 8192)."""
    torch, dev = torch_dev
    X, Z, XX = _synthetic(100 + p, 40000, 4, p)
    cfg = dict(X=X, Z=Z, XX=XX, d=0.05 * p, g=1e-4, n0=5, n=24, Nprime=9500)
    g, o = run_both(torch, dev, lagp, cfg, form="incremental")
    check(g, o, cfg, "incremental")


def test_explicit_dmma_one_cta_per_sm(torch_dev, lagp):
    """LAGP_DM_WARPS=16: the explicit DMMA kernel as one 16-warp CTA per SM (128-candidate
    tiles) against the oracle."""
    import os

    torch, dev = torch_dev
    cfg = make_config("C2", M=24, N=20000)
    old = os.environ.get("LAGP_DM_WARPS")
    os.environ["LAGP_DM_WARPS"] = "16"
    try:
        g, o = run_both(torch, dev, lagp, cfg, form="explicit")
    finally:
        if old is None:
            os.environ.pop("LAGP_DM_WARPS", None)
        else:
            os.environ["LAGP_DM_WARPS"] = old
    check(g, o, cfg, "explicit")


@pytest.mark.parametrize("env", [{"LAGP_V2_CPT": "2"}, {"LAGP_V2_CPT": "1"}, {"LAGP_V2_SFIRST": "1"},
                                 {"LAGP_V2_NOSTAGGER": "1"}, {"LAGP_INC_V1": "1"}, {"LAGP_NN_MMA": "1"},
                                 {"LAGP_NN_MMA": "0"}, {"LAGP_NN_CELLS": "0"}, {"LAGP_NN_CELLS": "2"},
                                 {"LAGP_NN_CR": "16"}, {"LAGP_NN_CR": "4096"}, {"LAGP_NN_Q": "4"},
                                 {"LAGP_NN_Q": "8"}, {"LAGP_NN_Q": "16"}])
def test_kernel_variants_agree(torch_dev, lagp, env):
    """Every A/B switch of the library (CTA shapes, tier order, phase order, v1
    kernel; NN: TF32 filter on/off, no spatial cells, the two-axis grid, multi-axis
    cells of 16 / 4096 rows, 4/8/16-query groups) against
    the oracle on the same C2 sample as the default path, with n = 64 so the
    shared-memory, tensor-memory and slab tiers are all in use."""
    import os

    torch, dev = torch_dev
    cfg = make_config("C2", M=24, N=20000, n=64)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        g, o = run_both(torch, dev, lagp, cfg, form="incremental")
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    check(g, o, cfg, "incremental")


def test_north_star_entry_point(torch_dev, lagp):
    """laGP_alc_batch itself — the north_star signature, called through ctypes
    with device data and every output — against the oracle; it resolves to the
    incremental form (LAGP_ALC_AUTO), which lagp_timing reports; pools beyond the
    incremental kernels resolve to the paper's explicit form."""
    import ctypes

    torch, dev = torch_dev
    cfg = make_config("C2", M=64, N=20000)
    X, Z, XX = (T(torch, dev, cfg[k]) for k in ("X", "Z", "XX"))
    M, n, n0 = XX.shape[0], cfg["n"], cfg["n0"]
    out = dict(idx=torch.empty((M, n), dtype=torch.int32, device=dev),
               mean=torch.empty(M, dtype=torch.float64, device=dev), s2=torch.empty(M, dtype=torch.float64, device=dev),
               var=torch.empty(M, dtype=torch.float64, device=dev), flags=torch.empty(M, dtype=torch.int32, device=dev),
               gaps=torch.empty((M, n - n0), dtype=torch.float64, device=dev))
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = lagp.lib().laGP_alc_batch(vp(X), X.shape[0], X.shape[1], vp(Z), vp(XX), M, cfg["d"], cfg["g"], n0, n,
                                   cfg["Nprime"], vp(out["idx"]), vp(out["mean"]), vp(out["s2"]), vp(out["var"]),
                                   vp(out["flags"]), vp(out["gaps"]),
                                   ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    assert st == lagp.LAGP_OK, lagp.last_error()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    o = oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"], cfg["d"], cfg["g"], n0, n, cfg["Nprime"])
    rep = check(g, o, cfg, "incremental", label="laGP_alc_batch")
    assert rep["identical"] == M
    r = lagp.alc_batch(X, Z, XX[:4], cfg["d"], cfg["g"], n0, n, cfg["Nprime"], timing=True)
    assert r["timing"]["alc_form"] == "incremental"
    assert torch.equal(r["idx"], out["idx"][:4])
    big = make_config("C5_2d", M=2, Nprime=12000, n=20)
    rb = lagp.alc_batch(*(T(torch, dev, big[k]) for k in ("X", "Z", "XX")), big["d"], big["g"], big["n0"], big["n"],
                        big["Nprime"], timing=True)
    assert rb["timing"]["alc_form"] == "incremental"  # the HBM-streaming kernel
