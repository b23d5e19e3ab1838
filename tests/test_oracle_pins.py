"""Pins for the CPU oracle (SURVEY.md §8c P1–P11).

Each test checks ``oracle/`` against something other than itself: the
definition of the greedy criterion computed by brute-force dense solves
(Fig 1 step 2(b), Eq (5), `eq:newv`), direct inversion, exhaustive sorting with
exact-arithmetic keys, the full-GP special case (Eq (1)-(2)), closed forms and
the worked examples in tests/golden/. No expected value comes from the CUDA path.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


# ---------------------------------------------------------------- brute force
def corr(A, B, d):
    A = np.atleast_2d(A)
    B = np.atleast_2d(B)
    D = ((A[:, None, :] - B[None, :, :]) ** 2).sum(-1)
    return np.exp(-D / d)


def v_of(XS, x, d, g):
    """v(x) = K(x,x) - k^T K^{-1} k on design XS, K(x,x) = 1+g (`eq:newv`)."""
    if len(XS) == 0:
        return 1.0 + g
    K = corr(XS, XS, d) + g * np.eye(len(XS))
    k = corr(XS, x, d)[:, 0]
    return 1.0 + g - k @ np.linalg.solve(K, k)


def exact_key(x, row):
    """fma-accumulated d^2 (k = 0..p-1), emulated exactly with rationals."""
    acc = 0.0
    for k in range(len(x)):
        diff = float(x[k]) - float(row[k])
        acc = float(Fraction(diff) * Fraction(diff) + Fraction(acc))
    return acc


def exact_nn(X, x, m):
    keys = [(exact_key(x, X[i]), i) for i in range(X.shape[0])]
    keys.sort()
    return np.array([i for _, i in keys[:m]], dtype=np.int32)


def brute_greedy(X, Z, x, d, g, n0, n, Nprime):
    """Fig 1 step 2 by definition: argmax_c v_j(x) - v_{j+1}(x) via dense solves."""
    pool = exact_nn(X, x, Nprime)
    chosen = [int(i) for i in pool[:n0]]
    gaps, best = [], []
    for _ in range(n0, n):
        vj = v_of(X[chosen], x, d, g)
        scores = []
        for c in pool:
            c = int(c)
            if c in chosen:
                continue
            scores.append((vj - v_of(X[chosen + [c]], x, d, g), -c))
        scores.sort(reverse=True)
        (d1, c1), (d2, _) = scores[0], scores[1] if len(scores) > 1 else (0.0, 0)
        gaps.append((d1 - max(d2, 0.0)) / d1)
        best.append(d1)
        chosen.append(-c1)
    XS = X[chosen]
    K = corr(XS, XS, d) + g * np.eye(len(chosen))
    h = corr(XS, x, d)[:, 0]
    Y = Z[chosen]
    b = np.linalg.solve(K, Y)
    psi = Y @ b
    mu = h @ b
    s2 = psi * (1 + g - h @ np.linalg.solve(K, h)) / len(chosen)
    return np.array(chosen), mu, s2, np.array(gaps), np.array(best)


# ----------------------------------------------------------------------- P4 NN
def test_nn_1d_example():
    """1-d design (0,1,2,3), x=1.1, m=2 -> rows 1 then 2."""
    X = np.array([[0.0], [1.0], [2.0], [3.0]])
    idx, d2 = oracle.nn(X, np.array([1.1]), 2)
    assert idx.tolist() == [1, 2]


@pytest.mark.parametrize("p,N,m,seed", [(8, 1000, 100, 1), (2, 500, 500, 2), (3, 300, 17, 3)])
def test_nn_exhaustive_exact_keys(p, N, m, seed):
    """P4: the pool equals an exhaustive sort by exactly-rounded fma keys (d^2, idx)."""
    rng = np.random.default_rng(seed)
    X = rng.random((N, p))
    x = rng.random(p)
    idx, d2 = oracle.nn(X, x, m)
    ref = exact_nn(X, x, m)
    assert idx.tolist() == ref.tolist()
    assert [exact_key(x, X[i]) for i in idx] == d2.tolist()


def test_nn_grid_ties_lowest_index():
    """R8: exact distance ties on a grid resolve to the lowest row index."""
    G = np.stack(np.meshgrid(np.arange(7.0), np.arange(5.0), indexing="ij"), -1).reshape(-1, 2)
    x = np.array([3.0, 2.0])
    for m in (1, 5, 9, 13, 21):
        idx, _ = oracle.nn(G, x, m)
        assert idx.tolist() == exact_nn(G, x, m).tolist()
    idx, _ = oracle.nn(G, x, 5)
    # centre first, then the 4 unit-distance neighbours in index order
    c = 3 * 5 + 2
    assert idx.tolist() == [c, c - 5, c - 1, c + 1, c + 5]


# --------------------------------------------------------- invert (a2 helper)
def test_invert_spd_matches_library():
    rng = np.random.default_rng(4)
    for n in (1, 2, 6, 20, 50):
        Xj = rng.random((n, 3))
        K = corr(Xj, Xj, 0.3) + 1e-4 * np.eye(n)
        Ki = oracle.invert_spd(K)
        ref = np.linalg.inv(K)
        assert np.linalg.norm(Ki - ref) / np.linalg.norm(ref) < 1e-9
        assert np.array_equal(Ki, Ki.T)


# ------------------------------------------------------------ P1/P2 ALC score
def kval(a, b, d):
    """K(a,b) with the same IEEE steps as the definition: fma-keyed d^2, /d, exp."""
    return math.exp(-exact_key(a, b) / d)


def exact_solve(A, b):
    """Gaussian elimination in exact rational arithmetic."""
    n = len(A)
    M = [[Fraction(A[i][j]) for j in range(n)] + [Fraction(b[i])] for i in range(n)]
    for c in range(n):
        piv = max(range(c, n), key=lambda r: abs(M[r][c]))
        M[c], M[piv] = M[piv], M[c]
        for r in range(c + 1, n):
            f = M[r][c] / M[c][c]
            if f:
                for k in range(c, n + 1):
                    M[r][k] -= f * M[c][k]
    x = [Fraction(0)] * n
    for i in range(n - 1, -1, -1):
        x[i] = (M[i][n] - sum(M[i][k] * x[k] for k in range(i + 1, n))) / M[i][i]
    return x


def v_exact(XS, x, d, g):
    """v(x) = 1 + g - k^T K^{-1} k exactly (rationals) for the given double entries."""
    n = len(XS)
    K = [[kval(XS[a], XS[b], d) + (g if a == b else 0.0) for b in range(n)] for a in range(n)]
    k = [kval(XS[a], x, d) for a in range(n)]
    s = exact_solve(K, k)
    return Fraction(1) + Fraction(g) - sum(Fraction(k[i]) * s[i] for i in range(n))


def _alc_instance(seed, glo, ghi):
    rng = np.random.default_rng(100 + seed)
    p = int(rng.integers(1, 5))
    j = int(rng.integers(1, 13))
    d = float(rng.uniform(0.2, 1.5))
    g = float(10 ** rng.uniform(glo, ghi))
    Xj = rng.random((j, p))
    cands = rng.random((12, p))
    x = rng.random(p)
    return p, j, d, g, Xj, cands, x


@pytest.mark.parametrize("seed", range(20))
def test_alc_scores_equal_exact_variance_difference(seed):
    """P1: Delta(x') = v_j(x) - v_{j+1}(x) (eq:newv, Eq 5), reference in exact
    rational arithmetic; well-conditioned draws (g >= 1e-2) so the explicit
    inverse's own rounding stays far below the 1e-9 bound."""
    p, j, d, g, Xj, cands, x = _alc_instance(seed, -2, -1)
    Kinv = np.linalg.inv(corr(Xj, Xj, d) + g * np.eye(j))
    dcf, dlit, minv = oracle.alc_scores(Xj, Kinv, cands, x, d, g)
    XL = [r for r in Xj]
    vj = v_exact(XL, x, d, g)
    ref = np.array([float(vj - v_exact(XL + [c], x, d, g)) for c in cands])
    scale = np.abs(ref).max()
    assert np.abs(dcf - ref).max() <= 1e-9 * scale
    # P2: Eq (5) literal = closed form up to roundoff
    assert np.abs(dlit - dcf).max() <= 1e-9 * scale
    # m_j^{-1}(x') is the Schur complement of Eq (6)
    for c, mc in zip(cands, minv):
        k = corr(Xj, c, d)[:, 0]
        assert abs(mc - (1 + g - k @ np.linalg.solve(corr(Xj, Xj, d) + g * np.eye(j), k))) < 1e-10
    assert (dcf >= 0).all()


@pytest.mark.parametrize("seed", range(6))
def test_alc_scores_ill_conditioned_within_inverse_noise(seed):
    """P1 at g down to 1e-4: the explicit-inverse error stays within the
    first-order bound eps * cond(K_j) * j / min(m^{-1}) (App A.6)."""
    p, j, d, g, Xj, cands, x = _alc_instance(seed, -4, -2)
    K = corr(Xj, Xj, d) + g * np.eye(j)
    Kinv = np.linalg.inv(K)
    dcf, _, minv = oracle.alc_scores(Xj, Kinv, cands, x, d, g)
    XL = [r for r in Xj]
    vj = v_exact(XL, x, d, g)
    ref = np.array([float(vj - v_exact(XL + [c], x, d, g)) for c in cands])
    bound = 64 * 2.2e-16 * np.linalg.cond(K) * j / minv.min()
    assert np.abs(dcf - ref).max() <= max(bound, 1e-12) * np.abs(ref).max()


def test_alc_selection_property():
    """P8: eta=0 and x itself among the candidates -> Delta(x) = v_j(x) is the max."""
    rng = np.random.default_rng(7)
    for _ in range(10):
        p = 2
        Xj = rng.random((5, p))
        x = rng.random(p)
        cands = np.vstack([rng.random((15, p)), x[None, :]])
        Kinv = np.linalg.inv(corr(Xj, Xj, 0.5))
        dcf, _, _ = oracle.alc_scores(Xj, Kinv, cands, x, 0.5, 0.0)
        assert int(np.argmax(dcf)) == 15
        vj = v_of(Xj, x, 0.5, 0.0)
        assert abs(dcf[15] - vj) <= 1e-8 * vj


def test_alc_far_candidate_scores_zero():
    """A candidate with no correlation to x or X_j reduces nothing: Delta = 0."""
    Xj = np.array([[0.0, 0.0], [0.1, 0.0]])
    Kinv = np.linalg.inv(corr(Xj, Xj, 0.01) + 1e-4 * np.eye(2))
    dcf, _, minv = oracle.alc_scores(Xj, Kinv, np.array([[50.0, 50.0]]), np.array([0.05, 0.0]), 0.01, 1e-4)
    assert dcf[0] == 0.0 and minv[0] == 1.0 + 1e-4


# ------------------------------------------------------------- P3 pinv update
@pytest.mark.parametrize("j", [1, 2, 5, 20, 49, 127])
def test_partitioned_inverse_matches_direct_inversion(j):
    rng = np.random.default_rng(j)
    p = 3
    d, g = 0.05, 1e-3
    XS = rng.random((j + 1, p))
    K1 = corr(XS, XS, d) + g * np.eye(j + 1)
    cond = np.linalg.cond(K1)
    assert cond <= 1e6
    Kinv = np.linalg.inv(K1[:j, :j])
    out, rc = oracle.pinv_update(Kinv, K1[:j, j], K1[j, j])
    assert rc == 0
    ref = np.linalg.inv(K1)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-8


# --------------------------------------------------- P5 full-GP special case
@pytest.mark.parametrize("seed", range(4))
def test_full_gp_when_n_equals_N(seed):
    """P5: n = N' = N => the local design is all of X and (mu, s2) = Eq (1)-(2)."""
    rng = np.random.default_rng(300 + seed)
    N, p = 24, 2
    X = rng.random((N, p))
    Z = np.sin(4 * X[:, 0]) + X[:, 1] ** 2
    x = rng.random(p)
    d, g = 0.2, 1e-3
    r = oracle.local_design(X, Z, x, d, g, 4, N, N)
    assert sorted(r["idx"].tolist()) == list(range(N))
    K = corr(X, X, d) + g * np.eye(N)
    k = corr(X, x, d)[:, 0]
    Ki_Y = np.linalg.solve(K, Z)
    mu = k @ Ki_Y  # Eq (1)
    psi = Z @ Ki_Y
    s2 = psi * (1 + g - k @ np.linalg.solve(K, k)) / N  # Eq (2)
    assert abs(r["mean"] - mu) <= 1e-9 * max(1.0, abs(mu))
    assert abs(r["s2"] - s2) <= 1e-8 * s2
    assert abs(r["var"] - s2 * N / (N - 2)) <= 1e-8 * s2


# ------------------------------------------------------------- P6 predict
def test_predict_interpolates_at_design_point_eta0():
    rng = np.random.default_rng(11)
    Xn = rng.random((10, 2))
    Yn = rng.normal(size=10)
    m, s2, var = oracle.predict(Xn, Yn, Xn[3], 0.3, 0.0)
    assert abs(m - Yn[3]) < 1e-8
    assert abs(s2) < 1e-10


def test_predict_far_field():
    rng = np.random.default_rng(12)
    Xn = rng.random((10, 2))
    Yn = rng.normal(size=10)
    g = 1e-3
    m, s2, var = oracle.predict(Xn, Yn, np.array([40.0, 40.0]), 0.1, g)
    K = corr(Xn, Xn, 0.1) + g * np.eye(10)
    psi = Yn @ np.linalg.solve(K, Yn)
    assert m == 0.0
    assert abs(s2 - psi * (1 + g) / 10) <= 1e-12 * s2
    assert abs(var - s2 * 10 / 8) <= 1e-12 * var


def test_predict_matches_dense_solve():
    rng = np.random.default_rng(13)
    for n in (3, 8, 50):
        Xn = rng.random((n, 3))
        Yn = rng.normal(size=n)
        x = rng.random(3)
        d, g = 0.4, 1e-4
        m, s2, var = oracle.predict(Xn, Yn, x, d, g)
        K = corr(Xn, Xn, d) + g * np.eye(n)
        k = corr(Xn, x, d)[:, 0]
        mu = k @ np.linalg.solve(K, Yn)
        ref = (Yn @ np.linalg.solve(K, Yn)) * (1 + g - k @ np.linalg.solve(K, k)) / n
        assert abs(m - mu) <= 1e-8 * max(1, abs(mu))
        assert abs(s2 - ref) <= 1e-7 * ref


# ------------------------------------------------ brute-force greedy (Fig 1)
@pytest.mark.parametrize("seed", range(12))
def test_greedy_loop_equals_bruteforce_definition(seed):
    """Fig 1 step 2 by definition (argmax of fresh-solve variance reductions)."""
    rng = np.random.default_rng(500 + seed)
    p = int(rng.integers(1, 5))
    N = int(rng.integers(20, 60))
    X = rng.random((N, p))
    Z = np.cos(3 * X).sum(1)
    x = rng.random(p)
    n0 = int(rng.integers(1, 5))
    n = n0 + int(rng.integers(2, 9))
    Nprime = int(rng.integers(n + 1, N + 1))
    d = float(rng.uniform(0.05, 0.6))
    g = 1e-3
    r = oracle.local_design(X, Z, x, d, g, n0, n, Nprime)
    idx, mu, s2, gaps, best = brute_greedy(X, Z, x, d, g, n0, n, Nprime)
    # identical trajectories unless the brute-force top-2 gap is at roundoff level
    for t in range(n):
        if t >= n0 and gaps[t - n0] < 1e-9:
            break
        assert r["idx"][t] == idx[t], (t, r["idx"], idx)
    else:
        assert abs(r["mean"] - mu) <= 1e-8 * max(1.0, abs(mu))
        assert abs(r["s2"] - s2) <= 1e-8 * s2
        np.testing.assert_allclose(r["best"], best, rtol=1e-7, atol=1e-12 * best.max())
        np.testing.assert_allclose(r["gaps"], gaps, rtol=1e-5, atol=1e-9)


# ------------------------------------------------------------- P7 telescoping
@pytest.mark.parametrize("seed", range(4))
def test_telescoping_variance(seed):
    """P7: v_n(x) = v_{n0}(x) - sum_j Delta_best(j), Delta >= 0 (App A.5)."""
    rng = np.random.default_rng(700 + seed)
    X = rng.random((400, 2))
    Z = X[:, 0]
    x = rng.random(2)
    d, g = 0.05, 1e-4
    n0, n = 6, 30
    r = oracle.local_design(X, Z, x, d, g, n0, n, 200)
    idx = r["idx"]
    v0 = v_of(X[idx[:n0]], x, d, g)
    vn = v_of(X[idx], x, d, g)
    assert (r["best"] >= 0).all()
    assert abs(vn - (v0 - r["best"].sum())) <= 1e-8 * v0
    # v_n from the returned s2: s2 = psi v_n / n
    K = corr(X[idx], X[idx], d) + g * np.eye(n)
    psi = Z[idx] @ np.linalg.solve(K, Z[idx])
    assert abs(r["s2"] - psi * vn / n) <= 1e-8 * r["s2"]


# ------------------------------------------------------ P9 determinism/order
def test_determinism_and_thread_invariance():
    rng = np.random.default_rng(9)
    X = rng.random((800, 3))
    Z = X.sum(1)
    XX = rng.random((16, 3))
    a = oracle.alc_batch(X, Z, XX, 0.1, 1e-4, 6, 20, 100, threads=1)
    b = oracle.alc_batch(X, Z, XX, 0.1, 1e-4, 6, 20, 100, threads=4)
    for k in ("idx", "mean", "s2", "var", "flags", "gaps", "best"):
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    # chunk composition: two halves concatenated == whole
    c1 = oracle.alc_batch(X, Z, XX[:7], 0.1, 1e-4, 6, 20, 100, threads=2)
    c2 = oracle.alc_batch(X, Z, XX[7:], 0.1, 1e-4, 6, 20, 100, threads=2)
    assert np.array_equal(np.vstack([c1["idx"], c2["idx"]]), a["idx"])
    assert np.array_equal(np.concatenate([c1["mean"], c2["mean"]]), a["mean"])


# ------------------------------------------------------- P10/P11 worked examples
def test_worked_example_WA():
    gold = json.load(open(GOLDEN))["W-A"]
    X = (np.arange(11) / 10.0)[:, None]
    Y = np.sin(2 * math.pi * X[:, 0])
    r = oracle.local_design(X, Y, np.array([0.43]), 0.1, 1e-4, 2, 5, 11)
    assert r["idx"].tolist() == gold["idx"]
    for v, ref, rt in zip(r["best"], gold["best_delta"], gold["best_delta_rtol"]):
        assert abs(v - ref) <= rt * ref
    assert np.allclose(r["gaps"], gold["gaps"], rtol=0, atol=1e-8)
    assert abs(r["mean"] - gold["mean"]) <= 1e-13
    assert abs(r["s2"] - gold["s2"]) <= 1e-10 * gold["s2"]
    assert abs(r["var"] - gold["var"]) <= 1e-10 * gold["var"]


def test_worked_example_WB():
    gold = json.load(open(GOLDEN))["W-B"]
    rng = np.random.default_rng(42)
    X = rng.random((30, 2))
    x = rng.random(2)
    Y = np.sin(5 * X[:, 0]) + np.cos(3 * X[:, 1])
    r = oracle.local_design(X, Y, x, 0.05, 1e-4, 3, 8, 30)
    assert r["idx"].tolist() == gold["idx"]
    assert oracle.nn(X, x, 8)[0].tolist() == gold["nn8"]
    assert abs(r["mean"] - gold["mean"]) <= 1e-12
    assert abs(r["s2"] - gold["s2"]) <= 1e-10 * gold["s2"]
    assert abs(r["var"] - gold["var"]) <= 1e-10 * gold["var"]
    # the greedy steps' best reductions and top-2 gaps (explicit-inverse noise: eps * cond)
    assert np.allclose(r["best"], gold["best_delta"], rtol=1e-8, atol=0)
    assert np.allclose(r["gaps"], gold["gaps"], rtol=0, atol=1e-8)


def test_worked_examples_regenerate():
    """tests/golden/worked_examples.json is what scripts/golden_worked_examples.py
    (60-digit decimal brute force, no oracle import) produces."""
    import subprocess
    import sys

    script = os.path.join(os.path.dirname(os.path.dirname(__file__)), "scripts", "golden_worked_examples.py")
    r = subprocess.run([sys.executable, script, "--check"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


# --------------------------------------------- degenerate cases (R12)
def test_exact_tie_picks_lowest_index_and_flags():
    X = np.array([[0.0], [0.1], [-0.1], [0.2], [-0.2]])
    Z = X[:, 0]
    r = oracle.local_design(X, Z, np.array([0.0]), 0.05, 1e-4, 1, 3, 5)
    assert r["idx"][:2].tolist() == [0, 1]
    assert r["gaps"][0] == 0.0
    assert r["flags"] & oracle.FLAG_NEAR_TIE


def test_exhausted_duplicates_eta0():
    X = np.array([[0.5, 0.5]] * 3)
    Z = np.array([1.0, 1.0, 1.0])
    r = oracle.local_design(X, Z, np.array([0.4, 0.5]), 0.1, 0.0, 1, 2, 3)
    assert r["idx"].tolist() == [0, -1]
    assert r["flags"] & oracle.FLAG_EXHAUSTED
    assert r["flags"] & oracle.FLAG_SENTINEL
    assert math.isnan(r["var"])  # df = j = 1 <= 2
    k = math.exp(-0.01 / 0.1)
    assert abs(r["mean"] - k * 1.0) < 1e-15
    assert abs(r["s2"] - 1.0 * (1.0 - k * k)) < 1e-15


def test_sentinel_skips_duplicate_but_continues():
    X = np.array([[0.0], [0.0], [0.3], [0.6], [0.9]])
    Z = X[:, 0]
    r = oracle.local_design(X, Z, np.array([0.05]), 0.1, 0.0, 1, 3, 5)
    assert r["flags"] & oracle.FLAG_SENTINEL
    assert not r["flags"] & oracle.FLAG_EXHAUSTED
    assert 1 not in r["idx"].tolist()


def test_score_noise_reference_pinned_to_decimal_brute_force():
    """oracle.score_noise (reading R18's tau_cfg): its long-double fresh-solve
    reference reproduces the 60-digit brute-force top-2 gaps of W-A and W-B, and
    its noise bounds the explicit-inverse error of the oracle's own best scores."""
    gold = json.load(open(GOLDEN))
    X = (np.arange(11) / 10.0)[:, None]
    Y = np.sin(2 * math.pi * X[:, 0])
    rng = np.random.default_rng(42)
    XB = rng.random((30, 2))
    xb = rng.random(2)
    YB = np.sin(5 * XB[:, 0]) + np.cos(3 * XB[:, 1])
    for key, (XS, YS, x, d, n0, n, Np) in {"W-A": (X, Y, np.array([0.43]), 0.1, 2, 5, 11),
                                            "W-B": (XB, YB, xb, 0.05, 3, 8, 30)}.items():
        r = oracle.local_design(XS, YS, x, d, 1e-4, n0, n, Np)
        noise, ref_gap = oracle.score_noise(XS, x, r["idx"], d, 1e-4, n0, n, Np)
        assert np.allclose(ref_gap, gold[key]["gaps"], rtol=0, atol=1e-12), key
        err = np.abs(r["best"] - np.array(gold[key]["best_delta"])) / np.array(gold[key]["best_delta"])
        assert (err <= noise * (1 + 1e-6) + 1e-15).all(), (key, err, noise)
        assert (noise > 0).all() and (noise < 1e-6).all()


def test_score_noise_small_when_well_conditioned():
    """With a large nugget K_j is well conditioned (kappa <= 1 + j/g, App A.6):
    the explicit-inverse scores agree with the fresh long-double solve to ~1e-13."""
    rng = np.random.default_rng(9)
    X = rng.random((200, 3))
    x = rng.random(3)
    r = oracle.local_design(X, np.zeros(200), x, 0.3, 0.5, 4, 20, 120)
    noise, gap = oracle.score_noise(X, x, r["idx"], 0.3, 0.5, 4, 20, 120)
    assert noise.max() < 1e-12
    assert np.allclose(gap, r["gaps"], rtol=0, atol=1e-12)
