"""Pins for row f3 of the oracle: separable lengthscales ("a separable
version via a vectorized theta parameter"; reading R23).

The oracle evaluates K(x, x') = exp(-sum_k (x_k - x'_k)^2 / theta_k) as the
isotropic correlation with theta = 1 on rescaled inputs x~_k = x_k / sqrt(theta_k)
(oracle.sep_scale). These tests check it against things other than itself: the
direct weighted-distance formula (numpy), a definition-level brute force of the
greedy criterion (fresh dense solves) built on that direct formula, the
isotropic special case, invariance under rescaling an input and its lengthscale
together, and an irrelevant dimension (theta_k -> infinity).
"""
import numpy as np
import pytest

import oracle


def sep_corr(A, B, theta):
    """K(a, b) = exp(-sum_k (a_k - b_k)^2 / theta_k), straight from the definition."""
    A = np.atleast_2d(A)
    B = np.atleast_2d(B)
    D = (((A[:, None, :] - B[None, :, :]) ** 2) / np.asarray(theta)[None, None, :]).sum(-1)
    return np.exp(-D)


def v_sep(XS, x, theta, g):
    if len(XS) == 0:
        return 1.0 + g
    K = sep_corr(XS, XS, theta) + g * np.eye(len(XS))
    k = sep_corr(XS, x, theta)[:, 0]
    return 1.0 + g - k @ np.linalg.solve(K, k)


def brute_greedy_sep(X, Z, x, theta, g, n0, n, Nprime):
    """Fig 1 step 2 by definition under the separable correlation: pool = N'
    nearest by the weighted distance, then argmax_c v_j(x) - v_{j+1}(x)."""
    w = ((X - x) ** 2 / np.asarray(theta)).sum(1)
    pool = np.lexsort((np.arange(len(X)), w))[:Nprime]
    chosen = [int(i) for i in pool[:n0]]
    gaps = []
    for _ in range(n0, n):
        vj = v_sep(X[chosen], x, theta, g)
        sc = sorted(((vj - v_sep(X[chosen + [int(c)]], x, theta, g), -int(c)) for c in pool if int(c) not in chosen),
                    reverse=True)
        d1, c1 = sc[0]
        d2 = sc[1][0] if len(sc) > 1 else 0.0
        gaps.append((d1 - max(d2, 0.0)) / d1)
        chosen.append(-c1)
    XS = X[chosen]
    K = sep_corr(XS, XS, theta) + g * np.eye(len(chosen))
    h = sep_corr(XS, x, theta)[:, 0]
    Y = Z[chosen]
    b = np.linalg.solve(K, Y)
    mu = h @ b
    s2 = (Y @ b) * (1 + g - h @ np.linalg.solve(K, h)) / len(chosen)
    return np.array(chosen), mu, s2, np.array(gaps)


def test_sep_correlation_matches_definition():
    rng = np.random.default_rng(3)
    for p in (1, 2, 3, 8):
        th = np.exp(rng.uniform(np.log(0.01), np.log(5.0), p))
        A, B = rng.random((40, p)), rng.random((30, p))
        As, Bs = oracle.sep_scale(A, th), oracle.sep_scale(B, th)
        K_iso = np.exp(-(((As[:, None, :] - Bs[None, :, :]) ** 2).sum(-1)))
        np.testing.assert_allclose(K_iso, sep_corr(A, B, th), rtol=1e-13, atol=1e-300)


def test_sep_scale_rejects_bad_theta():
    with pytest.raises(ValueError):
        oracle.sep_scale(np.zeros((3, 2)), [1.0])
    with pytest.raises(ValueError):
        oracle.sep_scale(np.zeros((3, 2)), [1.0, 0.0])


@pytest.mark.parametrize("seed", range(10))
def test_sep_greedy_equals_bruteforce_definition(seed):
    rng = np.random.default_rng(900 + seed)
    p = int(rng.integers(2, 5))
    N = int(rng.integers(25, 60))
    X = rng.random((N, p))
    Z = np.sin(4 * X[:, 0]) + X[:, -1] ** 2
    x = rng.random(p)
    th = np.exp(rng.uniform(np.log(0.03), np.log(2.0), p))
    n0 = int(rng.integers(1, 4))
    n = n0 + int(rng.integers(2, 8))
    Nprime = int(rng.integers(n + 1, N + 1))
    g = 1e-3
    r = oracle.alc_batch_sep(X, Z, x[None, :], th, g, n0, n, Nprime, threads=1)
    idx, mu, s2, gaps = brute_greedy_sep(X, Z, x, th, g, n0, n, Nprime)
    for t in range(n):
        if t >= n0 and gaps[t - n0] < 1e-9:
            return  # near tie at roundoff level: trajectories may legitimately part
        assert r["idx"][0][t] == idx[t], (t, r["idx"][0], idx)
    assert abs(r["mean"][0] - mu) <= 1e-8 * max(1.0, abs(mu))
    assert abs(r["s2"][0] - s2) <= 1e-8 * s2


def _problem(seed, N=400, M=6, p=3):
    rng = np.random.default_rng(seed)
    X = rng.random((N, p))
    Z = np.cos(3 * X).sum(1) + X[:, 0]
    XX = rng.random((M, p))
    return X, Z, XX


def test_sep_equal_lengthscales_is_isotropic():
    X, Z, XX = _problem(11)
    th = 0.07
    a = oracle.alc_batch_sep(X, Z, XX, [th] * 3, 1e-4, 6, 24, 120)
    b = oracle.alc_batch(X, Z, XX, th, 1e-4, 6, 24, 120)
    same = (a["idx"] == b["idx"]).all(1)
    assert same.sum() >= len(same) - 1
    np.testing.assert_allclose(a["mean"][same], b["mean"][same], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(a["s2"][same], b["s2"][same], rtol=1e-9)


def test_sep_rescaling_invariance():
    """Scaling input k by c and theta_k by c^2 leaves the correlation unchanged."""
    X, Z, XX = _problem(12)
    th = np.array([0.05, 0.3, 0.12])
    c = np.array([1.0, 4.0, 0.25])
    a = oracle.alc_batch_sep(X, Z, XX, th, 1e-4, 6, 24, 120)
    b = oracle.alc_batch_sep(X * c, Z, XX * c, th * c * c, 1e-4, 6, 24, 120)
    same = (a["idx"] == b["idx"]).all(1)
    assert same.sum() >= len(same) - 1
    np.testing.assert_allclose(a["mean"][same], b["mean"][same], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(a["s2"][same], b["s2"][same], rtol=1e-9)


def test_sep_irrelevant_dimension():
    """theta_k -> infinity removes input k: the p+1-dim problem equals the p-dim one."""
    X, Z, XX = _problem(13)
    rng = np.random.default_rng(5)
    th = np.array([0.05, 0.3, 0.12])
    X1 = np.hstack([X, rng.random((X.shape[0], 1))])
    XX1 = np.hstack([XX, rng.random((XX.shape[0], 1))])
    a = oracle.alc_batch_sep(X, Z, XX, th, 1e-4, 6, 24, 120)
    b = oracle.alc_batch_sep(X1, Z, XX1, np.append(th, 1e30), 1e-4, 6, 24, 120)
    np.testing.assert_array_equal(a["idx"], b["idx"])
    np.testing.assert_allclose(a["mean"], b["mean"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(a["s2"], b["s2"], rtol=1e-12)
