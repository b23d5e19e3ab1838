"""Pins for the row-f2 oracle (local MLE + multi-stage scheme, Fig 1 steps 3-4).

Every check compares the oracle with something other than itself: an
independent numpy evaluation of Eq (3) (slogdet + solve + lgamma), a worked
example, exact scaling identities, finite differences of the
numpy likelihood, a brute-force grid scan for the maximiser, and seeded GP
sample paths with a known lengthscale (statistical).
"""
import math

import numpy as np
import pytest

import oracle
from lagp_data import make_config


def np_loglik(X, Y, theta, eta):
    """Eq (3) evaluated independently: slogdet and a dense solve."""
    X = np.atleast_2d(X)
    n = X.shape[0]
    D = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    K = np.exp(-D / theta) + eta * np.eye(n)
    sign, logdet = np.linalg.slogdet(K)
    assert sign > 0
    psi = Y @ np.linalg.solve(K, Y)
    return math.lgamma(n / 2) - n / 2 * math.log(2 * math.pi) - 0.5 * logdet - n / 2 * math.log(psi / 2)


def data(seed, n=30, p=2):
    rng = np.random.default_rng(seed)
    X = rng.random((n, p))
    Y = np.sin(4 * X[:, 0]) + np.cos(3 * X[:, -1]) + 0.05 * rng.standard_normal(n)
    return X, Y


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("theta", [0.03, 0.2, 1.5])
def test_loglik_matches_direct_eq3(seed, theta):
    X, Y = data(seed, n=10 + 7 * seed, p=1 + seed % 3)
    l, _, _ = oracle.loglik(X, Y, theta, 1e-3)
    assert l == pytest.approx(np_loglik(X, Y, theta, 1e-3), rel=1e-10, abs=1e-10)


def test_loglik_worked_example_n1():
    # N=1, K=[[1]], y=sqrt(2) -> psi=2 -> l = -1/2 log 2
    l, _, _ = oracle.loglik(np.zeros((1, 2)), np.array([math.sqrt(2.0)]), 0.7, 0.0)
    assert l == pytest.approx(-0.5 * math.log(2.0), abs=1e-15)


@pytest.mark.parametrize("c", [2.0, 0.25, 8.0])
def test_loglik_response_scaling(c):
    # psi scales by c^2 -> l changes by -(n/2) log(c^2) exactly (powers of two: exact psi scaling)
    X, Y = data(3, n=25)
    l1, g1, h1 = oracle.loglik(X, Y, 0.3, 1e-4)
    l2, g2, h2 = oracle.loglik(X, c * Y, 0.3, 1e-4)
    assert l2 == pytest.approx(l1 - 25 / 2 * math.log(c * c), rel=1e-13, abs=1e-12)
    assert g2 == pytest.approx(g1, rel=1e-12, abs=1e-12)  # derivatives do not see the scale
    assert h2 == pytest.approx(h1, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("seed", range(8))
def test_gradient_matches_finite_differences(seed):
    # R20: dl/dtau against a central difference of the independent numpy l(exp(tau))
    X, Y = data(seed, n=12 + 4 * seed, p=1 + seed % 4)
    for theta in (0.05, 0.3, 2.0):
        _, g, h = oracle.loglik(X, Y, theta, 1e-3)
        t, d = math.log(theta), 1e-5
        fd = (np_loglik(X, Y, math.exp(t + d), 1e-3) - np_loglik(X, Y, math.exp(t - d), 1e-3)) / (2 * d)
        assert g == pytest.approx(fd, rel=1e-6, abs=1e-6)
        d2 = 2e-4
        fd2 = (np_loglik(X, Y, math.exp(t + d2), 1e-3) - 2 * np_loglik(X, Y, theta, 1e-3)
               + np_loglik(X, Y, math.exp(t - d2), 1e-3)) / d2 ** 2
        assert h == pytest.approx(fd2, rel=2e-4, abs=2e-4)


@pytest.mark.parametrize("seed", range(6))
def test_mle_is_the_grid_maximiser(seed):
    X, Y = data(seed, n=20 + 5 * seed, p=2)
    lo, hi, eta = 1e-3, 10.0, 1e-4
    th, lh, its, fl = oracle.mle(X, Y, 0.5, lo, hi, eta)
    assert lo <= th <= hi
    taus = np.linspace(math.log(lo), math.log(hi), 2001)
    grid = np.array([np_loglik(X, Y, math.exp(t), eta) for t in taus])
    assert lh == pytest.approx(np_loglik(X, Y, th, eta), rel=1e-10, abs=1e-10)
    assert lh >= grid.max() - 1e-9  # no grid point beats theta-hat
    if not fl & oracle.MLE_FLAG_BOUND:
        _, g, h = oracle.loglik(X, Y, th, eta)
        assert abs(g) <= 1e-7 * (1 + abs(lh))  # interior stationary point
        assert h < 0


def test_mle_postcondition_start_not_worse():
    for seed in range(10):
        X, Y = data(100 + seed, n=25, p=3)
        for t0 in (0.01, 0.3, 5.0):
            th, lh, _, _ = oracle.mle(X, Y, t0, 1e-3, 10.0, 1e-4)
            assert lh >= np_loglik(X, Y, t0, 1e-4) - 1e-12


def test_mle_flat_response_ends_on_a_bound():
    # constant Y with eta > 0 terminates at a boundary without error
    rng = np.random.default_rng(5)
    X = rng.random((20, 2))
    th, lh, its, fl = oracle.mle(X, np.full(20, 3.0), 0.2, 1e-3, 10.0, 1e-3)
    assert fl & oracle.MLE_FLAG_BOUND
    assert th == pytest.approx(10.0, rel=1e-12) or th == pytest.approx(1e-3, rel=1e-12)
    assert np.isfinite(lh)


def test_mle_recovers_gp_lengthscale():
    # SPEC S:101 (statistical, seeded): sample paths with theta = 0.5, N = 100, p = 1
    est = []
    for seed in range(20):
        rng = np.random.default_rng(1000 + seed)
        X = rng.random((100, 1))
        K = np.exp(-((X - X.T) ** 2) / 0.5) + 1e-6 * np.eye(100)
        Y = np.linalg.cholesky(K) @ rng.standard_normal(100)
        est.append(oracle.mle(X, Y, 0.1, 1e-3, 10.0, 1e-6)[0])
    assert 0.25 <= float(np.median(est)) <= 1.0


def test_local_fit_is_the_composition():
    # Fig 1: stage s = design with theta_x, then MLE started at theta_x; the
    # prediction uses the final theta on the last design
    cfg = make_config("C1", M=3)
    d0, lo, hi = cfg["d"], cfg["d"] / 100, cfg["d"] * 10
    fit = oracle.local_fit(cfg["X"], cfg["Z"], cfg["XX"], d0, lo, hi, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"],
                           stages=2)
    for i in range(3):
        th = d0
        for s in range(2):
            des = oracle.local_design(cfg["X"], cfg["Z"], cfg["XX"][i], th, cfg["g"], cfg["n0"], cfg["n"],
                                      cfg["Nprime"])
            ix = des["idx"]
            th = oracle.mle(cfg["X"][ix], cfg["Z"][ix], th, lo, hi, cfg["g"])[0]
            assert fit["theta"][s, i] == th
        assert (fit["idx"][i] == ix).all()
        m, s2, v = oracle.predict(cfg["X"][ix], cfg["Z"][ix], cfg["XX"][i], th, cfg["g"])
        assert (fit["mean"][i], fit["s2"][i], fit["var"][i]) == (m, s2, v)


def test_local_fit_stage_improves_likelihood():
    # l(theta-hat) on the stage's design >= l(incoming theta)
    cfg = make_config("C1", M=4)
    d0, lo, hi = cfg["d"], cfg["d"] / 100, cfg["d"] * 10
    for i in range(4):
        des = oracle.local_design(cfg["X"], cfg["Z"], cfg["XX"][i], d0, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
        Xn, Yn = cfg["X"][des["idx"]], cfg["Z"][des["idx"]]
        th, lh, _, _ = oracle.mle(Xn, Yn, d0, lo, hi, cfg["g"])
        assert lh >= np_loglik(Xn, Yn, d0, cfg["g"]) - 1e-12
