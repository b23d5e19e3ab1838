"""Seeded input generators for the workloads of SURVEY.md §8d (C1–C5).

Every array is generated with ``numpy.random.default_rng(seed)`` so the oracle
and the CUDA path see bit-identical inputs. Shapes, distributions and structure
follow the paper's workloads:

* C1 — 2-d toy surface, uniform design (PAPER.md P:763-765 borrows its 2-d
  function from Gramacy–Apley and does not restate it; we use a smooth surface).
* C2/C4 — 8-d borehole on Latin hypercube designs, "different random (Latin
  hypercube) samples" for design and predictive set.
* C3 — "LGBB-shaped" 3-d anisotropic grid design (dense in dim 1, coarse in
  dim 3) with a denser cell-centred predictive grid.
* C5 — candidate-set sweep designs (uniform 2-d, LHS 8-d).

θ ("d") and η ("g") are never given for these workloads (Fig 1 step 1 only
asks for "a sensible starting global θ"). DESIGN.md reading R13 freezes
g = 1e-4 and d = the 10% quantile of squared pairwise distances over a seeded
1,000-row subsample of X (``q10_lengthscale``).
"""
from __future__ import annotations

import math

import numpy as np

# Standard borehole input ranges (Worley 1987 / Morris et al. 1993 literature
# values; the paper cites the function without restating it).
_BOREHOLE_RANGES = np.array(
    [
        [0.05, 0.15],  # rw
        [100.0, 50000.0],  # r
        [63070.0, 115600.0],  # Tu
        [990.0, 1110.0],  # Hu
        [63.1, 116.0],  # Tl
        [700.0, 820.0],  # Hl
        [1120.0, 1680.0],  # L
        [9855.0, 12045.0],  # Kw
    ]
)


def uniform(n: int, p: int, seed: int) -> np.ndarray:
    """n iid uniform points in [0,1]^p."""
    return np.random.default_rng(seed).random((n, p))


def lhs(n: int, p: int, seed: int) -> np.ndarray:
    """Random Latin hypercube in [0,1]^p: one point per stratum per axis."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, p))
    for k in range(p):
        perm = rng.permutation(n)
        out[:, k] = (perm + rng.random(n)) / n
    return out


def borehole(X: np.ndarray) -> np.ndarray:
    """Borehole water-flow function on the unit cube (affine map to the ranges)."""
    lo, hi = _BOREHOLE_RANGES[:, 0], _BOREHOLE_RANGES[:, 1]
    Z = lo + X * (hi - lo)
    rw, r, Tu, Hu, Tl, Hl, L, Kw = (Z[:, k] for k in range(8))
    lr = np.log(r / rw)
    return 2.0 * math.pi * Tu * (Hu - Hl) / (lr * (1.0 + 2.0 * L * Tu / (lr * rw * rw * Kw) + Tu / Tl))


def surface2d(X: np.ndarray) -> np.ndarray:
    """Smooth 2-d test surface for C1."""
    return np.sin(2 * math.pi * X[:, 0]) * np.cos(2 * math.pi * X[:, 1]) + X[:, 0]


def lift_surface(X: np.ndarray) -> np.ndarray:
    """LGBB-like 'lift' response: abrupt transition near 'Mach 1'."""
    return np.tanh(12.0 * (X[:, 0] - 0.2)) + 0.5 * X[:, 1] - 0.2 * X[:, 2] ** 2


def lgbb_design(shape=(117, 54, 6), jitter_seed: int | None = None) -> np.ndarray:
    """Anisotropic 3-d grid, lexicographic row order (nodes at i/(n_k-1)).

    With ``jitter_seed`` each coordinate is perturbed by U(-1e-3, 1e-3)·spacing
    (variant C3j, which removes NN-boundary distance ties).
    """
    axes = [np.linspace(0.0, 1.0, s) for s in shape]
    G = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, len(shape))
    if jitter_seed is not None:
        rng = np.random.default_rng(jitter_seed)
        sp = np.array([1.0 / (s - 1) for s in shape])
        G = G + (rng.random(G.shape) * 2.0 - 1.0) * 1e-3 * sp
    return G


def lgbb_pred_grid(shape=(250, 200, 10)) -> np.ndarray:
    """Cell-centred predictive grid, denser than the design in every dimension."""
    axes = [(np.arange(s) + 0.5) / s for s in shape]
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, len(shape))


def q10_lengthscale(X: np.ndarray, seed: int, nsub: int = 1000) -> float:
    """d = 10% quantile of squared pairwise distances over a seeded subsample."""
    rng = np.random.default_rng(seed)
    m = min(nsub, X.shape[0])
    S = X[rng.choice(X.shape[0], m, replace=False)]
    D = ((S[:, None, :] - S[None, :, :]) ** 2).sum(-1)
    iu = np.triu_indices(m, 1)
    return float(np.quantile(D[iu], 0.10))


# name -> recipe. "M" is the full predictive-set size.
CONFIGS = {
    "C1": dict(kind="uniform2d", N=4000, M=100, p=2, n0=6, n=50, Nprime=500, seedX=101, seedXX=102),
    "C2": dict(kind="borehole", N=100_000, M=10_000, p=8, n0=6, n=50, Nprime=1000, seedX=201, seedXX=202),
    "C3": dict(kind="lgbb", N=37_908, M=500_000, p=3, n0=6, n=50, Nprime=1000, seedX=None, seedXX=None),
    "C3j": dict(kind="lgbb", N=37_908, M=500_000, p=3, n0=6, n=50, Nprime=1000, seedX=301, seedXX=None),
    "C4": dict(kind="borehole", N=1_000_000, M=1_000_000, p=8, n0=6, n=50, Nprime=1000, seedX=401, seedXX=402),
    "C5_2d": dict(kind="uniform2d", N=200_000, M=4096, p=2, n0=6, n=50, Nprime=1000, seedX=501, seedXX=503),
    "C5_8d": dict(kind="borehole", N=200_000, M=4096, p=8, n0=6, n=50, Nprime=1000, seedX=502, seedXX=503),
}


def make_config(name: str, M: int | None = None, N: int | None = None, **over) -> dict:
    """Materialise a config: X (N×p), Z (N), XX (M×p), d, g, n0, n, Nprime.

    ``M``/``N`` shrink the predictive set / design for test-sized cases (XX is
    then the first M rows of the full seeded set, so sampled parity on the
    full-size run sees the same rows). Extra keys override n0/n/Nprime/d/g.
    """
    r = dict(CONFIGS[name])
    r.update({k: v for k, v in over.items() if k in ("n0", "n", "Nprime", "d", "g")})
    Nd = r["N"] if N is None else N
    Mx = r["M"] if M is None else M
    p = r["p"]
    if r["kind"] == "uniform2d":
        X = uniform(Nd, p, r["seedX"])
        XX = uniform(Mx, p, r["seedXX"])
        Z = surface2d(X)
    elif r["kind"] == "borehole":
        X = lhs(Nd, p, r["seedX"])
        # an LHS of size M is not a prefix of an LHS of size M' > M; always draw
        # the full-size predictive LHS and slice, so test subsets match the bench.
        XX = lhs(max(r["M"], Mx), p, r["seedXX"])[:Mx]
        Z = borehole(X)
    elif r["kind"] == "lgbb":
        X = lgbb_design(jitter_seed=r["seedX"])
        if N is not None:
            X = X[:Nd]
        G = lgbb_pred_grid()
        if Mx < G.shape[0]:
            # seeded subsample of the dense grid (rows in ascending order)
            sel = np.sort(np.random.default_rng(303).choice(G.shape[0], Mx, replace=False))
            G = G[sel]
        XX = G
        Z = lift_surface(X)
    else:
        raise ValueError(r["kind"])
    d = over.get("d", None)
    if d is None:
        d = q10_lengthscale(X, seed=(r["seedX"] or 300) + 7)
    g = over.get("g", 1e-4)
    return dict(
        name=name,
        X=np.ascontiguousarray(X, dtype=np.float64),
        Z=np.ascontiguousarray(Z, dtype=np.float64),
        XX=np.ascontiguousarray(XX, dtype=np.float64),
        d=float(d),
        g=float(g),
        n0=int(r["n0"]),
        n=int(r["n"]),
        Nprime=int(r["Nprime"]),
    )
