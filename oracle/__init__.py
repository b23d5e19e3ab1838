"""CPU oracle for the greedy ALC local-design path (arXiv 1310.5182).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package. The product
path (paper_1310_5182_b200) never imports it and shares no code with it.

Thin ctypes marshalling over ``oracle/liblagp_oracle.so`` (plain C in
``lagp_oracle.c``; every function there cites the passage it follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lagp_oracle.c")
_LIB = os.path.join(_HERE, "liblagp_oracle.so")

FLAG_NEAR_TIE = 1
FLAG_SENTINEL = 2
FLAG_EXHAUSTED = 4
FLAG_NONFINITE = 8
MLE_FLAG_MAXIT = 32
MLE_FLAG_BOUND = 16
MLE_FLAG_FAIL = 64


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no implicit fp contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = [
            "gcc", "-O2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
            "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm",
        ]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        D = ctypes.POINTER(ctypes.c_double)
        I32 = ctypes.POINTER(ctypes.c_int32)
        U32 = ctypes.POINTER(ctypes.c_uint32)
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.oracle_nn.argtypes = [D, i64, i32, D, ctypes.c_int32, I32, D]
        _lib.oracle_invert_spd.argtypes = [i32, D, D]
        _lib.oracle_alc_scores.argtypes = [i32, i32, i32, D, D, D, D, dbl, dbl, D, D, D]
        _lib.oracle_pinv_update.argtypes = [i32, D, D, dbl, D]
        _lib.oracle_predict.argtypes = [i32, i32, D, D, D, dbl, dbl, D, D, D]
        _lib.oracle_local_design.argtypes = [D, i64, i32, D, D, dbl, dbl, i32, i32, i32,
                                             I32, D, D, D, U32, D, D, D]
        _lib.oracle_alc_batch.argtypes = [D, i64, i32, D, D, i64, dbl, dbl, i32, i32, i32, i32,
                                          I32, D, D, D, U32, D, D, D]
        _lib.oracle_loglik.argtypes = [i32, i32, D, D, dbl, dbl, i32, D, D, D]
        _lib.oracle_mle.argtypes = [i32, i32, D, D, dbl, dbl, dbl, dbl, D, D, ctypes.POINTER(ctypes.c_int), U32]
        _lib.oracle_sep_scale.argtypes = [D, i64, i32, D, D]
        _lib.oracle_sep_scale.restype = None
        _lib.oracle_local_fit_batch.argtypes = [D, i64, i32, D, D, i64, dbl, dbl, dbl, dbl, i32, i32, i32, i32,
                                                i32, I32, D, D, D, D, U32]
        _lib.oracle_score_noise.argtypes = [D, i64, i32, D, dbl, dbl, i32, i32, i32, I32, D, D]
        for f in ("oracle_score_noise", "oracle_nn", "oracle_invert_spd", "oracle_alc_scores", "oracle_pinv_update",
                  "oracle_predict", "oracle_local_design", "oracle_alc_batch", "oracle_loglik", "oracle_mle",
                  "oracle_local_fit_batch"):
            getattr(_lib, f).restype = ctypes.c_int
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def nn(X, x, m):
    """a1: exact m nearest rows by (d², index). Returns (idx int32[m], d2[m])."""
    X, pX = _d(X)
    x, px = _d(x)
    N, p = X.shape
    idx = np.empty(m, np.int32)
    d2 = np.empty(m, np.float64)
    rc = lib().oracle_nn(pX, N, p, px, m, _p(idx, ctypes.c_int32), _p(d2, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_nn rc={rc}")
    return idx, d2


def invert_spd(A):
    A, pA = _d(A)
    n = A.shape[0]
    out = np.empty((n, n))
    rc = lib().oracle_invert_spd(n, pA, _p(out, ctypes.c_double))
    if rc:
        raise np.linalg.LinAlgError(f"oracle_invert_spd rc={rc}")
    return out


def alc_scores(Xj, Kinv, cands, x, d, g):
    """a3 diagnostic: (delta_closed_form, delta_eq5_literal, m_inv) per candidate."""
    Xj, pXj = _d(Xj)
    Kinv, pK = _d(Kinv)
    cands, pc = _d(cands)
    x, px = _d(x)
    j, p = Xj.shape
    nc = cands.shape[0]
    dcf = np.empty(nc)
    dlit = np.empty(nc)
    minv = np.empty(nc)
    rc = lib().oracle_alc_scores(j, p, nc, pXj, pK, pc, px, d, g, _p(dcf, ctypes.c_double),
                                 _p(dlit, ctypes.c_double), _p(minv, ctypes.c_double))
    if rc:
        raise RuntimeError(rc)
    return dcf, dlit, minv


def pinv_update(Kinv, k, kdiag):
    """a4: K_{j+1}^{-1} from K_j^{-1}, k = k_j(x_new), kdiag = K(x_new,x_new)+eta."""
    Kinv, pK = _d(Kinv)
    k, pk = _d(k)
    j = Kinv.shape[0]
    out = np.empty((j + 1, j + 1))
    rc = lib().oracle_pinv_update(j, pK, pk, kdiag, _p(out, ctypes.c_double))
    return out, rc


def predict(Xn, Yn, x, d, g):
    """a5: (mean, s2, var) from a fresh Cholesky of K_n."""
    Xn, pX = _d(Xn)
    Yn, pY = _d(Yn)
    x, px = _d(x)
    n, p = Xn.shape
    m, s, v = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    rc = lib().oracle_predict(n, p, pX, pY, px, d, g, ctypes.byref(m), ctypes.byref(s), ctypes.byref(v))
    if rc:
        raise np.linalg.LinAlgError(f"oracle_predict rc={rc}")
    return m.value, s.value, v.value


def alc_batch(X, Z, XX, d, g, n0, n, Nprime, threads=0):
    """Full path for every row of XX (OpenMP over locations)."""
    X, pX = _d(X)
    Z, pZ = _d(Z)
    XX, pXX = _d(np.atleast_2d(XX))
    N, p = X.shape
    M = XX.shape[0]
    G = n - n0
    idx = np.empty((M, n), np.int32)
    mean = np.empty(M)
    s2 = np.empty(M)
    var = np.empty(M)
    flags = np.empty(M, np.uint32)
    gaps = np.empty((M, G))
    best = np.empty((M, G))
    s2acc = np.empty(M)
    used = lib().oracle_alc_batch(
        pX, N, p, pZ, pXX, M, d, g, n0, n, Nprime, threads,
        _p(idx, ctypes.c_int32), _p(mean, ctypes.c_double), _p(s2, ctypes.c_double),
        _p(var, ctypes.c_double), _p(flags, ctypes.c_uint32), _p(gaps, ctypes.c_double),
        _p(best, ctypes.c_double), _p(s2acc, ctypes.c_double))
    return dict(idx=idx, mean=mean, s2=s2, var=var, flags=flags, gaps=gaps, best=best,
                s2_acc=s2acc, threads=used)


def score_noise(X, x, idx, d, g, n0, n, Nprime):
    """Reading R18 (tau_cfg): along the oracle's own trajectory idx[n] for x, the
    per-step max |Delta_explicit - Delta_ref| / max Delta_ref between the oracle's
    explicit-K^{-1} scores and a fresh long-double solve of the same Eq (5)
    closed form, and the reference top-2 gap. Returns (noise, ref_gap), each
    [n - n0] (NaN after an exhaustion)."""
    X, pX = _d(X)
    x, px = _d(np.ravel(x))
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    N, p = X.shape
    noise = np.empty(n - n0)
    gap = np.empty(n - n0)
    rc = lib().oracle_score_noise(pX, N, p, px, d, g, n0, n, Nprime, _p(idx, ctypes.c_int32),
                                  _p(noise, ctypes.c_double), _p(gap, ctypes.c_double))
    if rc:
        raise RuntimeError(f"oracle_score_noise rc={rc}")
    return noise, gap


def sep_scale(X, theta):
    """Row f3: x~_k = x_k / sqrt(theta_k) (oracle_sep_scale), so that the separable
    correlation exp(-sum_k (x_k - x'_k)^2 / theta_k) is exp(-||x~ - x~'||^2)."""
    X, pX = _d(np.atleast_2d(X))
    th, pth = _d(np.asarray(theta, dtype=np.float64).ravel())
    N, p = X.shape
    if th.shape[0] != p or not np.all(th > 0):
        raise ValueError("theta must hold p positive lengthscales")
    out = np.empty_like(X)
    lib().oracle_sep_scale(pX, N, p, pth, _p(out, ctypes.c_double))
    return out


def alc_batch_sep(X, Z, XX, theta, g, n0, n, Nprime, threads=0):
    """Row f3: the full path (a1-a5) under the separable correlation with
    lengthscales theta[p]: the isotropic path with d = 1 on the rescaled inputs."""
    return alc_batch(sep_scale(X, theta), Z, sep_scale(XX, theta), 1.0, g, n0, n, Nprime, threads=threads)


def local_design(X, Z, x, d, g, n0, n, Nprime):
    r = alc_batch(X, Z, np.atleast_2d(x), d, g, n0, n, Nprime, threads=1)
    return {k: (v[0] if isinstance(v, np.ndarray) else v) for k, v in r.items()}


def loglik(Xn, Yn, d, g, deriv=True):
    """Eq (3) log likelihood on (Xn, Yn) and, with deriv, its first and second
    derivatives in tau = log(theta) (reading R20). Returns (l, dl, d2l); l = -inf
    when K is not SPD or psi <= 0."""
    Xn, pX = _d(np.atleast_2d(Xn))
    Yn, pY = _d(Yn)
    n, p = Xn.shape
    l, dl, d2l = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().oracle_loglik(n, p, pX, pY, d, g, 1 if deriv else 0, ctypes.byref(l), ctypes.byref(dl), ctypes.byref(d2l))
    return l.value, dl.value, d2l.value


def mle(Xn, Yn, d0, lo, hi, g):
    """Fig 1 step 3: theta-hat on (Xn, Yn) by the safeguarded Newton of reading
    R21. Returns (theta_hat, l(theta_hat), iterations, flags)."""
    Xn, pX = _d(np.atleast_2d(Xn))
    Yn, pY = _d(Yn)
    n, p = Xn.shape
    th, lh, it, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_int(), ctypes.c_uint32()
    lib().oracle_mle(n, p, pX, pY, d0, lo, hi, g, ctypes.byref(th), ctypes.byref(lh), ctypes.byref(it),
                     ctypes.byref(fl))
    return th.value, lh.value, it.value, fl.value


def local_fit(X, Z, XX, d0, lo, hi, g, n0, n, Nprime, stages=2, threads=0):
    """Fig 1 steps 1-5 (multi-stage: design, MLE, repeat, predict) for every row
    of XX. theta is stages x M (theta_x after each stage)."""
    if not 1 <= stages <= 16:
        raise ValueError("stages must be in [1, 16]")
    X, pX = _d(X)
    Z, pZ = _d(Z)
    XX, pXX = _d(np.atleast_2d(XX))
    N, p = X.shape
    M = XX.shape[0]
    idx = np.empty((M, n), np.int32)
    theta = np.empty((stages, M))
    mean = np.empty(M)
    s2 = np.empty(M)
    var = np.empty(M)
    flags = np.empty(M, np.uint32)
    used = lib().oracle_local_fit_batch(
        pX, N, p, pZ, pXX, M, d0, lo, hi, g, n0, n, Nprime, stages, threads,
        _p(idx, ctypes.c_int32), _p(theta, ctypes.c_double), _p(mean, ctypes.c_double),
        _p(s2, ctypes.c_double), _p(var, ctypes.c_double), _p(flags, ctypes.c_uint32))
    return dict(idx=idx, theta=theta, mean=mean, s2=s2, var=var, flags=flags, threads=used)
