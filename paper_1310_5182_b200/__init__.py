"""laGP on B200 — the greedy ALC local-design hot path of Gramacy, Niemi & Weiss,
"Massively parallel approximate Gaussian process regression" (arXiv 1310.5182).

Thin Python binding over the C ABI in ``include/lagp.h`` (``liblagp_b200.so``,
hand-written sm_100a CUDA). Every step of the path runs in the library's
kernels; this module only checks and marshals torch CUDA tensors (device memory,
the current stream) and, for ``alc_batch_dist``, uses torch.distributed for the
one collective (an all-gather of per-location results).

Names follow the paper: X (design), Z (responses), XX (predictive set 𝒳),
d = θ (lengthscale), g = η (nugget), n0, n, Nprime = N′.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import (  # noqa: F401
    ALC_AUTO,
    ALC_EXPLICIT,
    ALC_INCREMENTAL,
    FLAG_EXHAUSTED,
    FLAG_MLE_BOUND,
    FLAG_MLE_FAIL,
    FLAG_MLE_MAXIT,
    FLAG_NEAR_TIE,
    FLAG_NONFINITE,
    FLAG_SENTINEL,
    LAGP_EINVAL,
    LAGP_OK,
    LAGP_PARTIAL,
    NMAX,
    PMAX,
    Timing,
)

_LIB = None

FORMS = {"explicit": ALC_EXPLICIT, "incremental": ALC_INCREMENTAL, "explicit_dfma": _lib.ALC_EXPLICIT_DFMA,
         "auto": ALC_AUTO}


class LagpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"lagp status {status}: {msg}")
        self.status = status


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = _lib.load()
    return _LIB


def last_error() -> str:
    return lib().lagp_last_error().decode()


def abi_version() -> int:
    return lib().lagp_abi_version()


def release_workspace():
    """lagp_release_workspace: return the library's cached workspace memory on the
    current device to the driver."""
    _check(lib().lagp_release_workspace())


def _check(st: int, ok=(LAGP_OK,)):
    if st not in ok:
        raise LagpError(st, last_error())
    return st


def _dev(t: torch.Tensor, name: str, dtype=torch.float64) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype} (got {t.dtype})")
    return t.contiguous()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def alc_batch(X, Z, XX, d, g, n0, n, Nprime, form="auto", gaps=False, timing=False, out=None, theta=None):
    """laGP_alc_batch_ex on CUDA tensors. Returns a dict with idx [M×n] int32,
    mean, s2, var [M] float64, flags [M] int32 (uint32 bits), optionally
    gaps [M×(n-n0)] and the phase timing, plus ``status`` (OK or PARTIAL).
    ``form="auto"`` is laGP_alc_batch's choice (the incremental form where it
    applies, else the paper's explicit form); the timing names the form that ran.
    With ``theta`` (CUDA float64 [M]) every location uses its own lengthscale
    (laGP_alc_batch_theta); ``d`` is then only validated."""
    X = _dev(X, "X")
    Z = _dev(Z, "Z")
    XX = _dev(XX, "XX")
    dev = X.device
    N, p = X.shape
    M = XX.shape[0]
    if out is None:
        out = dict(
            idx=torch.empty((M, n), dtype=torch.int32, device=dev),
            mean=torch.empty(M, dtype=torch.float64, device=dev),
            s2=torch.empty(M, dtype=torch.float64, device=dev),
            var=torch.empty(M, dtype=torch.float64, device=dev),
            flags=torch.empty(M, dtype=torch.int32, device=dev),
        )
        if gaps:
            out["gaps"] = torch.empty((M, n - n0), dtype=torch.float64, device=dev)
    tm = Timing()
    if theta is None and form == "auto" and not timing:
        # the north_star entry point itself (LAGP_ALC_AUTO inside)
        st = lib().laGP_alc_batch(
            _ptr(X), N, p, _ptr(Z), _ptr(XX), M, float(d), float(g), int(n0), int(n), int(Nprime),
            _ptr(out["idx"]), _ptr(out["mean"]), _ptr(out["s2"]), _ptr(out["var"]), _ptr(out["flags"]),
            _ptr(out.get("gaps")), _stream(dev))
    elif theta is None:
        st = lib().laGP_alc_batch_ex(
            _ptr(X), N, p, _ptr(Z), _ptr(XX), M, float(d), float(g), int(n0), int(n), int(Nprime),
            _ptr(out["idx"]), _ptr(out["mean"]), _ptr(out["s2"]), _ptr(out["var"]), _ptr(out["flags"]),
            _ptr(out.get("gaps")), FORMS[form], ctypes.byref(tm) if timing else None, _stream(dev))
    else:
        theta = _dev(theta, "theta")
        if theta.shape != (M,):
            raise ValueError(f"theta must have shape ({M},)")
        st = lib().laGP_alc_batch_theta(
            _ptr(X), N, p, _ptr(Z), _ptr(XX), M, _ptr(theta), float(d), float(g), int(n0), int(n), int(Nprime),
            _ptr(out["idx"]), _ptr(out["mean"]), _ptr(out["s2"]), _ptr(out["var"]), _ptr(out["flags"]),
            _ptr(out.get("gaps")), FORMS[form], ctypes.byref(tm) if timing else None, _stream(dev))
    _check(st, (LAGP_OK, LAGP_PARTIAL))
    out["status"] = st
    if timing:
        out["timing"] = tm.as_dict()
    return out


def alc_batch_sep(X, Z, XX, theta, g, n0, n, Nprime, form="auto", gaps=False, timing=False):
    """laGP_alc_batch_sep (row f3): the full path under the separable correlation
    exp(-sum_k (x_k - x'_k)^2 / theta_k); ``theta`` is a sequence of p floats (host)."""
    X = _dev(X, "X")
    Z = _dev(Z, "Z")
    XX = _dev(XX, "XX")
    dev = X.device
    N, p = X.shape
    M = XX.shape[0]
    if len(theta) != p:
        raise ValueError(f"theta must hold p={p} lengthscales")
    th = (ctypes.c_double * p)(*[float(v) for v in theta])
    out = dict(idx=torch.empty((M, n), dtype=torch.int32, device=dev),
               mean=torch.empty(M, dtype=torch.float64, device=dev),
               s2=torch.empty(M, dtype=torch.float64, device=dev),
               var=torch.empty(M, dtype=torch.float64, device=dev),
               flags=torch.empty(M, dtype=torch.int32, device=dev))
    if gaps:
        out["gaps"] = torch.empty((M, n - n0), dtype=torch.float64, device=dev)
    tm = Timing()
    st = lib().laGP_alc_batch_sep(
        _ptr(X), N, p, _ptr(Z), _ptr(XX), M, th, float(g), int(n0), int(n), int(Nprime),
        _ptr(out["idx"]), _ptr(out["mean"]), _ptr(out["s2"]), _ptr(out["var"]), _ptr(out["flags"]),
        _ptr(out.get("gaps")), FORMS[form], ctypes.byref(tm) if timing else None, _stream(dev))
    _check(st, (LAGP_OK, LAGP_PARTIAL))
    out["status"] = st
    if timing:
        out["timing"] = tm.as_dict()
    return out


def mle(X, Z, XX, idx, d0, lo, hi, g, theta_in=None):
    """laGP_mle (row f2, Fig 1 step 3 + step 5): theta-hat of every local design
    idx [M×n] (CUDA int32) started at theta_in [M] (or d0), inside [lo, hi]; and
    the prediction at theta-hat. Returns theta, loglik, iters, flags, mean, s2, var."""
    X = _dev(X, "X")
    Z = _dev(Z, "Z")
    XX = _dev(XX, "XX")
    idx = _dev(idx, "idx", torch.int32)
    dev = X.device
    N, p = X.shape
    M, n = idx.shape
    if theta_in is not None:
        theta_in = _dev(theta_in, "theta_in")
    f64 = dict(dtype=torch.float64, device=dev)
    out = dict(theta=torch.empty(M, **f64), loglik=torch.empty(M, **f64),
               iters=torch.empty(M, dtype=torch.int32, device=dev),
               flags=torch.zeros(M, dtype=torch.int32, device=dev),
               mean=torch.empty(M, **f64), s2=torch.empty(M, **f64), var=torch.empty(M, **f64))
    st = lib().laGP_mle(_ptr(X), N, p, _ptr(Z), _ptr(XX), M, _ptr(idx), n, _ptr(theta_in), float(d0), float(lo),
                        float(hi), float(g), _ptr(out["theta"]), _ptr(out["loglik"]), _ptr(out["iters"]),
                        _ptr(out["flags"]), _ptr(out["mean"]), _ptr(out["s2"]), _ptr(out["var"]), _stream(dev))
    _check(st, (LAGP_OK, LAGP_PARTIAL))
    out["status"] = st
    return out


def local_fit(X, Z, XX, d0, lo, hi, g, n0, n, Nprime, stages=2, form="auto", timing=False):
    """laGP_local_fit (Fig 1 steps 1-5): NN pool once, then ``stages`` times
    {local design with theta_x, theta_x = MLE}, then the prediction. Returns idx
    (last design), theta [stages×M], mean, s2, var, flags, status (+ timing)."""
    X = _dev(X, "X")
    Z = _dev(Z, "Z")
    XX = _dev(XX, "XX")
    dev = X.device
    N, p = X.shape
    M = XX.shape[0]
    f64 = dict(dtype=torch.float64, device=dev)
    out = dict(idx=torch.empty((M, n), dtype=torch.int32, device=dev), theta=torch.empty((stages, M), **f64),
               mean=torch.empty(M, **f64), s2=torch.empty(M, **f64), var=torch.empty(M, **f64),
               flags=torch.empty(M, dtype=torch.int32, device=dev))
    tm = Timing()
    st = lib().laGP_local_fit(_ptr(X), N, p, _ptr(Z), _ptr(XX), M, float(d0), float(lo), float(hi), float(g),
                              int(n0), int(n), int(Nprime), int(stages), FORMS[form], _ptr(out["idx"]),
                              _ptr(out["theta"]), _ptr(out["mean"]), _ptr(out["s2"]), _ptr(out["var"]),
                              _ptr(out["flags"]), ctypes.byref(tm) if timing else None, _stream(dev))
    _check(st, (LAGP_OK, LAGP_PARTIAL))
    out["status"] = st
    if timing:
        out["timing"] = tm.as_dict()
    return out


def alc_batch_host(X, Z, XX, d, g, n0, n, Nprime, form="auto", out=None, device=None):
    """laGP_alc_batch_host: numpy (ideally pinned-backed) host arrays in and out;
    the host<->device copies happen inside the call (end-to-end API)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    XX = np.ascontiguousarray(XX, dtype=np.float64)
    N, p = X.shape
    M = XX.shape[0]
    if out is None:
        out = dict(idx=np.empty((M, n), np.int32), mean=np.empty(M), s2=np.empty(M), var=np.empty(M),
                   flags=np.empty(M, np.uint32))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    pp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = lib().laGP_alc_batch_host(
        pp(X), N, p, pp(Z), pp(XX), M, float(d), float(g), int(n0), int(n), int(Nprime),
        pp(out["idx"]), pp(out["mean"]), pp(out["s2"]), pp(out["var"]), pp(out["flags"]), None,
        FORMS[form], _stream(dev))
    _check(st, (LAGP_OK, LAGP_PARTIAL))
    out["status"] = st
    return out


def nn_pool(X, XX, Nprime, with_d2=False):
    """laGP_nn_pool: [M×Nprime] int32 pool sorted by (d^2, index) (+ d^2)."""
    X = _dev(X, "X")
    XX = _dev(XX, "XX")
    N, p = X.shape
    M = XX.shape[0]
    pool = torch.empty((M, Nprime), dtype=torch.int32, device=X.device)
    d2 = torch.empty((M, Nprime), dtype=torch.float64, device=X.device) if with_d2 else None
    _check(lib().laGP_nn_pool(_ptr(X), N, p, _ptr(XX), M, int(Nprime), _ptr(pool), _ptr(d2), _stream(X.device)))
    return (pool, d2) if with_d2 else pool


def alc_scores(Xj, Kinv, cands, cand_idx, x, d, g):
    """laGP_alc_scores (batched Fig 2 I/O): Xj [B×j×p], Kinv [B×j×j], cands
    [B×nc×p], cand_idx [B×nc] int32, x [B×p] -> (delta [B×nc], best [B], gap [B])."""
    Xj, Kinv, cands, x = (_dev(t, nm) for t, nm in ((Xj, "Xj"), (Kinv, "Kinv"), (cands, "cands"), (x, "x")))
    cand_idx = _dev(cand_idx, "cand_idx", torch.int32)
    B, j, p = Xj.shape
    nc = cands.shape[1]
    dev = Xj.device
    delta = torch.empty((B, nc), dtype=torch.float64, device=dev)
    best = torch.empty(B, dtype=torch.int32, device=dev)
    gap = torch.empty(B, dtype=torch.float64, device=dev)
    _check(lib().laGP_alc_scores(B, j, p, nc, _ptr(Xj), _ptr(Kinv), _ptr(cands), _ptr(cand_idx), _ptr(x),
                                 float(d), float(g), _ptr(delta), _ptr(best), _ptr(gap), _stream(dev)))
    return delta, best, gap


def pinv_update(Kinv, k, kdiag):
    """laGP_pinv_update: K_{j+1}^{-1} [B×(j+1)×(j+1)] from K_j^{-1} [B×j×j], k [B×j]."""
    Kinv = _dev(Kinv, "Kinv")
    k = _dev(k, "k")
    B, j, _ = Kinv.shape
    out = torch.empty((B, j + 1, j + 1), dtype=torch.float64, device=Kinv.device)
    _check(lib().laGP_pinv_update(B, j, _ptr(Kinv), _ptr(k), float(kdiag), _ptr(out), _stream(Kinv.device)))
    return out


def predict(Xn, Yn, x, d, g):
    """laGP_predict: Xn [B×n×p], Yn [B×n], x [B×p] -> (mean, s2, var) [B]."""
    Xn, Yn, x = _dev(Xn, "Xn"), _dev(Yn, "Yn"), _dev(x, "x")
    B, n, p = Xn.shape
    dev = Xn.device
    mean = torch.empty(B, dtype=torch.float64, device=dev)
    s2 = torch.empty(B, dtype=torch.float64, device=dev)
    var = torch.empty(B, dtype=torch.float64, device=dev)
    _check(lib().laGP_predict(B, n, p, _ptr(Xn), _ptr(Yn), _ptr(x), float(d), float(g), _ptr(mean), _ptr(s2),
                              _ptr(var), _stream(dev)))
    return mean, s2, var


def exp_nonpos(x):
    """laGP_exp_nonpos: the incremental kernels' exp for x <= 0, elementwise on a CUDA tensor."""
    x = _dev(x, "x").contiguous()
    y = torch.empty_like(x)
    _check(lib().laGP_exp_nonpos(_ptr(x), _ptr(y), x.numel(), _stream(x.device)))
    return y


def shard_bounds(M: int, rank: int, world: int):
    """Rank r of R gets rows [r*ceil(M/R), min(M, (r+1)*ceil(M/R))) of XX."""
    per = -(-M // world)
    lo = min(M, rank * per)
    return lo, min(M, lo + per), per


def alc_batch_dist(X, Z, XX, d, g, n0, n, Nprime, form="auto", group=None):
    """Multi-GPU path: every rank holds the full X, Z (replicated)
    and the full XX; rank r runs laGP_alc_batch on its contiguous shard of XX
    and one all-gather (NCCL over NVLink under the "nccl" backend) assembles
    the outputs in input order on every rank. Results are bit-identical to the
    single-GPU call (each location depends only on its own row)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    M = XX.shape[0]
    lo, hi, per = shard_bounds(M, rank, world)
    r = alc_batch(X, Z, XX[lo:hi], d, g, n0, n, Nprime, form=form)
    return gather_shards(r, M, group)


def gather_shards(r: dict, M: int, group=None) -> dict:
    """All-gather per-rank result shards (rows [lo, hi) of each rank, padded to
    ceil(M/R)) into full [M, ...] tensors in input order on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    _, _, per = shard_bounds(M, 0, world)
    nccl = dist.get_backend(group) == "nccl"

    def gather(t, fill):
        pad = torch.full((per,) + tuple(t.shape[1:]), fill, dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        if nccl:
            full = torch.empty((world * per,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(full, pad, group=group)
        else:  # gloo (CPU tests, or CUDA tensors staged through host memory)
            hp = pad.cpu()
            parts = [torch.empty_like(hp) for _ in range(world)]
            dist.all_gather(parts, hp, group=group)
            full = torch.cat(parts).to(t.device)
        return full[:M]

    return dict(idx=gather(r["idx"], -1), mean=gather(r["mean"], float("nan")),
                s2=gather(r["s2"], float("nan")), var=gather(r["var"], float("nan")),
                flags=gather(r["flags"], 0))
