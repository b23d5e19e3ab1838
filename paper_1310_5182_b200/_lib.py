"""ctypes declaration of include/lagp.h (argument marshalling only).

Loads the in-tree ``liblagp_b200.so``. There is no fallback: if the library is
missing, importing this module raises (build it with ``__graft_entry__.build()``
or ``python paper_1310_5182_b200/build.py``).
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liblagp_b200.so")

LAGP_OK, LAGP_PARTIAL, LAGP_EINVAL, LAGP_ECUDA, LAGP_ENOMEM = 0, 1, 2, 3, 4
FLAG_NEAR_TIE, FLAG_SENTINEL, FLAG_EXHAUSTED, FLAG_NONFINITE = 1, 2, 4, 8
FLAG_MLE_BOUND, FLAG_MLE_MAXIT, FLAG_MLE_FAIL = 16, 32, 64
ALC_EXPLICIT, ALC_INCREMENTAL, ALC_EXPLICIT_DFMA, ALC_AUTO = 0, 1, 2, 3
FORM_NAMES = {0: "explicit", 1: "incremental", 2: "explicit_dfma", 3: "auto"}
NMAX, PMAX = 128, 16

EXPORTS = (
    "laGP_alc_batch",
    "laGP_alc_batch_ex",
    "laGP_alc_batch_host",
    "laGP_nn_pool",
    "laGP_alc_scores",
    "laGP_pinv_update",
    "laGP_predict",
    "laGP_alc_batch_theta",
    "laGP_mle",
    "laGP_local_fit",
    "laGP_exp_nonpos",
    "laGP_alc_batch_sep",
    "lagp_release_workspace",
    "lagp_last_error",
    "lagp_abi_version",
)


class Timing(ctypes.Structure):
    _fields_ = [
        ("nn_ms", ctypes.c_float),
        ("alc_ms", ctypes.c_float),
        ("predict_ms", ctypes.c_float),
        ("total_ms", ctypes.c_float),
        ("launches", ctypes.c_int32),
        ("nn_fallbacks", ctypes.c_int32),
        ("alc_form", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("nn_filter_pairs", ctypes.c_int64),
        ("nn_sample_pairs", ctypes.c_int64),
        ("nn_exact_keys", ctypes.c_int64),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["alc_form"] = FORM_NAMES.get(d["alc_form"], d["alc_form"])
        return d


_vp, _i64, _i32, _dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: the sm_100a CUDA library is not built "
            "(run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    batch_args = [_vp, _i64, _i32, _vp, _vp, _i64, _dbl, _dbl, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
    lib.laGP_alc_batch.argtypes = batch_args + [_vp]
    lib.laGP_alc_batch_ex.argtypes = batch_args + [_i32, ctypes.POINTER(Timing), _vp]
    lib.laGP_alc_batch_host.argtypes = batch_args + [_i32, _vp]
    lib.laGP_nn_pool.argtypes = [_vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp, _vp]
    lib.laGP_alc_scores.argtypes = [_i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _vp, _vp, _vp, _vp]
    lib.laGP_pinv_update.argtypes = [_i32, _i32, _vp, _vp, _dbl, _vp, _vp]
    lib.laGP_predict.argtypes = [_i32, _i32, _i32, _vp, _vp, _vp, _dbl, _dbl, _vp, _vp, _vp, _vp]
    lib.laGP_alc_batch_theta.argtypes = [_vp, _i64, _i32, _vp, _vp, _i64, _vp, _dbl, _dbl, _i32, _i32, _i32,
                                         _vp, _vp, _vp, _vp, _vp, _vp, _i32, ctypes.POINTER(Timing), _vp]
    lib.laGP_mle.argtypes = [_vp, _i64, _i32, _vp, _vp, _i64, _vp, _i32, _vp, _dbl, _dbl, _dbl, _dbl,
                             _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    lib.laGP_local_fit.argtypes = [_vp, _i64, _i32, _vp, _vp, _i64, _dbl, _dbl, _dbl, _dbl, _i32, _i32, _i32,
                                   _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(Timing), _vp]
    lib.laGP_exp_nonpos.argtypes = [_vp, _vp, _i64, _vp]
    lib.laGP_alc_batch_sep.argtypes = [_vp, _i64, _i32, _vp, _vp, _i64, ctypes.POINTER(ctypes.c_double), _dbl,
                                       _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                       ctypes.POINTER(Timing), _vp]
    lib.lagp_release_workspace.argtypes = []
    for f in EXPORTS[:-2]:
        getattr(lib, f).restype = ctypes.c_int
    lib.lagp_last_error.argtypes = []
    lib.lagp_last_error.restype = ctypes.c_char_p
    lib.lagp_abi_version.argtypes = []
    lib.lagp_abi_version.restype = ctypes.c_int
    return lib
