"""ctypes binding of the in-tree C-ABI library ``libmaternfisher.so``.

The library is the whole compute path (sm_100a kernels + the C ABI declared in
``include/maternfisher.h``).  There is no CPU fallback: if the shared object is
missing the import fails, and every compute entry point returns MLE_CUDA_ERROR
when no GPU is visible, which the wrappers raise as ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libmaternfisher.so"

MLE_OK = 0
MLE_NOT_PD = 1
MLE_INVALID = 2
MLE_CUDA_ERROR = 3

WHICH = {"sigma": 0, "sigma2": 1, "alpha": 2, "nu": 3}
PHASES = ("gen", "potrf", "solve", "reduce", "total")

# Every symbol the public header declares (tests check the .so exports all of them).
EXPORTED = (
    "mle_version", "mle_last_error", "mle_device_count", "mle_ctx_create", "mle_ctx_destroy",
    "mle_ctx_n", "mle_ctx_set_values", "mle_loglik", "mle_eval_all", "mle_build",
    "mle_phase_times", "mle_cholesky", "mle_bessel_k", "mle_dnu_xnu_knu", "mle_matern_elem",
    "mle_eval_batch", "mle_simulate", "mle_release_cached_memory",
    "mle_kernel_profile", "mle_kernel_stats", "mle_ctx_cond_estimate", "mle_ctx_seq_derivs", "mle_dctx_create", "mle_dctx_destroy",
    "mle_dctx_layout", "mle_dctx_begin", "mle_dctx_factor", "mle_dctx_update",
    "mle_dctx_wblock", "mle_dctx_forward", "mle_dctx_right_operand", "mle_dctx_right",
    "mle_dctx_partials", "mle_launch_count", "mle_dnu_series", "mle_digamma",
    "mle_dctx_update_range", "mle_dctx_right_range", "mle_dctx_set_async", "mle_dctx_stream",
    "mle_dctx_wcache", "mle_dctx_panel_partials", "mle_dctx_2s_owner", "mle_dctx_2s_finish",
    "mle_dctx_2s_update_range", "mle_dctx_panel_slices", "mle_dctx_forward_range",
)

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
            "paper_2601_11437_b200/csrc); there is no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH))
    sig = {
        "mle_version": (ctypes.c_char_p, []),
        "mle_last_error": (ctypes.c_char_p, []),
        "mle_device_count": (ctypes.c_int, []),
        "mle_release_cached_memory": (ctypes.c_int, []),
        "mle_launch_count": (ctypes.c_int64, []),
        "mle_dnu_series": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64,
                                          ctypes.c_int, _dp]),
        "mle_digamma": (ctypes.c_int, [_dp, ctypes.c_int64, _dp]),
        "mle_kernel_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
        "mle_kernel_stats": (ctypes.c_int, [ctypes.c_void_p, _dp]),
        "mle_ctx_cond_estimate": (ctypes.c_int, [ctypes.c_void_p, _dp]),
        "mle_ctx_seq_derivs": (ctypes.c_int, [ctypes.c_void_p]),
        "mle_dctx_create": (ctypes.c_int, [_dp, _dp, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(_vp)]),
        "mle_dctx_destroy": (None, [_vp]),
        "mle_dctx_layout": (ctypes.c_int, [_vp, _i64p]),
        "mle_dctx_begin": (ctypes.c_int, [_vp, _dp, ctypes.c_int]),
        "mle_dctx_factor": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_update": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_wblock": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_forward": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_right_operand": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_right": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp]),
        "mle_dctx_partials": (ctypes.c_int, [_vp, _dp]),
        "mle_dctx_update_range": (ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_int,
                                                 ctypes.c_int]),
        "mle_dctx_right_range": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int,
                                                ctypes.c_int]),
        "mle_dctx_set_async": (ctypes.c_int, [_vp, ctypes.c_int]),
        "mle_dctx_stream": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
        "mle_dctx_wcache": (ctypes.c_int, [_vp, ctypes.c_int]),
        "mle_dctx_panel_partials": (ctypes.c_int, [_vp, _dp]),
        "mle_dctx_2s_owner": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_2s_finish": (ctypes.c_int, [_vp, ctypes.c_int]),
        "mle_dctx_2s_update_range": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int,
                                                    ctypes.c_int]),
        "mle_dctx_panel_slices": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
        "mle_dctx_forward_range": (ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_int,
                                                  ctypes.c_int]),
        "mle_ctx_create": (ctypes.c_int, [_dp, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                          ctypes.POINTER(_vp)]),
        "mle_ctx_destroy": (None, [_vp]),
        "mle_ctx_n": (ctypes.c_int64, [_vp]),
        "mle_ctx_set_values": (ctypes.c_int, [_vp, _dp]),
        "mle_loglik": (ctypes.c_int, [_vp, _dp, _dp, _i64p]),
        "mle_eval_all": (ctypes.c_int, [_vp, _dp, _dp, _dp, _dp, _i64p]),
        "mle_build": (ctypes.c_int, [_vp, _dp, ctypes.c_int, _dp]),
        "mle_eval_batch": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, _dp,
                                          ctypes.POINTER(ctypes.c_int), _dp, _i64p,
                                          ctypes.POINTER(ctypes.c_int)]),
        "mle_simulate": (ctypes.c_int, [_vp, _dp, _dp, _dp, _i64p]),
        "mle_phase_times": (ctypes.c_int, [_vp, _dp]),
        "mle_cholesky": (ctypes.c_int, [_dp, ctypes.c_int64, ctypes.c_int, _dp, _i64p]),
        "mle_bessel_k": (ctypes.c_int, [ctypes.c_double, _dp, ctypes.c_int64, ctypes.c_int, _dp]),
        "mle_dnu_xnu_knu": (ctypes.c_int, [ctypes.c_double, _dp, ctypes.c_int64, ctypes.c_int,
                                           _dp]),
        "mle_matern_elem": (ctypes.c_int, [_dp, ctypes.c_int, _dp, ctypes.c_int64, ctypes.c_int,
                                           _dp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def as_ptr(arr: np.ndarray):
    return arr.ctypes.data_as(_dp)


def last_error() -> str:
    msg = lib.mle_last_error()
    return msg.decode() if msg else ""


class NativeError(RuntimeError):
    """CUDA failure inside the engine (MLE_CUDA_ERROR)."""


def check(rc: int, pivot: int | None = None):
    """Map a C-ABI return code onto the reference's exception types."""
    if rc == MLE_OK:
        return
    if rc == MLE_NOT_PD:
        from .likelihood import NotPositiveDefinite

        raise NotPositiveDefinite(int(pivot if pivot is not None else -1))
    if rc == MLE_INVALID:
        raise ValueError(last_error())
    raise NativeError(last_error() or f"engine error {rc}")


def device_count() -> int:
    return int(lib.mle_device_count())


def release_cached_memory() -> None:
    """Hand the idle buffers of destroyed contexts back to the driver
    (mle_release_cached_memory)."""
    check(lib.mle_release_cached_memory())


def default_device() -> int:
    return int(os.environ.get("MLE_DEVICE", "0"))
