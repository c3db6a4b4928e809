"""K_nu and d/dnu[x^nu K_nu(x)] evaluated by the sm_100a kernels.

Mirrors the reference surface of ``pkg/src/maternmle/bessel.py`` for the hot-path
functions: ``bessel_k`` (bessel.py:80-100), ``dnu_xnu_knu`` (bessel.py:327-370),
``select_regime`` / ``BesselRegime`` (bessel.py:61-141; pure host logic that the
device dispatch implements per element).  Values are computed on the GPU by the
same device functions the covariance generation kernel uses.
"""

from __future__ import annotations

import enum
import math

import numpy as np

from . import _native as nat

__all__ = ["BesselRegime", "bessel_k", "dnu_xnu_knu", "select_regime",
           "SMALL_MID_SPLIT", "MID_LARGE_SPLIT", "INTEGER_BAND", "FD_LAG"]

SMALL_MID_SPLIT = 8.5    # bessel.py:46
MID_LARGE_SPLIT = 30.0   # bessel.py:47
INTEGER_BAND = 1e-6      # bessel.py:49
FD_LAG = 1e-9            # bessel.py:50


class BesselRegime(enum.Enum):
    """Evaluation strategy for a given (nu, x) (bessel.py:61-68)."""

    ZERO_ARG = "zero_arg"
    SMALL_X = "small_x"
    MID_X = "mid_x"
    LARGE_X = "large_x"
    FINITE_DIFF = "finite_diff"


def _near(v: float) -> bool:
    return abs(v - round(v)) <= INTEGER_BAND


def select_regime(nu: float, x: float) -> BesselRegime:
    """Unique regime of (nu, x); same predicates as bessel.py:126-141."""
    if x == 0.0:
        return BesselRegime.ZERO_ARG
    if x < SMALL_MID_SPLIT:
        return BesselRegime.FINITE_DIFF if _near(nu) else BesselRegime.SMALL_X
    if x < MID_LARGE_SPLIT:
        return BesselRegime.MID_X
    return BesselRegime.FINITE_DIFF if _near(nu + 0.5) else BesselRegime.LARGE_X


def _device_call(fn, first, x, device):
    x_arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    flat = x_arr.reshape(-1)
    out = np.empty_like(flat)
    dev = nat.default_device() if device is None else device
    nat.check(fn(first, nat.as_ptr(flat), flat.size, dev, nat.as_ptr(out)))
    return out.reshape(x_arr.shape)


def bessel_k(nu, x, device: int | None = None):
    """K_nu(x) on the GPU; K_nu = K_{-nu}; x > 0 and finite (bessel.py:80-100)."""
    if np.ndim(nu) != 0:
        nu_arr, x_arr = np.broadcast_arrays(np.asarray(nu, float), np.asarray(x, float))
        out = np.empty(nu_arr.shape)
        for v in np.unique(nu_arr):
            mask = nu_arr == v
            out[mask] = _device_call(nat.lib.mle_bessel_k, float(v), x_arr[mask], device)
        return out
    nu = float(nu)
    if not math.isfinite(nu):
        raise ValueError("bessel_k requires finite nu and x")
    out = _device_call(nat.lib.mle_bessel_k, nu, x, device)
    return float(np.asarray(out).reshape(-1)[0]) if np.ndim(x) == 0 else out


def dnu_xnu_knu(nu, x, device: int | None = None):
    """d/dnu [x^nu K_nu(x)] on the GPU with the four-regime dispatch (bessel.py:327-370)."""
    if not np.isscalar(nu) and np.asarray(nu).ndim > 0:
        raise ValueError("dnu_xnu_knu expects a scalar order nu")
    nu = float(nu)
    if not math.isfinite(nu) or nu <= 0.0:
        raise ValueError("dnu_xnu_knu requires nu > 0")
    out = _device_call(nat.lib.mle_dnu_xnu_knu, nu, x, device)
    return float(np.asarray(out).reshape(-1)[0]) if np.ndim(x) == 0 else out
