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
import warnings

import numpy as np

from . import _native as nat

__all__ = ["BesselRegime", "MidRangeSmallOrderWarning", "bessel_k", "case2_series",
           "case3_series", "case4_series", "digamma", "dnu_xnu_knu", "select_regime",
           "u_poly_coeffs", "SMALL_MID_SPLIT", "MID_LARGE_SPLIT", "MID_TRUNCATION_SPLIT",
           "INTEGER_BAND", "FD_LAG", "CASE2_TERMS", "CASE3_TERMS_NEAR", "CASE3_TERMS_FAR",
           "CASE4_TERMS"]

SMALL_MID_SPLIT = 8.5        # bessel.py:46
MID_LARGE_SPLIT = 30.0       # bessel.py:47
MID_TRUNCATION_SPLIT = 15.0  # bessel.py:48
INTEGER_BAND = 1e-6          # bessel.py:49
FD_LAG = 1e-9                # bessel.py:50
CASE2_TERMS = 20             # bessel.py:52
CASE3_TERMS_NEAR = 12        # bessel.py:53
CASE3_TERMS_FAR = 8          # bessel.py:54
CASE4_TERMS = 5              # bessel.py:55
SMALL_ORDER_WARN = 0.05      # bessel.py:240


class MidRangeSmallOrderWarning(UserWarning):
    """The mid-range (case-3) expansion was used with nu < 0.05 (bessel.py:72-77): the
    uniform asymptotic series has no stated validity floor in nu, so results are flagged."""


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


def _warn_small_order(nu: float):
    warnings.warn(f"mid-range order-derivative expansion used with nu={nu:g} < 0.05",
                  MidRangeSmallOrderWarning, stacklevel=3)


def dnu_xnu_knu(nu, x, device: int | None = None):
    """d/dnu [x^nu K_nu(x)] on the GPU with the four-regime dispatch (bessel.py:327-370)."""
    if not np.isscalar(nu) and np.asarray(nu).ndim > 0:
        raise ValueError("dnu_xnu_knu expects a scalar order nu")
    nu = float(nu)
    if not math.isfinite(nu) or nu <= 0.0:
        raise ValueError("dnu_xnu_knu requires nu > 0")
    xa = np.asarray(x, dtype=float)
    if nu < SMALL_ORDER_WARN and np.any((xa >= SMALL_MID_SPLIT) & (xa < MID_LARGE_SPLIT)):
        _warn_small_order(nu)  # raised by case3_series inside the dispatch (bessel.py:240-245)
    out = _device_call(nat.lib.mle_dnu_xnu_knu, nu, x, device)
    return float(np.asarray(out).reshape(-1)[0]) if np.ndim(x) == 0 else out


def _series(which_case, nu, x, device):
    nu = float(nu)
    out = _device_call(lambda first, xp, m, dev, op: nat.lib.mle_dnu_series(
        which_case, first, xp, m, dev, op), nu, x, device)
    return float(np.asarray(out).reshape(-1)[0]) if np.ndim(x) == 0 else out


def case2_series(nu: float, x, device: int | None = None):
    """Ascending series of d/dnu[x^nu K_nu(x)] alone, 0 < x < 8.5 and nu off the integers
    (bessel.py:184-223); ValueError outside that domain."""
    return _series(2, nu, x, device)


def case3_series(nu: float, x, device: int | None = None):
    """Uniform-asymptotic series alone, 8.5 <= x < 30, nu > 0 (bessel.py:226-283); warns
    MidRangeSmallOrderWarning for nu < 0.05 (bessel.py:240-245)."""
    xa = np.asarray(x, dtype=float)
    if not (np.all(xa >= SMALL_MID_SPLIT) and np.all(xa < MID_LARGE_SPLIT)):
        raise ValueError("case3_series requires 8.5 <= x < 30")
    if float(nu) <= 0.0:
        raise ValueError("case3_series requires nu > 0")
    if float(nu) < SMALL_ORDER_WARN:
        _warn_small_order(float(nu))
    return _series(3, nu, x, device)


def case4_series(nu: float, x, device: int | None = None):
    """Large-argument series alone, x >= 30, nu > 0 (bessel.py:286-318)."""
    return _series(4, nu, x, device)


def digamma(nu):
    """psi(nu); ValueError at the poles nu in {0, -1, -2, ...} (bessel.py:103-115).  Host
    arithmetic (the per-theta prologue's routine, long double)."""
    arr = np.ascontiguousarray(np.asarray(nu, dtype=np.float64))
    flat = arr.reshape(-1)
    out = np.empty_like(flat)
    nat.check(nat.lib.mle_digamma(nat.as_ptr(flat), flat.size, nat.as_ptr(out)))
    return float(out[0]) if np.isscalar(nu) else out.reshape(arr.shape)


def u_poly_coeffs(k_max: int):
    """Debye polynomials U_0..U_k_max as coefficient lists in p, U_k of length 3k+1
    (bessel.py:144-170: U_{k+1}(p) = p^2 (1 - p^2) U_k'(p) / 2 + (1/8) int_0^p (1 - 5 t^2)
    U_k(t) dt).  The engine's device tables are the same recursion (prologue.cpp)."""
    if k_max < 0:
        raise ValueError("k_max must be non-negative")
    out = [np.ones(1)]
    for k in range(1, k_max + 1):
        prev = np.concatenate([out[-1], np.zeros(3)])  # degree 3(k-1) -> room for 3k
        j = np.arange(1, 3 * k + 1, dtype=float)
        up1 = 0.5 * (j - 1.0 + 1.0 / (4.0 * j)) * prev[np.arange(0, 3 * k)]
        up3 = np.where(j >= 3, 0.5 * (j - 3.0 + 5.0 / (4.0 * j)) *
                       prev[np.maximum(np.arange(-2, 3 * k - 2), 0)], 0.0)
        out.append(np.concatenate([[0.0], up1 - up3]))
    return out
