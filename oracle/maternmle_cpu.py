"""numpy/scipy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Follows, in order:
  bessel.py:45-56      regime constants
  bessel.py:126-141    regime selection
  bessel.py:144-176    Debye U_k tables
  bessel.py:184-223    case 2 ascending series
  bessel.py:226-283    case 3 uniform asymptotics
  bessel.py:286-318    case 4 large-x series
  bessel.py:321-370    forward difference + dispatcher
  matern.py:100-125    C, dC/dalpha, dC/dnu at positive distance
  matern.py:171-203    dense assembly (pdist + squareform; the reference's np.unique
                       dedup changes no value, so it is omitted)
  likelihood.py:63-149 dpotrf, log-likelihood, Algorithm 3 score / Fisher
  optimizer.py:114-142 counting objective (used with paper_2601_11437_b200's host
                       Fisher-BT driver for CPU fits)
All arithmetic is float64 in the same operation order as the reference so that the
oracle reproduces it bit for bit (checked in tests/test_oracle.py).
"""

from __future__ import annotations

import math

import numpy as np
from scipy import special as sps
from scipy.linalg import solve_triangular
from scipy.linalg.lapack import dpotrf
from scipy.spatial.distance import pdist, squareform

LOG2 = math.log(2.0)
LOG_2PI = math.log(2.0 * math.pi)
SQRT_HALF_PI = math.sqrt(0.5 * math.pi)
SPLIT_SMALL, SPLIT_LARGE, SPLIT_TRUNC = 8.5, 30.0, 15.0
BAND, LAG = 1e-6, 1e-9
K2, K3_NEAR, K3_FAR, K4 = 20, 12, 8, 5


class NotPD(Exception):
    def __init__(self, pivot):
        self.pivot = pivot
        super().__init__(f"not positive definite at pivot {pivot}")


# --------------------------------------------------------------------- special functions
def near_int(v):
    return abs(v - round(v)) <= BAND


def regime(nu, x):
    """'zero' | 'small' | 'mid' | 'large' | 'fd' (bessel.py:126-141)."""
    if x == 0.0:
        return "zero"
    if x < SPLIT_SMALL:
        return "fd" if near_int(nu) else "small"
    if x < SPLIT_LARGE:
        return "mid"
    return "fd" if near_int(nu + 0.5) else "large"


def debye_tables(kmax=K3_NEAR):
    """U_k coefficient vectors by the recursion of bessel.py:144-170 and U_k'."""
    u = [np.array([1.0])]
    for k in range(kmax):
        prev = u[-1]
        nxt = np.zeros(3 * k + 4)
        for j in range(1, 3 * k + 4):
            c = 0.0
            if j - 1 < prev.size:
                c += 0.5 * (j - 1 + 1.0 / (4.0 * j)) * prev[j - 1]
            if 0 <= j - 3 < prev.size:
                c -= 0.5 * (j - 3 + 5.0 / (4.0 * j)) * prev[j - 3]
            nxt[j] = c
        u.append(nxt)
    du = [c[1:] * np.arange(1, c.size) if c.size > 1 else np.zeros(1) for c in u]
    return u, du


_U, _DU = debye_tables()


def small_series(nu, x):
    """bessel.py:184-223 (vectorised over x)."""
    gp = sps.gamma(nu)
    gn = -math.pi / (math.sin(math.pi * nu) * nu * gp)
    pp, pn = float(sps.digamma(nu)), float(sps.digamma(-nu))
    tlx = 2.0 * np.log(x)
    x2n = x ** (2.0 * nu)
    q = 0.25 * x * x
    pref = np.full_like(x, 0.5)
    g_p = g_n = 1.0
    d_p = d_n = 0.0
    acc = np.zeros_like(x)
    for k in range(K2 + 1):
        if k:
            pref = pref * q / k
            g_p /= nu + k
            g_n /= -nu + k
            d_p -= 1.0 / (nu + k)
            d_n -= 1.0 / (-nu + k)
        tp = 2.0 ** nu * (LOG2 + pp - d_n) * gp * g_n
        tn = 2.0 ** -nu * x2n * (-LOG2 + tlx - pn + d_p) * gn * g_p
        acc = acc + pref * (tp + tn)
    return acc


def mid_series(nu, x):
    """bessel.py:226-283 (vectorised over x)."""
    out = np.empty_like(x)
    for sel, kk in ((x < SPLIT_TRUNC, K3_NEAR), (x >= SPLIT_TRUNC, K3_FAR)):
        if not sel.any():
            continue
        xs = x[sel]
        zz = xs / nu
        rt = np.sqrt(1.0 + zz * zz)
        p = 1.0 / rt
        eta = rt + np.log(zz / (1.0 + rt))
        pre = xs ** nu * math.sqrt(math.pi / (2.0 * nu)) * np.exp(-nu * eta) / np.sqrt(rt)
        s_u = np.zeros_like(xs)
        s_ku = np.zeros_like(xs)
        s_du = np.zeros_like(xs)
        sg, npow = 1.0, 1.0
        for k in range(kk + 1):
            uv = np.polynomial.polynomial.polyval(p, _U[k])
            duv = np.polynomial.polynomial.polyval(p, _DU[k])
            s_u += sg * npow * uv
            s_ku += sg * (k * npow / nu) * uv
            s_du += sg * npow * duv
            sg = -sg
            npow /= nu
        br = math.log(nu) + np.log(1.0 + rt) - 1.0 / (2.0 * nu * (1.0 + zz * zz))
        out[sel] = (br * pre * s_u - pre * s_ku
                    + (xs * xs / nu ** 3) * (1.0 + zz * zz) ** -1.5 * pre * s_du)
    return out


def large_series(nu, x):
    """bessel.py:286-318 (vectorised over x)."""
    lx = np.log(x)
    tot = lx.copy()
    a, b = 1.0, 0.0
    xp = np.ones_like(x)
    f4 = 4.0 * nu * nu
    for k in range(1, K4 + 1):
        fac = f4 - (2 * k - 1) ** 2
        a *= fac / (8.0 * k)
        if a == 0.0:
            break
        b += 8.0 * nu / fac
        xp = xp / x
        tot = tot + xp * (lx + b) * a
    return SQRT_HALF_PI * x ** (nu - 0.5) * np.exp(-x) * tot


def fd_derivative(nu, x):
    """bessel.py:321-324."""
    return (x ** (nu + LAG) * sps.kv(nu + LAG, x) - x ** nu * sps.kv(nu, x)) / LAG


def dnu_xnu_knu(nu, x):
    """d/dnu [x^nu K_nu(x)] with the four-regime dispatch (bessel.py:327-370)."""
    nu = float(nu)
    if not math.isfinite(nu) or nu <= 0.0:
        raise ValueError("dnu_xnu_knu requires nu > 0")
    xa = np.atleast_1d(np.asarray(x, dtype=float))
    if np.any(xa < 0.0) or not np.all(np.isfinite(xa)):
        raise ValueError("dnu_xnu_knu requires finite x >= 0")
    out = np.zeros_like(xa)
    small = (xa > 0.0) & (xa < SPLIT_SMALL)
    mid = (xa >= SPLIT_SMALL) & (xa < SPLIT_LARGE)
    large = xa >= SPLIT_LARGE
    fd = np.zeros_like(small)
    if near_int(nu):
        fd, small = fd | small, small & False
    if near_int(nu + 0.5):
        fd, large = fd | large, large & False
    for sel, fn in ((small, small_series), (mid, mid_series), (large, large_series),
                    (fd, fd_derivative)):
        if sel.any():
            out[sel] = fn(nu, xa[sel])
    return float(out[0]) if np.ndim(x) == 0 else out.reshape(np.shape(x))


def bessel_k(nu, x):
    return sps.kv(np.abs(np.asarray(nu, float)), np.asarray(x, float))


# --------------------------------------------------------------------- covariance model
def cov_pos(h, th):
    """matern.py:100-104."""
    s2, al, nu = th
    u = h / al
    scale = s2 * 2.0 ** (1.0 - nu) / sps.gamma(nu)
    return scale * u ** nu * sps.kv(nu, u)


def dalpha_pos(h, th):
    """matern.py:107-111."""
    s2, al, nu = th
    u = h / al
    scale = 2.0 ** (1.0 - nu) / sps.gamma(nu) * s2 / al
    return scale * u ** (nu + 1.0) * sps.kv(nu - 1.0, u)


def dnu_pos(h, th):
    """matern.py:114-125."""
    s2, al, nu = th
    u = h / al
    q = 2.0 ** (1.0 - nu) / sps.gamma(nu)
    f = u ** nu * sps.kv(nu, u)
    return s2 * q * ((-math.log(2.0) - float(sps.digamma(nu))) * f + dnu_xnu_knu(nu, u))


KINDS = {
    "sigma": (lambda h, th: cov_pos(h, th), lambda th: th[0]),
    "sigma2": (lambda h, th: cov_pos(h, th) / th[0], lambda th: 1.0),
    "alpha": (dalpha_pos, lambda th: 0.0),
    "nu": (dnu_pos, lambda th: 0.0),
}


def elem(h, th, kind="sigma"):
    """C / dC at distances h with the zero-lag limit (matern.py:128-168)."""
    fn, zero = KINDS[kind]
    ha = np.atleast_1d(np.asarray(h, float))
    out = np.full(ha.shape, zero(th))
    pos = ha > 0.0
    if pos.any():
        out[pos] = fn(ha[pos], th)
    return float(out[0]) if np.ndim(h) == 0 else out.reshape(np.shape(h))


def matrix(locations, th, kind="sigma", nugget=0.0):
    """Dense symmetric n x n matrix (matern.py:171-203), optional nugget on Sigma's diagonal."""
    th = tuple(float(v) for v in th)
    cond = pdist(np.asarray(locations, float))
    fn, zero = KINDS[kind]
    vals = np.full(cond.shape, zero(th))
    pos = cond > 0.0
    if pos.any():
        vals[pos] = fn(cond[pos], th)
    mat = squareform(vals, checks=False)
    diag = zero(th) + (nugget if kind == "sigma" else 0.0)
    np.fill_diagonal(mat, diag)
    return mat


# --------------------------------------------------------------------- likelihood engine
def cholesky(sigma):
    """likelihood.py:63-78."""
    low, info = dpotrf(np.asarray(sigma, float), lower=1, clean=1, overwrite_a=0)
    if info != 0:
        raise NotPD(int(info) - 1)
    return low


def loglik(locations, z, th, nugget=0.0):
    """likelihood.py:81-89."""
    low = cholesky(matrix(locations, th, "sigma", nugget))
    y = solve_triangular(low, z, lower=True, check_finite=False)
    n = len(z)
    return -0.5 * n * LOG_2PI - float(np.sum(np.log(np.diag(low)))) - 0.5 * float(y @ y)


def trace_product(a, b):
    """likelihood.py:92-104."""
    mix = a + b.T
    return 0.5 * float(np.sum(mix * mix) - np.sum(a * a) - np.sum(b * b))


def eval_all(locations, z, th):
    """Algorithm 3 (likelihood.py:107-149): (loglik, grad[3], fisher[3,3])."""
    n = len(z)
    s2 = th[0]
    low = cholesky(matrix(locations, th, "sigma"))
    y = solve_triangular(low, z, lower=True, check_finite=False)
    quad = float(y @ y)
    ll = -0.5 * n * LOG_2PI - float(np.sum(np.log(np.diag(low)))) - 0.5 * quad
    w = solve_triangular(low, y, lower=True, trans="T", check_finite=False)
    grad = np.empty(3)
    fis = np.empty((3, 3))
    grad[0] = (quad - n) / (2.0 * s2)
    fis[0, 0] = n / (2.0 * s2 * s2)
    blocks = []
    for kind in ("alpha", "nu"):
        si = matrix(locations, th, kind)
        a = solve_triangular(low, solve_triangular(low, si, lower=True, check_finite=False),
                             lower=True, trans="T", check_finite=False)
        tr = float(np.trace(a))
        blocks.append((a, tr, -0.5 * tr + 0.5 * float(w @ (si @ w))))
    (aa, ta, ga), (an, tn, gn) = blocks
    grad[1], grad[2] = ga, gn
    fis[0, 1] = fis[1, 0] = ta / (2.0 * s2)
    fis[1, 1] = 0.5 * trace_product(aa, aa)
    fis[0, 2] = fis[2, 0] = tn / (2.0 * s2)
    fis[1, 2] = fis[2, 1] = 0.5 * trace_product(aa, an)
    fis[2, 2] = 0.5 * trace_product(an, an)
    return ll, grad, fis


def eval_all_nugget(locations, z, th, nugget):
    """NOT IN THE REFERENCE -- config-5 restatement ("Nugget" row).

    The reference has no nugget: its diagonal is hard-wired to sigma^2 (matern.py:186-188)
    and its sigma^2 closed forms (likelihood.py:129-130, 141, 145) assume
    dSigma/dsigma^2 = Sigma / sigma^2.  With Sigma_tau = Sigma + tau^2 I that no longer holds;
    dSigma_tau/dsigma^2 = (Sigma_tau - tau^2 I) / sigma^2 = R (the Matern correlation) is
    treated as a third derivative block with exactly the algorithm of likelihood.py:107-149:
    A_i = Sigma_tau^-1 S_i by two triangular solves (:134-135), g_i = -tr(A_i)/2 +
    w^T S_i w / 2 (:136-137), I_ij = trace_product(A_i, A_j) / 2 (:140-147).  nugget = 0 gives
    the reference's eval_all up to rounding (tests/test_oracle.py).  Parity is unpinned by
    construction: no reference output exists for this case.
    """
    n = len(z)
    s2 = th[0]
    low = cholesky(matrix(locations, th, "sigma", nugget))
    y = solve_triangular(low, z, lower=True, check_finite=False)
    quad = float(y @ y)
    ll = -0.5 * n * LOG_2PI - float(np.sum(np.log(np.diag(low)))) - 0.5 * quad
    w = solve_triangular(low, y, lower=True, trans="T", check_finite=False)
    blocks = []
    for kind in ("sigma2", "alpha", "nu"):
        si = matrix(locations, th, "sigma") / s2 if kind == "sigma2" else matrix(locations, th,
                                                                                   kind)
        a = solve_triangular(low, solve_triangular(low, si, lower=True, check_finite=False),
                             lower=True, trans="T", check_finite=False)
        blocks.append((a, -0.5 * float(np.trace(a)) + 0.5 * float(w @ (si @ w))))
    grad = np.array([g for _, g in blocks])
    fis = np.empty((3, 3))
    for i in range(3):
        for j in range(i, 3):
            fis[i, j] = fis[j, i] = 0.5 * trace_product(blocks[i][0], blocks[j][0])
    return ll, grad, fis


class CountingObjective:
    """optimizer.py:114-142 semantics over the oracle (CPU fits for parity tests)."""

    def __init__(self, locations, z, nugget=0.0):
        self.locations = np.asarray(locations, float)
        self.z = np.asarray(z, float)
        self.nugget = float(nugget)  # nugget > 0: config-5 restatement (eval_all_nugget)
        self.loglik_calls = 0
        self.grad_calls = 0

    def loglik(self, theta):
        self.loglik_calls += 1
        th = tuple(float(v) for v in theta)
        if not all(math.isfinite(v) and v > 0.0 for v in th):
            return -math.inf
        try:
            with np.errstate(over="ignore", under="ignore", invalid="ignore"):
                v = loglik(self.locations, self.z, th, self.nugget)
        except (NotPD, ValueError):
            return -math.inf
        return -math.inf if math.isnan(v) else v

    def eval_all(self, theta):
        self.loglik_calls += 1
        self.grad_calls += 1
        th = tuple(float(v) for v in theta)
        if not all(math.isfinite(v) and v > 0.0 for v in th):
            raise ValueError("theta components must be finite and > 0")
        with np.errstate(over="ignore", under="ignore", invalid="ignore"):
            if self.nugget > 0.0:
                return eval_all_nugget(self.locations, self.z, th, self.nugget)
            return eval_all(self.locations, self.z, th)
