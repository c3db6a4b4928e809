"""Exact log-likelihood, score and Fisher information on the GPU.

Drop-in for ``pkg/src/maternmle/likelihood.py``: ``NotPositiveDefinite``
(likelihood.py:41-51), ``LikelihoodEval`` (:54-60), ``cholesky_lower`` (:63-78),
``log_likelihood`` (:81-89), ``trace_product`` (:92-104) and ``grad_and_fisher``
(:107-149).  ``log_likelihood`` and ``grad_and_fisher`` run entirely on the
device (generation, Cholesky, solves and reductions); only theta goes down and
the scalars come back.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .matern import MaternParams, SpatialDataset

__all__ = [
    "NotPositiveDefinite",
    "LikelihoodEval",
    "cholesky_lower",
    "log_likelihood",
    "trace_product",
    "grad_and_fisher",
]


class NotPositiveDefinite(Exception):
    """Cholesky factorization failed; carries the zero-based failing pivot."""

    def __init__(self, pivot: int):
        self.pivot = pivot
        super().__init__(f"matrix not positive definite at pivot {pivot}")


@dataclass
class LikelihoodEval:
    """Log-likelihood, its gradient over (sigma2, alpha, nu), and I(theta)."""

    loglik: float
    grad: np.ndarray
    fisher: np.ndarray


def _theta_vec(theta) -> np.ndarray:
    return theta.as_array() if isinstance(theta, MaternParams) else MaternParams.from_array(
        theta).as_array()


def cholesky_lower(sigma, device: int | None = None) -> np.ndarray:
    """Lower-triangular L with L L^T = sigma, factored by the sm_100a kernels.

    Only the lower triangle of ``sigma`` is read; the strict upper triangle of the
    result is zero (LAPACK ``clean=1``).  Raises :class:`NotPositiveDefinite` with
    the 0-based failing pivot (likelihood.py:75-77).
    """
    a = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("cholesky_lower expects a square matrix")
    n = a.shape[0]
    out = np.empty_like(a)
    piv = ctypes.c_int64(-1)
    dev = nat.default_device() if device is None else device
    rc = nat.lib.mle_cholesky(nat.as_ptr(a), n, dev, nat.as_ptr(out), ctypes.byref(piv))
    nat.check(rc, piv.value)
    return out


def log_likelihood(data: SpatialDataset, theta) -> float:
    """Exact log-likelihood of the dataset under theta (likelihood.py:81-89)."""
    return data.engine().loglik(_theta_vec(theta))


def grad_and_fisher(data: SpatialDataset, theta) -> LikelihoodEval:
    """Log-likelihood, gradient and Fisher information in one device pass
    (likelihood.py:107-149; Algorithm 3 of the paper)."""
    ll, grad, fisher = data.engine().eval_all(_theta_vec(theta))
    return LikelihoodEval(loglik=ll, grad=grad, fisher=fisher)


def trace_product(a, b) -> float:
    """trace(AB) for square host matrices (likelihood.py:92-104).

    Utility only: the engine never forms these products (the Fisher entries are
    Frobenius inner products reduced on the device), so this is computed directly
    as sum(A * B^T) on the GPU through torch.
    """
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("trace_product expects square matrices")
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    import torch

    if not torch.cuda.is_available():
        raise nat.NativeError("trace_product needs a CUDA device (no CPU fallback)")
    ta = torch.as_tensor(a, device="cuda")
    tb = torch.as_tensor(b, device="cuda")
    return float((ta * tb.T).sum().item())
