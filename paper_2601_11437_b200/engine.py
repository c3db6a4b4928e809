"""Device-resident dataset handle over the C ABI (one ``mle_ctx`` per dataset and GPU).

This is the object behind :class:`~paper_2601_11437_b200.matern.SpatialDataset`
and the GPU :class:`~paper_2601_11437_b200.optimizer.LikelihoodObjective`.
Locations and values are copied to HBM once; every evaluation regenerates the
covariance tiles on the device from theta, so only theta crosses the host link
per call (plus the 13 result doubles coming back).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as nat


class Engine:
    """Owns one ``mle_ctx`` (locations + values resident on ``device``)."""

    def __init__(self, locations, values, device: int | None = None, nugget: float = 0.0):
        loc = np.ascontiguousarray(np.asarray(locations, dtype=np.float64))
        val = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        if loc.ndim != 2 or loc.shape[1] != 2:
            raise ValueError("locations must have shape (n, 2)")
        if val.shape != (loc.shape[0],):
            raise ValueError("values length must equal the number of locations")
        self.n = int(loc.shape[0])
        self.device = nat.default_device() if device is None else int(device)
        self.nugget = float(nugget)
        self._lock = threading.Lock()
        handle = ctypes.c_void_p()
        rc = nat.lib.mle_ctx_create(nat.as_ptr(loc), nat.as_ptr(val), self.n, self.device,
                                    self.nugget, ctypes.byref(handle))
        nat.check(rc)
        self._ctx = handle

    def close(self):
        ctx, self._ctx = getattr(self, "_ctx", None), None
        if ctx:
            nat.lib.mle_ctx_destroy(ctx)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_values(self, values):
        val = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        if val.shape != (self.n,):
            raise ValueError("values length must equal the number of locations")
        with self._lock:
            nat.check(nat.lib.mle_ctx_set_values(self._ctx, nat.as_ptr(val)))

    @staticmethod
    def _theta(theta) -> np.ndarray:
        th = np.ascontiguousarray(np.asarray(theta, dtype=np.float64).reshape(3))
        return th

    def loglik(self, theta) -> float:
        th = self._theta(theta)
        out = np.zeros(1)
        piv = ctypes.c_int64(-1)
        with self._lock:
            rc = nat.lib.mle_loglik(self._ctx, nat.as_ptr(th), nat.as_ptr(out), ctypes.byref(piv))
        nat.check(rc, piv.value)
        return float(out[0])

    def eval_all(self, theta):
        th = self._theta(theta)
        ll = np.zeros(1)
        grad = np.zeros(3)
        fisher = np.zeros(9)
        piv = ctypes.c_int64(-1)
        with self._lock:
            rc = nat.lib.mle_eval_all(self._ctx, nat.as_ptr(th), nat.as_ptr(ll), nat.as_ptr(grad),
                                      nat.as_ptr(fisher), ctypes.byref(piv))
        nat.check(rc, piv.value)
        return float(ll[0]), grad, fisher.reshape(3, 3)

    def simulate(self, theta, normals) -> np.ndarray:
        """z = L w with L the device Cholesky factor of Sigma(theta) (simulate.py:100-106)."""
        th = self._theta(theta)
        w = np.ascontiguousarray(np.asarray(normals, dtype=np.float64))
        if w.shape != (self.n,):
            raise ValueError("normals must have length n")
        z = np.empty(self.n)
        piv = ctypes.c_int64(-1)
        with self._lock:
            rc = nat.lib.mle_simulate(self._ctx, nat.as_ptr(th), nat.as_ptr(w), nat.as_ptr(z),
                                      ctypes.byref(piv))
        nat.check(rc, piv.value)
        return z

    def build(self, theta, which: str) -> np.ndarray:
        if which not in nat.WHICH:
            raise ValueError(f"which must be one of {sorted(nat.WHICH)}, got {which!r}")
        th = self._theta(theta)
        out = np.empty((self.n, self.n))
        with self._lock:
            rc = nat.lib.mle_build(self._ctx, nat.as_ptr(th), nat.WHICH[which], nat.as_ptr(out))
        nat.check(rc)
        return out

    def cond_estimate(self) -> float:
        """(max / min diag L)^2 of the last factorization (0.0 before any)."""
        out = np.zeros(1)
        nat.check(nat.lib.mle_ctx_cond_estimate(self._ctx, nat.as_ptr(out)))
        return float(out[0])

    @property
    def sequential_derivs(self) -> bool:
        """True when eval_all reduces the derivative blocks one at a time (they do not fit
        on the device beside the factor: config 5 on one B200; see mle_ctx_seq_derivs)."""
        return bool(nat.lib.mle_ctx_seq_derivs(self._ctx))

    def kernel_profile(self, enable: bool = True):
        """Serialise passes led by this engine and event-time every Ozaki GEMM / slicing."""
        nat.check(nat.lib.mle_kernel_profile(self._ctx, int(bool(enable))))

    def kernel_stats(self) -> dict:
        """Per-kernel sums of the last profiled pass (see mle_kernel_stats)."""
        out = np.zeros(13)  # MLE_KSTATS
        nat.check(nat.lib.mle_kernel_stats(self._ctx, nat.as_ptr(out)))
        return {"gemm_launches": int(out[0]), "gemm_ms": float(out[1]),
                "gemm_fp64_flops": float(out[2]), "gemm_int8_ops": float(out[3]),
                "slice_launches": int(out[4]), "slice_ms": float(out[5]),
                "slice_bytes": float(out[6]), "host_enqueue_ms": float(out[7]),
                "gpu_gap_ms": float(out[8]), "spec_wait_ms": float(out[9]),
                "gen_launches": int(out[10]), "gen_ms": float(out[11]),
                "gen_bytes": float(out[12])}

    def phase_times(self) -> dict:
        out = np.zeros(len(nat.PHASES) + 3)
        nat.check(nat.lib.mle_phase_times(self._ctx, nat.as_ptr(out)))
        rec = {f"{p}_ms": float(v) for p, v in zip(nat.PHASES, out)}
        rec["flops"] = float(out[len(nat.PHASES)])
        rec["gen_bytes"] = float(out[len(nat.PHASES) + 1])
        rec["launches"] = int(out[len(nat.PHASES) + 2])
        return rec
