"""One likelihood evaluation sharded over several GPUs (BASELINE configs 4-5).

The single-GPU engine keeps every N x N matrix of a dataset on one device.  Config 5
(n = 100,000 with a nugget: four 80 GB matrices) cannot; config 4 strong scaling splits one
factorization.  Here the padded matrices are cut into 512-column outer blocks owned
cyclically by the ranks (block b on rank b % world); each rank holds the full-height column
panels of Sigma -> L and of the derivative blocks for its blocks.  Per evaluation
(the algorithm of the single-GPU engine, with the panel traffic made explicit):

* Cholesky, right-looking: the owner of block b factors its panel and broadcasts
  P_b = L[c1:, b] as Ozaki int8 slices; every rank applies the trailing update to its panels.
* Forward sweep X = L^-1 S (eval_all): the owner of b builds W_b = [D_b^-1; -P_b D_b^-1] and
  broadcasts its slices; every rank updates its own columns -- no other traffic.
* Right sweep (lower half of X L^-T): the owner of b re-sends W_b and broadcasts the slices of
  X[:, b]; every rank updates its panels j >= b.
* Reductions: each rank sums over its panels; one all-reduce.

Data motion per evaluation is ~3 x 4 bytes per lower-triangle element (int8 slices), i.e.
~26 GB at n = 65,536 -- a few tens of ms on NVSwitch against ~10 s of tensor-core work.

Backend: ``CudaPanels`` drives the C-ABI (``mle_dctx_*``, libmaternfisher.so) on the rank's
GPU -- the only compute path.  The tests substitute a host FP64 restatement of the same block
steps (tests/dist_host_backend.py, built on the oracle) to exercise this driver and its
collectives with ``gloo`` on CPU (tests/test_multiproc.py).  Communicators:
``TorchComm`` (torch.distributed: NCCL on GPUs, gloo on CPU) and ``InProcessComm`` (several
ranks stepped by one process, e.g. on one GPU for tests).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from .likelihood import LikelihoodEval, NotPositiveDefinite
from .matern import MaternParams

__all__ = ["DistributedEngine", "DistributedObjective", "TorchComm", "InProcessComm", "CudaPanels",
           "results_from_sums"]

LOG_2PI = 1.8378770664093453  # likelihood.py:38
BLOCK = 512


def results_from_sums(sums, n, theta, nugget=0.0, derivs=True):
    """(loglik, grad, fisher) from the reduction sums -- the formulas of engine.cu's
    run_chunk (likelihood.py:85-89, 123-147; nugget block: DESIGN.md §4)."""
    s = np.asarray(sums, float)
    s2 = float(theta[0])
    logdet, quad = s[0], s[1]
    ll = -0.5 * n * LOG_2PI - logdet - 0.5 * quad
    if not derivs:
        return ll, None, None
    tr_a, tr_n, faa, fan, fnn = s[2], s[3], s[4], s[5], s[6]
    yby_a, yby_n = s[11], s[12]
    grad = np.empty(3)
    f = np.empty((3, 3))
    grad[1] = -0.5 * tr_a + 0.5 * yby_a
    grad[2] = -0.5 * tr_n + 0.5 * yby_n
    f[1, 1] = 0.5 * faa
    f[1, 2] = f[2, 1] = 0.5 * fan
    f[2, 2] = 0.5 * fnn
    if nugget == 0.0:
        grad[0] = (quad - n) / (2.0 * s2)
        f[0, 0] = n / (2.0 * s2 * s2)
        f[0, 1] = f[1, 0] = tr_a / (2.0 * s2)
        f[0, 2] = f[2, 0] = tr_n / (2.0 * s2)
    else:
        t = nugget
        tr_m, fam, fnm, fmm, yby_m = s[7], s[8], s[9], s[10], s[13]
        grad[0] = -0.5 * (n - t * tr_m) / s2 + 0.5 * (quad - t * yby_m) / s2
        f[0, 0] = 0.5 * (n - 2.0 * t * tr_m + t * t * fmm) / (s2 * s2)
        f[0, 1] = f[1, 0] = 0.5 * (tr_a - t * fam) / s2
        f[0, 2] = f[2, 0] = 0.5 * (tr_n - t * fnm) / s2
    return ll, grad, f


# --------------------------------------------------------------------------- communicators
class TorchComm:
    """torch.distributed collectives for the one rank this process hosts."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.local_ranks = [self.rank]

    def broadcast(self, bufs, src):
        self.dist.broadcast(bufs[0], src=src, group=self.group)
        if bufs[0].is_cuda:
            import torch

            torch.cuda.current_stream(bufs[0].device).synchronize()

    def all_reduce_sum(self, arrs):
        import torch

        t = torch.tensor(arrs[0], dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return [t.cpu().numpy()]


class InProcessComm:
    """Several ranks stepped by one process (all buffers visible): broadcast = copy."""

    def __init__(self, world):
        self.world = world
        self.local_ranks = list(range(world))

    def broadcast(self, bufs, src):
        for r, b in enumerate(bufs):
            if r != src:
                b.copy_(bufs[src])
        if bufs[src].is_cuda:
            import torch

            torch.cuda.synchronize(bufs[src].device)

    def all_reduce_sum(self, arrs):
        tot = np.sum(np.stack(arrs), axis=0)
        return [tot.copy() for _ in arrs]


# ------------------------------------------------------------------------------- backends
class CudaPanels:
    """One rank's panels on its GPU, through the mle_dctx_* C-ABI."""

    def __init__(self, locations, values, rank, world, device=0, nugget=0.0):
        import torch

        from . import _native as nat

        self.nat = nat
        self.torch = torch
        loc = np.ascontiguousarray(np.asarray(locations, float))
        z = np.ascontiguousarray(np.asarray(values, float))
        self.n = loc.shape[0]
        self.device = device
        self.nugget = float(nugget)
        h = ctypes.c_void_p()
        nat.check(nat.lib.mle_dctx_create(nat.as_ptr(loc), nat.as_ptr(z), self.n, device,
                                          self.nugget, rank, world, ctypes.byref(h)))
        self._d = h
        lay = np.zeros(7, dtype=np.int64)
        nat.check(nat.lib.mle_dctx_layout(self._d, lay.ctypes.data_as(nat._i64p)))
        self.N, self.nb, self.nmat = int(lay[0]), int(lay[1]), int(lay[5])
        self._bytes = {"P": int(lay[2]), "W": int(lay[3]), "X": int(lay[4])}

    def close(self):
        d, self._d = getattr(self, "_d", None), None
        if d:
            self.nat.lib.mle_dctx_destroy(d)

    __del__ = close

    def exchange(self, kind):
        return self.torch.empty(self._bytes[kind], dtype=self.torch.uint8,
                                device=f"cuda:{self.device}")

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    def begin(self, theta, derivs):
        th = np.ascontiguousarray(np.asarray(theta, float))
        self.nat.check(self.nat.lib.mle_dctx_begin(self._d, self.nat.as_ptr(th), int(derivs)))

    def factor(self, b, exch):
        self.nat.check(self.nat.lib.mle_dctx_factor(self._d, b, self._p(exch)))

    def update(self, b, exch):
        self.nat.check(self.nat.lib.mle_dctx_update(self._d, b, self._p(exch)))

    def wblock(self, b, exch):
        self.nat.check(self.nat.lib.mle_dctx_wblock(self._d, b, self._p(exch)))

    def forward(self, b, exch):
        self.nat.check(self.nat.lib.mle_dctx_forward(self._d, b, self._p(exch)))

    def right_operand(self, b, exch):
        self.nat.check(self.nat.lib.mle_dctx_right_operand(self._d, b, self._p(exch)))

    def right(self, b, exch_w, exch_x):
        self.nat.check(self.nat.lib.mle_dctx_right(self._d, b, self._p(exch_w),
                                                   self._p(exch_x)))

    def partials(self):
        out = np.zeros(16)
        self.nat.check(self.nat.lib.mle_dctx_partials(self._d, self.nat.as_ptr(out)))
        return out


# --------------------------------------------------------------------------------- driver
class DistributedEngine:
    """loglik / eval_all of one dataset over ``comm``'s ranks (the reference's surface)."""

    def __init__(self, locations, values, comm, nugget: float = 0.0, device: int = 0,
                 backend=None):
        """``backend(locations, values, rank, world, nugget)`` builds one rank's panels
        (default: :class:`CudaPanels` on ``device``; tests pass a host restatement)."""
        self.comm = comm
        self.nugget = float(nugget)
        world = comm.world
        make = backend or (lambda loc, z, r, w, t: CudaPanels(loc, z, r, w, device, t))
        self.ranks = [make(locations, values, r, world, nugget) for r in comm.local_ranks]
        self.local = list(comm.local_ranks)
        self.n = self.ranks[0].n
        self.nb = self.ranks[0].nb
        self.world = world
        self._ex = {k: [r.exchange(k) for r in self.ranks] for k in ("P", "W", "X")}

    def close(self):
        for r in self.ranks:
            r.close()

    def _owner(self, b):
        return b % self.world

    def _local(self, rank):
        return self.local.index(rank) if rank in self.local else None

    def _run(self, theta, derivs):
        th = MaternParams.from_array(theta).as_array()
        for r in self.ranks:
            r.begin(th, derivs)
        P, W, X = self._ex["P"], self._ex["W"], self._ex["X"]
        for b in range(self.nb):  # right-looking Cholesky
            o = self._owner(b)
            lo = self._local(o)
            if lo is not None:
                self.ranks[lo].factor(b, P[lo])
            if b + 1 < self.nb:
                self.comm.broadcast(P, o)
                for r, be in enumerate(self.ranks):
                    be.update(b, P[r])
        if derivs:
            for b in range(self.nb):  # forward sweep X = L^-1 S on every rank's own columns
                o = self._owner(b)
                lo = self._local(o)
                if lo is not None:
                    self.ranks[lo].wblock(b, W[lo])
                self.comm.broadcast(W, o)
                for r, be in enumerate(self.ranks):
                    be.forward(b, W[r])
            for b in range(self.nb):  # right sweep (lower half of X L^-T)
                o = self._owner(b)
                lo = self._local(o)
                if lo is not None:
                    self.ranks[lo].wblock(b, W[lo])
                    self.ranks[lo].right_operand(b, X[lo])
                self.comm.broadcast(W, o)
                self.comm.broadcast(X, o)
                for r, be in enumerate(self.ranks):
                    be.right(b, W[r], X[r])
        local = [be.partials() for be in self.ranks]
        parts = self.comm.all_reduce_sum(local)[0]
        if parts[14] > 0:
            # every failed rank reports its first failing pivot; the smallest wins (LAPACK)
            big = float(2 ** 52)
            vecs = []
            for r, p in zip(self.local, local):
                v = np.zeros(self.world)
                v[r] = p[15] if p[14] > 0 else big
                vecs.append(v)
            raise NotPositiveDefinite(int(np.min(self.comm.all_reduce_sum(vecs)[0])))
        return th, parts

    def loglik(self, theta) -> float:
        th, s = self._run(theta, False)
        return results_from_sums(s, self.n, th, self.nugget, derivs=False)[0]

    def eval_all(self, theta):
        th, s = self._run(theta, True)
        return results_from_sums(s, self.n, th, self.nugget)

    def grad_and_fisher(self, theta) -> LikelihoodEval:
        ll, g, f = self.eval_all(theta)
        return LikelihoodEval(loglik=ll, grad=g, fisher=f)


class DistributedObjective:
    """The reference's objective surface (optimizer.py:114-142) over a DistributedEngine:
    ``loglik`` counts one call and maps NotPositiveDefinite / ValueError / NaN to -inf;
    ``eval_all`` counts one call of each kind and propagates errors.  Every rank runs the
    same deterministic host loop (fisher_bt) over its own instance, so every call is a
    collective entered by all ranks in the same order."""

    def __init__(self, engine: DistributedEngine):
        self.engine = engine
        self.loglik_calls = 0
        self.grad_calls = 0

    def loglik(self, theta_vec) -> float:
        self.loglik_calls += 1
        try:
            value = self.engine.loglik(MaternParams.from_array(theta_vec).as_array())
        except (NotPositiveDefinite, ValueError):
            return -math.inf
        return -math.inf if math.isnan(value) else value

    def eval_all(self, theta_vec):
        self.loglik_calls += 1
        self.grad_calls += 1
        return self.engine.eval_all(MaternParams.from_array(theta_vec).as_array())
