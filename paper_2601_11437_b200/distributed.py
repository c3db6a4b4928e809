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
SUMS = 14  # MLE_DCTX_SUMS


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
        # stream-ordered (asynchronous) block steps need NCCL: its collectives are ordered on
        # the issuing CUDA stream; gloo copies through the host
        self.stream_ordered = dist.get_backend(group) == "nccl"

    def _src(self, src):
        """Group rank -> the global rank torch.distributed.broadcast expects."""
        if self.group is None:
            return src
        return self.dist.get_global_rank(self.group, src)

    def broadcast(self, bufs, src):
        """Blocking: returns when this rank's buffer holds the owner's bytes."""
        self.dist.broadcast(bufs[0], src=self._src(src), group=self.group)
        if bufs[0].is_cuda:
            import torch

            torch.cuda.current_stream(bufs[0].device).synchronize()

    def broadcast_on_stream(self, buf, src):
        """Enqueued on the current CUDA stream (NCCL); no host synchronisation."""
        self.dist.broadcast(buf, src=self._src(src), group=self.group)

    def all_reduce_sum(self, arrs):
        import torch

        t = torch.tensor(arrs[0], dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return [t.cpu().numpy()]


class InProcessComm:
    """Several ranks stepped by one process (all buffers visible): broadcast = copy."""

    stream_ordered = False

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
        self.rank, self.world = rank, world
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

    def update(self, b, exch, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        self.nat.check(self.nat.lib.mle_dctx_update_range(self._d, b, self._p(exch), lo, hi))

    def wblock(self, b, exch):
        """W_b on the owner (kept); exch None: no copy into an exchange buffer."""
        ptr = ctypes.c_void_p(None) if exch is None else self._p(exch)
        self.nat.check(self.nat.lib.mle_dctx_wblock(self._d, b, ptr))

    def forward(self, b, exch, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        self.nat.check(self.nat.lib.mle_dctx_forward_range(self._d, b, self._p(exch), lo, hi))

    def ts_owner(self, b, exch_x):
        self.nat.check(self.nat.lib.mle_dctx_2s_owner(self._d, b, self._p(exch_x)))

    def ts_finish(self, b):
        self.nat.check(self.nat.lib.mle_dctx_2s_finish(self._d, b))

    def ts_update(self, b, exch_x, exch_p, lo=0, hi=None):
        hi = self.nb if hi is None else hi
        self.nat.check(self.nat.lib.mle_dctx_2s_update_range(self._d, b, self._p(exch_x),
                                                             self._p(exch_p), lo, hi))

    def panel_slices(self, b, exch_p):
        self.nat.check(self.nat.lib.mle_dctx_panel_slices(self._d, b, self._p(exch_p)))

    def right_operand(self, b, exch):
        self.nat.check(self.nat.lib.mle_dctx_right_operand(self._d, b, self._p(exch)))

    def right(self, b, exch_w, exch_x, lo=0, hi=None):
        """exch_w None: W_b from this rank's W cache (wcache)."""
        hi = self.nb if hi is None else hi
        w = None if exch_w is None else self._p(exch_w)
        self.nat.check(self.nat.lib.mle_dctx_right_range(self._d, b, w, self._p(exch_x), lo,
                                                         hi))

    def wcache(self, on=True):
        """Keep every W_b (~3.5 N^2 bytes) for the right sweep; False if it does not fit."""
        rc = self.nat.lib.mle_dctx_wcache(self._d, int(bool(on)))
        if rc == self.nat.MLE_CUDA_ERROR:
            return False
        self.nat.check(rc)
        return bool(on)

    def set_async(self, on=True):
        self.nat.check(self.nat.lib.mle_dctx_set_async(self._d, int(bool(on))))

    def stream(self):
        """The rank's compute stream as a torch stream (its block steps run on it)."""
        h = ctypes.c_void_p()
        self.nat.check(self.nat.lib.mle_dctx_stream(self._d, ctypes.byref(h)))
        return self.torch.cuda.ExternalStream(h.value, device=f"cuda:{self.device}")

    def partials(self):
        out = np.zeros(16)
        self.nat.check(self.nat.lib.mle_dctx_partials(self._d, self.nat.as_ptr(out)))
        return out

    def panel_partials(self):
        """({block: 14 sums}, failed, pivot) for this rank's panels."""
        owned = list(range(self.rank, self.nb, self.world))
        out = np.zeros(len(owned) * SUMS + 2)
        self.nat.check(self.nat.lib.mle_dctx_panel_partials(self._d, self.nat.as_ptr(out)))
        per = {b: out[q * SUMS:(q + 1) * SUMS].copy() for q, b in enumerate(owned)}
        return per, out[-2] > 0, out[-1]


# --------------------------------------------------------------------------------- driver
class _Exchange:
    """Double-buffered exchange slots of one kind (P, W or X) and their ordering.

    Synchronous mode (gloo, in-process ranks, host backends): every block step has drained its
    stream, ``send`` is a blocking broadcast, nothing else to order.  Stream-ordered mode
    (NCCL; CudaPanels in async mode): a slot's broadcast runs on the rank's communication
    stream after (i) the owner's producing step (event on the compute stream) and (ii) the
    previous consumer of the slot (event); the consuming step waits for the broadcast's
    event -- so broadcasts of block b + 1 overlap the trailing GEMMs of block b."""

    def __init__(self, engine, kind):
        self.e = engine
        self.buf = [[r.exchange(kind) for r in engine.ranks] for _ in range(2)]
        self.free = [None, None]  # per slot: per local rank, event after the last consumer

    def slot(self, b):
        return self.buf[b % 2]

    def produced(self, b, r):
        """Owner r (local index) has queued the step that fills slot b."""
        if not self.e.async_steps:
            return None
        import torch

        ev = torch.cuda.Event()
        ev.record(self.e.streams[r])
        return ev

    def send(self, b, owner, ready):
        """Broadcast slot b from ``owner`` (group rank); ``ready`` = produced(...) or None."""
        bufs = self.slot(b)
        if not self.e.async_steps:
            self.e.comm.broadcast(bufs, owner)
            return
        import torch

        r = 0  # one local rank per process in stream-ordered mode
        cs = self.e.comm_streams[r]
        if ready is not None:
            cs.wait_event(ready)
        if self.free[b % 2] is not None:
            cs.wait_event(self.free[b % 2][r])
        with torch.cuda.stream(cs):
            self.e.comm.broadcast_on_stream(bufs[r], owner)
            ev = torch.cuda.Event()
            ev.record(cs)
        self.e.streams[r].wait_event(ev)

    def consumed(self, b):
        """Every consumer of slot b on this rank has been queued."""
        if not self.e.async_steps:
            return
        import torch

        evs = []
        for st in self.e.streams:
            ev = torch.cuda.Event()
            ev.record(st)
            evs.append(ev)
        self.free[b % 2] = evs


class DistributedEngine:
    """loglik / eval_all of one dataset over ``comm``'s ranks (the reference's surface)."""

    def __init__(self, locations, values, comm, nugget: float = 0.0, device: int = 0,
                 backend=None, overlap=None, wcache=None, solve=None):
        """``backend(locations, values, rank, world, nugget)`` builds one rank's panels
        (default: :class:`CudaPanels` on ``device``; tests pass a host restatement).

        ``overlap`` (default: on for NCCL with the CUDA backend): block steps are queued
        asynchronously and the panel / W / X broadcasts run on a communication stream under
        the trailing GEMMs.  ``wcache`` (default: on when the memory is there): every rank
        keeps the forward sweep's W_b for the right sweep instead of a second broadcast."""
        self.comm = comm
        self.nugget = float(nugget)
        world = comm.world
        make = backend or (lambda loc, z, r, w, t: CudaPanels(loc, z, r, w, device, t))
        self.ranks = [make(locations, values, r, world, nugget) for r in comm.local_ranks]
        self.local = list(comm.local_ranks)
        self.n = self.ranks[0].n
        self.nb = self.ranks[0].nb
        self.world = world
        can_async = (backend is None and getattr(comm, "stream_ordered", False)
                     and len(self.ranks) == 1)
        self.async_steps = can_async if overlap is None else (bool(overlap) and can_async)
        self.streams, self.comm_streams = [], []
        if self.async_steps:
            import torch

            for r in self.ranks:
                r.set_async(True)
                self.streams.append(r.stream())
                self.comm_streams.append(torch.cuda.Stream(device=r.device))
        self._ex = {k: _Exchange(self, k) for k in ("P", "W", "X")}
        # solve formulation, as in the single-context engine: the two-sided reduction from
        # N >= 16,384 (MLE_SOLVE=w|2s overrides), the full forward + right sweeps below
        import os

        env = os.environ.get("MLE_SOLVE")
        big_n = self.ranks[0].N
        self.solve = solve or (env if env in ("w", "2s") else ("2s" if big_n >= 16384 else "w"))
        if self.solve == "2s" and not all(hasattr(r, "ts_owner") for r in self.ranks):
            self.solve = "w"
        want = True if wcache is None else bool(wcache)
        self.wcache = False
        if want and all(hasattr(r, "wcache") for r in self.ranks):
            ok = [r.wcache(True) for r in self.ranks]
            # every rank must agree (the right sweep's broadcast pattern depends on it)
            votes = self.comm.all_reduce_sum([np.array([1.0 if o else 0.0]) for o in ok])[0]
            self.wcache = float(votes[0]) > world - 0.5
            if not self.wcache:
                for r in self.ranks:
                    r.wcache(False)

    def close(self):
        for r in self.ranks:
            r.close()

    def _owner(self, b):
        return b % self.world

    def _local(self, rank):
        return self.local.index(rank) if rank in self.local else None

    def _others(self, b_next):
        """Range pieces of the blocks other than b_next: [(0, b_next), (b_next + 1, nb)]."""
        return [(0, b_next), (b_next + 1, self.nb)]

    def _run(self, theta, derivs):
        th = MaternParams.from_array(theta).as_array()
        for r in self.ranks:
            r.begin(th, derivs)
        self._cholesky()
        if derivs and self.solve == "2s":
            self._two_sided()
            self._deferred_sweep()
        elif derivs:
            self._forward_sweep()
            self._right_sweep()
        # Per-panel sums placed in a (blocks x sums) array (zeros elsewhere: adding them is
        # exact), one all-reduce, then the panels added in block order: the result does not
        # depend on the number of ranks or on who owns what.
        width = SUMS + 2
        vecs, fails = [], []
        for r, be in zip(self.local, self.ranks):
            v = np.zeros((self.nb + 1) * width)
            if hasattr(be, "panel_partials"):
                per, failed, pivot = be.panel_partials()
                for b, sums in per.items():
                    v[b * width:b * width + SUMS] = sums
            else:  # host restatement backends: one row per rank
                p = be.partials()
                v[r * width:r * width + SUMS] = p[:SUMS]
                failed, pivot = p[14] > 0, p[15]
            v[self.nb * width + SUMS] = 1.0 if failed else 0.0
            vecs.append(v)
            fails.append((failed, pivot))
        tot = self.comm.all_reduce_sum(vecs)[0].reshape(self.nb + 1, width)
        parts = np.zeros(16)
        for b in range(self.nb):
            parts[:SUMS] += tot[b, :SUMS]
        if tot[self.nb, SUMS] > 0:
            # every failed rank reports its first failing pivot; the smallest wins (LAPACK)
            big = float(2 ** 52)
            piv = []
            for r, (failed, pivot) in zip(self.local, fails):
                v = np.zeros(self.world)
                v[r] = pivot if failed else big
                piv.append(v)
            raise NotPositiveDefinite(int(np.min(self.comm.all_reduce_sum(piv)[0])))
        return th, parts

    # Right-looking Cholesky with look-ahead: the owner of block b + 1 applies block b's update
    # to its panel b + 1 first, factors it and sends P_{b+1}; the remaining updates of block b
    # (every rank) run while P_{b+1} is in flight.  Panel updates are independent GEMMs, so
    # the split changes no arithmetic.
    def _cholesky(self):
        P, nb = self._ex["P"], self.nb

        def factor_and_send(b):
            o = self._owner(b)
            lo = self._local(o)
            ready = None
            if lo is not None:
                self.ranks[lo].factor(b, P.slot(b)[lo])
                ready = P.produced(b, lo)
            if b + 1 < nb:
                P.send(b, o, ready)

        factor_and_send(0)
        for b in range(nb - 1):
            nxt = b + 1
            on = self._local(self._owner(nxt))
            for r, be in enumerate(self.ranks):
                if r == on:
                    be.update(b, P.slot(b)[r], nxt, nxt + 1)
            factor_and_send(nxt)
            for r, be in enumerate(self.ranks):
                pieces = self._others(nxt) if r == on else [(0, nb)]
                for lo, hi in pieces:
                    be.update(b, P.slot(b)[r], lo, hi)
            P.consumed(b)

    # Forward sweep X = L^-1 S: W_b depends only on L, so the owner of b + 1 builds and sends
    # W_{b+1} ahead of block b's GEMMs.
    def _forward_sweep(self):
        W, nb = self._ex["W"], self.nb

        def build_and_send(b):
            o = self._owner(b)
            lo = self._local(o)
            ready = None
            if lo is not None:
                self.ranks[lo].wblock(b, W.slot(b)[lo])
                ready = W.produced(b, lo)
            W.send(b, o, ready)

        build_and_send(0)
        for b in range(nb):
            if b + 1 < nb:
                build_and_send(b + 1)
            for r, be in enumerate(self.ranks):
                be.forward(b, W.slot(b)[r])
            W.consumed(b)

    # Right sweep (lower half of X L^-T): the owner of b + 1 applies block b to its panel
    # b + 1 first, slices X[:, b+1] and sends it; W_b comes from the W cache (or is re-sent).
    def _right_sweep(self):
        W, X, nb = self._ex["W"], self._ex["X"], self.nb

        def operand_and_send(b):
            o = self._owner(b)
            lo = self._local(o)
            ready = None
            if lo is not None:
                if not self.wcache:
                    self.ranks[lo].wblock(b, W.slot(b)[lo])
                self.ranks[lo].right_operand(b, X.slot(b)[lo])
                ready = X.produced(b, lo)
            if not self.wcache:
                W.send(b, o, ready)
            X.send(b, o, ready)

        def wb(b, r):
            return None if self.wcache else W.slot(b)[r]

        operand_and_send(0)
        for b in range(nb):
            nxt = b + 1
            on = self._local(self._owner(nxt)) if nxt < nb else None
            if nxt < nb:
                for r, be in enumerate(self.ranks):
                    if r == on:
                        be.right(b, wb(b, r), X.slot(b)[r], nxt, nxt + 1)
                operand_and_send(nxt)
            for r, be in enumerate(self.ranks):
                pieces = self._others(nxt) if r == on else [(0, nb)]
                for lo, hi in pieces:
                    be.right(b, wb(b, r), X.slot(b)[r], lo, hi)
            X.consumed(b)
            if not self.wcache:
                W.consumed(b)

    # Two-sided reduction (the single-context solves_2s recurrence) on the
    # panels: the owner of block b runs steps (1)-(3) on its panel and sends the slices of S21
    # and of P_b = L21; every rank applies the syr2k (4) to its panels j > b; the owner
    # finishes with (5).  Look-ahead: the owner of b + 1 updates that panel first.
    def _two_sided(self):
        X, P, nb = self._ex["X"], self._ex["P"], self.nb

        def owner_step(b):
            o = self._owner(b)
            lo = self._local(o)
            ready = None
            if lo is not None:
                self.ranks[lo].wblock(b, None)  # D_b^-1 and W_b (kept for the deferred sweep)
                self.ranks[lo].ts_owner(b, X.slot(b)[lo])
                if b + 1 < nb:
                    self.ranks[lo].panel_slices(b, P.slot(b)[lo])
                ready = X.produced(b, lo)
            if b + 1 < nb:
                X.send(b, o, ready)
                P.send(b, o, ready)

        owner_step(0)
        for b in range(nb):
            o = self._local(self._owner(b))
            if b + 1 >= nb:
                break
            if o is not None:
                self.ranks[o].ts_finish(b)
            nxt = b + 1
            on = self._local(self._owner(nxt))
            for r, be in enumerate(self.ranks):
                if r == on:
                    be.ts_update(b, X.slot(b)[r], P.slot(b)[r], nxt, nxt + 1)
            owner_step(nxt)
            for r, be in enumerate(self.ranks):
                pieces = self._others(nxt) if r == on else [(0, nb)]
                for lo, hi in pieces:
                    be.ts_update(b, X.slot(b)[r], P.slot(b)[r], lo, hi)
            X.consumed(b)
            P.consumed(b)

    # Deferred sweep: S21 <- L22^-1 S21 for every block column, as the block-inverse forward
    # sweep restricted to the panels left of each row block; W_b goes out once.
    def _deferred_sweep(self):
        W, nb = self._ex["W"], self.nb
        for b in range(1, nb):
            o = self._owner(b)
            lo = self._local(o)
            ready = None
            if lo is not None:
                self.ranks[lo].wblock(b, W.slot(b)[lo])  # recomputed: ~0.3% of the work
                ready = W.produced(b, lo)
            W.send(b, o, ready)
            for r, be in enumerate(self.ranks):
                be.forward(b, W.slot(b)[r], 0, b)
            W.consumed(b)

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
