"""Lock-step batched evaluation for several concurrent Fisher-BT fits.

Replicate fits (BASELINE config 2: five fields of n = 3,600) are independent, and each
Fisher-BT step issues one loglik or eval_all at a time (optimizer.py:345-375).  Instead of
running the fits one after another, or on five streams that each leave most of the GPU
idle at this size, every fit runs its unchanged host loop in its own thread while its
objective hands each evaluation request to a shared :class:`BatchCoordinator`.  When all
live fits have a request pending, the last one to arrive runs them as ONE batched pass
through ``mle_eval_batch`` (each kernel launch covers all datasets), then every fit resumes
with its own result.  Counters, -inf mapping and exception behaviour per fit are exactly
those of :class:`~paper_2601_11437_b200.fisher_bt.LikelihoodObjective`, and the batched
kernels compute each item with the same arithmetic as a single evaluation, so every fit is
bit-identical to running it alone.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import _native as nat
from .fisher_bt import FisherBTConfig, OptResult, fisher_bt
from .likelihood import NotPositiveDefinite
from .matern import MaternParams, SpatialDataset

__all__ = ["BatchCoordinator", "BatchedObjective", "eval_batch", "fit_many"]

LOGLIK, EVAL_ALL = 1, 2


def eval_batch(engines, thetas, modes):
    """One batched pass over several engines (same device and size class).

    Returns a list with, per request, ``(rc, pivot, loglik, grad, fisher)``.
    """
    count = len(engines)
    ctxs = (ctypes.c_void_p * count)(*[e._ctx for e in engines])
    th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float64).reshape(count, 3))
    md = (ctypes.c_int * count)(*[int(m) for m in modes])
    res = np.zeros((count, 13))
    piv = np.full(count, -1, dtype=np.int64)
    rcs = (ctypes.c_int * count)()
    locks = [e._lock for e in engines]
    for lk in locks:
        lk.acquire()
    try:
        rc = nat.lib.mle_eval_batch(ctxs, count, nat.as_ptr(th), md, nat.as_ptr(res),
                                    piv.ctypes.data_as(nat._i64p), rcs)
    finally:
        for lk in locks:
            lk.release()
    nat.check(rc)
    return [(int(rcs[i]), int(piv[i]), float(res[i, 0]), res[i, 1:4].copy(),
             res[i, 4:13].reshape(3, 3).copy()) for i in range(count)]


class BatchCoordinator:
    """Gathers one request per live client and runs them as one batch."""

    def __init__(self, clients: int):
        self._cv = threading.Condition()
        self._live = clients
        self._pending = {}
        self._results = {}
        self._error = None
        self.batches = 0
        self.requests = 0
        self.eval_passes = 0
        # device-side accounting of every batch (CUDA events on the launching stream)
        self.acc = {"flops": 0.0, "gen_ms": 0.0, "potrf_ms": 0.0, "solve_ms": 0.0,
                    "reduce_ms": 0.0, "gen_bytes": 0.0, "launches": 0, "host_enqueue_ms": 0.0}

    def _run_locked_batch(self):
        # Alignment policy: while some clients wait on a cheap loglik (gen + Cholesky) and
        # others on an eval_all (derivatives + solves), run only the logliks; the eval_all
        # requests then meet in one full pass instead of paying the solve sweeps' latency
        # chain once per straggler.  Every pass makes progress, so no client starves.
        ids = sorted(self._pending)
        cheap = [i for i in ids if self._pending[i][2] == LOGLIK]
        if cheap and len(cheap) < len(ids):
            ids = cheap
        else:
            self.eval_passes += int(any(self._pending[i][2] == EVAL_ALL for i in ids))
        reqs = [self._pending.pop(i) for i in ids]
        self._cv.release()
        try:
            try:
                out = eval_batch([r[0] for r in reqs], [r[1] for r in reqs],
                                 [r[2] for r in reqs])
                err = None
                p = reqs[0][0].phase_times()  # batch-level (same on every member)
                p["host_enqueue_ms"] = reqs[0][0].kernel_stats()["host_enqueue_ms"]
                for key in self.acc:
                    self.acc[key] += p[key]
            except Exception as exc:  # CUDA failures reach every client
                out, err = None, exc
        finally:
            self._cv.acquire()
        self.batches += 1
        self.requests += len(reqs)
        for k, i in enumerate(ids):
            self._results[i] = err if err is not None else out[k]
        self._cv.notify_all()

    def request(self, client: int, engine, theta, mode):
        with self._cv:
            self._pending[client] = (engine, np.asarray(theta, dtype=np.float64), mode)
            if len(self._pending) == self._live:
                self._run_locked_batch()
            while client not in self._results:
                self._cv.wait()
            out = self._results.pop(client)
        if isinstance(out, Exception):
            raise out
        return out

    def retire(self):
        with self._cv:
            self._live -= 1
            if self._live > 0 and len(self._pending) == self._live:
                self._run_locked_batch()


class BatchedObjective:
    """Objective with the reference surface whose evaluations go through a coordinator."""

    def __init__(self, data: SpatialDataset, coord: BatchCoordinator, client: int):
        self.data = data
        self.coord = coord
        self.client = client
        self.loglik_calls = 0
        self.grad_calls = 0

    def loglik(self, theta_vec) -> float:
        self.loglik_calls += 1
        try:
            th = MaternParams.from_array(theta_vec).as_array()
        except ValueError:
            return -math.inf
        rc, piv, ll, _, _ = self.coord.request(self.client, self.data.engine(), th, LOGLIK)
        if rc != nat.MLE_OK:  # NotPositiveDefinite / ValueError -> -inf (optimizer.py:131-134)
            return -math.inf
        return -math.inf if math.isnan(ll) else ll

    def eval_all(self, theta_vec):
        self.loglik_calls += 1
        self.grad_calls += 1
        th = MaternParams.from_array(theta_vec).as_array()
        rc, piv, ll, grad, fisher = self.coord.request(self.client, self.data.engine(), th,
                                                       EVAL_ALL)
        if rc == nat.MLE_NOT_PD:
            raise NotPositiveDefinite(piv)
        if rc != nat.MLE_OK:
            raise ValueError(nat.last_error())
        return ll, grad, fisher


def fit_many(datasets, cfg: FisherBTConfig, objectives_out=None, coordinator_out=None):
    """Run one Fisher-BT fit per dataset concurrently with lock-step batched evaluation.

    Returns the list of :class:`OptResult` (same order as ``datasets``).
    """
    coord = BatchCoordinator(len(datasets))
    if coordinator_out is not None:
        coordinator_out.append(coord)
    objs = [BatchedObjective(d, coord, i) for i, d in enumerate(datasets)]
    results: list = [None] * len(datasets)
    errors: list = [None] * len(datasets)

    def work(i):
        try:
            results[i] = fisher_bt(datasets[i], cfg, objective=objs[i])
        except BaseException as exc:  # surfaced after join
            errors[i] = exc
        finally:
            coord.retire()

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(datasets))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    if objectives_out is not None:
        objectives_out.extend(objs)
    return results
