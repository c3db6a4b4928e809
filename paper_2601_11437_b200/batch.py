"""Lock-step batched evaluation for several concurrent Fisher-BT fits.

Replicate fits (BASELINE config 2: five fields of n = 3,600) are independent, and each
Fisher-BT step issues one loglik or eval_all at a time (optimizer.py:345-375).  Instead of
running the fits one after another, or on five streams that each leave most of the GPU
idle at this size, :func:`fit_many` runs every fit as the request generator
``fisher_bt_gen`` (the unchanged host algorithm) and answers the pending requests of all
live fits with ONE batched pass through ``mle_eval_batch`` (each kernel launch covers all
datasets), from a single host thread.  Counters, -inf mapping and exception behaviour per
fit are exactly those of :class:`~paper_2601_11437_b200.fisher_bt.LikelihoodObjective`, and
the batched kernels compute each item with the same arithmetic as a single evaluation, so
every fit is bit-identical to running it alone.

:class:`BatchCoordinator` / :class:`BatchedObjective` offer the same batching to callers that
run their own objective-calling loops in threads.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

from . import _native as nat
from .fisher_bt import FisherBTConfig, OptResult, fisher_bt
from .likelihood import NotPositiveDefinite
from .matern import MaternParams, SpatialDataset

__all__ = ["BatchCoordinator", "BatchedObjective", "LockstepStats", "eval_batch", "fit_many"]

LOGLIK, EVAL_ALL = 1, 2
LOGLIK_MODE, EVAL_MODE = LOGLIK, EVAL_ALL  # mle_eval_batch modes


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


def _loglik_value(rc, ll):
    """loglik's mapping (optimizer.py:129-134): NotPositiveDefinite / ValueError / NaN -> -inf;
    a CUDA failure is raised, never mapped."""
    if rc in (nat.MLE_NOT_PD, nat.MLE_INVALID):
        return -math.inf
    if rc != nat.MLE_OK:
        raise RuntimeError(f"CUDA failure in a batched log-likelihood: {nat.last_error()}")
    return -math.inf if math.isnan(ll) else ll


def _unique_thetas(thetas):
    """(valid unique theta arrays in first-seen order, item -> unique index or None)."""
    order, where, slot = [], {}, []
    for t in thetas:
        try:
            th = MaternParams.from_array(t).as_array()
        except ValueError:
            slot.append(None)
            continue
        key = th.tobytes()
        if key not in where:
            where[key] = len(order)
            order.append(th)
        slot.append(where[key])
    return order, slot


def batched_logliks(data: SpatialDataset, thetas):
    """Log-likelihoods of one dataset at several independent theta, as batched passes over
    the dataset's engine and its helper contexts (SpatialDataset.engines).  Equal theta are
    evaluated once (the engine is deterministic); invalid theta give -inf without a pass.
    Every value is bit-identical to a single ``log_likelihood`` call."""
    order, slot = _unique_thetas(thetas)
    vals = []
    if order:
        engines = data.engines(len(order))
        for start in range(0, len(order), len(engines)):
            chunk = order[start:start + len(engines)]
            out = eval_batch(engines[:len(chunk)], chunk, [LOGLIK_MODE] * len(chunk))
            vals.extend(_loglik_value(rc, ll) for rc, _, ll, _, _ in out)
    return [-math.inf if k is None else vals[k] for k in slot]


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
                    "reduce_ms": 0.0, "gen_bytes": 0.0, "launches": 0, "host_enqueue_ms": 0.0,
                    "gpu_gap_ms": 0.0, "spec_wait_ms": 0.0}

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
                ks = reqs[0][0].kernel_stats()
                for key in ("host_enqueue_ms", "gpu_gap_ms", "spec_wait_ms"):
                    p[key] = ks[key]
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


class _Counters:
    """Per-fit call counters with the reference objective's semantics (optimizer.py:127-138)."""

    def __init__(self, data: SpatialDataset):
        self.data = data
        self.loglik_calls = 0
        self.grad_calls = 0


class LockstepStats:
    """Accounting of a lock-step run (same fields as BatchCoordinator)."""

    def __init__(self):
        self.batches = 0
        self.requests = 0
        self.eval_passes = 0
        self.acc = {"flops": 0.0, "gen_ms": 0.0, "potrf_ms": 0.0, "solve_ms": 0.0,
                    "reduce_ms": 0.0, "gen_bytes": 0.0, "launches": 0, "host_enqueue_ms": 0.0,
                    "gpu_gap_ms": 0.0, "spec_wait_ms": 0.0}


def fit_many(datasets, cfg: FisherBTConfig, objectives_out=None, coordinator_out=None,
             groups=None, return_exceptions=False):
    """Run one Fisher-BT fit per dataset concurrently with lock-step batched evaluation.

    Every fit is the request generator ``fisher_bt_gen`` (the unchanged Algorithm 1); a host
    thread collects the pending request of every live fit of its group and answers them with
    ONE batched engine pass (``mle_eval_batch``), so no thread hand-offs sit between GPU passes.
    Alignment policy as in :class:`BatchCoordinator`: while some fits wait on a loglik and
    others on an eval_all, only the logliks run.  Counters, -inf mapping and exceptions per fit
    are those of :class:`~paper_2601_11437_b200.fisher_bt.LikelihoodObjective`; each fit is
    bit-identical to running it alone.  Returns the list of :class:`OptResult` (same order as
    ``datasets``).

    ``groups``: the fits are split (interleaved) into this many lock-step groups, each driven
    by its own host thread on disjoint contexts, so one group's latency-bound Cholesky overlaps
    the other's tensor-core solves on the GPU.  Default: 2 for four or more fits (env
    ``MLE_FIT_GROUPS`` overrides), else 1.
    """
    n = len(datasets)
    if groups is None:
        env = os.environ.get("MLE_FIT_GROUPS")
        groups = int(env) if env else (2 if n >= 4 else 1)
    groups = max(1, min(int(groups), n)) if n else 1
    if groups == 1:
        return _finish(_fit_group(datasets, cfg, objectives_out, coordinator_out),
                       return_exceptions)
    parts = [list(range(g, n, groups)) for g in range(groups)]
    res = [None] * groups
    objs = [[] for _ in range(groups)]
    stats = [[] for _ in range(groups)]
    errors = []

    def work(g):
        try:
            res[g] = _fit_group([datasets[i] for i in parts[g]], cfg, objs[g], stats[g])
        except BaseException as exc:  # re-raised in the caller's thread
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(g,)) for g in range(groups)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    results = [None] * n
    counters = [None] * n
    for g, idx in enumerate(parts):
        for j, i in enumerate(idx):
            results[i] = res[g][j]
            counters[i] = objs[g][j]
    if objectives_out is not None:
        objectives_out.extend(counters)
    if coordinator_out is not None:
        for st in stats:
            coordinator_out.extend(st)
    return _finish(results, return_exceptions)


def _finish(results, return_exceptions):
    """Every fit has run to its end.  A failed fit's slot holds its exception
    (``return_exceptions``), or the first failed fit in dataset order raises -- what running
    the fits one after another would raise first."""
    if return_exceptions:
        return [r.exc if isinstance(r, _FitFailure) else r for r in results]
    for r in results:
        if isinstance(r, _FitFailure):
            raise r.exc
    return results


def _fit_group(datasets, cfg: FisherBTConfig, objectives_out=None, coordinator_out=None):
    """One lock-step group of :func:`fit_many`, driven by the calling thread.

    A fit's own failure (InitializationFailed, or NotPositiveDefinite out of eval_all) ends
    that fit only: it is re-raised from :func:`fit_many` after every other fit of the group
    has finished, exactly as running the fits one by one would surface it first."""
    from .fisher_bt import EVAL_ALL, LOGLIK, LOGLIK_MANY, fisher_bt_gen

    stats = LockstepStats()
    if coordinator_out is not None:
        coordinator_out.append(stats)
    cnt = [_Counters(d) for d in datasets]
    gens = [fisher_bt_gen(cfg, c) for c in cnt]
    results: list = [None] * len(datasets)
    pending = {}

    def advance(i, how, value):
        try:
            pending[i] = how(value) if how is not None else next(gens[i])
        except StopIteration as stop:
            pending.pop(i, None)
            results[i] = stop.value
        except Exception as exc:  # this fit failed; the others go on
            pending.pop(i, None)
            results[i] = _FitFailure(exc)

    for i in range(len(gens)):
        advance(i, None, None)
    while pending:
        ids = sorted(pending)
        cheap = [i for i in ids if pending[i][0] != EVAL_ALL]
        if cheap and len(cheap) < len(ids):
            ids = cheap
        else:
            stats.eval_passes += int(any(pending[i][0] == EVAL_ALL for i in ids))
        answers = {}
        items = []  # (fit, engine, theta, mode, unique slot)
        many = {}   # fit -> (item slots, per-theta unique index)
        for i in ids:
            kind, theta_vec = pending[i]
            c = cnt[i]
            if kind == LOGLIK_MANY:
                c.loglik_calls += len(theta_vec)
                order, slot = _unique_thetas(theta_vec)
                engines = datasets[i].engines(len(order)) if order else []
                first = len(items)
                for k, th in enumerate(order):
                    items.append((i, engines[k % len(engines)], th, LOGLIK_MODE))
                many[i] = (first, len(order), slot)
                continue
            c.loglik_calls += 1
            if kind == EVAL_ALL:
                c.grad_calls += 1
            try:
                th = MaternParams.from_array(theta_vec).as_array()
            except ValueError as exc:  # loglik -> -inf; eval_all raises (optimizer.py:131-138)
                answers[i] = (-math.inf, None) if kind == LOGLIK else (None, exc)
                continue
            items.append((i, datasets[i].engine(), th,
                          LOGLIK_MODE if kind == LOGLIK else EVAL_MODE))
        # rounds: an engine appears at most once per batched pass
        outs = [None] * len(items)
        todo = list(range(len(items)))
        while todo:
            seen, run, later = set(), [], []
            for k in todo:
                (run if id(items[k][1]) not in seen else later).append(k)
                seen.add(id(items[k][1]))
            todo = later
            try:
                out = eval_batch([items[k][1] for k in run], [items[k][2] for k in run],
                                 [items[k][3] for k in run])
                p = items[run[0]][1].phase_times()
                ks = items[run[0]][1].kernel_stats()
                for key in ("host_enqueue_ms", "gpu_gap_ms", "spec_wait_ms"):
                    p[key] = ks[key]
                for key in stats.acc:
                    stats.acc[key] += p[key]
                for k, o in zip(run, out):
                    outs[k] = o
            except Exception as exc:  # CUDA failures reach every fit of the pass
                for k in run:
                    outs[k] = exc
            stats.batches += 1
            stats.requests += len(run)
        for k, (i, _, _, mode) in enumerate(items):
            if i in many:
                continue
            o = outs[k]
            if isinstance(o, Exception):
                answers[i] = (None, o)
                continue
            rc, piv, ll, grad, fisher = o
            if mode == LOGLIK_MODE:
                ok = rc == nat.MLE_OK and not math.isnan(ll)
                answers[i] = (ll if ok else -math.inf, None)
            elif rc == nat.MLE_NOT_PD:
                answers[i] = (None, NotPositiveDefinite(piv))
            elif rc != nat.MLE_OK:
                answers[i] = (None, ValueError(nat.last_error()))
            else:
                answers[i] = ((ll, grad, fisher), None)
        for i, (first, count, slot) in many.items():
            try:
                vals = []
                for k in range(first, first + count):
                    o = outs[k]
                    if isinstance(o, Exception):
                        raise o
                    vals.append(_loglik_value(o[0], o[2]))
                answers[i] = ([-math.inf if s is None else vals[s] for s in slot], None)
            except Exception as exc:
                answers[i] = (None, exc)
        for i in ids:
            value, exc = answers[i]
            if exc is not None:
                advance(i, gens[i].throw, exc)
            else:
                advance(i, gens[i].send, value)
    if objectives_out is not None:
        objectives_out.extend(cnt)
    return results


class _FitFailure:
    """A fit of a lock-step group that raised (kept until the group has finished)."""

    def __init__(self, exc):
        self.exc = exc
