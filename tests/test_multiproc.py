"""Multi-rank host logic on CPU (gloo, world_size 2): bench.py's sharded arm (every rank
running the same Fisher-BT loop over the DistributedEngine, stepped per Fisher iteration, and
the max-over-ranks reduction of the timing), and the DistributedEngine driver itself with a
host restatement of the block steps."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _bench_worker(rank, world, port, out):
    """One rank of bench.py's sharded arm (N > 1) on CPU: every rank runs the same host
    Fisher-BT loop, stepped one Fisher iteration at a time (bench.FitStepper), over a
    DistributedObjective whose engine is the host restatement of the block steps; then the
    max-over-ranks time / sum reductions the whole-job value uses."""
    import sys

    import numpy as np

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import bench
    from dist_host_backend import HostPanels
    from oracle import maternmle_cpu as O
    import paper_2601_11437_b200 as m
    from paper_2601_11437_b200.distributed import (DistributedEngine, DistributedObjective,
                                                   TorchComm)

    rng = np.random.default_rng(5)
    n = 700  # N = 1024: 2 outer blocks, one per rank
    loc = m.jittered_grid(27, 1)[:n]
    z = O.cholesky(O.matrix(loc, (1.0, 0.15, 0.9))) @ rng.standard_normal(n)
    eng = DistributedEngine(loc, z, TorchComm(), backend=HostPanels)
    th0 = m.MaternParams(0.8, 0.1, 0.7)
    cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
    stepper = bench.FitStepper(lambda: DistributedObjective(eng), cfg)
    thetas = []
    while not stepper.done:
        stepper.step()
        thetas.append(stepper.obj.grad_calls)
    res = stepper.done[0]
    gathered = [None] * world
    dist.all_gather_object(gathered, (res.theta_hat.as_array().tolist(), res.grad_calls,
                                      res.loglik_calls, res.termination.value))
    t = torch.tensor([10.0 + rank, 20.0 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put((gathered, t.tolist(), (loc, z, th0.as_array().tolist())))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_sharded_fit_two_ranks():
    import numpy as np

    import paper_2601_11437_b200 as m
    from oracle import maternmle_cpu as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax, (loc, z, th0) = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert gathered[0] == gathered[1]  # identical deterministic loop on every rank
    assert tmax == [11.0, 40.0]
    # the same fit on the CPU oracle objective: same counts and termination, same theta-hat
    cfg = m.FisherBTConfig(theta_lower=m.MaternParams(*th0), theta_upper=m.MaternParams(*th0))
    ref = m.fisher_bt(None, cfg, objective=O.CountingObjective(loc, z))
    th, g, ll, term = gathered[0]
    assert (g, ll, term) == (ref.grad_calls, ref.loglik_calls, ref.termination.value)
    np.testing.assert_allclose(th, ref.theta_hat.as_array(), rtol=1e-9)


def test_fit_stepper_matches_full_fit():
    """bench.FitStepper: one step = exactly one eval_all; stepping reproduces fisher_bt."""
    import bench
    import numpy as np

    import paper_2601_11437_b200 as m
    from oracle import maternmle_cpu as O

    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "config1_seed0_data.npz"))
    loc, z = d["loc"], d["z"]
    th0 = m.MaternParams(0.5, 0.05, 1.0)
    cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
    full = m.fisher_bt(None, cfg, objective=O.CountingObjective(loc, z))
    st = bench.FitStepper(lambda: O.CountingObjective(loc, z), cfg)
    steps = 0
    while not st.done:
        before = st.obj.grad_calls
        st.step()
        steps += 1
        assert st.done or st.obj.grad_calls == before + 1
    r = st.done[0]
    assert steps == full.grad_calls
    assert (r.grad_calls, r.loglik_calls) == (full.grad_calls, full.loglik_calls)
    np.testing.assert_array_equal(r.theta_hat.as_array(), full.theta_hat.as_array())


def _dist_worker(rank, world, port, out):
    """One rank of DistributedEngine over gloo with the host restatement of the block steps."""
    import sys

    import numpy as np

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    from dist_host_backend import HostPanels
    from oracle import maternmle_cpu as O
    from paper_2601_11437_b200.distributed import DistributedEngine, TorchComm

    rng = np.random.default_rng(3)
    n = 1200  # N = 1536: 3 outer blocks over 2 ranks (uneven ownership)
    loc = rng.uniform(size=(n, 2))
    th = (1.1, 0.12, 1.4)
    z = O.cholesky(O.matrix(loc, th)) @ rng.standard_normal(n)
    comm = TorchComm()
    eng = DistributedEngine(loc, z, comm, backend=HostPanels)
    res = eng.eval_all(th)
    ll = eng.loglik(th)
    tau2 = 1e-3
    engn = DistributedEngine(loc, z, comm, nugget=tau2, backend=HostPanels)
    resn = engn.eval_all(th)
    # the two-sided reduction on the panels (the single-context path from N >= 16,384)
    res2 = DistributedEngine(loc, z, comm, backend=HostPanels, solve="2s").eval_all(th)
    res2n = DistributedEngine(loc, z, comm, nugget=tau2, backend=HostPanels,
                              solve="2s").eval_all(th)
    # a failing factorization: coincident locations -> NotPositiveDefinite on every rank
    bad = loc.copy()
    bad[900] = bad[899]
    try:
        DistributedEngine(bad, z, comm, backend=HostPanels).loglik(th)
        pivot = None
    except Exception as exc:  # NotPositiveDefinite
        pivot = getattr(exc, "pivot", repr(exc))
    if rank == 0:
        out.put((res[0], res[1].tolist(), res[2].tolist(), ll, resn[0], resn[1].tolist(),
                 resn[2].tolist(), pivot, [res2[0], res2[1].tolist(), res2[2].tolist()],
                 [res2n[0], res2n[1].tolist(), res2n[2].tolist()]))
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_engine_driver_gloo():
    """DistributedEngine (config 4/5 sharding) over 2 gloo ranks == the oracle's eval_all,
    with and without a nugget; a singular Sigma fails on every rank at the same pivot."""
    import numpy as np

    from oracle import maternmle_cpu as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ll, g, f, ll2, lln, gn, fn, pivot, two, twon = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    n = 1200
    loc = rng.uniform(size=(n, 2))
    th = (1.1, 0.12, 1.4)
    z = O.cholesky(O.matrix(loc, th)) @ rng.standard_normal(n)
    ref = O.eval_all(loc, z, th)
    assert ll == pytest.approx(ref[0], rel=1e-11)
    assert ll2 == pytest.approx(O.loglik(loc, z, th), rel=1e-11)
    np.testing.assert_allclose(g, ref[1], rtol=1e-8)
    np.testing.assert_allclose(f, ref[2], rtol=1e-10)
    refn = O.eval_all_nugget(loc, z, th, 1e-3)
    assert lln == pytest.approx(refn[0], rel=1e-11)
    np.testing.assert_allclose(gn, refn[1], rtol=1e-8)
    np.testing.assert_allclose(fn, refn[2], rtol=1e-10)
    assert pivot == 900
    # two-sided path (solve="2s"), with and without the nugget
    assert two[0] == pytest.approx(ref[0], rel=1e-11)
    np.testing.assert_allclose(two[1], ref[1], rtol=1e-8)
    np.testing.assert_allclose(two[2], ref[2], rtol=1e-10)
    assert twon[0] == pytest.approx(refn[0], rel=1e-11)
    np.testing.assert_allclose(twon[1], refn[1], rtol=1e-8)
    np.testing.assert_allclose(twon[2], refn[2], rtol=1e-10)
