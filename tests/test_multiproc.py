"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): disjoint replica
sharding (weak scaling, no data-path collective) and the max-over-ranks / sum-over-ranks
reductions that produce the whole-job value."""

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


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    seeds = bench.replica_seeds(rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    t = torch.tensor([10.0 + rank, 20.0 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([11.0 + rank], dtype=torch.float64)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((gathered, t.tolist(), c.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_sharding_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax, csum = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert gathered[0] == [0, 1, 2, 3, 4]
    assert gathered[1] == [5, 6, 7, 8, 9]
    assert not set(gathered[0]) & set(gathered[1])
    assert tmax == [11.0, 40.0]
    assert csum == [23.0]


@pytest.mark.parametrize("rank", [0, 1, 3, 7])
def test_replica_seed_blocks(rank):
    import bench

    s = bench.replica_seeds(rank)
    assert s == list(range(5 * rank, 5 * rank + 5))


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
                 resn[2].tolist(), pivot))
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
    ll, g, f, ll2, lln, gn, fn, pivot = q.get(timeout=300)
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
