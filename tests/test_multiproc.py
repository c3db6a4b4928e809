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
