"""The distributed engine's CUDA panels (mle_dctx_*) on the one GPU of the test box: world 1,
and several ranks stepped in one process (InProcessComm: the broadcasts become device copies),
against the single-context engine.  The multi-process driver itself is covered with gloo in
tests/test_multiproc.py; here every block step runs the real sm_100a kernels."""

import numpy as np
import pytest

from conftest import config_data
from test_gpu_likelihood import score_scale

pytestmark = pytest.mark.gpu


def _ref(gpu, loc, z, th, nugget=0.0):
    eng = gpu.Engine(loc, z, nugget=nugget)
    out = eng.eval_all(np.asarray(th, float))
    ll = eng.loglik(np.asarray(th, float) * np.array([1.0, 1.0, 1.0]))
    eng.close()
    return out, ll


@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("solve", ["w", "2s"])
def test_cuda_panels_match_engine(gpu, world, solve):
    from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm

    loc, z = config_data("config2", 1)  # n = 3,600 -> N = 4,096: 8 blocks
    th = (1.0, 0.2, 1.5)
    (ll, g, f), ll_only = _ref(gpu, loc, z, th)
    eng = DistributedEngine(loc, z, InProcessComm(world), solve=solve)
    assert eng.solve == solve
    dll, dg, df = eng.eval_all(th)
    assert dll == pytest.approx(ll, rel=1e-12)
    # same kernels and slice counts, but N is padded to 512 (vs 128) and the final sums run in
    # a different order (per-panel partials vs the single-context reduction): compare the score
    # on its component scale, as the parity tests do
    scale = score_scale(th, len(z), g, f)
    assert np.all(np.abs(dg - g) <= 1e-9 * scale), (dg, g, scale)
    np.testing.assert_allclose(df, f, rtol=1e-10)
    assert eng.loglik(th) == pytest.approx(ll_only, rel=1e-12)
    eng.close()


def test_cuda_panels_nugget_and_failure(gpu):
    from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm

    rng = np.random.default_rng(2)
    loc = gpu.gmm_locations(1500, 2)
    z = rng.standard_normal(1500)
    th = (0.9, 0.08, 1.013)
    (ll, g, f), _ = _ref(gpu, loc, z, th, nugget=1e-4)
    for solve in ("w", "2s"):
        eng = DistributedEngine(loc, z, InProcessComm(2), nugget=1e-4, solve=solve)
        dll, dg, df = eng.eval_all(th)
        assert dll == pytest.approx(ll, rel=1e-12)
        np.testing.assert_allclose(df, f, rtol=1e-9)
        scale = score_scale(th, len(z), g, f)
        assert np.all(np.abs(dg - g) <= 1e-8 * scale), (solve, dg, g, scale)
        eng.close()
    eng = DistributedEngine(loc, z, InProcessComm(2), nugget=1e-4)
    dll, dg, df = eng.eval_all(th)
    assert dll == pytest.approx(ll, rel=1e-12)
    np.testing.assert_allclose(df, f, rtol=1e-9)
    # distributed vs single-context on a hard case (GMM clusters, config-5 theta): the
    # north-star score bound
    scale = score_scale(th, len(z), g, f)
    assert np.all(np.abs(dg - g) <= 1e-8 * scale), (dg, g, scale)
    eng.close()
    # coincident first pair: an exactly zero pivot (sigma^2 = 1) in block 0 (rank 0); every
    # rank must report the failure (deep coincident pairs are rounding-dependent in any
    # blocked Cholesky, the reference's LAPACK dpotrf included)
    bad = loc.copy()
    bad[1] = bad[0]
    eng = DistributedEngine(bad, z, InProcessComm(2))
    with pytest.raises(gpu.NotPositiveDefinite) as info:
        eng.loglik((1.0, 0.1, 0.5))
    assert info.value.pivot == 1
    eng.close()


def test_results_do_not_depend_on_world_size(gpu):
    """Per-panel partial sums added in block order (distributed.py): 1, 2 and 3 ranks give
    bit-identical log-likelihood, score and Fisher -- so a fit takes the same path on any
    number of GPUs.  Also with and without the W cache (no second W broadcast)."""
    from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm

    loc, z = config_data("config2", 3)
    th = (0.9, 0.15, 1.3)
    outs = []
    for world, wc in ((1, True), (2, True), (3, True), (3, False)):
        eng = DistributedEngine(loc, z, InProcessComm(world), wcache=wc, solve="w")
        assert eng.wcache == wc
        outs.append((eng.eval_all(th), eng.loglik(th)))
        eng.close()
    (ll0, g0, f0), l0 = outs[0]
    for (ll, g, f), l in outs[1:]:
        assert ll == ll0 and l == l0
        np.testing.assert_array_equal(g, g0)
        np.testing.assert_array_equal(f, f0)


def _nccl_world1(q, port):
    """World-1 NCCL process: the stream-ordered (asynchronous) schedule -- block steps queued
    without host drains, broadcasts on the communication stream behind events -- must give
    the synchronous schedule's results bit for bit."""
    import os
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from conftest import config_data as cd
    from paper_2601_11437_b200.distributed import DistributedEngine, TorchComm

    loc, z = cd("config2", 2)
    th = (1.0, 0.2, 1.5)
    res = []
    for solve in ("w", "2s"):
        a = DistributedEngine(loc, z, TorchComm(), overlap=True, solve=solve)
        b = DistributedEngine(loc, z, TorchComm(), overlap=False, solve=solve)
        ra, rb = a.eval_all(th), b.eval_all(th)
        la, lb = a.loglik(th), b.loglik(th)
        res.append((a.async_steps, b.async_steps, ra[0] == rb[0], bool(np.all(ra[1] == rb[1])),
                    bool(np.all(ra[2] == rb[2])), la == lb))
        a.close()
        b.close()
    q.put(res)
    dist.destroy_process_group()


def test_stream_ordered_schedule_nccl_world1(gpu):
    import torch.multiprocessing as mp

    from test_multiproc import _free_port

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1, args=(q, _free_port()))
    p.start()
    out = q.get(timeout=600)
    p.join(60)
    for res in out:  # full sweeps, two-sided
        assert res[0] is True and res[1] is False
        assert all(res[2:]), res


def _gloo_cuda_rank(rank, world, port, q):
    """One rank of a 2-process gloo job, both ranks' panels on cuda:0 (the CUDA block steps
    in two processes; gloo moves the CUDA exchange buffers through the host)."""
    import os
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import config_data as cd
    from paper_2601_11437_b200.distributed import DistributedEngine, TorchComm

    loc, z = cd("config2", 1)
    th = (1.0, 0.2, 1.5)
    eng = DistributedEngine(loc, z, TorchComm())
    ll, g, f = eng.eval_all(th)
    l2 = eng.loglik(th)
    eng.close()
    if rank == 0:
        q.put((ll, g.tolist(), f.tolist(), l2))
    dist.barrier()
    dist.destroy_process_group()


def test_cuda_panels_two_processes_gloo(gpu):
    """CudaPanels in two processes (gloo) == the same engine stepped in one process."""
    import torch.multiprocessing as mp

    from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm
    from test_multiproc import _free_port

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_cuda_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ll, g, f, l2 = q.get(timeout=900)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    loc, z = config_data("config2", 1)
    th = (1.0, 0.2, 1.5)
    ref = DistributedEngine(loc, z, InProcessComm(1))
    rl, rg, rf = ref.eval_all(th)
    assert ll == rl and l2 == ref.loglik(th)
    np.testing.assert_array_equal(g, rg)
    np.testing.assert_array_equal(f, rf)
    ref.close()


def test_two_sided_panels_do_not_depend_on_world_size(gpu):
    """The sharded two-sided path: 1, 2 and 3 ranks bit-identical."""
    from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm

    loc, z = config_data("config2", 3)
    th = (0.9, 0.15, 1.3)
    outs = []
    for world in (1, 2, 3):
        eng = DistributedEngine(loc, z, InProcessComm(world), solve="2s")
        outs.append(eng.eval_all(th))
        eng.close()
    for ll, g, f in outs[1:]:
        assert ll == outs[0][0]
        np.testing.assert_array_equal(g, outs[0][1])
        np.testing.assert_array_equal(f, outs[0][2])
