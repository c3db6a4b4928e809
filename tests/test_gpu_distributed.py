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
def test_cuda_panels_match_engine(gpu, world):
    from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm

    loc, z = config_data("config2", 1)  # n = 3,600 -> N = 4,096: 8 blocks
    th = (1.0, 0.2, 1.5)
    (ll, g, f), ll_only = _ref(gpu, loc, z, th)
    eng = DistributedEngine(loc, z, InProcessComm(world))
    dll, dg, df = eng.eval_all(th)
    assert dll == pytest.approx(ll, rel=1e-12)
    # the distributed sweeps use 8-slice operands, the single-context engine 7 (and N is padded
    # to 512 vs 128): compare the score on its component scale, as the parity tests do
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
    eng = DistributedEngine(loc, z, InProcessComm(2), nugget=1e-4)
    dll, dg, df = eng.eval_all(th)
    assert dll == pytest.approx(ll, rel=1e-12)
    np.testing.assert_allclose(df, f, rtol=1e-9)
    # 8-slice distributed sweeps vs 7-slice single-context sweeps on a hard case (GMM
    # clusters, config-5 theta): the north-star score bound
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
