"""The two-sided blocked reduction (engine.cu solves_2s: the sygst recurrence + the deferred
forward sweep on the strictly lower block part; n^3 instead of 4 n^3 / 3 flops per derivative
block) against the reference's goldens, and against the full-sweep formulation (solves_w)."""

import os

import numpy as np
import pytest

from conftest import config_data, load_json
from test_gpu_likelihood import check_eval, score_scale

pytestmark = pytest.mark.gpu


@pytest.fixture
def two_sided():
    old = os.environ.get("MLE_SOLVE")
    os.environ["MLE_SOLVE"] = "2s"
    yield
    if old is None:
        del os.environ["MLE_SOLVE"]
    else:
        os.environ["MLE_SOLVE"] = old


def test_two_sided_small_and_config_goldens(gpu, golden_small, two_sided):
    arrays, ev = golden_small
    floors = load_json("small_floor.json")
    for name, recs in ev["cases"].items():
        loc, z = arrays[f"{name}_loc"], arrays[f"{name}_z"]
        data = gpu.SpatialDataset(loc, z)
        for k, rec in enumerate(recs):
            if "not_pd_pivot" in rec:
                continue
            check_eval(gpu, data, rec, loc.shape[0], floor=floors[name][k]["floor"])
        data.release()
    for cfg in ("config1", "config2", "config3"):
        loc, z = config_data(cfg)
        data = gpu.SpatialDataset(loc, z)
        for rec in load_json(f"{cfg}_evals.json"):
            check_eval(gpu, data, rec, loc.shape[0])
        data.release()


def test_two_sided_matches_full_sweeps(gpu):
    loc, z = config_data("config2", 2)
    out = {}
    for mode in ("w", "2s"):
        os.environ["MLE_SOLVE"] = mode
        try:
            eng = gpu.Engine(loc, z)
            out[mode] = eng.eval_all(np.array([1.0, 0.2, 1.5]))
            eng.close()
        finally:
            del os.environ["MLE_SOLVE"]
    (lw, gw, fw), (l2, g2, f2) = out["w"], out["2s"]
    assert l2 == lw  # the log-likelihood does not involve the solves
    scale = score_scale((1.0, 0.2, 1.5), len(z), gw, fw)
    assert np.all(np.abs(g2 - gw) <= 1e-10 * scale), (g2, gw)
    np.testing.assert_allclose(f2, fw, rtol=1e-10)


def test_two_sided_nugget(gpu, two_sided):
    """Nugget items add the third block M = L^-1 L^-T (S = I): same recurrence."""
    rng = np.random.default_rng(2)
    loc = gpu.gmm_locations(1500, 2)
    z = rng.standard_normal(1500)
    th = np.array([0.9, 0.08, 1.013])
    got = gpu.Engine(loc, z, nugget=1e-4).eval_all(th)
    os.environ["MLE_SOLVE"] = "w"
    ref = gpu.Engine(loc, z, nugget=1e-4).eval_all(th)
    os.environ["MLE_SOLVE"] = "2s"
    assert got[0] == ref[0]
    scale = score_scale(th, len(z), ref[1], ref[2])
    assert np.all(np.abs(got[1] - ref[1]) <= 1e-9 * scale), (got[1], ref[1])
    np.testing.assert_allclose(got[2], ref[2], rtol=1e-9)


def test_two_sided_batched_is_bit_identical_to_single(gpu, two_sided):
    """Several datasets in one batched pass (mle_eval_batch: every launch covers all items)
    on the two-sided path give each item's single-evaluation result bit for bit."""
    sets = [config_data("config2", s) for s in range(3)]
    engines = [gpu.Engine(loc, z) for loc, z in sets]
    thetas = [np.array([1.0, 0.2, 1.5]), np.array([0.9, 0.15, 1.3]), np.array([1.1, 0.22, 1.7])]
    batched = gpu.eval_batch(engines, thetas, [2, 2, 2])
    for eng, th, (rc, piv, ll, g, f) in zip(engines, thetas, batched):
        assert rc == 0
        single = gpu.Engine(*sets[engines.index(eng)]).eval_all(th)
        assert ll == single[0]
        np.testing.assert_array_equal(g, single[1])
        np.testing.assert_array_equal(f, single[2])
    for e in engines:
        e.close()
