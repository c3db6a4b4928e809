"""Host Fisher-BT driver logic (CPU): L9 design, damped scoring step, relaxed Armijo,
Nelder-Mead and the main loop, driven by analytic surrogate objectives exactly as the
reference's own optimizer tests inject them (reference tests/test_optimizer.py)."""

import math

import numpy as np
import pytest

import paper_2601_11437_b200 as m

LO = m.MaternParams(0.01, 0.01, 0.01)
HI = m.MaternParams(5.0, 5.0, 2.0)


class Bowl:
    """Concave quadratic with exact curvature as the information matrix."""

    def __init__(self, peak, curv):
        self.peak = np.asarray(peak, float)
        self.curv = np.asarray(curv, float)
        self.loglik_calls = 0
        self.grad_calls = 0

    def _value(self, th):
        d = np.asarray(th, float) - self.peak
        return -0.5 * float(d @ self.curv @ d)

    def loglik(self, th):
        self.loglik_calls += 1
        return self._value(th)

    def eval_all(self, th):
        self.loglik_calls += 1
        self.grad_calls += 1
        d = np.asarray(th, float) - self.peak
        return self._value(th), -self.curv @ d, self.curv.copy()


def cfg(**kw):
    return m.FisherBTConfig(theta_lower=LO, theta_upper=HI, **kw)


def test_l9_rows():
    rows = m.l9_candidates(LO, HI)
    assert len(rows) == 9
    assert rows[0] == m.MaternParams(2.505, 2.505, 1.005)
    assert rows[1].alpha == pytest.approx(0.84166667, abs=1e-8)
    assert rows[1].nu == pytest.approx(0.34166667, abs=1e-8)
    lo, hi = LO.as_array(), HI.as_array()
    levels = [0.5 * lo + 0.5 * hi, 5 / 6 * lo + 1 / 6 * hi, 1 / 6 * lo + 5 / 6 * hi]
    for c in range(3):
        counts = [sum(math.isclose(r.as_array()[c], lv[c], rel_tol=1e-12) for r in rows)
                  for lv in levels]
        assert counts == [3, 3, 3]


def test_degenerate_cube_repeats_start():
    th = m.MaternParams(1.0, 0.5, 0.7)
    for r in m.l9_candidates(th, th):
        np.testing.assert_allclose(r.as_array(), th.as_array(), rtol=1e-15)


def test_fisher_step_cases():
    np.testing.assert_allclose(m.fisher_step(np.array([2.0, 4.0, 8.0]), np.diag([2.0, 4.0, 8.0])),
                               [1, 1, 1], atol=1e-14)
    rng = np.random.default_rng(2)
    for _ in range(5):
        r = rng.standard_normal((3, 3))
        info = r @ r.T + 0.1 * np.eye(3)
        g = rng.standard_normal(3)
        np.testing.assert_allclose(info @ m.fisher_step(g, info), g, rtol=1e-10, atol=1e-12)
    info = np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    step = m.fisher_step(np.array([1.0, 1.0, 0.5]), info)
    np.testing.assert_allclose(info @ step, [1.0, 1.0, 0.5], atol=1e-3)
    with pytest.raises(m.SingularInformation):
        m.fisher_step(np.array([1.0, 0.0, 0.0]), np.zeros((3, 3)))


def test_armijo():
    g, p = np.array([0.2, 0.0, 0.0]), np.array([1.0, 0.0, 0.0])
    assert m.armijo_relaxed(-100.0, -100.5, g, p, cfg())
    assert not m.armijo_relaxed(-100.502, -100.5, g, p, cfg())
    assert m.armijo_relaxed(-50.0, -50.0, np.zeros(3), np.zeros(3), cfg())


def test_nelder_mead_on_bowl():
    obj = Bowl([1.2, 0.4, 0.9], np.diag([4.0, 9.0, 1.0]))
    th, calls = m.nelder_mead(None, m.MaternParams(0.8, 0.75, 0.5), 1e-9, objective=obj)
    np.testing.assert_allclose(th.as_array(), [1.2, 0.4, 0.9], atol=1e-4)
    assert calls == obj.loglik_calls


def test_nelder_mead_infinite_tol_returns_start():
    obj = Bowl([1.2, 0.4, 0.9], np.eye(3))
    th, calls = m.nelder_mead(None, m.MaternParams(0.8, 0.09, 0.45), math.inf, objective=obj)
    assert th == m.MaternParams(0.8, 0.09, 0.45)
    assert calls == 4


def test_one_step_on_bowl():
    res = m.fisher_bt(None, cfg(), objective=Bowl([1.5, 0.8, 0.6], np.diag([2.0, 3.0, 5.0])))
    np.testing.assert_allclose(res.theta_hat.as_array(), [1.5, 0.8, 0.6], atol=1e-12)
    assert res.termination is m.Termination.GRADIENT_TOL
    assert not res.used_fallback
    assert len(res.iterate_trace) == 2
    assert res.loglik_calls == 9 + 1 + 1 + 1 and res.grad_calls == 2


def test_budget_forces_fallback_on_bowl():
    res = m.fisher_bt(None, cfg(max_grad_calls=0), objective=Bowl([1.5, 0.8, 0.6], np.eye(3)))
    assert res.used_fallback
    assert res.fisher_phase_grad_calls == 1


def test_initialization_failure():
    class Dead(Bowl):
        def loglik(self, th):
            self.loglik_calls += 1
            return -math.inf

    with pytest.raises(m.InitializationFailed):
        m.fisher_bt(None, cfg(), objective=Dead([1, 1, 1], np.eye(3)))


def test_config_validation():
    with pytest.raises(ValueError):
        m.FisherBTConfig(theta_lower=HI, theta_upper=LO)
    with pytest.raises(ValueError):
        cfg(grad_tol=0.0)
    with pytest.raises(ValueError):
        cfg(nm_tol=-1.0)
    with pytest.raises(ValueError):
        cfg(max_halvings=-1)


def test_params_validation():
    with pytest.raises(ValueError):
        m.MaternParams(0.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        m.MaternParams(1.0, 1.0, math.nan)
    th = m.MaternParams(1.5, 0.2, 0.7)
    assert m.MaternParams.from_array(th.as_array()) == th


def test_dataset_validation():
    with pytest.raises(ValueError):
        m.SpatialDataset(np.zeros((0, 2)), np.zeros(0))
    with pytest.raises(ValueError):
        m.SpatialDataset(np.zeros((3, 3)), np.zeros(3))
    with pytest.raises(ValueError):
        m.SpatialDataset(np.zeros((3, 2)), np.zeros(4))
    with pytest.raises(ValueError):
        m.SpatialDataset(np.array([[0.0, np.inf]]), np.zeros(1))


def test_regime_partition():
    for nu in np.linspace(0.01, 3.0, 61):
        for x in np.linspace(0.0, 100.0, 201):
            r = m.select_regime(nu, x)
            near_i = abs(nu - round(nu)) <= 1e-6
            near_h = abs(nu + 0.5 - round(nu + 0.5)) <= 1e-6
            if x == 0.0:
                exp = m.BesselRegime.ZERO_ARG
            elif x < 8.5:
                exp = m.BesselRegime.FINITE_DIFF if near_i else m.BesselRegime.SMALL_X
            elif x < 30.0:
                exp = m.BesselRegime.MID_X
            else:
                exp = m.BesselRegime.FINITE_DIFF if near_h else m.BesselRegime.LARGE_X
            assert r is exp


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_driver_matches_live_reference_driver(reference, seed):
    """Same surrogate objective through the reference's fisher_bt and ours: identical
    trajectory, counters and termination (including the Nelder-Mead shift)."""
    rng = np.random.default_rng(seed)
    r = rng.standard_normal((3, 3))
    curv = r @ r.T + 0.5 * np.eye(3)
    peak = rng.uniform(0.5, 1.5, 3)

    class Warped(Bowl):
        def _value(self, th):  # non-quadratic so several iterations / halvings happen
            d = np.asarray(th, float) - self.peak
            return -0.5 * float(d @ self.curv @ d) - 0.3 * float(np.sum(d ** 4))

    for kw in ({}, {"max_grad_calls": 2}, {"max_loglik_calls": 12}):
        ours = m.fisher_bt(None, cfg(**kw), objective=Warped(peak, curv))
        theirs_cfg = reference.FisherBTConfig(
            theta_lower=reference.MaternParams(0.01, 0.01, 0.01),
            theta_upper=reference.MaternParams(5.0, 5.0, 2.0), **kw)
        theirs = reference.fisher_bt(None, theirs_cfg, objective=Warped(peak, curv))
        np.testing.assert_array_equal(ours.theta_hat.as_array(), theirs.theta_hat.as_array())
        assert ours.loglik_calls == theirs.loglik_calls
        assert ours.grad_calls == theirs.grad_calls
        assert ours.termination.value == theirs.termination.value
        assert ours.used_fallback == theirs.used_fallback
        assert len(ours.iterate_trace) == len(theirs.iterate_trace)


def test_bench_algorithmic_flop_counts():
    """bench.py's roofline numerator (block sums) against the closed forms of SURVEY §8(d):
    Cholesky n^3/3; per derivative block n^3 + n^3/3 (full sweeps) or 2n^3/3 + n^3/3 (two-sided)."""
    import bench

    n = 65536
    chol = bench.gemm_algorithmic_flops(n, "loglik")
    w = bench.gemm_algorithmic_flops(n, "eval_all", path="w")
    two = bench.gemm_algorithmic_flops(n, "eval_all", path="2s")
    assert abs(chol / (n ** 3 / 3) - 1) < 0.03
    assert abs(w / (3 * n ** 3) - 1) < 0.02
    assert abs(two / (7 * n ** 3 / 3) - 1) < 0.03
    assert bench.solve_path(65536) == "2s" and bench.solve_path(3600) == "w"
