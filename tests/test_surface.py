"""Drop-in surface beyond the evaluation path (CPU): digamma, the Debye tables, the
series' domain errors, and the simulate module's plan logic -- against the oracle and, in the
build container, the reference package itself (bessel.py:72-176, simulate.py:34-128)."""

import warnings

import numpy as np
import pytest
from scipy import special as sps

import paper_2601_11437_b200 as m
from oracle import maternmle_cpu as O


def test_digamma_values_and_poles():
    x = np.array([1e-3, 0.05, 0.5, 1.0, 1.3, 2.5, 7.0, 50.0, 1e4, -0.5, -1.25, -7.5])
    got = m.digamma(x)
    np.testing.assert_allclose(got, sps.digamma(x), rtol=2e-15, atol=0)
    assert m.digamma(1.0) == pytest.approx(-0.5772156649015329, rel=1e-15)
    assert isinstance(m.digamma(0.5), float)
    for pole in (0.0, -1.0, -3.0):
        with pytest.raises(ValueError):
            m.digamma(pole)
    with pytest.raises(ValueError):
        m.digamma(np.array([0.5, -2.0]))


def test_u_poly_coeffs_matches_oracle_tables():
    mine = m.u_poly_coeffs(12)
    ref_u, _ = O.debye_tables(12)
    assert len(mine) == 13
    for k, (a, b) in enumerate(zip(mine, ref_u)):
        assert a.shape == (3 * k + 1,)
        np.testing.assert_array_equal(a, b)
    assert m.u_poly_coeffs(0)[0].tolist() == [1.0]
    with pytest.raises(ValueError):
        m.u_poly_coeffs(-1)


def test_u_poly_coeffs_and_plans_match_reference(reference):
    for a, b in zip(m.u_poly_coeffs(12), reference.u_poly_coeffs(12)):
        np.testing.assert_array_equal(a, b)
    for scheme in ("UNIFORM_RANDOM", "UNIT_GRID"):
        p = m.SimulationPlan(n=64, theta_true=m.MaternParams(1.0, 0.1, 0.5),
                             location_scheme=getattr(m.LocationScheme, scheme), rng_seed=9,
                             domain=(0.0, 2.0, -1.0, 1.0))
        q = reference.SimulationPlan(n=64, theta_true=reference.MaternParams(1.0, 0.1, 0.5),
                                     location_scheme=getattr(reference.LocationScheme, scheme),
                                     rng_seed=9, domain=(0.0, 2.0, -1.0, 1.0))
        np.testing.assert_array_equal(m.gen_locations(p), reference.gen_locations(q))
    th = m.MaternParams(1.3, 0.2, 0.7)
    assert m.microergodic(th) == reference.microergodic(reference.MaternParams(1.3, 0.2, 0.7))
    assert m.replicate_seed(7, 3, 1) == reference.replicate_seed(7, 3, 1)
    assert m.GENERATOR_ID == reference.GENERATOR_ID
    assert m.digamma(0.37) == pytest.approx(reference.digamma(0.37), rel=2e-15)


def test_plan_errors():
    th = m.MaternParams(1.0, 0.1, 0.5)
    with pytest.raises(m.PlanError):
        m.SimulationPlan(n=1, theta_true=th)
    with pytest.raises(m.PlanError):
        m.SimulationPlan(n=10, theta_true=th)  # grid needs a perfect square
    with pytest.raises(m.PlanError):
        m.SimulationPlan(n=9, theta_true=th, replicates=0)
    with pytest.raises(m.PlanError):
        m.SimulationPlan(n=9, theta_true=th, domain=(1.0, 0.0, 0.0, 1.0))
    assert issubclass(m.PlanError, ValueError)
    assert m.microergodic(m.MaternParams(1.0, 1e-300, 5.0)) == float("inf")


def test_series_domain_errors_before_device_work():
    with pytest.raises(ValueError):
        m.case2_series(0.7, np.array([1.0, 9.0]))
    with pytest.raises(ValueError):
        m.case2_series(1.0000001, 1.0)  # nu inside the integer band
    with pytest.raises(ValueError):
        m.case3_series(0.7, 31.0)
    with pytest.raises(ValueError):
        m.case3_series(-0.5, 10.0)
    with pytest.raises(ValueError):
        m.case4_series(0.7, 29.0)
    assert issubclass(m.MidRangeSmallOrderWarning, UserWarning)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        with pytest.raises(ValueError):
            m.case4_series(0.0, 40.0)
