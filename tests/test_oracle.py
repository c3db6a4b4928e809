"""The CPU oracle is pinned to the reference: golden fixtures (everywhere) and the live
reference package (build container only).  CPU-only."""

import math

import numpy as np
import pytest

from conftest import config_data, fit_golden, load_json
from oracle import maternmle_cpu as O


def test_dnu_grid_matches_reference_outputs_bitwise(bessel_golden):
    for p in bessel_golden["grid"]:
        assert O.dnu_xnu_knu(p["nu"], p["x"]) == p["dnu_ref"], p


def test_dnu_grid_vs_mpmath_acceptance_criterion_1(bessel_golden):
    # reference acceptance criterion 1: rel err <= 1e-6 on the 200-point grid
    worst = max(abs(O.dnu_xnu_knu(p["nu"], p["x"]) - p["dnu_mp"]) / (1 + abs(p["dnu_mp"]))
                for p in bessel_golden["grid"])
    assert worst <= 1e-6


def test_dnu_spots(bessel_golden):
    for s in bessel_golden["spots"]:
        assert O.dnu_xnu_knu(s["nu"], s["x"]) == s["dnu_ref"], s
        assert O.regime(s["nu"], s["x"]) == {"small_x": "small", "mid_x": "mid",
                                             "large_x": "large", "finite_diff": "fd",
                                             "zero_arg": "zero"}[s["regime"]]


def test_bessel_k_spots(bessel_golden):
    for s in bessel_golden["k_spots"]:
        assert float(O.bessel_k(s["nu"], s["x"])) == s["k_ref"]
        assert abs(O.bessel_k(s["nu"], s["x"]) - s["k_mp"]) <= 1e-12 * s["k_mp"]


def test_debye_tables_closed_forms():
    u, du = O.debye_tables(2)
    np.testing.assert_allclose(u[1], [0.0, 1.0 / 8.0, 0.0, -5.0 / 24.0], atol=1e-15)
    np.testing.assert_allclose(u[2], np.array([0, 0, 81, 0, -462, 0, 385]) / 1152.0, atol=1e-15)


def test_matrices_match_golden_bitwise(golden_small):
    arrays, ev = golden_small
    thetas = ev["thetas"]
    for name in ev["cases"]:
        if f"{name}_t0_sigma" not in arrays:
            continue
        loc = arrays[f"{name}_loc"]
        for ti in range(4):
            assert np.array_equal(O.matrix(loc, thetas[ti], "sigma"), arrays[f"{name}_t{ti}_sigma"])
            for w in ("sigma2", "alpha", "nu"):
                assert np.array_equal(O.matrix(loc, thetas[ti], w), arrays[f"{name}_t{ti}_{w}"]), (
                    name, ti, w)


def test_evaluations_match_golden(golden_small):
    arrays, ev = golden_small
    for name, recs in ev["cases"].items():
        loc, z = arrays[f"{name}_loc"], arrays[f"{name}_z"]
        for rec in recs:
            th = tuple(rec["theta"])
            if "not_pd_pivot" in rec:
                with pytest.raises(O.NotPD) as info:
                    O.loglik(loc, z, th)
                assert info.value.pivot == rec["not_pd_pivot"]
                continue
            assert O.loglik(loc, z, th) == pytest.approx(rec["loglik"], rel=1e-14, abs=0)
            ll, g, f = O.eval_all(loc, z, th)
            assert ll == pytest.approx(rec["eval_loglik"], rel=1e-14)
            np.testing.assert_allclose(g, rec["grad"], rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(f, rec["fisher"], rtol=1e-12)


def test_config1_evaluations_match_golden():
    loc, z = config_data("config1")
    for rec in load_json("config1_evals.json"):
        ll, g, f = O.eval_all(loc, z, tuple(rec["theta"]))
        assert ll == pytest.approx(rec["eval_loglik"], rel=1e-13)
        np.testing.assert_allclose(f, rec["fisher"], rtol=1e-10)


def test_config1_fit_with_host_driver_matches_reference_fit():
    """Host Fisher-BT driver (product host logic) over the oracle objective reproduces the
    reference's own fit on config 1 exactly (same arithmetic on both sides)."""
    from paper_2601_11437_b200 import FisherBTConfig, MaternParams, fisher_bt

    gold = fit_golden("config1")
    loc, z = config_data("config1")
    th0 = MaternParams(*gold["theta0"])
    res = fisher_bt(None, FisherBTConfig(theta_lower=th0, theta_upper=th0),
                    objective=O.CountingObjective(loc, z))
    assert res.grad_calls == gold["grad_calls"]
    assert res.loglik_calls == gold["loglik_calls"]
    assert res.termination.value == gold["termination"]
    # LAPACK's blocked summation order depends on the OpenBLAS thread count, so the fit is
    # reproduced to ~1e-11 rather than bit for bit across thread counts.
    np.testing.assert_allclose(res.theta_hat.as_array(), gold["theta_hat"], rtol=1e-9)
    assert res.loglik_at_hat == pytest.approx(gold["loglik_at_hat"], rel=1e-13)


def test_oracle_vs_live_reference(reference):
    rng = np.random.default_rng(42)
    for _ in range(3):
        n = int(rng.integers(5, 60))
        loc = rng.uniform(size=(n, 2))
        th = tuple(rng.uniform(0.2, 1.8, size=3))
        data = reference.SpatialDataset(loc, rng.standard_normal(n))
        p = reference.MaternParams(*th)
        for w in ("sigma2", "alpha", "nu"):
            assert np.array_equal(O.matrix(loc, th, w), reference.build_dcov_matrix(data, p, w))
        assert np.array_equal(O.matrix(loc, th), reference.build_cov_matrix(data, p))
        ev = reference.grad_and_fisher(data, p)
        ll, g, f = O.eval_all(loc, data.values, th)
        assert ll == ev.loglik
        np.testing.assert_array_equal(f, ev.fisher)
    for nu in (0.3, 1.0, 1.5, 2.7):
        xs = np.array([0.0, 1e-3, 0.4, 3.0, 8.4, 8.6, 14.0, 16.0, 29.0, 31.0, 50.0])
        np.testing.assert_array_equal(O.dnu_xnu_knu(nu, xs), reference.dnu_xnu_knu(nu, xs))


def test_reference_bessel_oracle_pins_mpmath_golden(reference, bessel_golden):
    """Our mpmath golden agrees with the reference's own frozen quadrature oracle."""
    import json
    from pathlib import Path

    path = Path("/root/reference/pkg/tests/data/bessel_oracle.json")
    theirs = json.loads(path.read_text())
    ours = {(p["nu"], p["x"]): p["dnu_mp"] for p in bessel_golden["grid"]}
    for p in theirs["grid"]:
        key = (p["nu"], p["x"])
        assert key in ours
        assert abs(ours[key] - p["dnu"]) <= 1e-9 * (1 + abs(p["dnu"]))


def test_domain_errors():
    with pytest.raises(ValueError):
        O.dnu_xnu_knu(0.0, 1.0)
    with pytest.raises(ValueError):
        O.dnu_xnu_knu(0.5, -1.0)
    assert O.dnu_xnu_knu(0.7, 0.0) == 0.0
    assert math.isinf(O.CountingObjective(np.zeros((2, 2)), np.zeros(2)).loglik([1.0, 0.1, 0.5]))


def test_nugget_restatement_pins():
    """eval_all_nugget (config 5, not in the reference): tau^2 = 0 reproduces the reference
    algorithm's eval_all, and the sigma^2 score matches a central difference of the
    nugget log-likelihood."""
    from oracle import maternmle_cpu as O

    rng = np.random.default_rng(7)
    loc = rng.uniform(size=(120, 2))
    th = (1.1, 0.15, 1.3)
    z = O.cholesky(O.matrix(loc, th)) @ rng.standard_normal(120)
    a, b = O.eval_all(loc, z, th), O.eval_all_nugget(loc, z, th, 0.0)
    assert b[0] == pytest.approx(a[0], rel=1e-13)
    np.testing.assert_allclose(b[1], a[1], rtol=1e-10)
    np.testing.assert_allclose(b[2], a[2], rtol=1e-10)
    tau2 = 1e-2
    ll, g, f = O.eval_all_nugget(loc, z, th, tau2)
    assert ll == pytest.approx(O.loglik(loc, z, th, tau2), rel=1e-14)
    for i in range(3):
        h = 1e-6 * th[i]
        tp, tm = list(th), list(th)
        tp[i] += h
        tm[i] -= h
        fd = (O.loglik(loc, z, tp, tau2) - O.loglik(loc, z, tm, tau2)) / (2 * h)
        assert g[i] == pytest.approx(fd, rel=1e-5, abs=1e-6)
    np.testing.assert_array_equal(f, f.T)
    assert np.all(np.linalg.eigvalsh(f) > 0)
