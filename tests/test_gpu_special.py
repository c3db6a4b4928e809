"""CUDA special functions vs the golden vectors (reference outputs + 40-digit mpmath)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_bessel_k_grid(gpu, bessel_golden):
    nus = np.array([p["nu"] for p in bessel_golden["grid"]])
    xs = np.array([p["x"] for p in bessel_golden["grid"]])
    k_mp = np.array([p["k_mp"] for p in bessel_golden["grid"]])
    k_ref = np.array([p["k_ref"] for p in bessel_golden["grid"]])
    got = gpu.bessel_k(nus, xs)
    # Temme/CF2 in FP64 is within a few ulp of the 40-digit value; scipy's AMOS kv (the
    # reference) itself deviates by up to ~7e-14 near x = 2.
    assert np.max(np.abs(got - k_mp) / k_mp) <= 5e-15
    assert np.max(np.abs(got - k_ref) / k_ref) <= 2e-13


def test_bessel_k_spots_and_closed_forms(gpu, bessel_golden):
    for s in bessel_golden["k_spots"]:
        assert gpu.bessel_k(s["nu"], s["x"]) == pytest.approx(s["k_mp"], rel=2e-14)
    xs = np.linspace(0.05, 30.0, 200)
    closed = np.sqrt(np.pi / (2 * xs)) * np.exp(-xs)
    np.testing.assert_allclose(gpu.bessel_k(0.5, xs), closed, rtol=1e-14)
    for nu in np.linspace(0.0, 3.0, 31):
        for x in (0.01, 0.5, 3.0, 25.0):
            assert gpu.bessel_k(nu, x) == gpu.bessel_k(-nu, x)


def test_dnu_grid(gpu, bessel_golden):
    worst_mp = worst_ref = 0.0
    for nu in sorted({p["nu"] for p in bessel_golden["grid"]}):
        pts = [p for p in bessel_golden["grid"] if p["nu"] == nu]
        xs = np.array([p["x"] for p in pts])
        got = gpu.dnu_xnu_knu(nu, xs)
        mp_ = np.array([p["dnu_mp"] for p in pts])
        ref = np.array([p["dnu_ref"] for p in pts])
        worst_mp = max(worst_mp, np.max(np.abs(got - mp_) / (1 + np.abs(mp_))))
        worst_ref = max(worst_ref, np.max(np.abs(got - ref) / (1 + np.abs(ref))))
    assert worst_mp <= 1e-6      # reference acceptance criterion 1
    assert worst_ref <= 1e-9     # parity with the reference's own outputs


def test_dnu_spots(gpu, bessel_golden):
    for s in bessel_golden["spots"]:
        got = gpu.dnu_xnu_knu(s["nu"], s["x"])
        if s["regime"] == "finite_diff":
            # the reference's lag-1e-9 forward difference carries ~1e-6 relative noise
            assert abs(got - s["dnu_ref"]) <= 1e-5 * (1 + abs(s["dnu_ref"]))
            assert abs(got - s["dnu_mp"]) <= 1e-5 * (1 + abs(s["dnu_mp"]))
        else:
            assert abs(got - s["dnu_ref"]) <= 1e-9 * (1 + abs(s["dnu_ref"])), s
            assert abs(got - s["dnu_mp"]) <= 1e-6 * (1 + abs(s["dnu_mp"])), s


def test_dnu_zero_and_domain(gpu):
    assert gpu.dnu_xnu_knu(0.7, 0.0) == 0.0
    out = gpu.dnu_xnu_knu(0.77, np.array([0.0, 0.5, 5.0, 10.0, 31.0]))
    for x, v in zip([0.0, 0.5, 5.0, 10.0, 31.0], out):
        assert v == gpu.dnu_xnu_knu(0.77, x)
    with pytest.raises(ValueError):
        gpu.dnu_xnu_knu(0.0, 1.0)
    with pytest.raises(ValueError):
        gpu.dnu_xnu_knu(0.5, -1.0)
    with pytest.raises(ValueError):
        gpu.bessel_k(0.5, -1.0)
    with pytest.raises(ValueError):
        gpu.bessel_k(math.nan, 1.0)


def test_case4_half_integer(gpu):
    # nu = 1/2 near-half-integer band at x >= 30 uses the forward difference; nu = 0.3 the
    # large-x series; both must track the 40-digit value.
    x = 35.0
    closed = math.sqrt(math.pi / 2.0) * math.exp(-x) * math.log(x)
    assert gpu.dnu_xnu_knu(0.5, x) == pytest.approx(closed, rel=1e-5)


def test_matern_elementwise_closed_forms(gpu):
    h = np.linspace(0.01, 5.0, 200)
    np.testing.assert_allclose(gpu.matern_cov(h, (1.0, 0.1, 0.5)), np.exp(-h / 0.1), rtol=1e-12)
    np.testing.assert_allclose(gpu.matern_cov(h, (2.0, 1.0, 1.5)), 2 * (1 + h) * np.exp(-h),
                               rtol=1e-12)
    assert gpu.matern_cov(0.0, (3.2, 1.7, 1.9)) == 3.2
    assert gpu.dcov_dsigma2(0.0, (1.7, 0.2, 0.8)) == 1.0
    assert gpu.dcov_dalpha(0.0, (1.0, 0.3, 1.2)) == 0.0
    assert gpu.dcov_dnu(0.0, (1.0, 0.3, 1.2)) == 0.0
    assert gpu.dcov_dalpha(0.1, (1.0, 0.1, 0.5)) == pytest.approx(10 * math.exp(-1), rel=1e-12)
    grid = np.arange(0.0, 5.0 + 1e-9, 0.01)
    for th in ((1.0, 0.1, 0.5), (0.3, 0.7, 1.3), (2.0, 0.25, 2.4)):
        v = gpu.matern_cov(grid, th)
        assert np.all(np.diff(v) <= 0.0) and np.all(v[1:] > 0.0) and np.all(v <= th[0])
    with pytest.raises(ValueError):
        gpu.matern_cov(-0.1, (1.0, 0.1, 0.5))


def test_matern_derivatives_vs_oracle(gpu):
    from oracle import maternmle_cpu as O

    rng = np.random.default_rng(3)
    h = rng.uniform(0.0, 2.0, 4000)
    for th in ((1.0, 0.3, 1.2), (0.7, 0.05, 0.4), (1.5, 0.05, 0.8), (1.0, 0.2, 1.5),
               (0.9, 0.08, 2.6)):
        for kind, fn in (("sigma", gpu.matern_cov), ("sigma2", gpu.dcov_dsigma2),
                         ("alpha", gpu.dcov_dalpha), ("nu", gpu.dcov_dnu)):
            got, ref = fn(h, th), O.elem(h, th, kind)
            scale = np.max(np.abs(ref))
            # The reference's case-2 series (bessel.py:213-222) cancels catastrophically as
            # x -> 8.5: its own error vs 40-digit truth reaches 8e-8 relative there (nu=2.6,
            # x=8.4), i.e. ~2e-9 of max|dC/dnu|; two roundings of that formula differ by as much.
            tol = 1e-12 if kind != "nu" else 1e-8
            assert np.max(np.abs(got - ref)) <= tol * scale, (th, kind)


def _case2_term_mass(O, nu, x):
    """sum_k |term_k| of the case-2 series (the oracle's loop with absolute values)."""
    import math

    from scipy import special as sps

    gp = sps.gamma(nu)
    gn = -math.pi / (math.sin(math.pi * nu) * nu * gp)
    pp, pn = float(sps.digamma(nu)), float(sps.digamma(-nu))
    tlx, x2n, q = 2.0 * np.log(x), x ** (2.0 * nu), 0.25 * x * x
    pref, g_p, g_n, d_p, d_n = np.full_like(x, 0.5), 1.0, 1.0, 0.0, 0.0
    mass = np.zeros_like(x)
    for k in range(O.K2 + 1):
        if k:
            pref = pref * q / k
            g_p /= nu + k
            g_n /= -nu + k
            d_p -= 1.0 / (nu + k)
            d_n -= 1.0 / (-nu + k)
        tp = 2.0 ** nu * (O.LOG2 + pp - d_n) * gp * g_n
        tn = 2.0 ** -nu * x2n * (-O.LOG2 + tlx - pn + d_p) * gn * g_p
        mass = mass + pref * (np.abs(tp) + np.abs(tn))
    return mass


def test_case_series_vs_oracle(gpu):
    """case2/3/4_series on their own domains vs the oracle's restatement of bessel.py:184-318."""
    from oracle import maternmle_cpu as O

    x2 = np.geomspace(1e-3, 8.49, 60)
    x3 = np.linspace(8.5, 29.99, 60)
    x4 = np.geomspace(30.0, 300.0, 40)
    for nu in (0.3, 0.77, 1.5, 2.2):
        got = gpu.case2_series(nu, x2)
        ref = O.small_series(nu, x2)
        # the 21-term series cancels (bessel.py:213-222): its terms reach ~1e6 near x = 8.5
        # (nu = 2.2) while the sum is O(1), so two correct summation orders differ by
        # ~1e-16 x sum |terms| (measured: 2.8e-10 absolute at x = 8.49, nu = 2.2)
        assert np.all(np.abs(got - ref) <= 5e-14 * (1 + _case2_term_mass(O, nu, x2))), nu
        np.testing.assert_allclose(gpu.case3_series(nu, x3), O.mid_series(nu, x3),
                                   rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(gpu.case4_series(nu, x4), O.large_series(nu, x4),
                                   rtol=1e-12, atol=1e-300)
    assert isinstance(gpu.case4_series(1.5, 40.0), float)
    # half-integer nu: the a_k product vanishes and the series stops early (bessel.py:311-313)
    np.testing.assert_allclose(gpu.case4_series(0.5, x4), O.large_series(0.5, x4), rtol=1e-13)


def test_mid_range_small_order_warning(gpu):
    with pytest.warns(gpu.MidRangeSmallOrderWarning):
        gpu.case3_series(0.03, np.array([9.0, 12.0]))
    with pytest.warns(gpu.MidRangeSmallOrderWarning):
        gpu.dnu_xnu_knu(0.03, np.array([1.0, 9.0]))
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("error")
        gpu.dnu_xnu_knu(0.03, np.array([1.0, 40.0]))  # no mid-range element: no warning
        gpu.case3_series(0.06, 9.0)


def test_simulate_grf_alias(gpu):
    """simulate_grf (simulate.py:100-106) draws z = L u with the reference's seeded normals."""
    from oracle import maternmle_cpu as O

    loc = gpu.jittered_grid(12, 3)
    th = gpu.MaternParams(1.2, 0.15, 0.9)
    z = gpu.simulate_grf(loc, th, 5)
    ref = O.cholesky(O.matrix(loc, th.as_array())) @ np.random.default_rng(5).standard_normal(144)
    np.testing.assert_allclose(z, ref, rtol=1e-11, atol=1e-12)
