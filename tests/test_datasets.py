"""Pinned workload generators (CPU)."""

import numpy as np
from scipy.spatial.distance import pdist

import paper_2601_11437_b200 as m
from conftest import config_data


def test_jittered_grid_properties():
    for side in (5, 30, 60):
        loc = m.jittered_grid(side, 3)
        h = 1.0 / side
        assert loc.shape == (side * side, 2)
        ii, jj = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
        base = np.column_stack([(ii.ravel() + 0.5) * h, (jj.ravel() + 0.5) * h])
        assert np.all(np.abs(loc - base) <= 0.4 * h)
        assert pdist(loc).min() >= 0.2 * h - 1e-15
        np.testing.assert_array_equal(loc, m.jittered_grid(side, 3))


def test_committed_config_locations_are_the_generator_output():
    for name, seeds in (("config1", (0,)), ("config2", (0, 1, 2, 3, 4))):
        wl = m.WORKLOADS[name]
        for s in seeds:
            loc, z = config_data(name, s)
            np.testing.assert_array_equal(loc, wl.locations(s))
            assert z.shape == (wl.n,)


def test_gmm_locations():
    loc = m.gmm_locations(5000, 0)
    assert loc.shape == (5000, 2)
    assert np.all((loc[:, 0] >= 0) & (loc[:, 0] <= 1.5) & (loc[:, 1] >= 0) & (loc[:, 1] <= 1))
    assert pdist(loc).min() >= 1e-9
    np.testing.assert_array_equal(loc, m.gmm_locations(5000, 0))


def test_workload_table():
    assert [m.WORKLOADS[f"config{i}"].n for i in range(1, 6)] == [900, 3600, 16384, 65536, 100000]
    assert m.WORKLOADS["config2"].seeds == (0, 1, 2, 3, 4)
