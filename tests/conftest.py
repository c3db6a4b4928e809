"""Shared fixtures.  ``-m "not gpu"`` runs on CPU (oracle vs golden, host logic,
C-ABI exports, gloo multi-process); ``-m gpu`` runs the CUDA parity tests."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")
    config.addinivalue_line("markers", "slow: long-running")


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def golden_small():
    return np.load(GOLDEN / "small.npz"), load_json("small_evals.json")


@pytest.fixture(scope="session")
def bessel_golden():
    return load_json("bessel_golden.json")


def config_data(name, seed=0):
    d = np.load(GOLDEN / f"{name}_seed{seed}_data.npz")
    return d["loc"], d["z"]


def fit_golden(name, seed=0):
    path = GOLDEN / f"{name}_seed{seed}_fit.json"
    return json.loads(path.read_text()) if path.exists() else None


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference package (only in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference tree not present (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import maternmle

    return maternmle


def fd_regime(theta, locations=None):
    """theta whose nu sits in the reference's finite-difference band (bessel.py:126-141):
    nu within 1e-6 of an integer (case-2 range, x < 8.5), or of a half-integer when some
    u = h / alpha >= 30 can occur (case-4 range; bounded by the locations' bounding-box
    diagonal when the locations are given)."""
    nu = theta[2]
    if abs(nu - round(nu)) <= 1e-6:
        return True
    if abs(nu + 0.5 - round(nu + 0.5)) > 1e-6:
        return False
    if locations is None:
        return True
    loc = np.asarray(locations, float)
    diag = float(np.hypot(*(loc.max(axis=0) - loc.min(axis=0)))) if len(loc) > 1 else 0.0
    return diag / theta[1] >= 30.0


@pytest.fixture(scope="session")
def gpu():
    import paper_2601_11437_b200 as m

    if m.device_count() < 1:
        pytest.fail("gpu-marked test but no CUDA device is visible")
    return m


os.environ.setdefault("OPENBLAS_NUM_THREADS", "4")
