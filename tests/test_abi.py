"""The C-ABI library loads, exports every symbol include/maternfisher.h declares, and
rejects bad arguments without touching a GPU.  CPU-only (no compute calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2601_11437_b200 as m
from paper_2601_11437_b200 import _native as nat

HEADER = Path(__file__).resolve().parent.parent / "include" / "maternfisher.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(mle_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(nat.EXPORTED)


def test_version_and_device_count():
    assert b"sm_100a" in nat.lib.mle_version()
    assert nat.lib.mle_device_count() >= 0


def test_invalid_arguments_rejected_before_device_work():
    out = np.zeros(1)
    x = np.array([-1.0])
    assert nat.lib.mle_bessel_k(0.5, nat.as_ptr(x), 1, 0, nat.as_ptr(out)) == nat.MLE_INVALID
    assert nat.lib.mle_dnu_xnu_knu(0.0, nat.as_ptr(np.array([1.0])), 1, 0,
                                   nat.as_ptr(out)) == nat.MLE_INVALID
    bad = np.array([1.0, -0.1, 0.5])
    assert nat.lib.mle_matern_elem(nat.as_ptr(bad), 0, nat.as_ptr(np.array([0.1])), 1, 0,
                                   nat.as_ptr(out)) == nat.MLE_INVALID
    h = ctypes.c_void_p()
    loc = np.zeros((1, 2))
    assert nat.lib.mle_ctx_create(nat.as_ptr(loc), nat.as_ptr(np.zeros(1)), 0, 0, 0.0,
                                  ctypes.byref(h)) == nat.MLE_INVALID
    nanv = np.array([np.nan])
    assert nat.lib.mle_ctx_create(nat.as_ptr(loc), nat.as_ptr(nanv), 1, 0, 0.0,
                                  ctypes.byref(h)) == nat.MLE_INVALID
    with pytest.raises(ValueError):
        m.bessel_k(0.5, 0.0)
    with pytest.raises(ValueError):
        m.dnu_xnu_knu(-0.5, 1.0)


@pytest.mark.skipif(m.device_count() > 0, reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    """Without a GPU every compute entry point errors: there is no CPU fallback."""
    with pytest.raises(nat.NativeError):
        m.bessel_k(0.5, 1.0)
    data = m.SpatialDataset(np.array([[0.0, 0.0], [0.1, 0.0]]), np.zeros(2))
    with pytest.raises(nat.NativeError):
        m.log_likelihood(data, (1.0, 0.1, 0.5))
    obj = m.LikelihoodObjective(data)
    with pytest.raises(nat.NativeError):  # CUDA failures are never mapped to -inf
        obj.loglik([1.0, 0.1, 0.5])


def test_sharded_entry_points_reject_null_handles():
    """The rank-sharded C-ABI (mle_dctx_*) validates its handle before any device work."""
    out = np.zeros(32)
    h = ctypes.c_void_p()
    assert nat.lib.mle_dctx_set_async(None, 1) == nat.MLE_INVALID
    assert nat.lib.mle_dctx_stream(None, ctypes.byref(h)) == nat.MLE_INVALID
    assert nat.lib.mle_dctx_wcache(None, 1) == nat.MLE_INVALID
    assert nat.lib.mle_dctx_update_range(None, 0, None, 0, 1) == nat.MLE_INVALID
    assert nat.lib.mle_dctx_right_range(None, 0, None, None, 0, 1) == nat.MLE_INVALID
    assert nat.lib.mle_dctx_panel_partials(None, nat.as_ptr(out)) == nat.MLE_INVALID
    assert nat.lib.mle_dctx_create(nat.as_ptr(np.zeros((2, 2))), nat.as_ptr(np.zeros(2)), 2, 0,
                                   0.0, 2, 2, ctypes.byref(h)) == nat.MLE_INVALID  # rank >= world
