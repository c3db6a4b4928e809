"""The ctypes binding INTEGRATION.md §1 tells a maintainer to paste into the reference
(``maternmle/gpu.py``), executed as written:

* CPU (here): against the unmodified reference's own modules (its relative imports resolved
  to ``maternmle.likelihood`` / ``maternmle.matern``), the objective builds and, with no GPU,
  fails loudly instead of falling back;
* GPU: the same code drives a Fisher-BT fit (the reference's algorithm; on the GPU box the
  reference tree is absent, so the driver is this package's bit-identical ``fisher_bt`` and
  the two relative imports resolve to its identical ``NotPositiveDefinite`` / ``MaternParams``)
  and must reproduce the reference's golden config-1 fit."""

import re
import types
from pathlib import Path

import numpy as np
import pytest

from conftest import config_data, fit_golden

DOC = Path(__file__).resolve().parent.parent / "INTEGRATION.md"


def snippet_source():
    text = DOC.read_text()
    sec = text[text.index("## 1."):text.index("## 2.")]
    blocks = re.findall(r"```python\n(.*?)```", sec, flags=re.S)
    return blocks[0]


def load_snippet(likelihood_mod, matern_mod, lib_path):
    src = snippet_source()
    src = src.replace("from .likelihood import NotPositiveDefinite",
                      "NotPositiveDefinite = _likelihood.NotPositiveDefinite")
    src = src.replace("from .matern import MaternParams", "MaternParams = _matern.MaternParams")
    src = src.replace('"/path/to/paper_2601_11437_b200/libmaternfisher.so"', repr(str(lib_path)))
    mod = types.ModuleType("gpu_snippet")
    mod.__dict__.update(_likelihood=likelihood_mod, _matern=matern_mod)
    exec(compile(src, str(DOC), "exec"), mod.__dict__)
    return mod


def test_snippet_against_reference_modules_fails_loudly_without_gpu(reference):
    import paper_2601_11437_b200 as m
    from maternmle import likelihood, matern

    mod = load_snippet(likelihood, matern, m.LIB_PATH)
    assert hasattr(mod, "GpuLikelihoodObjective")
    if m.device_count() > 0:
        pytest.skip("a GPU is visible: the GPU test covers this")
    loc, z = config_data("config1")
    with pytest.raises(RuntimeError):
        mod.GpuLikelihoodObjective(matern.SpatialDataset(loc, z))


@pytest.mark.gpu
def test_snippet_objective_reproduces_reference_fit(gpu):
    from paper_2601_11437_b200 import likelihood, matern

    mod = load_snippet(likelihood, matern, gpu.LIB_PATH)
    gold = fit_golden("config1", 0)
    loc, z = config_data("config1")
    data = gpu.SpatialDataset(loc, z)
    obj = mod.GpuLikelihoodObjective(data)
    th0 = gpu.MaternParams(*gold["theta0"])
    res = gpu.fisher_bt(data, gpu.FisherBTConfig(theta_lower=th0, theta_upper=th0),
                        objective=obj)
    assert (res.grad_calls, res.loglik_calls) == (gold["grad_calls"], gold["loglik_calls"])
    assert obj.loglik_calls == gold["loglik_calls"] and obj.grad_calls == gold["grad_calls"]
    assert res.termination.value == gold["termination"]
    np.testing.assert_allclose(res.theta_hat.as_array(), gold["theta_hat"], rtol=1e-6)
    assert res.loglik_at_hat == pytest.approx(gold["loglik_at_hat"], rel=1e-10)
    # failure conventions: invalid theta -> -inf (counted), eval_all propagates
    assert obj.loglik(np.array([1.0, -1.0, 0.5])) == -np.inf
    with pytest.raises(ValueError):
        obj.eval_all(np.array([1.0, -1.0, 0.5]))
