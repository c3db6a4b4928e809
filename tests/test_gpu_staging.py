"""Operand staging of the DMMA GEMM (linalg.cu dgemm_kernel) and the NVTX switch.

The switches are read once per process, so every variant runs in its own interpreter:

* MLE_DGEMM_STAGE unset (bulk copies on an mbarrier ring for kBNK products, cp.async for
  kBKN), =cpasync (Ampere-style everywhere), =bulk (bulk copies everywhere): same stages'
  contents and the same k order, so log-likelihood, score and Fisher matrix must be
  bit-identical -- on ragged sizes (edge tiles), the config-1 / config-2 goldens' data (full
  sweeps) and an n = 16,384 grid (two-sided path; the size at which a missing proxy fence
  before the stage release showed up as wrong factors);
* MLE_NVTX=1 (phase ranges) changes no result;
* MLE_GEN_STAGE=0 / 2 (gen.cu: the generation kernels read their table coefficients from
  global memory only / both kernels stage the tile's table intervals in shared memory; by
  default only the derivative kernel stages): same coefficients and Horner order, so every
  generated element -- and with it every result -- must be bit-identical.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(repo)r)
import paper_2601_11437_b200 as m
out = {}
def bits(res):
    ll, g, f = res[:3]
    return [float(ll).hex()] + [float(x).hex() for x in np.ravel(g)] + [float(x).hex() for x in np.ravel(f)]
rng = np.random.default_rng(3)
for n in (131, 700, 1153):
    side = int(np.ceil(np.sqrt(n)))
    loc = m.jittered_grid(side, 1)[:n]
    z = rng.standard_normal(n)
    e = m.Engine(loc, z)
    out["ragged%%d" %% n] = bits(e.eval_all((0.9, 0.15, 0.7))) + [float(e.loglik((1.1, 0.1, 1.3))).hex()]
# unordered random locations: a generation tile's pairs span many table intervals (more than
# the shared-memory staging holds: the per-tile fallback to global loads), plus two coincident
# points' neighbourhood handled by the exact path (a tiny nugget keeps Sigma factorizable)
locr = rng.random((700, 2))
locr[17] = locr[400]
er = m.Engine(locr, rng.standard_normal(700), nugget=1e-3)
out["random700"] = bits(er.eval_all((0.8, 0.02, 1.2))) + [float(er.loglik((1.0, 0.3, 0.4))).hex()]
for name, th in (("config1", (1.0, 0.1, 0.5)), ("config2", (1.0, 0.2, 1.5))):
    d = np.load(%(repo)r + "/tests/golden/" + name + "_seed0_data.npz")
    out[name] = bits(m.Engine(d["loc"], d["z"]).eval_all(th))
d = np.load(%(repo)r + "/tests/golden/config3_seed0_data.npz")
e3 = m.Engine(d["loc"], d["z"])
out["config3"] = bits(e3.eval_all((1.5, 0.05, 0.8))) + [float(e3.loglik((3.0, 0.05, 0.8))).hex()]
print("RESULT " + json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ)
    for k in ("MLE_DGEMM_STAGE", "MLE_NVTX", "MLE_GEN_STAGE"):
        env.pop(k, None)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD % {"repo": str(REPO)}], env=env,
                       capture_output=True, text=True, timeout=600)
    lines = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and lines, (env_extra, p.stdout[-1500:], p.stderr[-1500:])
    return json.loads(lines[0][7:])


@pytest.fixture(scope="module")
def default_bits(gpu):
    return _run({})


@pytest.mark.parametrize("env", [{"MLE_DGEMM_STAGE": "cpasync"}, {"MLE_DGEMM_STAGE": "bulk"},
                                 {"MLE_NVTX": "1"}, {"MLE_GEN_STAGE": "0"},
                                 {"MLE_GEN_STAGE": "2"}],
                         ids=["cpasync", "bulk", "nvtx", "gen-global", "gen-staged-both"])
def test_staging_variants_bit_identical(default_bits, env):
    got = _run(env)
    for key, ref in default_bits.items():
        assert got[key] == ref, (env, key)
