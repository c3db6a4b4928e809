"""Sequential-derivative mode (engine.cu eval_all_seq; config 5 on one B200): eval_all
reduces the derivative blocks one at a time in a single work matrix, parks finished blocks
in the unused upper triangles and streams W_b block by block.  Per block it runs the same
generation and the same two-sided reduction as the batched path, so at sizes where both fit
the two must agree to rounding of the final sums (the log-likelihood bit for bit).

The mode is fixed when a context is created (MLE_SEQ_DERIVS=1 forces it, with the two-sided
path forced by MLE_SOLVE=2s below n = 16,384), so each variant runs in its own interpreter.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(repo)r)
import paper_2601_11437_b200 as m
out = {}
rng = np.random.default_rng(11)
def pack(res):
    ll, g, f = res[:3]
    return [float(ll)] + [float(x) for x in np.ravel(g)] + [float(x) for x in np.ravel(f)]
for name, n, nugget, th in (("grid1300", 1300, 0.0, (0.9, 0.12, 0.8)),
                            ("grid1300_nugget", 1300, 1e-3, (0.9, 0.12, 0.8)),
                            ("ragged777", 777, 0.0, (1.2, 0.2, 1.4)),
                            ("gmm2100_nugget", 2100, 1e-6, (0.9, 0.08, 1.0))):
    if name.startswith("gmm"):
        loc = m.gmm_locations(n, 5)
    else:
        side = int(np.ceil(np.sqrt(n)))
        loc = m.jittered_grid(side, 2)[:n]
    z = rng.standard_normal(n)
    e = m.Engine(loc, z, nugget=nugget)
    out.setdefault("modes", []).append(bool(e.sequential_derivs))
    a = pack(e.eval_all(th))                 # factor + blocks
    b = pack(e.eval_all(th))                 # resident factor + blocks
    ll = float(e.loglik(th))
    c = pack(e.eval_all(tuple(x * 1.01 for x in th)))
    out[name] = {"first": a, "again": b, "loglik": ll, "moved": c}
# a full fit (config-1 data) through the objective surface
d = np.load(%(repo)r + "/tests/golden/config1_seed0_data.npz")
data = m.SpatialDataset(d["loc"], d["z"])
th0 = m.MaternParams(0.5, 0.05, 1.0)
res = m.fisher_bt(data, m.FisherBTConfig(theta_lower=th0, theta_upper=th0))
out["fit"] = {"theta": res.theta_hat.as_array().tolist(), "grad_calls": res.grad_calls,
              "loglik_calls": res.loglik_calls, "termination": res.termination.value,
              "loglik": float(res.loglik_at_hat)}
print("RESULT " + json.dumps(out))
"""


def _run(seq):
    env = dict(os.environ)
    env["MLE_SOLVE"] = "2s"
    env["MLE_SEQ_DERIVS"] = "1" if seq else "0"
    p = subprocess.run([sys.executable, "-c", CHILD % {"repo": str(REPO)}], env=env,
                       capture_output=True, text=True, timeout=900)
    lines = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and lines, (seq, p.stdout[-1500:], p.stderr[-1500:])
    return json.loads(lines[0][7:])


@pytest.fixture(scope="module")
def both(gpu):
    return _run(False), _run(True)


def _close(a, b, n):
    a, b = np.asarray(a), np.asarray(b)
    assert a[0] == b[0]  # log-likelihood: the same pass
    # the score is a difference of two O(n) terms: compare on that scale (as the golden tests)
    assert np.all(np.abs(a[1:4] - b[1:4]) <= 1e-11 * np.maximum(np.abs(b[1:4]), 10.0 * n)), (a, b)
    assert np.all(np.abs(a[4:] - b[4:]) <= 1e-11 * np.abs(b[4:])), (a[4:], b[4:])


@pytest.mark.parametrize("case,n", [("grid1300", 1300), ("grid1300_nugget", 1300),
                                    ("ragged777", 777), ("gmm2100_nugget", 2100)])
def test_sequential_blocks_match_batched(both, case, n):
    std, seq = both
    for key in ("first", "again", "moved"):
        _close(seq[case][key], std[case][key], n)
    assert seq[case]["loglik"] == std[case]["loglik"]
    # resident factor: identical to the evaluation that factored
    assert seq[case]["again"] == seq[case]["first"]


def test_modes_are_what_the_switch_says(both):
    std, seq = both
    assert std["modes"] == [False] * 4 and seq["modes"] == [True] * 4


def test_sequential_fit_matches_batched(both):
    std, seq = both
    assert seq["fit"]["grad_calls"] == std["fit"]["grad_calls"]
    assert seq["fit"]["loglik_calls"] == std["fit"]["loglik_calls"]
    assert seq["fit"]["termination"] == std["fit"]["termination"]
    assert np.allclose(seq["fit"]["theta"], std["fit"]["theta"], rtol=1e-9, atol=0)
    assert abs(seq["fit"]["loglik"] - std["fit"]["loglik"]) <= 1e-12 * abs(std["fit"]["loglik"])
