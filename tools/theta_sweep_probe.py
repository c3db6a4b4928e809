"""Table vs exact generation vs the CPU oracle over a seeded theta sweep (the set of
tests/test_gpu_likelihood.py::test_oracle_parity_theta_sweep): deviations of the
log-likelihood, score (of its component scale) and Fisher entries."""
import os
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
import paper_2601_11437_b200 as m  # noqa: E402
from oracle import maternmle_cpu as O  # noqa: E402
from test_gpu_likelihood import score_scale  # noqa: E402

rng = np.random.default_rng(41)
loc = m.jittered_grid(14, 5)
n = loc.shape[0]
z = rng.standard_normal(n)
thetas = [(float(s2), float(a), float(nu)) for s2, a, nu in zip(
    rng.uniform(0.2, 5.0, 12), rng.uniform(0.02, 0.15, 12), rng.uniform(0.15, 2.2, 12))]
thetas += [(1.0, 0.1, 0.5), (2.0, 0.05, 1.5), (0.7, 0.12, 1.001), (1.5, 0.03, 0.4999)]
for th in thetas:
    ll, g, f = O.eval_all(loc, z, th)
    row = []
    for tab in ("1", "0"):
        os.environ["MLE_GEN_TABLE"] = tab
        ev = m.Engine(loc, z).eval_all(np.array(th))
        sc = score_scale(th, n, ev[1], ev[2])
        row.append((abs(ev[0] - ll) / abs(ll), np.max(np.abs(ev[1] - g) / sc),
                    np.max(np.abs(ev[2] - f) / np.abs(f))))
    print("theta=(%.3f, %.4f, %.4f)  table: ll %.1e score %.1e fisher %.1e | exact: ll %.1e score %.1e fisher %.1e"
          % (th + row[0] + row[1]))
