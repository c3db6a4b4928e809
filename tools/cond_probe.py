"""Conditioning estimates (max/min diag L)^2 on the bench data and harder cases."""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
import paper_2601_11437_b200 as m  # noqa: E402
from conftest import config_data  # noqa: E402

for s in range(5):
    loc, z = config_data("config2", s)
    e = m.Engine(loc, z)
    for th in ((1.0, 0.2, 1.5), (0.8, 0.1, 1.0)):
        e.loglik(np.array(th))
        print(f"config2 seed {s} theta {th}: cond_est {e.cond_estimate():.3e}")
from oracle import maternmle_cpu as O  # noqa: E402
loc = m.gmm_locations(1500, 2)
z = np.random.default_rng(2).standard_normal(1500)
for tau in (0.0, 1e-6, 1e-4):
    e = m.Engine(loc, z, nugget=tau)
    try:
        e.loglik(np.array([0.9, 0.08, 1.013]))
        print(f"gmm1500 nugget {tau}: cond_est {e.cond_estimate():.3e}")
    except Exception as exc:
        print("gmm", tau, exc)
