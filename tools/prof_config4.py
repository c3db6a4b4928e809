"""Profiling driver at BASELINE config 4 (n = 65,536): one Fisher iteration as the bench
times it -- a line-search loglik at a new theta (generation + Cholesky) followed by eval_all
at that theta (factor cache: derivative generation + both solve sweeps + reductions).

    python tools/prof_config4.py            (under ncu: launch list / --set full capture)
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_11437_b200 as m  # noqa: E402

wl = m.WORKLOADS["config4"]
loc = wl.locations(0)
z = m.simulate_field(loc, wl.theta_true, 0)
data = m.SpatialDataset(loc, z)
eng = data.engine()
eng.loglik(np.array([1.0, 0.1, 1.0]))           # warm-up (buffers, tables)
th = np.array(wl.theta_true, float) * np.array([1.01, 0.99, 1.0])
ll = eng.loglik(th)
p1 = eng.phase_times()
ev = eng.eval_all(th)
p2 = eng.phase_times()
print("loglik", ll, p1)
print("eval_all", ev[0], p2)
