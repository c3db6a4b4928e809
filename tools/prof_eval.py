"""Profiling driver: one eval_all + one loglik at config-2 size after warm-up."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_11437_b200 as m  # noqa: E402

n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 60
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
loc = m.jittered_grid(n_side, 0)
z = np.random.default_rng(0).standard_normal(loc.shape[0])
data = m.SpatialDataset(loc, z)
th = (1.0, 0.2, 1.5)
for _ in range(warm):
    data.engine().eval_all(th)
    data.engine().loglik(th)
ev = data.engine().eval_all(th)
p1 = data.engine().phase_times()
ll = data.engine().loglik(th)
p2 = data.engine().phase_times()
print("eval_all", p1)
print("loglik", p2)
