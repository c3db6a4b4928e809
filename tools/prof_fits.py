"""Profiling driver: the five config-2 fits once (after one warm-up fit set), lock-step batched."""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

data = []
for s in range(5):
    d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
    data.append(m.SpatialDataset(d["loc"], d["z"]))
th0 = m.MaternParams(0.8, 0.1, 1.0)
cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for r in range(reps + 1):
    coords = []
    res = m.fit_many(data, cfg, coordinator_out=coords)
    print(r, coords[0].acc, coords[0].batches, coords[0].eval_passes, flush=True)
