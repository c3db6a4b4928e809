"""Profiling driver: one batched eval_all over the five config-2 replicas (after warm-up)."""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
data = []
for s in range(5):
    d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
    data.append(m.SpatialDataset(d["loc"], d["z"]))
eng = [d.engine() for d in data]
th = np.array([1.0, 0.2, 1.5])
for r in range(reps + 1):
    m.eval_batch(eng, [th * (1 + 1e-9 * r)] * 5, [mode] * 5)
    print(r, eng[0].phase_times())
