"""Batched loglik / eval_all pass times (5 config-2 replicas) with and without look-ahead."""
import os
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
eng = [d.engine() for d in data]
th = np.array([1.0, 0.2, 1.5])
for la in ("1", "0", "1"):
    os.environ["MLE_LOOKAHEAD"] = la
    for mode, name in ((1, "loglik"), (2, "eval_all")):
        ts = []
        for r in range(6):
            t = th * (1 + 1e-7 * (r + 1) * (3 if mode == 1 else 1))
            m.eval_batch(eng, [t] * 5, [mode] * 5)
            p = eng[0].phase_times()
            ts.append((p["total_ms"], p["potrf_ms"], p["solve_ms"]))
        ts = np.median(np.array(ts[1:]), axis=0)
        print(f"lookahead={la} {name:8s} total {ts[0]:.3f} ms  potrf {ts[1]:.3f}  solve {ts[2]:.3f}")
