"""Config-3 / intermediate-size log-likelihood and eval_all times against the far trailing
update's grid cap (MLE_FAR_CTAS, read once per process): min of 5 runs each.

    MLE_FAR_CTAS=132 python tools/far_ctas_probe.py 128
"""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_11437_b200 as m  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 128
loc = m.jittered_grid(side, 0)
z = m.simulate_field(loc, (1.5, 0.05, 0.8), 0)
eng = m.SpatialDataset(loc, z).engine()
th = np.array([1.5, 0.05, 0.8])
eng.loglik(th)
out = {}
for name in ("loglik", "eval_all"):
    ts = []
    for r in range(5):
        thr = th * (1 + 1e-9 * (r + 1))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = getattr(eng, name)(thr)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    out[name + "_ms"] = round(min(ts), 3)
    out[name + "_bits"] = float(res if name == "loglik" else res[0]).hex()
print("FARPROBE", os.environ.get("MLE_FAR_CTAS", "default"), side * side, out)
