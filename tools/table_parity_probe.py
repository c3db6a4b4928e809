"""ll deviation vs the golden small evaluations: exact generation vs generation tables."""
import json
import os
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as gpu  # noqa: E402

arr = np.load(REPO / "tests" / "golden" / "small.npz")
ev = json.loads((REPO / "tests" / "golden" / "small_evals.json").read_text())
for mode in ("0", "1"):
    os.environ["MLE_GEN_TABLE"] = mode
    worst = []
    for name, recs in ev["cases"].items():
        loc, z = arr[f"{name}_loc"], arr[f"{name}_z"]
        data = gpu.SpatialDataset(loc, z)
        for rec in recs:
            if "not_pd_pivot" in rec:
                continue
            ll = gpu.log_likelihood(data, rec["theta"])
            worst.append((abs(ll - rec["loglik"]) / abs(rec["loglik"]), name, rec["theta"], len(z)))
    worst.sort(reverse=True)
    print("MLE_GEN_TABLE", mode)
    for w in worst[:6]:
        print("  rel %.2e  %s theta=%s n=%d" % w)
