"""Ill-conditioned golden probe: GPU log-likelihood of the small goldens vs the reference,
under the generation / GEMM variants selected by the environment (MLE_GEN_TABLE,
MLE_FP64_GEMM).  Prints one JSON line per (case, theta) with the relative deviation and
the condition estimate of the device factor."""
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

arrays = np.load(REPO / "tests/golden/small.npz")
ev = json.loads((REPO / "tests/golden/small_evals.json").read_text())
for name, recs in ev["cases"].items():
    data = m.SpatialDataset(arrays[f"{name}_loc"], arrays[f"{name}_z"])
    for rec in recs:
        if "loglik" not in rec:
            continue
        ll = m.log_likelihood(data, rec["theta"])
        cond = data.engine().cond_estimate()
        print(json.dumps({"case": name, "theta": rec["theta"], "rel": (ll - rec["loglik"]) / abs(rec["loglik"]),
                          "cond_est": cond}))
