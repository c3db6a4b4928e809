"""Config-2 (seed 0) log-likelihood under the engine variants selected by the environment,
against the reference goldens (config2_evals.json): prints the relative deviations."""
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

d = np.load(REPO / "tests/golden/config2_seed0_data.npz")
ev = json.loads((REPO / "tests/golden/config2_evals.json").read_text())
data = m.SpatialDataset(d["loc"], d["z"])
for th in ([1.0, 0.2, 1.5], ev[0]["theta"], ev[1]["theta"]):
    ll, g, f = data.engine().eval_all(np.array(th))
    ref = [r for r in ev if r["theta"] == list(th)]
    rel = (ll - ref[0]["eval_loglik"]) / abs(ref[0]["eval_loglik"]) if ref else None
    print(json.dumps({"theta": th, "ll": ll, "rel_vs_golden": rel}))
