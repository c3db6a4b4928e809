"""Config-3 / config-4 Fisher-BT fits with both solve formulations (MLE_SOLVE=w: full sweeps,
MLE_SOLVE=2s: two-sided reduction): the same call counts, termination and theta_hat within
1e-6 is the size-independent check that the faster formulation does not change the fit.

    python tools/fit_paths_probe.py config4 > out.json
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_11437_b200 as m  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
wl = m.WORKLOADS[name]
npz = Path(__file__).resolve().parent.parent / "tests" / "golden" / f"{name}_seed0_data.npz"
if npz.exists():
    d = np.load(npz)
    loc, z = d["loc"], d["z"]
else:
    loc = wl.locations(0)
    z = m.simulate_field(loc, wl.theta_true, 0)
th0 = m.MaternParams(*wl.theta0)
cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
out = {"config": name}
for path in ("2s", "w"):
    os.environ["MLE_SOLVE"] = path
    data = m.SpatialDataset(loc, z)
    t0 = time.perf_counter()
    r = m.fisher_bt(data, cfg)
    out[path] = {"seconds": time.perf_counter() - t0, "grad_calls": r.grad_calls,
                 "loglik_calls": r.loglik_calls, "termination": r.termination.value,
                 "theta_hat": r.theta_hat.as_array().tolist(), "loglik_at_hat": r.loglik_at_hat,
                 "fisher_at_hat": np.asarray(r.fisher_at_hat).tolist()}
    data.release()
a, b = np.array(out["2s"]["theta_hat"]), np.array(out["w"]["theta_hat"])
out["theta_hat_rel_diff"] = float(np.max(np.abs(a - b) / np.abs(b)))
out["same_counts"] = (out["2s"]["grad_calls"], out["2s"]["loglik_calls"],
                      out["2s"]["termination"]) == (out["w"]["grad_calls"],
                                                    out["w"]["loglik_calls"],
                                                    out["w"]["termination"])
print(json.dumps(out, indent=1))
