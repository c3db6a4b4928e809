"""Generation at BASELINE config 4 (n = 65,536) under the kernel-profiling pass: gen_ms /
GB/s of one loglik (Sigma) and one eval_all (derivative pair), plus the results' bits, so two
builds / switches (e.g. MLE_GEN_STAGE=0 vs 1) can be compared across processes.

    MLE_GEN_STAGE=0 python tools/gen_config4_probe.py [config3]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2601_11437_b200 as m  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
wl = m.WORKLOADS[name]
loc = wl.locations(0)
z = m.simulate_field(loc, wl.theta_true, 0)
eng = m.SpatialDataset(loc, z).engine()
eng.loglik(np.array(wl.theta_true, float))  # warm-up (buffers, tables)
th = np.array(wl.theta_true, float) * np.array([1.01, 0.99, 1.0])
out = {"workload": name}
eng.kernel_profile(True)
ll = eng.loglik(th)
ks = eng.kernel_stats()
out["sigma_gen_ms"] = ks["gen_ms"]
out["sigma_gen_gbs"] = ks["gen_bytes"] / (ks["gen_ms"] * 1e-3) / 1e9
ev = eng.eval_all(th)
ks = eng.kernel_stats()
out["derivs_gen_ms"] = ks["gen_ms"]
out["derivs_gen_gbs"] = ks["gen_bytes"] / (ks["gen_ms"] * 1e-3) / 1e9
eng.kernel_profile(False)
out["bits"] = ([float(ll).hex(), float(ev[0]).hex()] + [float(x).hex() for x in np.asarray(ev[1]).ravel()]
               + [float(x).hex() for x in np.asarray(ev[2]).ravel()])
print("GENPROBE " + json.dumps(out))
