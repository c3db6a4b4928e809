"""The rank-sharded engine at config 4's full size (n = 65,536) with two ranks stepped in one
process on one B200 (InProcessComm: the broadcasts are device copies), against the
single-context engine: log-likelihood, score and Fisher at theta_true.  Memory: the two
ranks' panels together are the three 34.5 GB matrices, plus a W cache each.

    python tools/dist_config4_check.py > out.json
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_2601_11437_b200 as m  # noqa: E402
from paper_2601_11437_b200.distributed import DistributedEngine, InProcessComm  # noqa: E402
from test_gpu_likelihood import score_scale  # noqa: E402

wl = m.WORKLOADS["config4"]
loc = wl.locations(0)
z = m.simulate_field(loc, wl.theta_true, 0)
th = np.array(wl.theta_true, float)
eng = m.Engine(loc, z)
t0 = time.perf_counter()
ll, g, f = eng.eval_all(th)
t_single = time.perf_counter() - t0
eng.close()
m._native.lib.mle_release_cached_memory()
out = {"n": wl.n, "theta": th.tolist(), "single": {"loglik": ll, "grad": g.tolist(),
                                                    "fisher": f.tolist(), "seconds": t_single}}
for world in (2,):
    d = DistributedEngine(loc, z, InProcessComm(world))
    t0 = time.perf_counter()
    dl, dg, df = d.eval_all(th)
    dt = time.perf_counter() - t0
    dll = d.loglik(th)
    d.close()
    scale = score_scale(th, wl.n, g, f)
    out[f"world{world}"] = {
        "loglik": dl, "grad": dg.tolist(), "fisher": df.tolist(), "loglik_only": dll,
        "seconds_sequential_ranks": dt, "wcache": True,
        "loglik_rel": abs(dl - ll) / abs(ll),
        "score_rel_scale": (np.abs(dg - g) / scale).tolist(),
        "fisher_rel": float(np.max(np.abs(df - f) / np.abs(f)))}
print(json.dumps(out, indent=1))
