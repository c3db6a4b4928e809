"""Where do the non-device milliseconds of a fit step go?  Wraps eval_batch with timers."""
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402
from paper_2601_11437_b200 import batch as B  # noqa: E402

data = []
for s in range(5):
    d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
    data.append(m.SpatialDataset(d["loc"], d["z"]))
th0 = m.MaternParams(0.8, 0.1, 1.0)
cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
orig = B.eval_batch
acc = {"calls": 0, "eval_batch_s": 0.0}


def timed_eval_batch(*a, **k):
    t0 = time.perf_counter()
    out = orig(*a, **k)
    acc["eval_batch_s"] += time.perf_counter() - t0
    acc["calls"] += 1
    return out


B.eval_batch = timed_eval_batch
_c_call = B.nat.lib.mle_eval_batch
acc["c_s"] = 0.0


def timed_c_call(*a):
    t0 = time.perf_counter()
    rc = _c_call(*a)
    acc["c_s"] += time.perf_counter() - t0
    return rc


B.nat.lib.mle_eval_batch = timed_c_call
for r in range(3):
    acc.update(calls=0, eval_batch_s=0.0, c_s=0.0)
    coords = []
    t0 = time.perf_counter()
    B.fit_many(data, cfg, coordinator_out=coords)
    wall = time.perf_counter() - t0
    a = coords[0].acc
    dev = a["gen_ms"] + a["potrf_ms"] + a["solve_ms"] + a["reduce_ms"]
    print(f"step wall {1e3*wall:.1f} ms | in eval_batch {1e3*acc['eval_batch_s']:.1f} ms "
          f"({acc['calls']} calls) | device phases {dev:.1f} ms | host enqueue "
          f"{a['host_enqueue_ms']:.1f} ms | GPU idle between passes {a['gpu_gap_ms']:.1f} ms "
          f"+ spec/upload wait {a['spec_wait_ms']:.1f} ms "
          f"| in C call {1e3*acc['c_s']:.1f} ms | python outside eval_batch "
          f"{1e3*(wall-acc['eval_batch_s']):.1f} ms")
