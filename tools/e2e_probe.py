"""Where does the end-to-end step spend time?  Context create / first eval / fits / release."""
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

host = []
for s in range(5):
    d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
    host.append((d["loc"], d["z"]))
th = np.array([1.0, 0.2, 1.5])
for it in range(3):
    t0 = time.perf_counter()
    ds = [m.SpatialDataset(loc, z) for loc, z in host]
    eng = [d.engine() for d in ds]
    t1 = time.perf_counter()
    m.eval_batch(eng, [th] * 5, [2] * 5)
    t2 = time.perf_counter()
    m.eval_batch(eng, [th * (1 + 1e-9)] * 5, [2] * 5)
    t3 = time.perf_counter()
    for d in ds:
        d.release()
    t4 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.1f} ms, first eval_all batch {1e3*(t2-t1):.1f} ms, "
          f"second {1e3*(t3-t2):.1f} ms, release {1e3*(t4-t3):.1f} ms", flush=True)
