"""Config 4 (n = 65,536): the derivative blocks of one eval_all (factor resident), batched
(both blocks in every launch) vs sequential-derivative mode (MLE_SEQ_DERIVS=1: one block at
a time).  Each mode in its own process (the mode is fixed at context creation)."""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent


def child():
    import numpy as np
    sys.path.insert(0, str(REPO))
    import paper_2601_11437_b200 as m
    wl = m.WORKLOADS["config4"]
    loc = wl.locations(0)
    z = m.simulate_field(loc, wl.theta_true, 0)
    eng = m.Engine(loc, z)
    th = np.array(wl.theta_true)
    out = {"sequential": bool(eng.sequential_derivs)}
    for rep in range(2):
        t = th * (1 + 1e-3 * rep)
        t0 = time.perf_counter()
        ll = eng.loglik(t)
        t1 = time.perf_counter()
        ev = eng.eval_all(t)
        t2 = time.perf_counter()
        out[f"rep{rep}"] = {"loglik_s": t1 - t0, "blocks_s": t2 - t1,
                            "blocks_tflops": 2 * 65536.0 ** 3 / (t2 - t1) / 1e12,
                            "grad": [float(x) for x in ev[1]]}
    print("RESULT " + json.dumps(out))


if "--child" in sys.argv:
    child()
else:
    for mode in ("0", "1"):
        env = dict(os.environ, MLE_SEQ_DERIVS=mode)
        p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True,
                           text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        print(mode, line[0][7:] if line else (p.stdout[-800:], p.stderr[-800:]))
