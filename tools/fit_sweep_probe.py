"""Fisher-BT fits on seeded small fields: the GPU objective against the CPU oracle's objective
under the same host loop (call counts, termination, theta_hat, loglik_at_hat)."""
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402
from oracle import maternmle_cpu as O  # noqa: E402

CASES = [
    ("gmm300", lambda: m.gmm_locations(300, 11), (1.2, 0.05, 0.6), (1.0, 0.1, 1.0), None),
    ("grid324", lambda: m.jittered_grid(18, 3), (0.8, 0.12, 1.8), (0.5, 0.05, 1.0), None),
    ("gmm300-L9", lambda: m.gmm_locations(300, 12), (1.5, 0.07, 0.9), (0.5, 0.03, 0.4), (2.0, 0.2, 1.6)),
    ("unif350", lambda: np.random.default_rng(4).uniform(size=(350, 2)), (2.0, 0.03, 0.35), (1.0, 0.1, 1.0), None),
]


def run_cases():
    out = []
    for name, mk, th_true, lo, hi in CASES:
        loc = mk()
        low = O.cholesky(O.matrix(loc, th_true, "sigma"))
        z = low @ np.random.default_rng(99).standard_normal(len(loc))
        cfg = m.FisherBTConfig(theta_lower=m.MaternParams(*lo),
                               theta_upper=m.MaternParams(*(hi or lo)))
        t0 = time.time()
        ref = m.fisher_bt(m.SpatialDataset(loc, z), cfg, objective=O.CountingObjective(loc, z))
        t1 = time.time()
        res = m.fisher_bt(m.SpatialDataset(loc, z), cfg)
        out.append((name, ref, res, t1 - t0, time.time() - t1))
    return out


if __name__ == "__main__":
    for name, ref, res, tc, tg in run_cases():
        same = (res.grad_calls, res.loglik_calls, res.termination) == (ref.grad_calls, ref.loglik_calls, ref.termination)
        dth = np.max(np.abs(res.theta_hat.as_array() - ref.theta_hat.as_array()) / np.abs(ref.theta_hat.as_array()))
        print(name, "counts/termination equal:", same, (ref.grad_calls, ref.loglik_calls, ref.termination),
              (res.grad_calls, res.loglik_calls, res.termination), "theta_hat rel dev %.1e" % dth,
              "ll dev %.1e" % (abs(res.loglik_at_hat - ref.loglik_at_hat) / abs(ref.loglik_at_hat)),
              "theta_hat", np.round(ref.theta_hat.as_array(), 5), "cpu %.1fs gpu %.2fs" % (tc, tg))
