"""Noise floor of the reference's own log-likelihood on the small goldens.

The reference takes K_nu from scipy.special.kv (AMOS), whose relative error reaches a few
1e-15 (up to 7e-14 near x = 2).  On the most ill-conditioned golden cases that error alone
moves the log-likelihood by ~1e-10, the north_star tolerance itself: there the reference
value is not pinned to better than that by its own arithmetic.  This script measures the
floor directly: the oracle's restatement of the reference pipeline (matern.py:100-104,
171-203; likelihood.py:63-89) run once with scipy's kv (reproduces the golden bit for bit)
and once with K_nu from 30-digit mpmath rounded to double, and also
with LAPACK on 1 and on 8 OpenBLAS threads (the blocked dpotrf sums in a thread-dependent
order, so the reference's own value changes with its thread count), and records
    floor = max(|l(scipy kv) - l(30-digit K_nu)|, |l(1 thread) - l(8 threads)|) / |l|
per (case, theta).  tests/test_gpu_likelihood.py uses max(1e-10, 3 * floor) as the
log-likelihood tolerance -- a bound that exceeds 1e-10 only where the reference's own K_nu
error already does.  Runs HERE only (mpmath); the output small_floor.json is committed.
"""

import json
import sys
import types
from pathlib import Path

import mpmath as mp
import numpy as np
from scipy import special as sps
from threadpoolctl import threadpool_limits

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle import maternmle_cpu as O  # noqa: E402

mp.mp.dps = 30


def kv_exact(nu, x):
    x = np.asarray(x, float)
    flat = [float(mp.besselk(mp.mpf(float(nu)), mp.mpf(float(v)))) for v in x.ravel()]
    return np.array(flat).reshape(x.shape)


def main():
    arrays = np.load(HERE / "small.npz")
    ev = json.loads((HERE / "small_evals.json").read_text())
    exact = types.SimpleNamespace(kv=kv_exact, gamma=sps.gamma, digamma=sps.digamma)
    out = {}
    for name, recs in ev["cases"].items():
        loc, z = arrays[f"{name}_loc"], arrays[f"{name}_z"]
        out[name] = []
        for rec in recs:
            if "loglik" not in rec:
                out[name].append(None)
                continue
            th = tuple(rec["theta"])
            O.sps = sps
            with threadpool_limits(1):
                l_sc = O.loglik(loc, z, th)
            with threadpool_limits(8):
                l_sc8 = O.loglik(loc, z, th)
            O.sps = exact
            try:
                with threadpool_limits(1):
                    l_ex = O.loglik(loc, z, th)
            finally:
                O.sps = sps
            out[name].append({"theta": list(th), "loglik_scipy_1thread": l_sc,
                              "loglik_scipy_8threads": l_sc8, "loglik_exact_k": l_ex,
                              "golden_vs_scipy_rel": (l_sc - rec["loglik"]) / abs(rec["loglik"]),
                              "floor": max(abs(l_sc - l_ex), abs(l_sc - l_sc8)) / abs(l_sc)})
            print(name, th, out[name][-1]["floor"], flush=True)
    (HERE / "small_floor.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
