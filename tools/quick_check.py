"""First-light GPU check against the committed golden fixtures (developer tool)."""

import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

G = REPO / "tests" / "golden"


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


bg = json.loads((G / "bessel_golden.json").read_text())
worst_k = worst_d = worst_dref = 0.0
for p in bg["grid"]:
    k = m.bessel_k(p["nu"], p["x"])
    d = m.dnu_xnu_knu(p["nu"], p["x"])
    worst_k = max(worst_k, abs(k - p["k_ref"]) / abs(p["k_ref"]))
    worst_d = max(worst_d, abs(d - p["dnu_mp"]) / (1 + abs(p["dnu_mp"])))
    worst_dref = max(worst_dref, abs(d - p["dnu_ref"]) / (1 + abs(p["dnu_ref"])))
print(f"bessel grid: K vs scipy {worst_k:.2e}; dnu vs mpmath {worst_d:.2e}; dnu vs ref {worst_dref:.2e}")

sm = np.load(G / "small.npz")
ev = json.loads((G / "small_evals.json").read_text())
thetas = ev["thetas"]
for name in ev["cases"]:
    loc, z = sm[f"{name}_loc"], sm[f"{name}_z"]
    data = m.SpatialDataset(loc, z)
    msg = [name, f"n={loc.shape[0]}"]
    if f"{name}_t0_sigma" in sm:
        w = 0.0
        for ti in range(4):
            th = thetas[ti]
            w = max(w, rel(m.build_cov_matrix(data, th), sm[f"{name}_t{ti}_sigma"]))
            for which in ("sigma2", "alpha", "nu"):
                got = m.build_dcov_matrix(data, th, which)
                ref = sm[f"{name}_t{ti}_{which}"]
                err = np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)
                w = max(w, err)
        msg.append(f"matrices {w:.1e}")
    worst_ll = worst_g = worst_f = 0.0
    for rec in ev["cases"][name]:
        th = rec["theta"]
        if "not_pd_pivot" in rec:
            try:
                m.log_likelihood(data, th)
                msg.append("NOTPD-MISSED")
            except m.NotPositiveDefinite as e:
                msg.append(f"notpd {e.pivot} vs {rec['not_pd_pivot']}")
            continue
        ll = m.log_likelihood(data, th)
        worst_ll = max(worst_ll, abs(ll - rec["loglik"]) / abs(rec["loglik"]))
        r = m.grad_and_fisher(data, th)
        worst_ll = max(worst_ll, abs(r.loglik - rec["eval_loglik"]) / abs(rec["eval_loglik"]))
        worst_g = max(worst_g, float(np.max(np.abs(r.grad - rec["grad"]) /
                                            (1 + np.abs(rec["grad"])))))
        worst_f = max(worst_f, rel(r.fisher, rec["fisher"]))
    msg.append(f"ll {worst_ll:.1e} grad {worst_g:.1e} fisher {worst_f:.1e}")
    print(" ".join(msg))

# cholesky vs numpy
rng = np.random.default_rng(1)
for n in (1, 2, 130, 300):
    a = rng.standard_normal((n, n))
    spd = a @ a.T + n * np.eye(n)
    L = m.cholesky_lower(spd)
    print("chol", n, rel(L[np.tril_indices(n)], np.linalg.cholesky(spd)[np.tril_indices(n)]))
try:
    m.cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
except m.NotPositiveDefinite as e:
    print("indefinite pivot", e.pivot, "(expect 1)")

c1 = np.load(G / "config1_seed0_data.npz")
data = m.SpatialDataset(c1["loc"], c1["z"])
for rec in json.loads((G / "config1_evals.json").read_text()):
    r = m.grad_and_fisher(data, rec["theta"])
    print("config1", rec["theta"], "ll", abs(r.loglik - rec["eval_loglik"]) / abs(rec["eval_loglik"]),
          "grad", np.abs(r.grad - rec["grad"]), "fisher", rel(r.fisher, rec["fisher"]))
fit = json.loads((G / "config1_seed0_fit.json").read_text())
th0 = m.MaternParams(*fit["theta0"])
t0 = time.perf_counter()
res = m.fisher_bt(data, m.FisherBTConfig(theta_lower=th0, theta_upper=th0))
wall = time.perf_counter() - t0
print("fit1", res.theta_hat.as_array(), fit["theta_hat"], rel(res.theta_hat.as_array(), fit["theta_hat"]),
      res.grad_calls, fit["grad_calls"], res.loglik_calls, fit["loglik_calls"], res.termination.value,
      fit["termination"], f"{wall:.3f}s {res.grad_calls / wall:.1f} it/s")

for side in (60, 128):
    loc = m.jittered_grid(side, 0)
    z = np.random.default_rng(0).standard_normal(side * side)
    data = m.SpatialDataset(loc, z)
    th = (1.0, 0.1, 1.2)
    eng = data.engine()
    for rep in range(3):
        t0 = time.perf_counter()
        eng.eval_all(th)
        t1 = time.perf_counter()
    pt = eng.phase_times()
    t2 = time.perf_counter()
    eng.loglik(th)
    t3 = time.perf_counter()
    pl = eng.phase_times()
    print(f"n={side*side}: eval_all {1e3*(t1-t0):.1f} ms", {k: round(v, 3) for k, v in pt.items()},
          f"TF/s(potrf+solve)={pt['flops']/((pt['potrf_ms']+pt['solve_ms'])*1e-3)/1e12:.2f}",
          f"gen GB/s={pt['gen_bytes']/(pt['gen_ms']*1e-3)/1e9:.1f}",
          f"| loglik {1e3*(t3-t2):.1f} ms", {k: round(v, 3) for k, v in pl.items()})
