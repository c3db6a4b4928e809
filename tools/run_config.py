"""Full Fisher-BT fit of a BASELINE config on one GPU, with a timed single-iteration
breakdown (gen / Cholesky / solves / reductions).  Writes one JSON record to stdout.

    python tools/run_config.py config3 [--breakdown-only]
    python tools/run_config.py config5 --loglik-only
    python tools/run_config.py config4 --breakdown-only --kernel-profile

--loglik-only: the one-GPU share of a config that does not fit eval_all on one B200
(config 5: Sigma, three derivative blocks and M are 4 x 80 GB): field simulation, then
log-likelihoods at theta_true and two nearby thetas (Sigma 80 GB + factor slices 17.5 GB).
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402


def main():
    name = sys.argv[1]
    only_breakdown = "--breakdown-only" in sys.argv
    wl = m.WORKLOADS[name]
    seed = wl.seeds[0]
    t0 = time.perf_counter()
    loc = wl.locations(seed)
    z = m.simulate_field(loc, wl.theta_true, seed)
    t_sim = time.perf_counter() - t0
    data = m.SpatialDataset(loc, z, nugget=wl.nugget)
    eng = data.engine()
    rec = {"config": name, "n": wl.n, "theta_true": wl.theta_true, "theta0": wl.theta0,
           "nugget": wl.nugget, "simulate_s": t_sim}
    if "--loglik-only" in sys.argv:
        rec["loglik"] = []
        for scale in ((1.0, 1.0, 1.0), (1.0, 1.05, 1.0), (1.1, 1.0, 0.95)):
            th = np.array(wl.theta_true, float) * np.array(scale)
            t0 = time.perf_counter()
            ll = eng.loglik(th)
            wall = time.perf_counter() - t0
            p = eng.phase_times()
            rec["loglik"].append({"theta": th.tolist(), "loglik": ll, "wall_s": wall,
                                  "phases_ms": p,
                                  "potrf_tflops": p["flops"] / (p["potrf_ms"] * 1e-3) / 1e12})
        print(json.dumps(rec))
        return
    # single-iteration breakdown at theta_true: a factoring eval_all and a loglik
    th = np.array(wl.theta_true, float)
    t0 = time.perf_counter()
    ll, g, f = eng.eval_all(th)
    rec["eval_all_wall_s"] = time.perf_counter() - t0
    rec["eval_all_phases_ms"] = eng.phase_times()
    p = rec["eval_all_phases_ms"]
    rec["eval_all_factor_solve_tflops"] = p["flops"] / ((p["potrf_ms"] + p["solve_ms"]) * 1e-3) / 1e12
    t0 = time.perf_counter()
    eng.loglik(th * np.array([1.0, 1.0 + 1e-9, 1.0]))
    rec["loglik_wall_s"] = time.perf_counter() - t0
    rec["loglik_phases_ms"] = eng.phase_times()
    rec["loglik_potrf_tflops"] = rec["loglik_phases_ms"]["flops"] / (
        rec["loglik_phases_ms"]["potrf_ms"] * 1e-3) / 1e12
    rec["at_theta_true"] = {"loglik": ll, "grad": g.tolist(), "fisher": f.tolist()}
    if "--kernel-profile" in sys.argv:
        # one factoring eval_all serialised on one stream with CUDA events around every
        # generation / slicing / Ozaki GEMM launch (mle_kernel_profile): per-kernel rates
        eng.kernel_profile(True)
        eng.eval_all(th * np.array([1.0, 1.0 - 1e-9, 1.0]))
        ks = eng.kernel_stats()
        eng.kernel_profile(False)
        rec["kernel_profile"] = {
            "stats": ks,
            "gen_gbs": ks["gen_bytes"] / (ks["gen_ms"] * 1e-3) / 1e9,
            "slice_gbs": ks["slice_bytes"] / (ks["slice_ms"] * 1e-3) / 1e9,
            "ozgemm_int8_tops": ks["gemm_int8_ops"] / (ks["gemm_ms"] * 1e-3) / 1e12,
            "ozgemm_fp64_equiv_tflops": ks["gemm_fp64_flops"] / (ks["gemm_ms"] * 1e-3) / 1e12,
        }
    if not only_breakdown:
        th0 = m.MaternParams(*wl.theta0)
        cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
        t0 = time.perf_counter()
        res = m.fisher_bt(data, cfg)
        wall = time.perf_counter() - t0
        rec["fit"] = {"theta_hat": res.theta_hat.as_array().tolist(),
                      "loglik_at_hat": res.loglik_at_hat, "grad_calls": res.grad_calls,
                      "loglik_calls": res.loglik_calls, "termination": res.termination.value,
                      "used_fallback": res.used_fallback, "wall_s": wall,
                      "fisher_it_per_s": res.grad_calls / wall}
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
