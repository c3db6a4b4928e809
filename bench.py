"""Benchmark: Fisher-BT iterations/s on BASELINE config 4 (n = 65,536), the largest
configuration that fits one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3]): 256 x 256 jittered grid on [0, 1]^2 (seed 0), one FP64
field z = L w drawn on the GPU at theta_true = (1.0, 0.1, 1.2), Fisher-BT from the pinned
theta0 = (1.0, 0.1, 1.0) (degenerate L9 cube) with the reference's rules
(optimizer.py:331-412).  A step = one Fisher iteration: the host loop runs until its next
eval_all has been answered (the line-search logliks before it, and for a fit's first step its
L9 start, belong to that step).  When a fit converges the next one starts from theta0 on the
same resident data, so any K is a sequence of real Fisher iterations.

Own arm ("ours"), one process per GPU (torchrun for N > 1):
  N = 1: the single-context engine (SpatialDataset -> mle_ctx: all matrices on one GPU);
  N > 1: the sharded engine (DistributedEngine over NCCL: 512-column block-cyclic panels,
         int8-slice panel broadcasts), every rank running the same host loop -- strong
         scaling: the same fit at every N.
  value = Fisher iterations / device time of the K timed steps (max over ranks), inputs
          resident in HBM; e2e = one complete fit through the public API from host numpy
          arrays (dataset upload inside the timed region, results read back).
  roofline: the dominant kernel (the Ozaki FP64 GEMM on tcgen05 int8) in a kernel-profiled
          eval_all, ALGORITHMIC flops of its launches (SURVEY §8(d) block sums: Cholesky
          n^3 / 3 + per derivative block n^3 for the two-sided reduction used at this size;
          gemm_algorithmic_flops) x 28 int8 slice products / summed launch durations, against
          2 x MEASURED_PEAKS bf16 (int8 dense = twice bf16 dense; the sustained figure: the
          GEMMs run for seconds inside a step).
Reference arm (--impl reference): the reference's own CPU algorithm (oracle port of maternmle:
numpy / scipy / OpenBLAS on all host cores), rank 0 only.  A config-4 Fisher iteration is
hours of CPU (one Sigma generation alone ~20 min single-threaded), so each step times a
bounded sample of every phase at the config-4 theta and sizes and extrapolates (labelled):
generation per pair x pairs, dpotrf / dtrsm at their measured flop rates x flops, the
memory-bound assembly / traces x n^2; iteration = one eval_all + rho logliks, rho from the
fit's own call counts.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

import numpy as np  # noqa: E402

GOLDEN = REPO / "tests" / "golden"
# The headline workload.  MLE_BENCH_CONFIG / MLE_DIST_BACKEND exist only to validate the
# sharded code path end to end where N GPUs are not available (e.g. two gloo ranks sharing
# one GPU on a smaller config); a bench line produced that way is labelled in "config".
CONFIG = os.environ.get("MLE_BENCH_CONFIG", "config4")
DIST_BACKEND = os.environ.get("MLE_DIST_BACKEND", "nccl")
METRIC = "Fisher-BT iterations/s at n"
# tcgen05.mma kind::i8 issue-rate ceiling measured on this pool's B200 (tools/umma_rate,
# profiles/r01_umma_rate.txt), reported beside the MEASURED_PEAKS-derived peak.
INT8_PIPE_TOPS = 4485.0
FP64_PEAK_TFLOPS = 36.08  # cuBLAS DGEMM 16384^3, this pool's B200 (profiles/r01_fp64_peaks.txt)
OZ_PRODUCTS = 28          # int8 slice products per FP64-emulated product (7 slices)
# Reference call mix per Fisher iteration at config 4 (loglik-only calls / grad calls) from the
# config-4 fit on the GPU engine (identical host loop; profiles/r01_config4_fit.json: 8 grad
# calls, 24 loglik calls incl. the 8 eval_all -> 16 loglik-only, L9 included).
CONFIG4_RHO = 16.0 / 8.0


def workload_desc(world):
    if CONFIG != "config4":  # validation runs only (see CONFIG)
        return {"workload": f"VALIDATION RUN on {CONFIG} (not the headline workload)",
                "engine": "single-context" if world == 1 else
                f"sharded DistributedEngine over {world} ranks ({DIST_BACKEND})"}
    return {"workload": "config4: n=65536 jittered 256x256 grid on [0,1]^2 (seed 0), one FP64 "
                        "field z=Lw at theta_true=(1.0,0.1,1.2), Fisher-BT from theta0=(1.0,0.1,"
                        "1.0) (degenerate L9 cube) to ||grad||<=1e-3; step = one Fisher "
                        "iteration (eval_all + its line-search logliks)",
            "n": 65536, "engine": "single-context" if world == 1 else
            f"sharded DistributedEngine over {world} ranks (NCCL)",
            "nb": 128, "outer_block": 512,
            "l2": "inputs larger than L2: three 34.5 GB matrices"}


def config_inputs(name, seed=0, device=0):
    """Locations and z (golden z where the reference could draw it, else the GPU draw)."""
    import paper_2601_11437_b200 as m

    path = GOLDEN / f"{name}_seed{seed}_data.npz"
    if path.exists():
        d = np.load(path)
        return d["loc"], d["z"]
    wl = m.WORKLOADS[name]
    loc = wl.locations(seed)
    return loc, m.simulate_field(loc, wl.theta_true, seed, device=device)


class FitStepper:
    """Runs Fisher-BT (the package's request-generator driver, fisher_bt.py) one Fisher
    iteration at a time; restarts from theta0 when a fit ends."""

    def __init__(self, make_objective, cfg):
        self.make_objective = make_objective
        self.cfg = cfg
        self.done = []
        self._start()

    def _start(self):
        from paper_2601_11437_b200.fisher_bt import fisher_bt_gen

        self.obj = self.make_objective()
        self.gen = fisher_bt_gen(self.cfg, self.obj)
        self.req = next(self.gen)

    def step(self):
        from paper_2601_11437_b200.fisher_bt import EVAL_ALL, _answer

        while True:
            kind, theta = self.req
            ans = _answer(self.obj, kind, theta)
            try:
                self.req = self.gen.send(ans)
            except StopIteration as stop:
                self.done.append(stop.value)
                self._start()
            if kind == EVAL_ALL:
                return


class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


TWO_SIDED_MIN_N = 16384  # engine.cu kTwoSidedMinN: eval_all's solve formulation by size


def solve_path(n):
    env = os.environ.get("MLE_SOLVE")
    if env in ("w", "2s"):
        return env
    big_n = -(-(n + 1) // 128) * 128
    return "2s" if big_n >= TWO_SIDED_MIN_N else "w"


def gemm_algorithmic_flops(n, mode, path=None, nderiv=2, blk=512):
    """Standard-count FP64 flops of one evaluation's Ozaki GEMM launches, as
    block sums over the 512-column outer blocks (c0 = b blk, c1 = c0 + blk):
      Cholesky trailing updates (lower):  sum (n - c1)^2 blk                        ~ n^3 / 3
      eval_all, per derivative block, path "w" (solves_w):
        forward sweep X = L^-1 S:         sum 2 (n - c0) blk n                      ~ n^3
        right sweep (lower half):         sum (n - c0)^2 blk                        ~ n^3 / 3
      path "2s" (solves_2s, the sygst recurrence):
        syr2k trailing updates:           sum 2 (n - c1)^2 blk                      ~ 2 n^3 / 3
        panel products (2), (3), (5):     sum 3 x 2 (n - c1) blk^2                  ~ 3 blk n^2
        deferred forward sweep (lower):   sum 2 (n - c0) blk c0                     ~ n^3 / 3
    The Cholesky's 128-wide DMMA steps inside each block (not Ozaki launches) are excluded."""
    path = path or solve_path(n)
    chol = derv = 0.0
    for b in range(-(-n // blk)):
        c0 = b * blk
        c1 = min(n, c0 + blk)
        chol += float(n - c1) ** 2 * blk
        if path == "w":
            derv += 2.0 * (n - c0) * blk * n + float(n - c0) ** 2 * blk
        else:
            derv += 2.0 * float(n - c1) ** 2 * blk + 6.0 * (n - c1) * blk * blk \
                + 2.0 * (n - c0) * blk * c0
    return chol + (nderiv * derv if mode == "eval_all" else 0.0)


def kernel_profile(engine, theta, n, peaks):
    """One eval_all with every Ozaki GEMM / slicing / generation launch event-timed on the
    (serialised) launching stream; algorithmic work per launch class / summed durations."""
    engine.kernel_profile(True)
    try:
        engine.eval_all(np.asarray(theta, float))
        ks = engine.kernel_stats()
    finally:
        engine.kernel_profile(False)
    alg = gemm_algorithmic_flops(n, "eval_all")
    gemm_s = ks["gemm_ms"] * 1e-3
    pt = engine.phase_times()
    int8_peak = 2.0 * peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 2250.0))
    achieved = alg * OZ_PRODUCTS / gemm_s / 1e12
    return {
        "ozgemm_launches": ks["gemm_launches"], "ozgemm_ms": ks["gemm_ms"],
        "ozgemm_avg_launch_ms": ks["gemm_ms"] / max(1, ks["gemm_launches"]),
        "ozgemm_algorithmic_fp64_flops": alg,
        "ozgemm_executed_fp64_flops": ks["gemm_fp64_flops"],
        "ozgemm_executed_over_algorithmic": ks["gemm_fp64_flops"] / alg,
        "ozgemm_alg_int8_tops": achieved,
        "ozgemm_alg_fp64_equiv_tflops": alg / gemm_s / 1e12,
        "ozgemm_executed_int8_tops": ks["gemm_int8_ops"] / gemm_s / 1e12,
        "int8_peak_tops": int8_peak,
        "slice_ms": ks["slice_ms"], "slice_gbs": ks["slice_bytes"] / max(1e-9, ks["slice_ms"]
                                                                         * 1e-3) / 1e9,
        "solve_path": solve_path(n),
        "eval_all_ms": pt["total_ms"],
        # the reference's own work per eval_all (dpotrf + four n x n dtrsm: 13 n^3 / 3,
        # likelihood.py:121-135) over this engine's eval_all time: algorithm changes show
        # as speed-ups here, not as inflated TFLOP/s in the roofline
        "reference_equivalent_tflops": 13.0 * float(n) ** 3 / 3.0 / (pt["total_ms"] * 1e-3)
                                       / 1e12,
        "gen_ms": ks["gen_ms"],
        "gen_gbs": ks["gen_bytes"] / (ks["gen_ms"] * 1e-3) / 1e9 if ks["gen_ms"] else 0.0,
    }


# ----------------------------------------------------------------------------- CPU side
def use_all_host_threads():
    """torchrun exports OMP_NUM_THREADS=1 to its workers: give the CPU arms' BLAS / LAPACK
    every core this process may run on again (the reference arm is timed 'with all the host
    threads it can use')."""
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=len(os.sched_getaffinity(0)), user_api="blas")
    except Exception:
        pass


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info

        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            return int(info[0]["num_threads"])
    except Exception:
        pass
    return os.cpu_count() or 1


def cpu_config4_sample(pairs=400_000, n_lin=6144, seed=0):
    """The reference algorithm (oracle port: numpy / scipy / OpenBLAS, reference operation
    order) on a bounded sample of every phase of a config-4 Fisher iteration, extrapolated.

    * generation (single-threaded numpy/scipy ufuncs, as in the reference): C, dC/dalpha,
      dC/dnu (matern.py:100-125) on `pairs` uniformly drawn config-4 location pairs at
      theta_true, seconds per pair x n (n - 1) / 2 pairs;
    * dpotrf (likelihood.py:75) and dtrsm (solve_triangular, :134-135) at n_lin on all host
      cores: measured flop rates x n^3/3 and 4 x n^3 (two n x n solves per derivative block);
    * the memory-bound rest (squareform assembly, trace_product's A + B^T, :92-104) timed at
      n_lin and scaled by n^2;
    iteration = eval_all + rho x loglik (rho = CONFIG4_RHO)."""
    from scipy.linalg import solve_triangular
    from scipy.linalg.lapack import dpotrf
    from scipy.spatial.distance import squareform

    import paper_2601_11437_b200.datasets as ds
    from oracle import maternmle_cpu as O

    n = 65536
    th = (1.0, 0.1, 1.2)
    rng = np.random.default_rng(seed)
    loc = ds.jittered_grid(256, 0)
    i = rng.integers(0, n, size=pairs)
    j = rng.integers(0, n, size=pairs)
    keep = i != j
    h = np.hypot(*(loc[i[keep]] - loc[j[keep]]).T)
    t = {}
    for kind in ("sigma", "alpha", "nu"):
        t0 = time.perf_counter()
        O.elem(h, th, kind)
        t[kind] = (time.perf_counter() - t0) / h.size
    npairs = n * (n - 1) / 2.0
    gen_s = {k: v * npairs for k, v in t.items()}
    # LAPACK rates on all host cores
    a = rng.standard_normal((n_lin, n_lin))
    spd = a @ a.T / n_lin + np.eye(n_lin)
    t0 = time.perf_counter()
    low, info = dpotrf(spd, lower=1, clean=1, overwrite_a=0)
    t_potrf = time.perf_counter() - t0
    rhs = rng.standard_normal((n_lin, n_lin))
    t0 = time.perf_counter()
    solve_triangular(low, rhs, lower=True, check_finite=False)
    t_trsm = time.perf_counter() - t0
    potrf_rate = n_lin ** 3 / 3.0 / t_potrf
    trsm_rate = float(n_lin) ** 3 / t_trsm
    # memory-bound assembly and trace products, per element
    cond = rng.random(n_lin * (n_lin - 1) // 2)
    t0 = time.perf_counter()
    sq = squareform(cond, checks=False)
    t_sq = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.trace_product(sq, rhs)
    t_tp = time.perf_counter() - t0
    per_el_sq, per_el_tp = t_sq / n_lin ** 2, t_tp / n_lin ** 2
    nn = float(n) * n
    potrf_s = n ** 3 / 3.0 / potrf_rate
    trsm_s = float(n) ** 3 / trsm_rate
    loglik_s = gen_s["sigma"] + per_el_sq * nn + potrf_s + 2 * float(n) ** 2 / trsm_rate * 1.0
    eval_all_s = (gen_s["sigma"] + gen_s["alpha"] + gen_s["nu"] + 3 * per_el_sq * nn + potrf_s
                  + 4 * trsm_s + 3 * per_el_tp * nn)
    iter_s = eval_all_s + CONFIG4_RHO * loglik_s
    return {"value": 1.0 / iter_s, "iteration_s": iter_s, "eval_all_s": eval_all_s,
            "loglik_s": loglik_s, "gen_s_per_matrix": gen_s, "potrf_s": potrf_s,
            "trsm_s_each": trsm_s, "potrf_gflops": potrf_rate / 1e9,
            "trsm_gflops": trsm_rate / 1e9, "sample_pairs": int(h.size), "n_lin": n_lin}


def reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import maternmle_cpu as O  # noqa: F401  (imports / BLAS warm-up)

    use_all_host_threads()
    for _ in range(args.warmup):
        cpu_config4_sample(pairs=50_000, n_lin=1024)
    samples, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        samples.append(cpu_config4_sample())
        walls.append(time.perf_counter() - t0)
    val = statistics.median(s["value"] for s in samples)
    cores = cpu_cores()
    s0 = samples[len(samples) // 2]
    sample = ("per step: the reference algorithm (oracle port, numpy/scipy/OpenBLAS) timed on "
              "%d config-4 location pairs (C, dC/dalpha, dC/dnu at theta_true; generation "
              "single-threaded as in the reference) and dpotrf / dtrsm / assembly / trace "
              "products at n=%d on %d threads, EXTRAPOLATED to n=65536 (pairs x per-pair time, "
              "n^3 flops / measured rate, n^2 x per-element time); iteration = eval_all + "
              "%.1f loglik" % (s0["sample_pairs"], s0["n_lin"], cores, CONFIG4_RHO))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(1), "extrapolated": True,
            "cpu_baseline": {"value": val, "unit": "it/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "detail": s0,
            "measured_reference": measured_reference()}
    print(json.dumps(line), flush=True)


def measured_reference():
    """What the unmodified reference itself measured where it could run (committed goldens,
    made by tests/golden/make_golden.py in the build container, 8 cores): the calibration
    points next to the extrapolation above."""
    out = {}
    path = GOLDEN / "config3_evals.json"
    if path.exists():
        recs = json.loads(path.read_text())
        out["config3_log_likelihood_plus_grad_and_fisher_s"] = [r.get("cpu_wall_s")
                                                                for r in recs]
    fits = []
    for seed in range(5):
        fp = GOLDEN / f"config2_seed{seed}_fit.json"
        if fp.exists():
            f = json.loads(fp.read_text())
            fits.append({"seed": seed, "seconds": f["cpu_wall_s"], "grad_calls": f["grad_calls"],
                         "it_per_s": f["grad_calls"] / f["cpu_wall_s"]})
    if fits:
        out["config2_full_fits"] = fits
    fp = GOLDEN / "config3_seed0_fit.json"
    if fp.exists():
        f = json.loads(fp.read_text())
        out["config3_full_fit"] = {"seconds": f["cpu_wall_s"], "grad_calls": f["grad_calls"],
                                   "it_per_s": f["grad_calls"] / f["cpu_wall_s"]}
    out["note"] = ("reference package (maternmle, numpy/scipy/OpenBLAS) on 8 build-container "
                   "cores; generation single-threaded")
    return out


# ----------------------------------------------------------------------------- GPU side
def extra_single_gpu(m, device):
    """Context numbers on the smaller configs (not the headline): one config-3 fit (n=16,384)
    and the five config-2 replicate fits batched."""
    out = {}
    import torch

    loc, z = config_inputs("config3", 0, device)
    wl = m.WORKLOADS["config3"]
    th0 = m.MaternParams(*wl.theta0)
    cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
    data = m.SpatialDataset(loc, z, device=device)
    m.fisher_bt(data, cfg)  # warm (buffers, tables)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = m.fisher_bt(data, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out["config3_fit"] = {"n": wl.n, "grad_calls": r.grad_calls, "loglik_calls": r.loglik_calls,
                          "seconds": dt, "it_per_s": r.grad_calls / dt,
                          "theta_hat": r.theta_hat.as_array().tolist()}
    data.release()
    wl2 = m.WORKLOADS["config2"]
    sets = [m.SpatialDataset(*config_inputs("config2", s, device), device=device)
            for s in wl2.seeds]
    th0 = m.MaternParams(*wl2.theta0)
    cfg2 = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
    m.fit_many(sets, cfg2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = m.fit_many(sets, cfg2)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    g = sum(x.grad_calls for x in res)
    out["config2_five_fits"] = {"grad_calls": g, "seconds": dt, "it_per_s": g / dt}
    for d in sets:
        d.release()
    if os.environ.get("MLE_BENCH_CONFIG5", "1") != "0":
        try:
            out["config5_one_gpu"] = config5_one_gpu(m, device)
        except Exception as exc:  # 165 GB: never at the expense of the other context numbers
            out["config5_one_gpu"] = {"error": repr(exc)}
    return out


def config5_one_gpu(m, device):
    """BASELINE config 5 (n = 100,000, nugget 1e-6) on this one GPU in the engine's
    sequential-derivative mode: one log-likelihood and one eval_all
    (factor resident: the three derivative blocks, 3 n^3 flops), timed once each."""
    import gc

    import torch

    gc.collect()
    m.release_cached_memory()
    wl = m.WORKLOADS["config5"]
    loc = wl.locations(0)
    z = m.simulate_field(loc, wl.theta_true, 0, device=device, nugget=wl.nugget)
    data = m.SpatialDataset(loc, z, device=device, nugget=wl.nugget)
    eng = data.engine()
    th = wl.theta_true
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ll = eng.loglik(th)
    t1 = time.perf_counter()
    ev = eng.eval_all(th)
    t2 = time.perf_counter()
    nd = float(wl.n)
    rec = {"n": wl.n, "nugget": wl.nugget, "sequential_derivs": bool(eng.sequential_derivs),
           "loglik_s": t1 - t0, "loglik_fp64_equiv_tflops": nd ** 3 / 3.0 / (t1 - t0) / 1e12,
           "eval_all_blocks_s": t2 - t1,
           "blocks_fp64_equiv_tflops": 3.0 * nd ** 3 / (t2 - t1) / 1e12,
           "loglik": float(ll), "eval_all_loglik_identical": float(ev[0]) == float(ll)}
    data.release()
    m.release_cached_memory()
    return rec


def ours_arm(args, rank, world, local_rank):
    import torch

    import paper_2601_11437_b200 as m
    from paper_2601_11437_b200.distributed import (DistributedEngine, DistributedObjective,
                                                   TorchComm)

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    wl = m.WORKLOADS[CONFIG]
    loc = wl.locations(0)
    # z = L w at theta_true (simulate.py:100-106): drawn once on rank 0's GPU, shared
    zt = torch.zeros(wl.n, dtype=torch.float64, device="cuda")
    if rank == 0:
        zt.copy_(torch.from_numpy(m.simulate_field(loc, wl.theta_true, 0, device=local_rank)))
    if dist is not None:
        dist.broadcast(zt, 0)
    z = zt.cpu().numpy()
    th0 = m.MaternParams(*wl.theta0)
    cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)

    def make_backend(host_loc, host_z):
        if world == 1:
            data = m.SpatialDataset(host_loc, host_z, device=local_rank)
            return data, (lambda: m.LikelihoodObjective(data))
        eng = DistributedEngine(host_loc, host_z, TorchComm(), device=local_rank)
        return eng, (lambda: DistributedObjective(eng))

    handle, make_obj = make_backend(loc, z)
    stepper = FitStepper(make_obj, cfg)

    def barrier_sync():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn):
        barrier_sync()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        out = fn()
        torch.cuda.synchronize()
        stop.record()
        stop.synchronize()
        return out, start.elapsed_time(stop)

    for _ in range(args.warmup):
        stepper.step()
    from paper_2601_11437_b200 import _native as nat

    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = nat.lib.mle_launch_count()
    step_ms = []
    ll0 = stepper.obj.loglik_calls + sum(r.loglik_calls for r in stepper.done)
    for k in range(args.steps):
        _, ms = timed(stepper.step)
        step_ms.append(ms)
        if rank == 0:
            print(f"[bench] step {k} {ms:.1f} ms", file=sys.stderr, flush=True)
    clk = clocks.stop()
    launches = nat.lib.mle_launch_count() - launches0
    ll_calls = stepper.obj.loglik_calls + sum(r.loglik_calls for r in stepper.done) - ll0

    # end-to-end: one complete fit from host numpy arrays through the public API (dataset
    # upload, every evaluation, results read back) -- inside the timed region
    e2e_box = {}

    def e2e_fit():
        h, mk = make_backend(loc.copy(), z.copy())
        e2e_box["res"] = m.fisher_bt(None, cfg, objective=mk())
        if world == 1:
            h.release()
        else:
            h.close()

    if world == 1:
        handle.release()  # free the timed run's matrices before the e2e fit allocates its own
    else:
        handle.close()
    _, e2e_ms = timed(e2e_fit)
    res = e2e_box["res"]
    tot_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([tot_ms, e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, e2e_ms = float(t[0]), float(t[1])
    if rank != 0:
        return
    value = args.steps / (tot_ms * 1e-3)
    e2e_value = res.grad_calls / (e2e_ms * 1e-3)
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) \
        if (REPO / "MEASURED_PEAKS.json").exists() else {}
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_desc(world),
        "fits": {"loglik_calls_in_timed_steps": ll_calls,
                 "completed_fits_so_far": len(stepper.done),
                 "theta_hat_e2e_fit": res.theta_hat.as_array().tolist(),
                 "grad_calls_e2e_fit": res.grad_calls, "loglik_calls_e2e_fit": res.loglik_calls,
                 "termination_e2e_fit": res.termination.value},
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "it/s",
                "h2d_bytes_per_step": int(loc.nbytes + z.nbytes),
                "d2h_bytes_per_step": int(res.loglik_calls * (9 * 8 + 4 + 8)),
                "what": "one complete config-4 fit per e2e step (dataset upload from host "
                        "arrays, L9 start, every Fisher iteration, results to host)"},
    }
    if world == 1:
        data = m.SpatialDataset(loc, z, device=local_rank)
        kp = kernel_profile(data.engine(), wl.theta_true, wl.n, peaks)
        tpath = REPO / "profiles" / "r02_ozgemm_traffic.json"
        traffic = json.loads(tpath.read_text()) if tpath.exists() else {}
        launches_per_eval = data.engine().phase_times()["launches"]
        data.release()
        line["roofline"] = {
            "bound": "tensor", "unit": "TFLOP/s", "achieved": kp["ozgemm_alg_int8_tops"],
            "peak": kp["int8_peak_tops"], "frac": kp["ozgemm_alg_int8_tops"] / kp["int8_peak_tops"],
            "traffic": traffic.get("traffic_bytes_per_launch"),
            "kernel": "ozgemm_persistent_kernel<64,7,2> (Ozaki FP64 GEMM on tcgen05.mma kind::i8)"
                      ": ALGORITHMIC FP64 flops of one config-4 eval_all's GEMM launches (block "
                      "sums of the solve path used, bench.gemm_algorithmic_flops) x 28 int8 "
                      "slice products / summed launch durations (CUDA events on the launching "
                      "stream, kernel-profiling pass)",
            "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (int8 dense = 2 x bf16 "
                           "dense; sustained: the GEMMs run for seconds inside a step)",
            "traffic_source": traffic.get("source", "no ncu capture committed"),
            "traffic_launch_ms": traffic.get("launch_ms"),
            "int8_pipe_microbench_tops": INT8_PIPE_TOPS,
            "fp64_equiv_tflops_algorithmic": kp["ozgemm_alg_fp64_equiv_tflops"],
            "fp64_dmma_peak_tflops": FP64_PEAK_TFLOPS}
        line["kernels"] = kp
        gpath = REPO / "profiles" / "r02_gen_ncu.json"
        if gpath.exists():  # ncu of the generation kernels (same build): FP64 pipe, L1, DRAM
            g = json.loads(gpath.read_text())
            line["kernels"]["generation_ncu"] = {
                "fp64_pipe_pct_derivs": g["derivs_fp64_pipe_pct"],
                "fp64_pipe_pct_sigma": g["sigma_fp64_pipe_pct"],
                "l1tex_pct_derivs": g["derivs_l1tex_pct"],
                "dram_write_over_algorithmic": g["derivs_dram_write_bytes"]
                / g["derivs_algorithmic_bytes"],
                "hbm_frac": kp["gen_gbs"] / peaks.get("hbm_gbs", 6548.5) if kp["gen_gbs"]
                else None,
                "bound": g["bound"], "source": g["source"]}
        line["kernels"]["launches_per_profiled_eval_all"] = launches_per_eval
        try:
            line["context"] = extra_single_gpu(m, local_rank)
        except Exception as exc:  # context numbers must not sink the headline
            line["context"] = {"error": repr(exc)}
        if not args.no_cpu_baseline:
            use_all_host_threads()
            cpu = cpu_config4_sample()
            line["cpu_baseline"] = {
                "value": cpu["value"], "unit": "it/s", "cores": cpu_cores(), "kind": "port",
                "sample": "reference algorithm (oracle port) on %d config-4 pairs + LAPACK / "
                          "memory-bound phases at n=%d, EXTRAPOLATED to one config-4 Fisher "
                          "iteration (eval_all + %.1f loglik): %.0f s" % (
                              cpu["sample_pairs"], cpu["n_lin"], CONFIG4_RHO,
                              cpu["iteration_s"])}
    line["gpu_launches"] = int(launches)  # rank 0's kernels in the timed steps (mle_launch_count)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if DIST_BACKEND != "nccl":  # validation: more ranks than GPUs share them
            local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if DIST_BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(DIST_BACKEND)
    try:
        ours_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
