"""Benchmark: Fisher-BT iterations/s on BASELINE config 2 (n = 3,600, 5 replicate fits).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Own arm ("ours"): one process per GPU (torchrun for N > 1).  Each rank runs its own five
replicate Fisher-BT fits of config 2 (weak scaling: rank r fits seeds 5r..5r+4; rank 0 uses
the golden seeds 0-4; no data-path collective).  The five host loops run concurrently and
their evaluations are executed in lock step as batched GPU passes (paper_2601_11437_b200.
fit_many -> mle_eval_batch).  A step = all five fits from theta0 to convergence.
  value  = sum of grad_calls (Fisher iterations) over all ranks / max-over-ranks step time,
           inputs resident in HBM (datasets created and warmed before timing);
  e2e    = same metric through the public API from host numpy buffers: every step creates
           the datasets (H2D of locations and z), runs the fits and reads results back.
Reference arm (--impl reference): the reference's own CPU algorithm (oracle port of
maternmle: numpy / scipy / OpenBLAS on all host cores) on the same config, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
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
CONFIG = "config2"
THETA0 = (0.8, 0.1, 1.0)
N_REPLICAS = 5
# tcgen05.mma kind::i8 issue-rate ceiling measured on this pool's B200 with tools/umma_rate
# (the ozgemm k-block MMA sequence, operands resident in SMEM, 1888 MHz): 4485 TOPS burst;
# with random operands the clock settles at 1649-1761 MHz (sw_power_cap) -> 3624-3870 TOPS
# (profiles/r01_umma_rate.txt).  Reported beside the MEASURED_PEAKS-derived peak.
INT8_PIPE_TOPS = 4485.0
FP64_PEAK_TFLOPS = 36.08  # cuBLAS DGEMM 16384^3, this pool's B200 (profiles/r01_fp64_peaks.txt)
METRIC = "Fisher-BT iterations/s at n"


def workload_desc():
    return {"workload": "config2: n=3600 jittered 60x60 grid on [0,1]^2, true theta=(1.0,0.2,"
                        "1.5), 5 replicate FP64 fields per GPU, Fisher-BT from theta0=(0.8,0.1,"
                        "1.0) to ||grad||<=1e-3 (reference stopping rule)",
            "n": 3600, "replicas_per_gpu": N_REPLICAS, "nb": 128, "outer_block": 512,
            "l2": "inputs larger than L2: 3 x 110 MB matrices per replica, 5 replicas"}


def replica_seeds(rank: int):
    """Weak scaling: rank r owns seeds 5r..5r+4 (no data-path collective)."""
    return [N_REPLICAS * rank + s for s in range(N_REPLICAS)]


def load_replica(seed, device):
    """Locations and z for one replica (golden z for seeds 0-4, GPU-simulated otherwise)."""
    import paper_2601_11437_b200 as m

    path = GOLDEN / f"{CONFIG}_seed{seed}_data.npz"
    if path.exists():
        d = np.load(path)
        return d["loc"], d["z"]
    wl = m.WORKLOADS[CONFIG]
    loc = wl.locations(seed)
    return loc, m.simulate_field(loc, wl.theta_true, seed, device=device)


def run_fits(datasets, coords=None):
    """All replicas from THETA0, lock-step batched (one launch sequence covers them all)."""
    import paper_2601_11437_b200 as m

    th0 = m.MaternParams(*THETA0)
    cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
    return m.fit_many(datasets, cfg, coordinator_out=coords)


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
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


def isolated_phase_rates(datasets, theta, reps=4):
    """Batched eval_all / loglik over all replicas on one stream, CUDA events on it.
    Two thetas alternate so every evaluation refactors (no factor-cache hits)."""
    import paper_2601_11437_b200 as m

    engines = [d.engine() for d in datasets]
    th_a = np.asarray(theta, float)
    th_b = th_a * np.array([1.0, 1.0 + 1e-7, 1.0])
    th_c = th_a * np.array([1.0, 1.0 - 1e-7, 1.0])
    out = {"eval": [], "loglik": []}
    for r in range(reps + 1):
        for mode, key in ((2, "eval"), (1, "loglik")):
            th = (th_a if (r % 2 == 0) else th_b) if mode == 2 else th_c * (1.0 + 1e-9 * r)
            m.eval_batch(engines, [th] * len(engines), [mode] * len(engines))
            p = engines[0].phase_times()
            if r > 0:
                out[key].append(p)
    # kernel profiling pass: one stream, CUDA events around every Ozaki GEMM / slicing launch
    engines[0].kernel_profile(True)
    kst = []
    for r in range(2):
        m.eval_batch(engines, [th_a if r % 2 == 0 else th_b] * len(engines), [2] * len(engines))
        kst.append(engines[0].kernel_stats())
    engines[0].kernel_profile(False)
    ks = {k: sum(d[k] for d in kst) for k in kst[0]}
    ev, ll = out["eval"], out["loglik"]
    fac_ms = sum(p["potrf_ms"] + p["solve_ms"] for p in ev)
    fac_fl = sum(p["flops"] for p in ev)
    return {
        "batch": len(engines),
        "eval_factor_solve_tflops": fac_fl / (fac_ms * 1e-3) / 1e12,
        "eval_ms": statistics.median(p["total_ms"] for p in ev),
        "eval_phases_ms": {k: statistics.median(p[k] for p in ev)
                           for k in ("gen_ms", "potrf_ms", "solve_ms", "reduce_ms")},

        "loglik_ms": statistics.median(p["total_ms"] for p in ll),
        "loglik_potrf_tflops": sum(p["flops"] for p in ll) / (
            sum(p["potrf_ms"] for p in ll) * 1e-3) / 1e12,
        "launches_per_batched_eval": ev[-1]["launches"],
        "kernels": {
            "ozgemm_launches_per_eval": ks["gemm_launches"] / len(kst),
            "ozgemm_ms_per_eval": ks["gemm_ms"] / len(kst),
            "ozgemm_int8_tops": ks["gemm_int8_ops"] / (ks["gemm_ms"] * 1e-3) / 1e12,
            "ozgemm_fp64_equiv_tflops": ks["gemm_fp64_flops"] / (ks["gemm_ms"] * 1e-3) / 1e12,
            "slice_ms_per_eval": ks["slice_ms"] / len(kst),
            "slice_gbs": ks["slice_bytes"] / (ks["slice_ms"] * 1e-3) / 1e9,
            # covariance + derivative generation (tables + element kernels), algorithmic
            # bytes = 8 B per lower-triangle element per matrix written
            "gen_ms_per_eval": ks["gen_ms"] / len(kst),
            "gen_gbs": ks["gen_bytes"] / (ks["gen_ms"] * 1e-3) / 1e9 if ks["gen_ms"] else 0.0,
        },
    }


# ----------------------------------------------------------------------------- CPU side
def cpu_iteration_sample(reps=1):
    """Oracle (reference algorithm: numpy/scipy/OpenBLAS) time of one mean Fisher iteration of
    config 2 = one eval_all + rho loglik calls, rho = (loglik_calls - grad_calls) / grad_calls
    of the reference's own config-2 fits (golden, seeds 0-4)."""
    from oracle import maternmle_cpu as O

    fits = [json.loads((GOLDEN / f"{CONFIG}_seed{s}_fit.json").read_text()) for s in range(5)]
    g = sum(f["grad_calls"] for f in fits)
    rho = (sum(f["loglik_calls"] for f in fits) - g) / g
    d = np.load(GOLDEN / f"{CONFIG}_seed0_data.npz")
    loc, z = d["loc"], d["z"]
    th = (1.0, 0.2, 1.5)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.eval_all(loc, z, th)
        t1 = time.perf_counter()
        O.loglik(loc, z, th)
        t2 = time.perf_counter()
        times.append((t1 - t0) + rho * (t2 - t1))
    t_iter = statistics.median(times)
    return {"value": 1.0 / t_iter, "t_eval_all_s": t1 - t0, "t_loglik_s": t2 - t1, "rho": rho}


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info

        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            return int(info[0]["num_threads"])
    except Exception:
        pass
    return os.cpu_count() or 1


def reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import maternmle_cpu as O  # noqa: F401  (imports / BLAS warm-up)

    samples = [cpu_iteration_sample(1) for _ in range(args.steps)]
    val = statistics.median(s["value"] for s in samples)
    cores = cpu_cores()
    sample = ("per step: one config-2 eval_all + rho=%.3f loglik at n=3600 (the reference "
              "fits' mean evaluation mix per Fisher iteration); generation single-threaded "
              "numpy/scipy as in the reference, LAPACK on %d threads; warm-up = imports only"
              % (samples[0]["rho"], cores))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / val, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_desc(),
            "cpu_baseline": {"value": val, "unit": "it/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "detail": {"t_eval_all_s": samples[-1]["t_eval_all_s"],
                       "t_loglik_s": samples[-1]["t_loglik_s"]}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU side
def ours_arm(args, rank, world, local_rank):
    import torch

    import paper_2601_11437_b200 as m

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

    seeds = replica_seeds(rank)
    host = [load_replica(s, local_rank) for s in seeds]
    datasets = [m.SpatialDataset(loc, z, device=local_rank) for loc, z in host]

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
        run_fits(datasets)

    clocks = ClockSampler(local_rank)
    clocks.start()
    coords, step_ms, grad_calls, loglik_calls = [], [], 0, 0
    for _ in range(args.steps):
        res, ms = timed(lambda: run_fits(datasets, coords))
        step_ms.append(ms)
        print(f"[bench] step {ms:.1f} ms; device phases {coords[-1].acc}", file=sys.stderr,
              flush=True)
        grad_calls += sum(r.grad_calls for r in res)
        loglik_calls += sum(r.loglik_calls for r in res)
    clk = clocks.stop()
    last_fits = res

    # end-to-end: host arrays -> public API -> results on host, every step
    h2d = sum(loc.nbytes + z.nbytes for loc, z in host)
    e2e_ms, e2e_grad, e2e_evals = [], 0, 0
    e2e_coords = []

    def e2e_step():
        ds = [m.SpatialDataset(loc, z, device=local_rank) for loc, z in host]
        r = run_fits(ds, e2e_coords)
        for d in ds:
            d.release()
        return r

    # one untimed warm-up: the first contexts of this size populate the engine's buffer
    # cache (later create/destroy cycles reuse those buffers instead of cudaMalloc/cudaFree)
    e2e_step()
    for _ in range(max(1, args.steps)):
        res_e2e, ms = timed(e2e_step)
        e2e_ms.append(ms)
        print(f"[bench] e2e step {ms:.1f} ms; device phases {e2e_coords[-1].acc}",
              file=sys.stderr, flush=True)
        e2e_grad += sum(r.grad_calls for r in res_e2e)
        e2e_evals += sum(r.loglik_calls for r in res_e2e)

    tot_ms, tot_e2e = sum(step_ms), sum(e2e_ms)
    if dist is not None:
        t = torch.tensor([tot_ms, tot_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c = torch.tensor([grad_calls, e2e_grad, loglik_calls], dtype=torch.float64, device="cuda")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        tot_ms, tot_e2e = float(t[0]), float(t[1])
        grad_all, e2e_grad_all, ll_all = (float(v) for v in c)
    else:
        grad_all, e2e_grad_all, ll_all = float(grad_calls), float(e2e_grad), float(loglik_calls)
    if rank != 0:
        return

    value = grad_all / (tot_ms * 1e-3)
    e2e_value = e2e_grad_all / (tot_e2e * 1e-3)
    acc = {k: sum(c.acc[k] for c in coords) for k in coords[0].acc}
    batches = sum(c.batches for c in coords)
    iso = isolated_phase_rates(datasets, m.WORKLOADS[CONFIG].theta_true)
    achieved = iso["eval_factor_solve_tflops"]
    kern = iso["kernels"]
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) \
        if (REPO / "MEASURED_PEAKS.json").exists() else {}
    int8_peak = 2.0 * peaks.get("bf16_tflops", 2250.0)
    ncu_traffic = None
    tfile = REPO / "profiles" / "ozgemm_traffic.json"
    if tfile.exists():
        ncu_traffic = json.loads(tfile.read_text())
    # per request: 9 result doubles + failure flag (4 B) + pivot (8 B) come back to the host
    d2h = int(e2e_evals / max(1, len(e2e_ms)) * (9 * 8 + 4 + 8))
    in_fit_tflops = acc["flops"] / ((acc["potrf_ms"] + acc["solve_ms"]) * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_desc(),
        "roofline": {
            "bound": "tensor", "unit": "TFLOP/s", "achieved": kern["ozgemm_int8_tops"],
            "peak": int8_peak, "frac": kern["ozgemm_int8_tops"] / int8_peak,
            "traffic": ncu_traffic["dram_bytes"] if ncu_traffic else None,
            "kernel": "ozgemm_persistent_kernel<64, 7, 2> (Ozaki FP64 trailing-update GEMM on "
                      "tcgen05.mma kind::i8, 128x64 tiles in CTA pairs sharing A): int8 tensor "
                      "ops = 28 slice products (7 balanced base-256 slices) x 2 x 128 x 128 x K "
                      "per 128x128 tile, summed over every launch of a batched eval_all of the 5 "
                      "replicas, / the sum of the launches' CUDA-event durations (profiling "
                      "pass, one stream)",
            "fp64_equiv_tflops": kern["ozgemm_fp64_equiv_tflops"],
            "int8_pipe_microbench_tops": INT8_PIPE_TOPS,
            "frac_of_int8_pipe_microbench": kern["ozgemm_int8_tops"] / INT8_PIPE_TOPS,
            "peak_source": "int8 dense tcgen05 rate = 2 x MEASURED_PEAKS.json bf16_tflops "
                           "(burst; sm_100 int8 dense is twice bf16 dense)",
            "traffic_source": ncu_traffic.get("source") if ncu_traffic else None},
        "fp64_dmma_peak_tflops": FP64_PEAK_TFLOPS,
        "fp64_tflops_chol_solve": achieved,
        "fp64_tflops_chol_solve_in_fits": in_fit_tflops,
        "gen_hbm_gbs": kern["gen_gbs"],
        # per-kernel roofline fractions (north_star: "per-kernel roofline fractions at 1 GPU")
        "kernel_rooflines": {
            "ozgemm_int8_tensor": kern["ozgemm_int8_tops"] / int8_peak,
            "cholesky_solve_fp64_vs_dmma_peak": achieved / FP64_PEAK_TFLOPS,
            "slicing_hbm": kern["slice_gbs"] / peaks.get("hbm_gbs", 6555.0),
            "generation_hbm_algorithmic": kern["gen_gbs"] / peaks.get("hbm_gbs", 6555.0),
            "hbm_peak_gbs": peaks.get("hbm_gbs", 6555.0),
            "note": "ozgemm vs 2 x MEASURED_PEAKS bf16 (int8 dense); Cholesky+solves as "
                    "standard-count FP64 flops / phase time vs the 36.08 TF/s DGEMM peak "
                    "(>1: the Ozaki emulation beats the FP64 pipe); slicing and generation "
                    "as algorithmic bytes / kernel time vs MEASURED_PEAKS hbm_gbs"},
        "gpu_launches": int(acc["launches"]),
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "it/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "fits": {"grad_calls_per_step": grad_all / args.steps,
                 "loglik_calls_per_step": ll_all / args.steps,
                 "batched_passes_per_step": batches / args.steps,
                 "eval_passes_per_step": sum(c.eval_passes for c in coords) / args.steps,
                 "device_ms_per_step": {k: acc[k] / args.steps
                                        for k in ("gen_ms", "potrf_ms", "solve_ms",
                                                  "reduce_ms")},
                 "theta_hat_rank0": [r.theta_hat.as_array().tolist() for r in last_fits]},
        "isolated": iso,
    }
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_iteration_sample(1)
        line["cpu_baseline"] = {
            "value": cpu["value"], "unit": "it/s", "cores": cpu_cores(), "kind": "port",
            "sample": "one config-2 eval_all + rho=%.3f loglik (reference algorithm, numpy/"
                      "scipy/OpenBLAS) = one mean Fisher iteration; eval_all %.2fs, loglik "
                      "%.2fs" % (cpu["rho"], cpu["t_eval_all_s"], cpu["t_loglik_s"])}
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

        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        ours_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
