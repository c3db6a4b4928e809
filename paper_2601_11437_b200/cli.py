"""Command-line front end over the GPU engine: the reference's ``maternmle`` CLI surface
(cli.py:1-17, 452-505) with every evaluation on the B200 objective.

    python -m paper_2601_11437_b200 estimate DATA [--method fisher-bt|nelder-mead|both]
                                                   [--lower a,b,c] [--upper a,b,c]
                                                   [--seed S] [--out F] [--trace]
    python -m paper_2601_11437_b200 simulate OUT --n N --theta s2,a,nu [--seed S]
                                                 [--scheme grid|uniform]
    python -m paper_2601_11437_b200 benchmark --theta s2,a,nu ... --n N ... [--m M]
                                              [--methods ...] [--jobs J] --out-dir DIR
    python -m paper_2601_11437_b200 loglik DATA --theta s2,a,nu [--out F]

Formats and codes follow the reference:

* datasets: CSV with header ``x,y,z``, 17 significant digits, LF (cli.py:83-117); for
  n >= 65,536 a CSV is ~3 MB per 65k rows and slow to parse, so a path ending in ``.npz``
  (arrays ``loc`` (n, 2) and ``z`` (n,)) is read / written instead -- the same numbers,
  binary;
* results: the RunRecord JSON of cli.py:133-151 (theta_hat, std_errors from diag(I^-1) or a
  reason, loglik, call counts, wall_time, termination, seed, optional trace);
* benchmark: per-replicate ``run_t{ti}_n{n}_r{rep}.json`` plus ``summary.csv`` with the
  reference's columns (cli.py:285-390), replicate seeds from ``replicate_seed``;
* exit codes: 0 success, 2 parse / plan errors, 3 optimization failure (cli.py:15-16).

B200-first differences: the replicates of one benchmark cell are fitted together
(:func:`~paper_2601_11437_b200.batch.fit_many`: one batched engine pass per lock step,
results bit-identical to one-by-one fits), and ``--jobs`` spreads cells over the visible GPUs
(one host thread per GPU) instead of CPU worker processes.
"""

from __future__ import annotations

import argparse
import concurrent.futures
import csv
import json
import sys
import time
from pathlib import Path

import numpy as np

from . import _native as nat
from .batch import fit_many
from .fisher_bt import (FisherBTConfig, InitializationFailed, LikelihoodObjective,
                        SingularInformation, fisher_bt, nelder_mead)
from .likelihood import NotPositiveDefinite, grad_and_fisher
from .matern import MaternParams, SpatialDataset
from .simulate import (GENERATOR_ID, LocationScheme, PlanError, SimulationPlan, gen_locations,
                       microergodic, replicate_seed, simulate_grf)

__all__ = ["main", "build_parser", "read_dataset", "write_dataset", "parse_theta",
           "run_method", "run_benchmark", "DatasetFormatError"]

DEFAULT_LOWER = "0.01,0.01,0.01"   # cli.py:52-53 (the paper's initialization cube)
DEFAULT_UPPER = "5,5,2"
SUMMARY_COLUMNS = ["theta_set", "n", "method", "param", "mean", "sd", "mean_loglik_deficit",
                   "mean_loglik_calls", "mean_grad_calls", "mean_wall_time"]
EXIT_OK, EXIT_PARSE, EXIT_OPT = 0, 2, 3


class DatasetFormatError(Exception):
    """A malformed dataset file; ``line`` is 1-based (cli.py:69-73)."""

    def __init__(self, path, line, message):
        self.path, self.line = path, line
        super().__init__(f"{path}: line {line}: {message}")


def parse_theta(text: str) -> MaternParams:
    fields = str(text).split(",")
    if len(fields) != 3:
        raise ValueError(f"expected 3 comma-separated values, got {text!r}")
    return MaternParams(*(float(f) for f in fields))


def _theta_dict(p: MaternParams) -> dict:
    return {"sigma2": p.sigma2, "alpha": p.alpha, "nu": p.nu}


# ------------------------------------------------------------------------------ datasets
def read_dataset(path, device: int | None = None) -> SpatialDataset:
    """``x,y,z`` CSV (or ``.npz`` with ``loc`` / ``z``) -> a device-resident SpatialDataset."""
    path = str(path)
    if path.endswith(".npz"):
        try:
            with np.load(path) as d:
                loc, z = np.asarray(d["loc"], float), np.asarray(d["z"], float)
        except (KeyError, ValueError) as exc:
            raise DatasetFormatError(path, 1, f"npz needs arrays 'loc' and 'z' ({exc})")
        try:
            return SpatialDataset(loc, z, device=device)
        except ValueError as exc:
            raise DatasetFormatError(path, 1, str(exc))
    with open(path, "r", encoding="utf-8") as fh:
        if fh.readline().strip() != "x,y,z":
            raise DatasetFormatError(path, 1, "expected header 'x,y,z'")
        rows = []
        for lineno, raw in enumerate(fh, start=2):
            text = raw.strip()
            if not text:
                continue
            parts = text.split(",")
            if len(parts) != 3:
                raise DatasetFormatError(path, lineno, f"expected 3 fields, got {len(parts)}")
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2])))
            except ValueError:
                raise DatasetFormatError(path, lineno, "non-numeric field")
    if not rows:
        raise DatasetFormatError(path, 2, "no data rows")
    arr = np.array(rows, dtype=float)
    try:
        return SpatialDataset(arr[:, :2], arr[:, 2], device=device)
    except ValueError as exc:
        raise DatasetFormatError(path, 2, str(exc))


def write_dataset(path, locations, values):
    path = str(path)
    loc = np.asarray(locations, float)
    z = np.asarray(values, float)
    if path.endswith(".npz"):
        np.savez(path, loc=loc, z=z)
        return
    lines = ["x,y,z\n"] + [f"{x:.17g},{y:.17g},{v:.17g}\n" for (x, y), v in zip(loc, z)]
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.writelines(lines)


# ------------------------------------------------------------------------------- records
def _std_errors(fisher):
    """sqrt(diag(I^-1)) when I is positive definite, else (None, reason) (cli.py:120-130)."""
    info = np.asarray(fisher, float)
    try:
        np.linalg.cholesky(info)
        cov = np.linalg.inv(info)
    except np.linalg.LinAlgError:
        return None, "information_not_positive_definite"
    d = np.diag(cov)
    if not np.all(np.isfinite(d)) or np.any(d <= 0.0):
        return None, "information_not_positive_definite"
    return [float(v) for v in np.sqrt(d)], None


def _record(method, theta_hat, fisher, loglik, loglik_calls, grad_calls, wall, termination,
            seed, trace=None):
    se, why = _std_errors(fisher)
    rec = {"method": method, "theta_hat": _theta_dict(theta_hat), "std_errors": se,
           "loglik": loglik, "loglik_calls": loglik_calls, "grad_calls": grad_calls,
           "wall_time": wall, "termination": termination, "seed": seed}
    if why is not None:
        rec["std_errors_reason"] = why
    if trace is not None:
        rec["trace"] = trace
    return rec


def _fisher_record(res, wall, seed, with_trace=False):
    trace = ([[p.sigma2, p.alpha, p.nu, ll] for p, ll in res.iterate_trace]
             if with_trace else None)
    return _record("fisher-bt", res.theta_hat, res.fisher_at_hat, res.loglik_at_hat,
                   res.loglik_calls, res.grad_calls, wall, res.termination.value, seed, trace)


def run_method(data: SpatialDataset, method: str, cfg: FisherBTConfig, seed: int,
               with_trace: bool = False) -> dict:
    """One estimation method on one dataset -> RunRecord (cli.py:154-198)."""
    t0 = time.perf_counter()
    if method == "fisher-bt":
        res = fisher_bt(data, cfg)
        return _fisher_record(res, time.perf_counter() - t0, seed, with_trace)
    if method == "nelder-mead":
        # NM from the cube's midpoint, then one grad_and_fisher at its optimum
        mid = MaternParams.from_array(0.5 * (cfg.theta_lower.as_array()
                                             + cfg.theta_upper.as_array()))
        obj = LikelihoodObjective(data)
        theta_hat, calls = nelder_mead(data, mid, cfg.nm_tol, objective=obj)
        ev = grad_and_fisher(data, theta_hat)
        return _record(method, theta_hat, ev.fisher, ev.loglik, calls + 1, 1,
                       time.perf_counter() - t0, "nm_converged", seed)
    raise ValueError(f"unknown method {method!r}")


def _methods_for(flag: str):
    return ["fisher-bt", "nelder-mead"] if flag == "both" else [flag]


def _emit_json(document, out_path):
    text = json.dumps(document, indent=2) + "\n"
    if out_path:
        Path(out_path).write_text(text, encoding="utf-8")
    else:
        sys.stdout.write(text)


def _err(exc):
    print(f"error: {exc}", file=sys.stderr)


# ------------------------------------------------------------------------------ commands
def cmd_estimate(args) -> int:
    try:
        data = read_dataset(args.input)
        cfg = FisherBTConfig(theta_lower=parse_theta(args.lower),
                             theta_upper=parse_theta(args.upper))
    except (OSError, DatasetFormatError, ValueError) as exc:
        _err(exc)
        return EXIT_PARSE
    records = []
    for method in _methods_for(args.method):
        try:
            records.append(run_method(data, method, cfg, args.seed, with_trace=args.trace))
        except (InitializationFailed, SingularInformation) as exc:
            _err(f"optimization failed: {exc}")
            return EXIT_OPT
    _emit_json({"input": str(args.input), "records": records}, args.out)
    return EXIT_OK


def cmd_simulate(args) -> int:
    try:
        theta = parse_theta(args.theta)
        plan = SimulationPlan(n=args.n, theta_true=theta,
                              location_scheme=LocationScheme(args.scheme), rng_seed=args.seed)
        loc = gen_locations(plan)
        z = simulate_grf(loc, theta, args.seed)
    except (PlanError, ValueError) as exc:
        _err(exc)
        return EXIT_PARSE
    write_dataset(args.out, loc, z)
    meta = {"theta_true": _theta_dict(theta), "seed": args.seed, "scheme": args.scheme,
            "n": args.n, "generator": GENERATOR_ID}
    Path(str(args.out) + ".meta.json").write_text(json.dumps(meta, indent=2) + "\n",
                                                  encoding="utf-8")
    return EXIT_OK


def cmd_loglik(args) -> int:
    try:
        data = read_dataset(args.input)
        theta = parse_theta(args.theta)
    except (OSError, DatasetFormatError, ValueError) as exc:
        _err(exc)
        return EXIT_PARSE
    try:
        ev = grad_and_fisher(data, theta)
    except NotPositiveDefinite as exc:
        _err(exc)
        return EXIT_OPT
    _emit_json({"theta": _theta_dict(theta), "loglik": ev.loglik,
                "grad": [float(g) for g in ev.grad],
                "fisher": [[float(v) for v in row] for row in ev.fisher]}, args.out)
    return EXIT_OK


# ----------------------------------------------------------------------------- benchmark
def _cell(theta, n, ti, ni, replicates, methods, lower, upper, master_seed, scheme, device):
    """All replicates of one (theta_true, n) cell on one GPU: Fisher-BT fits batched in lock
    step (fit_many), Nelder-Mead one by one.  Per-replicate records as cli.py:256-282."""
    cfg = FisherBTConfig(theta_lower=MaternParams(*lower), theta_upper=MaternParams(*upper))
    seeds = [replicate_seed(master_seed, ti, ni, rep) for rep in range(replicates)]
    sets = []
    for seed in seeds:
        plan = SimulationPlan(n=n, theta_true=theta, location_scheme=LocationScheme(scheme),
                              rng_seed=seed)
        loc = gen_locations(plan)
        sets.append(SpatialDataset(loc, simulate_grf(loc, theta, seed, device=device),
                                   device=device))
    recs = [[] for _ in seeds]
    for method in methods:
        if method == "fisher-bt":
            t0 = time.perf_counter()
            fits = fit_many(sets, cfg, return_exceptions=True)
            wall = (time.perf_counter() - t0) / len(sets)  # the batch's time, per replicate
            for k, res in enumerate(fits):
                if isinstance(res, (InitializationFailed, SingularInformation)):
                    recs[k].append({"method": method, "seed": seeds[k], "error": str(res)})
                elif isinstance(res, Exception):
                    raise res
                else:
                    recs[k].append(_fisher_record(res, wall, seeds[k]))
        else:
            for k, data in enumerate(sets):
                try:
                    recs[k].append(run_method(data, method, cfg, seeds[k]))
                except (InitializationFailed, SingularInformation) as exc:
                    recs[k].append({"method": method, "seed": seeds[k], "error": str(exc)})
    for d in sets:
        d.release()
    return [{"theta_index": ti, "n_index": ni, "replicate": rep, "records": recs[rep]}
            for rep in range(replicates)]


def run_benchmark(theta_sets, sizes, replicates, methods, lower, upper, master_seed, jobs=1,
                  scheme="grid", out_dir=None):
    """Full-factorial study (theta_true x n x replicate x method) -> (results, summary rows);
    reproducible under any job count (seeds from (master, theta index, n index, replicate))."""
    cells = [(ti, th, ni, n) for ti, th in enumerate(theta_sets) for ni, n in enumerate(sizes)]
    for _, th, _, n in cells:  # plan errors before any GPU work (exit code 2)
        SimulationPlan(n=n, theta_true=th, location_scheme=LocationScheme(scheme))
    ndev = max(1, nat.device_count())
    workers = max(1, min(int(jobs), ndev, len(cells)))

    def run(k):
        ti, th, ni, n = cells[k]
        return _cell(th, n, ti, ni, replicates, methods, lower, upper, master_seed, scheme,
                     device=k % workers)

    if workers > 1:
        with concurrent.futures.ThreadPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(run, range(len(cells))))
    else:
        parts = [run(k) for k in range(len(cells))]
    results = sorted((r for p in parts for r in p),
                     key=lambda r: (r["theta_index"], r["n_index"], r["replicate"]))
    summary = _summarize(results, theta_sets, sizes, methods)
    if out_dir is not None:
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        for r in results:
            name = f"run_t{r['theta_index']}_n{sizes[r['n_index']]}_r{r['replicate']}.json"
            (out / name).write_text(json.dumps(r, indent=2) + "\n", encoding="utf-8")
        with open(out / "summary.csv", "w", encoding="utf-8", newline="\n") as fh:
            w = csv.writer(fh, lineterminator="\n")
            w.writerow(SUMMARY_COLUMNS)
            w.writerows(summary)
    return results, summary


def _summarize(results, theta_sets, sizes, methods):
    """Per-cell mean / SD over successful replicates; the log-likelihood deficit is measured
    from the best value any method reached on the same dataset (cli.py:336-390)."""
    rows = []
    fmt = "{:.17g}".format
    for ti, th in enumerate(theta_sets):
        label = f"{th.sigma2:g},{th.alpha:g},{th.nu:g}"
        for ni, n in enumerate(sizes):
            cell = [r for r in results if r["theta_index"] == ti and r["n_index"] == ni]
            for method in methods:
                est = {"sigma2": [], "alpha": [], "nu": [], "micro": []}
                deficit, ll_calls, g_calls, walls = [], [], [], []
                for r in cell:
                    ok = [x for x in r["records"] if "error" not in x]
                    rec = next((x for x in ok if x["method"] == method), None)
                    if rec is None:
                        continue
                    hat = rec["theta_hat"]
                    p = MaternParams(hat["sigma2"], hat["alpha"], hat["nu"])
                    for key, v in (("sigma2", p.sigma2), ("alpha", p.alpha), ("nu", p.nu),
                                   ("micro", microergodic(p))):
                        est[key].append(v)
                    deficit.append(max(x["loglik"] for x in ok) - rec["loglik"])
                    ll_calls.append(rec["loglik_calls"])
                    g_calls.append(rec["grad_calls"])
                    walls.append(rec["wall_time"])
                if not deficit:
                    continue
                for param, vals in est.items():
                    a = np.asarray(vals, float)
                    with np.errstate(invalid="ignore"):
                        sd = float(np.std(a, ddof=1)) if a.size > 1 else float("nan")
                    rows.append([label, n, method, param, fmt(float(np.mean(a))), fmt(sd),
                                 fmt(float(np.mean(deficit))), fmt(float(np.mean(ll_calls))),
                                 fmt(float(np.mean(g_calls))), fmt(float(np.mean(walls)))])
    return rows


def cmd_benchmark(args) -> int:
    try:
        thetas = [parse_theta(t) for t in args.theta]
        lo, hi = parse_theta(args.lower), parse_theta(args.upper)
    except ValueError as exc:
        _err(exc)
        return EXIT_PARSE
    try:
        run_benchmark(thetas, args.n, args.m, _methods_for(args.methods), tuple(lo.as_array()),
                      tuple(hi.as_array()), args.seed, jobs=args.jobs, scheme=args.scheme,
                      out_dir=args.out_dir)
    except PlanError as exc:
        _err(exc)
        return EXIT_PARSE
    return EXIT_OK


# --------------------------------------------------------------------------------- parser
def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="paper_2601_11437_b200",
        description="Exact Matern maximum-likelihood estimation on B200 (maternmle CLI).")
    sub = ap.add_subparsers(dest="command", required=True)
    methods = ["fisher-bt", "nelder-mead", "both"]

    p = sub.add_parser("estimate", help="fit Matern parameters to a dataset")
    p.add_argument("input", help="x,y,z CSV (or .npz with loc, z)")
    p.add_argument("--method", choices=methods, default="fisher-bt")
    p.add_argument("--lower", default=DEFAULT_LOWER, help="initialization cube lower corner")
    p.add_argument("--upper", default=DEFAULT_UPPER, help="initialization cube upper corner")
    p.add_argument("--seed", type=int, default=0, help="seed recorded in the result")
    p.add_argument("--out", default=None, help="result JSON path (default: stdout)")
    p.add_argument("--trace", action="store_true", help="include accepted iterates")
    p.set_defaults(func=cmd_estimate)

    p = sub.add_parser("simulate", help="draw one synthetic dataset")
    p.add_argument("out", help="output path (.csv, or .npz for large n)")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--theta", required=True, help="true parameters sigma2,alpha,nu")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--scheme", choices=["grid", "uniform"], default="grid")
    p.set_defaults(func=cmd_simulate)

    p = sub.add_parser("benchmark", help="factorial Monte-Carlo estimation study")
    p.add_argument("--theta", action="append", required=True, help="sigma2,alpha,nu (repeat)")
    p.add_argument("--n", action="append", type=int, required=True, help="size (repeat)")
    p.add_argument("--m", type=int, default=50, help="replicates per cell")
    p.add_argument("--methods", choices=methods, default="both")
    p.add_argument("--lower", default=DEFAULT_LOWER)
    p.add_argument("--upper", default=DEFAULT_UPPER)
    p.add_argument("--seed", type=int, default=0, help="master seed")
    p.add_argument("--jobs", type=int, default=1, help="GPUs to spread cells over")
    p.add_argument("--scheme", choices=["grid", "uniform"], default="grid")
    p.add_argument("--out-dir", required=True, help="directory for records and summary.csv")
    p.set_defaults(func=cmd_benchmark)

    p = sub.add_parser("loglik", help="loglik / grad / Fisher at fixed parameters")
    p.add_argument("input", help="x,y,z CSV (or .npz with loc, z)")
    p.add_argument("--theta", required=True, help="parameters sigma2,alpha,nu")
    p.add_argument("--out", default=None, help="result JSON path (default: stdout)")
    p.set_defaults(func=cmd_loglik)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
