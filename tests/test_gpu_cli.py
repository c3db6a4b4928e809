"""The command line on the GPU engine vs the reference's golden outputs: ``loglik`` at the
config-1 golden theta, ``estimate`` reproducing the reference's config-1 fit (RunRecord
fields), ``simulate`` -> ``estimate`` through the CSV and .npz formats, and a tiny
``benchmark`` (records + summary.csv with the reference's columns)."""

import csv
import json

import numpy as np
import pytest

from conftest import config_data, fit_golden, load_json

pytestmark = pytest.mark.gpu


def test_loglik_command_vs_golden(gpu, tmp_path):
    from paper_2601_11437_b200 import cli

    loc, z = config_data("config1")
    data = tmp_path / "c1.csv"
    cli.write_dataset(data, loc, z)
    rec = load_json("config1_evals.json")[0]
    out = tmp_path / "ll.json"
    th = ",".join(repr(v) for v in rec["theta"])
    assert cli.main(["loglik", str(data), "--theta", th, "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["loglik"] == pytest.approx(rec["eval_loglik"], rel=1e-10)
    np.testing.assert_allclose(doc["fisher"], rec["fisher"], rtol=1e-8)


def test_estimate_command_reproduces_reference_fit(gpu, tmp_path):
    from paper_2601_11437_b200 import cli

    gold = fit_golden("config1", 0)
    loc, z = config_data("config1")
    data = tmp_path / "c1.npz"
    cli.write_dataset(data, loc, z)
    t0 = ",".join(repr(v) for v in gold["theta0"])
    out = tmp_path / "fit.json"
    assert cli.main(["estimate", str(data), "--lower", t0, "--upper", t0, "--trace",
                     "--out", str(out)]) == 0
    rec = json.loads(out.read_text())["records"][0]
    assert rec["method"] == "fisher-bt"
    assert rec["grad_calls"] == gold["grad_calls"]
    assert rec["loglik_calls"] == gold["loglik_calls"]
    assert rec["termination"] == gold["termination"]
    hat = [rec["theta_hat"][k] for k in ("sigma2", "alpha", "nu")]
    np.testing.assert_allclose(hat, gold["theta_hat"], rtol=1e-6)
    assert len(rec["std_errors"]) == 3 and len(rec["trace"]) == len(gold["iterate_trace"])


def test_simulate_estimate_and_benchmark(gpu, tmp_path):
    from paper_2601_11437_b200 import cli

    sim = tmp_path / "s.csv"
    assert cli.main(["simulate", str(sim), "--n", "256", "--theta", "1,0.1,0.8",
                     "--seed", "3", "--scheme", "uniform"]) == 0
    meta = json.loads((tmp_path / "s.csv.meta.json").read_text())
    assert meta["n"] == 256 and meta["scheme"] == "uniform"
    out = tmp_path / "e.json"
    assert cli.main(["estimate", str(sim), "--method", "both", "--out", str(out)]) == 0
    recs = json.loads(out.read_text())["records"]
    assert [r["method"] for r in recs] == ["fisher-bt", "nelder-mead"]
    bdir = tmp_path / "bench"
    assert cli.main(["benchmark", "--theta", "1,0.1,0.5", "--n", "64", "--m", "3",
                     "--methods", "fisher-bt", "--out-dir", str(bdir)]) == 0
    runs = sorted(bdir.glob("run_t0_n64_r*.json"))
    assert len(runs) == 3
    rows = list(csv.reader(open(bdir / "summary.csv")))
    assert rows[0] == cli.SUMMARY_COLUMNS
    assert {r[3] for r in rows[1:]} == {"sigma2", "alpha", "nu", "micro"}
    # batched replicate fits == one-by-one fits
    for p in runs:
        r = json.loads(p.read_text())
        rec = r["records"][0]
        if "error" in rec:
            continue
        seed = rec["seed"]
        plan = gpu.SimulationPlan(n=64, theta_true=gpu.MaternParams(1, 0.1, 0.5),
                                  rng_seed=seed)
        loc = gpu.gen_locations(plan)
        data = gpu.SpatialDataset(loc, gpu.simulate_grf(loc, gpu.MaternParams(1, 0.1, 0.5),
                                                        seed))
        lo, hi = (gpu.MaternParams(*map(float, cli.DEFAULT_LOWER.split(","))),
                  gpu.MaternParams(*map(float, cli.DEFAULT_UPPER.split(","))))
        res = gpu.fisher_bt(data, gpu.FisherBTConfig(theta_lower=lo, theta_upper=hi))
        assert [rec["theta_hat"][k] for k in ("sigma2", "alpha", "nu")] == \
            res.theta_hat.as_array().tolist()
        assert rec["loglik_calls"] == res.loglik_calls
