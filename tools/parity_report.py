"""Measured deviation of the CUDA engine from every reference golden evaluation.

    python tools/parity_report.py [out.json]

For each golden record (tests/golden/*_evals.json: reference log_likelihood / grad_and_fisher
at pinned theta) prints the log-likelihood relative deviation, the score deviation relative to
its component scale and the Fisher entrywise relative deviation, split into
nu-dependent and other entries, and flags records in the reference's forward-difference
band (nu within 1e-6 of an integer, bessel.py:126-141).  Used to pin the test tolerances
(tests/test_gpu_likelihood.py) to measured numbers."""

import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

import paper_2601_11437_b200 as m  # noqa: E402
from conftest import GOLDEN, config_data, fd_regime  # noqa: E402
from test_gpu_likelihood import score_scale  # noqa: E402


def deviations(data, rec, n):
    th = rec["theta"]
    ll = m.log_likelihood(data, th)
    ev = m.grad_and_fisher(data, th)
    g, f = np.array(rec["grad"]), np.array(rec["fisher"])
    sc = score_scale(th, n, ev.grad, ev.fisher)
    dg = np.abs(ev.grad - g) / sc
    df = np.abs(ev.fisher - f) / np.abs(f)
    nu_mask = np.zeros((3, 3), bool)
    nu_mask[2, :] = nu_mask[:, 2] = True
    return {"theta": th, "fd_band": fd_regime(th, data.locations),
            "loglik_rel": abs(ll - rec["loglik"]) / abs(rec["loglik"]),
            "eval_loglik_rel": abs(ev.loglik - rec["eval_loglik"]) / abs(rec["eval_loglik"]),
            "score_rel_scale": dg.tolist(),
            "fisher_rel_nu": float(df[nu_mask].max()),
            "fisher_rel_other": float(df[~nu_mask].max())}


def main():
    out = []
    for name in ("config1", "config2", "config3"):
        path = GOLDEN / f"{name}_evals.json"
        if not path.exists():
            continue
        loc, z = config_data(name)
        data = m.SpatialDataset(loc, z)
        for rec in json.loads(path.read_text()):
            d = deviations(data, rec, loc.shape[0])
            d["config"] = name
            out.append(d)
            print(json.dumps(d), flush=True)
        data.release()
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
