"""A/B of an engine switch given as ENV=VALUE pairs: each variant runs in its own process
(the switches are read once per process), evaluates config 1 / config 2 (batched, loglik and
eval_all) / config 3 and prints results as hex bits plus timings; the parent compares bits.

  python tools/stage_ab.py MLE_DGEMM_STAGE=cpasync MLE_DGEMM_STAGE=bulk
"""
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

    out = {}
    # config 2 batched passes (the latency-bound chain)
    data = []
    for s in range(5):
        d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
        data.append(m.SpatialDataset(d["loc"], d["z"]))
    eng = [d.engine() for d in data]
    th = np.array([1.0, 0.2, 1.5])
    import torch
    for mode, name in ((1, "loglik"), (2, "eval_all")):
        ts = []
        for r in range(12):
            thr = th * (1 + 1e-9 * r)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = m.eval_batch(eng, [thr] * 5, [mode] * 5)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        out[f"config2_batched_{name}_ms"] = sorted(ts)[len(ts) // 2]
        out[f"config2_batched_{name}_phases"] = eng[0].phase_times()
    bits = []
    for e in eng:
        ll, gr, fi = e.eval_all(th)[:3]
        bits += [float(ll).hex()] + [float(x).hex() for x in np.asarray(gr).ravel()]
        bits += [float(x).hex() for x in np.asarray(fi).ravel()]
    out["config2_bits"] = bits
    # config 3 single evaluation (two-sided path)
    d = np.load(REPO / "tests" / "golden" / "config3_seed0_data.npz")
    ds = m.SpatialDataset(d["loc"], d["z"])
    e3 = ds.engine()
    th3 = (1.5, 0.05, 0.8)
    ts = []
    for r in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev = e3.eval_all(tuple(x * (1 + 1e-9 * r) for x in th3))
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    out["config3_eval_all_ms"] = min(ts)
    out["config3_phases"] = e3.phase_times()
    ll, gr, fi = e3.eval_all(th3)[:3]
    out["config3_bits"] = ([float(ll).hex()] + [float(x).hex() for x in np.asarray(gr).ravel()]
                           + [float(x).hex() for x in np.asarray(fi).ravel()])
    print("RESULT " + json.dumps(out))


def main():
    variants = sys.argv[1:]
    res = {}
    variants = [f"{i}:{v}" for i, v in enumerate(variants)]
    for v in variants:
        env = dict(os.environ)
        for kv in v.split(":", 1)[1].split(","):
            k, val = kv.split("=", 1)
            env[k] = val
        p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True,
                           text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(v, "FAILED", p.stdout[-2000:], p.stderr[-2000:])
            continue
        res[v] = json.loads(line[0][7:])
    base = variants[0]
    for v in variants:
        if v not in res:
            continue
        r = res[v]
        same2 = r["config2_bits"] == res[base]["config2_bits"] if base in res else None
        same3 = r["config3_bits"] == res[base]["config3_bits"] if base in res else None
        print(json.dumps({"variant": v, "bits_equal_config2": same2, "bits_equal_config3": same3,
                          **{k: r[k] for k in r if not k.endswith("_bits")}}))


if __name__ == "__main__":
    child() if "--child" in sys.argv else main()
