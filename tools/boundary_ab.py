"""A/B of the Cholesky's chain-first outer boundary (MLE_BOUNDARY_SPLIT=1 default vs 0):
results must be bit-identical (same per-tile arithmetic in the same order)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(REPO))
    import paper_2601_11437_b200 as m

    out = []
    for name, seed in (("config2", 0), ("config3", 0)):
        d = np.load(REPO / "tests" / "golden" / f"{name}_seed{seed}_data.npz")
        data = m.SpatialDataset(d["loc"], d["z"])
        for th in ((1.0, 0.2, 1.5), (0.9, 0.08, 0.7)):
            ll, g, f = data.engine().eval_all(np.array(th))
            out += [ll, *g, *f.ravel(), data.engine().loglik(np.array(th) * 1.01)]
        data.release()
    np.save(sys.argv[2], np.array(out))
    sys.exit(0)
res = {}
for flag in ("1", "0"):
    env = dict(os.environ, **{os.environ.get("AB_VAR", "MLE_BOUNDARY_SPLIT"): flag})
    path = f"/tmp/ab_{flag}.npy"
    subprocess.run([sys.executable, __file__, "child", path], env=env, check=True)
    res[flag] = np.load(path)
print("bit-identical:", bool(np.array_equal(res["1"], res["0"])),
      "max rel diff:", float(np.max(np.abs(res["1"] - res["0"]) / np.abs(res["0"]))))
