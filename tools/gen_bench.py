"""Generation throughput probe: the bench's kernel-profiling pass (one stream, CUDA events
around every generation / Ozaki GEMM / slicing launch) over a batched config-2 eval_all."""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402

data = []
for s in range(5):
    d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
    data.append(m.SpatialDataset(d["loc"], d["z"]))
eng = [d.engine() for d in data]
th = np.array([1.0, 0.2, 1.5])
for r in range(3):
    m.eval_batch(eng, [th * (1 + 1e-7 * r)] * 5, [2] * 5)
eng[0].kernel_profile(True)
for r in range(4):
    m.eval_batch(eng, [th * (1 + 1e-7 * (r % 2))] * 5, [2] * 5)
    ks = eng[0].kernel_stats()
    print({k: round(v, 4) if isinstance(v, float) else v for k, v in ks.items()})
    print("gen GB/s", ks["gen_bytes"] / (ks["gen_ms"] * 1e-3) / 1e9,
          "slice GB/s", ks["slice_bytes"] / (ks["slice_ms"] * 1e-3) / 1e9)
eng[0].kernel_profile(False)
