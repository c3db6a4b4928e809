"""Where the diagonal-tile chain loses time inside a batched config-2 loglik pass (five
n = 3,600 replicas): every potrf_diag_kernel CTA's globaltimer stamps (entry, tile loaded,
pivot blocks done, inverse done, exit; mle_diag_trace) next to the pass's launch completion
timeline (MLE_TRACE).

    MLE_TRACE=gpurun_out/diag_pass_trace.txt python tools/diag_trace_probe.py > out.txt
"""
import ctypes
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402
from paper_2601_11437_b200 import _native as nat  # noqa: E402

lib = nat.lib
lib.mle_diag_trace.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p,
                               ctypes.POINTER(ctypes.c_longlong)]
data = []
for s in range(5):
    d = np.load(REPO / "tests" / "golden" / f"config2_seed{s}_data.npz")
    data.append(m.SpatialDataset(d["loc"], d["z"]))
eng = [d.engine() for d in data]
th = np.array([1.0, 0.2, 1.5])
for r in range(3):  # warm-up (buffers, tables)
    m.eval_batch(eng, [th * (1 + 1e-9 * r)] * 5, [1] * 5)
cap = 4096
assert lib.mle_diag_trace(1, cap, None, None) == 0
m.eval_batch(eng, [th * 1.01] * 5, [1] * 5)  # one batched loglik pass (factoring)
print("pass", eng[0].phase_times())
buf = np.zeros((cap, 6), dtype=np.int64)
cnt = ctypes.c_longlong(0)
assert lib.mle_diag_trace(0, 0, buf.ctypes.data, ctypes.byref(cnt)) == 0
rec = buf[: cnt.value]
rec = rec[np.argsort(rec[:, 0])]
t0 = rec[0, 0]
print(f"{cnt.value} diag CTAs (one per dataset per tile)")
print("tile sm  start_us  load_us  pivots_us  inverse_us  store_us  total_us  gap_from_prev_tile_end_us")
prev_end = None
for tile in sorted(set(rec[:, 5] % 1000)):
    rows = rec[rec[:, 5] % 1000 == tile]
    st = rows[:, 0].min()
    en = rows[:, 4].max()
    d = np.median(np.diff(rows[:, :5], axis=1), axis=0) / 1e3
    gap = (st - prev_end) / 1e3 if prev_end is not None else 0.0
    print(f"{tile:4d} {int(rows[0, 5] // 1000):3d} {(st - t0) / 1e3:9.1f} {d[0]:8.1f} {d[1]:10.1f} "
          f"{d[2]:11.1f} {d[3]:9.1f} {(en - st) / 1e3:9.1f} {gap:10.1f}")
    prev_end = en
