"""Developer probe: do two replica groups fitted from two host threads overlap on the GPU
(one group's latency-bound Cholesky under the other's tensor-core solves)?
Prints the wall time of fit_many over all 5 config-2 replicas (one thread) against
splits into concurrent groups, and checks that every fit is bit-identical."""
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2601_11437_b200 as m  # noqa: E402

host = [bench.load_replica(s, 0) for s in range(5)]
ds = [m.SpatialDataset(loc, z, device=0) for loc, z in host]


def timed(fn, reps=3):
    fn()
    best = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        best.append(time.perf_counter() - t0)
    return min(best), out


def split(groups):
    def run():
        res = [None] * len(groups)

        def work(i, g):
            res[i] = bench.run_fits([ds[j] for j in g])
        th = [threading.Thread(target=work, args=(i, g)) for i, g in enumerate(groups)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        flat = {}
        for g, r in zip(groups, res):
            for j, x in zip(g, r):
                flat[j] = x
        return [flat[j] for j in range(5)]
    return run


t1, ref = timed(lambda: bench.run_fits(ds))
g = sum(r.grad_calls for r in ref)
print(f"one group of 5: {t1*1e3:.1f} ms  {g / t1:.1f} it/s")
for groups in ([[0, 1, 2], [3, 4]], [[0, 2, 4], [1, 3]], [[0], [1], [2], [3], [4]],
               [[0, 1], [2, 3], [4]]):
    t, out = timed(split(groups))
    same = all(np.array_equal(a.theta_hat.as_array(), b.theta_hat.as_array()) and
               a.grad_calls == b.grad_calls for a, b in zip(ref, out))
    print(f"groups {groups}: {t*1e3:.1f} ms  {g / t:.1f} it/s  identical={same}")
