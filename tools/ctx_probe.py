import sys, time
sys.path.insert(0, '.')
import numpy as np
import bench
import paper_2601_11437_b200 as m
host = [bench.load_replica(s, 0) for s in range(5)]
th0 = m.MaternParams(0.8, 0.1, 1.0)
for rep in range(4):
    t0 = time.perf_counter()
    ds = [m.SpatialDataset(loc, z, device=0) for loc, z in host]
    t1 = time.perf_counter()
    e = [d.engine() for d in ds]
    t2 = time.perf_counter()
    m.eval_batch(e, [np.array([0.8,0.1,1.0])]*5, [1]*5)
    t3 = time.perf_counter()
    for d in ds: d.release()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms  engine {1e3*(t2-t1):.2f}  first loglik pass {1e3*(t3-t2):.2f}  release {1e3*(t4-t3):.2f}")
