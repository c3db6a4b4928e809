import os, sys, json, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import config_data
import paper_2601_11437_b200 as gpu
loc, z = config_data('config2', 2)
d = json.load(open('tests/golden/config2_seed2_fit.json'))
np.set_printoptions(precision=17)
for S in ('6', '7'):
    os.environ['MLE_SOLVE_SLICES'] = S
    for gemm in ('ozaki', 'dmma'):
        os.environ['MLE_FP64_GEMM'] = gemm
        for th, _ in d['iterate_trace'][-2:]:
            r = gpu.Engine(loc, z).eval_all(np.array(th))
            print(S, gemm, repr(r[0]), r[1].tolist(), np.linalg.norm(r[1]))
