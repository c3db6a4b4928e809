import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2601_11437_b200 as gpu
from oracle import maternmle_cpu as O
th = (0.9, 0.08, 1.013)
for tau2 in (0.0, 1e-6, 1e-2):
    loc = gpu.gmm_locations(700, 3)
    z = O.cholesky(O.matrix(loc, th, "sigma", tau2)) @ np.random.default_rng(3).standard_normal(700)
    ref = O.eval_all_nugget(loc, z, th, tau2) if tau2 > 0 else O.eval_all(loc, z, th)
    ev = gpu.grad_and_fisher(gpu.SpatialDataset(loc, z, nugget=tau2), th)
    print(tau2, "grad diff", ev.grad - ref[1], "ll rel", abs(ev.loglik - ref[0]) / abs(ref[0]),
          "fisher rel", np.max(np.abs(ev.fisher - ref[2]) / np.abs(ref[2])))
