"""Config 4 / 5 with the distributed engine: one rank per GPU.

    python -m torch.distributed.run --standalone --nproc-per-node G tools/run_distributed.py \
        config4 [--fit] [--evals K]

Rank 0 draws the field (single-GPU engine: z = L w needs only Sigma, which fits one B200 up
to n ~ 100k) and broadcasts it; every rank builds its column panels and all ranks run the same
deterministic host loop.  Prints one JSON record from rank 0 (times are max over ranks).
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import paper_2601_11437_b200 as m  # noqa: E402
from paper_2601_11437_b200.distributed import DistributedEngine, TorchComm  # noqa: E402
from paper_2601_11437_b200.fisher_bt import drive, fisher_bt_gen  # noqa: E402


class _Objective:
    """Counting objective over the distributed engine (optimizer.py:114-142 semantics)."""

    def __init__(self, eng):
        self.eng = eng
        self.loglik_calls = 0
        self.grad_calls = 0

    def loglik(self, theta):
        self.loglik_calls += 1
        try:
            v = self.eng.loglik(theta)
        except (m.NotPositiveDefinite, ValueError):
            return -np.inf
        return -np.inf if np.isnan(v) else v

    def eval_all(self, theta):
        self.loglik_calls += 1
        self.grad_calls += 1
        return self.eng.eval_all(theta)


def _max_over_ranks(x):
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    name = sys.argv[1]
    fit = "--fit" in sys.argv
    evals = int(sys.argv[sys.argv.index("--evals") + 1]) if "--evals" in sys.argv else 1
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    wl = m.WORKLOADS[name]
    seed = wl.seeds[0]
    loc = wl.locations(seed)
    zt = torch.zeros(wl.n, dtype=torch.float64, device="cuda")
    if rank == 0:
        zt.copy_(torch.from_numpy(m.simulate_field(loc, wl.theta_true, seed, device=local)))
    dist.broadcast(zt, 0)
    z = zt.cpu().numpy()
    eng = DistributedEngine(loc, z, TorchComm(), nugget=wl.nugget, device=local)
    th = np.array(wl.theta_true, float)
    rec = {"config": name, "n": wl.n, "world": world, "nb": eng.nb}
    ts = []
    for r in range(evals):
        dist.barrier()
        t0 = time.perf_counter()
        ll, g, f = eng.eval_all(th)  # no factor cache in the distributed engine
        ts.append(_max_over_ranks(time.perf_counter() - t0))
    rec["eval_all_s"] = ts
    dist.barrier()
    t0 = time.perf_counter()
    eng.loglik(th * (1 + 3e-9))
    rec["loglik_s"] = _max_over_ranks(time.perf_counter() - t0)
    rec["at_theta_true"] = {"loglik": ll, "grad": g.tolist(), "fisher": f.tolist()}
    if fit:
        th0 = m.MaternParams(*wl.theta0)
        cfg = m.FisherBTConfig(theta_lower=th0, theta_upper=th0)
        obj = _Objective(eng)
        dist.barrier()
        t0 = time.perf_counter()
        res = drive(fisher_bt_gen(cfg, obj), obj)
        wall = _max_over_ranks(time.perf_counter() - t0)
        rec["fit"] = {"theta_hat": res.theta_hat.as_array().tolist(),
                      "loglik_at_hat": res.loglik_at_hat, "grad_calls": res.grad_calls,
                      "loglik_calls": res.loglik_calls, "termination": res.termination.value,
                      "wall_s": wall, "fisher_it_per_s": res.grad_calls / wall}
    if rank == 0:
        print(json.dumps(rec), flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
