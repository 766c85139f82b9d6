"""Replica dedup on one GPU standing in for a 2- and 4-GPU placement: the root's
NVLink bytes with and without it (executor stats only)."""
import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.api import Executor, RoutingPlan
_, grow = S.config3(2)
plan = RoutingPlan.from_scenario(grow, allow_oversourced=True)
for n_gpus in (2, 4):
    for dd in (False, True):
        ex = [Executor(plan, n_gpus=n_gpus, gpu=g, device=0) for g in range(n_gpus)]
        keep = []
        for side in (0, 1):
            n = plan.summary.src_world if side == 0 else plan.summary.dst_world
            for r in range(n):
                for b in range(6):
                    _, nb, g = ex[0].buffer(side, r, b)
                    if nb:
                        t = torch.zeros(nb, dtype=torch.uint8, device="cuda"); keep.append(t)
                        for e in ex: e.bind(side, r, b, t.data_ptr(), nb)
        for e in ex:
            e.set_replica_dedup(dd); e.prepare()
        print(n_gpus, dd, [(round(e.stats().remote_bytes/1e9,2), round(e.stats().dup_bytes/1e9,2), round(e.stats().local_bytes/1e9,2)) for e in ex])
        del ex, keep
        torch.cuda.empty_cache()
