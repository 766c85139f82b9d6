"""SPEC execute modes on the Table 4 geometry (AC9):
LLaMA-2 13B (TP,PP,DP) (2,8,1) <-> (2,2,4), 16 virtual ranks on N GPUs.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/ablation.py [--layers 8]

Modes: naive (one NCCL message per op, sequential), sync (buffered, one XOR step at a
time), async (buffered, all steps of a stage at once) and fused (the product: one-sided
NVLink/HBM stores, no staging). Every run is verified bit-exact. One JSON line.
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import RoutingPlan  # noqa: E402
from paper_2605_18815_b200.runtime import StagedTransition, Transition, dist_env  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = S.table4(args.layers)
    seed = 0x7AB4
    out = {}
    for name, s in (("s1_to_s2", sc), ("s2_to_s1", sc.reversed())):
        plan = RoutingPlan.from_scenario(s, allow_oversourced=True)
        res = {}
        for mode in ("fused", "async", "sync", "naive"):
            tr = Transition(plan, world, rank, local, alloc=False)
            keep = []
            for side in (A.SIDE_SRC, A.SIDE_DST):
                nr = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
                for r in range(nr):
                    for b in range(6):
                        _, n, g = tr.ex.buffer(side, r, b)
                        if n and g == rank:
                            t = torch.zeros(n, dtype=torch.uint8, device="cuda")
                            keep.append(t)
                            tr.ex.bind(side, r, b, t.data_ptr(), n)
            if mode == "fused":
                tr.connect()
                run = tr.run
            else:
                run = StagedTransition(plan, tr.ex, world, rank, mode=mode).run
            tr.ex.fill(A.SIDE_SRC, seed)
            times = []
            for i in range(args.reps + 1):
                torch.cuda.synchronize()
                dist.barrier()
                t0 = time.perf_counter()
                run()
                torch.cuda.synchronize()
                dist.barrier()
                if i:
                    times.append(time.perf_counter() - t0)
            bad = tr.ex.verify(A.SIDE_DST, seed)[0]
            t = torch.tensor([min(times), float(bad)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[mode] = {"seconds": round(t[0].item(), 5), "verified_mismatches": int(t[1].item())}
            del tr, keep
            torch.cuda.synchronize()
        res["bytes_moved"] = plan.bytes_moved()
        res["ordering_async<sync<naive"] = res["async"]["seconds"] < res["sync"]["seconds"] < res["naive"]["seconds"]
        out[name] = res
    if rank == 0:
        print(json.dumps({"geometry": "PAPER Table 4: LLaMA-2 13B (TP,PP,DP) (2,8,1) <-> (2,2,4), 16 virtual ranks",
                          "layers": args.layers, "n_gpus": world, "results": out}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
