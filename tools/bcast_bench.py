"""Broadcast promotion over NVLS multicast on BASELINE config 3's grow (Llama-3-8B
DP4 -> DP8, ZeRO-1): the joiners' parameters (every DP replica needs the whole model)
go from the root GPU as ONE multicast store stream instead of one push per joiner.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bcast_bench.py [--layers L]

All variants run on the same multi-GPU arena (VMM buffers, shared by descriptors) and
are verified bit-exact against canon (destinations cleared first). Prints one JSON line
(rank 0) with the forward transition time (max over ranks) of: per-destination pushes,
multicast, replica dedup (a region crosses NVLink once per destination GPU and is copied
to the other replica ranks there after a barrier), and dedup + multicast.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Arena, RoutingPlan  # noqa: E402
from paper_2605_18815_b200.runtime import (Transition, dist_env, exchange_arena, global_stage_cuts,  # noqa: E402
                                           run_dedup_early, setup_multicast)


def run_once(ex, stream, world, dedup, early=None):
    """One transition: fused/multicast pushes, then (replica dedup, on EVERY rank so the
    collectives stay matched) a barrier and the copies on each destination GPU. early =
    (side stream, gloo group): the copies start after the primaries' pushes and overlap
    the rest (runtime.run_dedup_early)."""
    if early is not None:
        run_dedup_early(ex, stream, early[0], early[1])
        return
    ex.run(stream.cuda_stream)
    if dedup:
        torch.cuda.synchronize()
        dist.barrier()
        ex.run_dup(stream.cuda_stream)


def timed(ex, stream, reps, world, dedup, early=None):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_once(ex, stream, world, dedup, early)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    mine = torch.tensor([min(ts)], dtype=torch.float64, device="cuda")
    per = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(per, mine)
    t = torch.tensor([min(ts), sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist() + [[round(x.item(), 3) for x in per]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--chunk-mb", type=int, default=512,
                    help="arena chunk (multicast binds chunk by chunk; 512 MiB = the recommended granularity)")
    ap.add_argument("--variants", default="push,multicast,dedup,dedup_multicast,dedup_early,dedup_early_multicast",
                    help="comma-separated subset to run")
    args = ap.parse_args()
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _, grow = S.config3(args.layers)
    plan = RoutingPlan.from_scenario(grow)
    arena = Arena.multi(plan, None, world, rank, local, chunk_bytes=args.chunk_mb << 20, groups=1)
    exchange_arena(arena, rank, world, tag=f"{os.environ.get('MASTER_PORT', '0')}-bcast")
    tr = Transition(plan, world, rank, local, alloc=False)
    arena.bind(tr.ex, None, global_stage_cuts(arena, world))
    ex = tr.ex
    stream = torch.cuda.current_stream()
    seed = 0xB0CA57
    out = {"workload": f"llama3-8b (L={args.layers}) dp4->dp8 zero1 grow (config 3)", "n_gpus": world,
           "chunk_mb": args.chunk_mb,
           "plan_bytes": plan.bytes_moved()}

    ctrl = dist.new_group(backend="gloo")
    side = torch.cuda.Stream()

    def variant(name, dedup, multicast, early=False):
        ex.set_replica_dedup(dedup, early=early)
        ear = (side, ctrl) if early else None
        mcs = []
        groups = ex.bcast_groups()
        if multicast and groups:
            mcs = setup_multicast(arena, ex, rank, world, local, tag=f"{os.environ.get('MASTER_PORT', '0')}-{name}",
                                  min_payload=1 << 20)
        ex.prepare()
        ex.fill(A.SIDE_DST, seed ^ 0x5A5A)  # cleared: the check proves this variant delivered them
        ex.fill(A.SIDE_SRC, seed)
        torch.cuda.synchronize()
        dist.barrier()
        run_once(ex, stream, world, dedup, ear)
        torch.cuda.synchronize()
        dist.barrier()
        bad = ex.verify(A.SIDE_DST, seed)[0] + ex.verify(A.SIDE_SRC, seed)[0]
        ms_min, ms_avg, per = timed(ex, stream, args.reps, world, dedup, ear)
        st = ex.stats()
        t = torch.tensor([bad], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        out[name] = {"ms_min": round(ms_min, 3), "ms_avg": round(ms_avg, 3), "mismatches": int(t.item()),
                     "ms_per_rank": per, "remote_gb_rank0": round(st.remote_bytes / 1e9, 2),
                     "mc_gb_rank0": round(st.mc_bytes / 1e9, 2), "dup_gb_rank0": round(st.dup_bytes / 1e9, 2),
                     "multicast_groups": len(mcs)}
        if name == "multicast":
            out["bcast_groups"] = [{"id": g.id, "root_rank": g.root_rank, "root_gpu": g.root_gpu, "slot": g.slot,
                                    "member_gpus": list(g.member_gpu[: g.n_members]),
                                    "member_ranks": list(g.member_rank[: g.n_members]),
                                    "payload_gb": round(g.payload_bytes / 1e9, 3)} for g in groups]
        for m in mcs:  # unbind before the next variant rebinds
            m.close()
        for g in groups:
            if g.root_gpu == rank and mcs:
                ex.set_multicast(g.id, 0)

    todo = args.variants.split(",")
    for name, dedup, multicast, early in (("push", False, False, False), ("multicast", False, True, False),
                                          ("dedup", True, False, False), ("dedup_multicast", True, True, False),
                                          ("dedup_early", True, False, True),
                                          ("dedup_early_multicast", True, True, True)):
        if name in todo:
            variant(name, dedup, multicast, early)
    if "push" in out:
        out["speedup_vs_push"] = {k: round(out["push"]["ms_min"] / out[k]["ms_min"], 3)
                                  for k in ("multicast", "dedup", "dedup_multicast", "dedup_early", "dedup_early_multicast")
                                  if k in out}
    del ex, tr, arena
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
