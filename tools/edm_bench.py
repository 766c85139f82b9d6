"""BASELINE config 3: Llama-3-8B elastic shrink / grow DP8 -> DP4 -> DP8 with the
Elastic Device Manager overlapping new-world preparation with old-layout training.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/edm_bench.py [--layers L]

Per direction: (1) blocking mode: prepare, then switch (nothing overlapped);
(2) overlapped mode: prepare on the EDM side thread while the training loop keeps
running bf16 GEMM steps on its own stream; switch when ready. Prints one JSON line
with the SPEC accounting (exposed, overlapped, ratio) for both modes.
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
from paper_2605_18815_b200.edm import ElasticDeviceManager, overlap_accounting  # noqa: E402
from paper_2605_18815_b200.runtime import (Transition, init_dist, local_ranks, run_dedup_early,  # noqa: E402
                                           setup_multicast, share_buffers)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--gemm", type=int, default=8192)
    ap.add_argument("--balance", action="store_true",
                    help="grow with balance_fanout (reference PlanOptions): joiners spread over the replicas")
    ap.add_argument("--dedup", action="store_true",
                    help="replica dedup: the grow's parameters cross NVLink once per destination GPU")
    ap.add_argument("--dedup-early", action="store_true",
                    help="--dedup with the replica copies overlapping the tail of the pushes")
    ap.add_argument("--multicast", action="store_true",
                    help="state in shareable VMM buffers; the grow's parameter broadcast over NVLS multicast")
    ap.add_argument("--placement", default="matched", choices=["matched", "contiguous"],
                    help="8 devices on fewer GPUs: matched puts one device of the 4-rank world (and its DP8 "
                         "partner) on each GPU; contiguous puts devices 2g, 2g+1 on GPU g (round 1)")
    ap.add_argument("--no-nccl-comms", action="store_true",
                    help="skip the new world's NCCL communicators (always skipped when ranks share a GPU)")
    args = ap.parse_args()
    args.dedup = args.dedup or args.dedup_early
    rank, world, local, shared = init_dist()
    # NCCL refuses two ranks of one communicator on one GPU
    nccl_comms = not args.no_nccl_comms and not shared
    early = (torch.cuda.Stream(), dist.new_group(backend="gloo")) if args.dedup_early else None
    shrink, grow = S.config3(args.layers)
    if args.placement == "matched" and 1 < world < 8 and 4 % world == 0:
        # devices share GPUs (8 devices on `world` GPUs): spread the 4-rank world over every
        # GPU (device d and its old-world partner d + 4 on GPU d % world), so each process
        # hosts its share of the new world, and relabel the identity world maps so the
        # executor's contiguous blocks are those groups (runtime.colocated_world)
        import dataclasses

        from paper_2605_18815_b200.runtime import colocated_world
        groups = [sorted([d for d in range(4) if d % world == g] + [d + 4 for d in range(4) if d % world == g])
                  for g in range(world)]
        w = colocated_world(groups)
        shrink = dataclasses.replace(shrink, world_src=w[:8], world_dst=w[:4])
        grow = dataclasses.replace(grow, world_src=w[:4], world_dst=w[:8])
    grow.balance = args.balance
    edm = ElasticDeviceManager()
    train_stream = torch.cuda.Stream()
    a = torch.randn(args.gemm, args.gemm, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(args.gemm, args.gemm, device="cuda", dtype=torch.bfloat16)

    def train_step():
        with torch.cuda.stream(train_stream):
            for _ in range(4):
                torch.matmul(a, b)
        train_stream.synchronize()

    # step cost of the old layout's training loop
    for _ in range(3):
        train_step()
    t0 = time.perf_counter()
    for _ in range(5):
        train_step()
    step_s = (time.perf_counter() - t0) / 5

    state = {}
    nbuild = [0]

    def build_for(sc):
        def build(ctrl):
            t = {}
            t0 = time.perf_counter()
            edm.get_or_create_groups(sc.dst)
            plan = RoutingPlan.from_scenario(sc, allow_oversourced=True)
            t["plan_s"] = time.perf_counter() - t0
            tr = Transition(plan, world, rank, local, alloc=False)
            if nccl_comms:
                # the new world's NCCL communicators, natively and non-blocking on this side
                # thread (the training loop keeps its own NCCL group busy meanwhile)
                t1 = time.perf_counter()
                mine = local_ranks(plan, tr.ex, A.SIDE_DST) or [0]
                info = edm.create_nccl_comms(sc.dst, rank, world, local, member_rank=mine[0], group=ctrl)
                t["nccl_comms_s"] = time.perf_counter() - t1
                t["nccl_init_s"], t["nccl_split_s"], t["nccl_cache_hit"] = info["init_s"], info["split_s"], info["cache_hit"]
            tr.ex.set_replica_dedup(args.dedup, early=args.dedup_early)
            keep = []
            if args.multicast:
                # VMM state buffers shared by descriptor; the current state is the source
                adopt = {(A.SIDE_SRC, k[1], k[2]): v for k, v in state.items()}
                nbuild[0] += 1  # same sequence on every rank: a rank-independent socket tag
                tag = f"{os.environ.get('MASTER_PORT', '0')}-{sc.name}-{nbuild[0]}"
                shared = share_buffers(tr, rank, world, local, tag=tag, group=ctrl, adopt=adopt)
                t["alloc_s"] = time.perf_counter() - t0 - t["plan_s"]
                mcs = setup_multicast(shared, tr.ex, rank, world, local, tag=tag, min_payload=1 << 20, group=ctrl)
                t["multicast_groups"] = len(mcs)
                keep = [shared, mcs]
                tr.ex.prepare()
                t["total_s"] = time.perf_counter() - t0
                return tr, keep, t
            for side in (A.SIDE_SRC, A.SIDE_DST):
                nr = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
                for r in range(nr):
                    for bb in range(6):
                        _, n, g = tr.ex.buffer(side, r, bb)
                        if not n or g != rank:
                            continue
                        key = (id(sc), side, r, bb)
                        if side == A.SIDE_SRC and ("cur", r, bb) in state:
                            buf = state[("cur", r, bb)]
                        else:
                            buf = torch.empty(n, dtype=torch.uint8, device="cuda")
                        keep.append(buf)
                        tr.ex.bind(side, r, bb, buf.data_ptr(), n)
            t["alloc_s"] = time.perf_counter() - t0 - t["plan_s"]
            if world > 1:
                blob = tr.ex.ipc_export()
                blobs = [None] * world
                dist.all_gather_object(blobs, blob, group=ctrl)
                for x in blobs:
                    tr.ex.ipc_import(x)
            tr.ex.prepare()
            st = tr.ex.stats()
            t["remote_gb"], t["dup_gb"] = round(st.remote_bytes / 1e9, 2), round(st.dup_bytes / 1e9, 2)
            t["total_s"] = time.perf_counter() - t0
            return tr, keep, t
        return build

    results = {}
    seed = 0xED

    def release(keep, buffers=True):
        """Multicast objects unbind before the buffers they bind go away."""
        if not args.multicast or not keep:
            return
        for m in keep[1]:
            m.close()
        if buffers:
            for k, v in keep[0].items():
                if not (k[0] == A.SIDE_SRC and ("cur", k[1], k[2]) in state):
                    v.close()
    # the DP8 state lives in its own buffers first
    first = RoutingPlan.from_scenario(shrink)
    ex0 = Transition(first, world, rank, local, alloc=False).ex
    for r in range(first.summary.src_world):
        for bb in range(6):
            _, n, g = ex0.buffer(A.SIDE_SRC, r, bb)
            if n and g == rank:
                if args.multicast:
                    from paper_2605_18815_b200.api import VmmBuffer
                    state[("cur", r, bb)] = VmmBuffer.alloc(local, n)
                    ex0.bind(A.SIDE_SRC, r, bb, state[("cur", r, bb)].ptr, n)
                else:
                    state[("cur", r, bb)] = torch.empty(n, dtype=torch.uint8, device="cuda")
                    ex0.bind(A.SIDE_SRC, r, bb, state[("cur", r, bb)].data_ptr(), n)
    ex0.fill(A.SIDE_SRC, seed)
    del ex0
    for name, sc in (("shrink_dp8_to_dp4", shrink), ("grow_dp4_to_dp8", grow)):
        out = {}
        for mode in ("blocking", "overlapped"):
            torch.cuda.synchronize()
            dist.barrier()
            edm.prepare_async(build_for(sc))
            window_steps = 0
            t_win = time.perf_counter()
            if mode == "overlapped":
                while not edm.ready():
                    train_step()
                    window_steps += 1
            tr, keep, tprep = edm.wait()
            window_s = time.perf_counter() - t_win if mode == "overlapped" else 0.0
            # all ranks must have finished preparing before anyone writes into peers
            flag = torch.ones(1, device="cuda")
            dist.all_reduce(flag)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if early is not None:  # replica copies overlap the tail of the pushes
                run_dedup_early(tr.ex, torch.cuda.current_stream(), early[0], early[1])
            else:
                tr.run()
            torch.cuda.synchronize()
            dist.barrier()
            if args.dedup and early is None:  # the replica copies on each destination GPU, after the pushes everywhere
                tr.ex.run_dup()
                torch.cuda.synchronize()
                dist.barrier()
            switch_s = time.perf_counter() - t0
            bad = tr.ex.verify(A.SIDE_DST, seed)[0]
            if nccl_comms:
                # the new world's communicators work: an all-reduce over the world and each
                # dimension sums to the communicator's size
                sizes = {"world": edm.check_nccl_comm(sc.dst)}
                for d in ("dp", "tp", "pp"):
                    sizes[d] = edm.check_nccl_comm(sc.dst, d)
                tprep["nccl_allreduce_sizes"] = sizes
                if sizes["world"] != world:
                    bad += 1
                if mode == "blocking":  # the overlapped run builds the new world from scratch
                    edm.destroy_nccl_comms(sc.dst)
            init = torch.tensor([edm.init_s, window_s, switch_s, float(bad)], dtype=torch.float64, device="cuda")
            dist.all_reduce(init, op=dist.ReduceOp.MAX)
            init_s, window_s, switch_s, bad = init.tolist()
            acc = overlap_accounting(init_s, switch_s, window_s=window_s, mode=mode)
            acc.update(window_train_steps=window_steps, train_step_s=step_s, verified_mismatches=int(bad),
                       bytes_moved=tr.plan.bytes_moved(), prepare_breakdown_rank0=tprep)
            out[mode] = acc
            if mode == "blocking":  # free the blocking run's new layout before the overlapped one
                release(keep)
                del tr, keep
                torch.cuda.synchronize()
            else:
                last = (tr, keep)
        # the new layout becomes the current state for the next event
        tr, keep = last
        state.clear()
        if args.multicast:
            for k, v in keep[0].items():
                if k[0] == A.SIDE_DST:
                    state[("cur", k[1], k[2])] = v
            release(keep, buffers=False)
            # the old layout (the adopted sources) is dead after the switch
            for k, v in keep[0].items():
                if k[0] != A.SIDE_DST:
                    v.close()
        else:
            for r in range(tr.plan.summary.dst_world):
                for bb in range(6):
                    p, n, g = tr.ex.buffer(A.SIDE_DST, r, bb)
                    if n and g == rank:
                        for t in keep:
                            if t.data_ptr() == p:
                                state[("cur", r, bb)] = t
        results[name] = out
        # the old layout is gone after the switch: drop every reference to its buffers
        del tr, keep, last
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"config": "BASELINE config 3: Llama-3-8B DP8->DP4->DP8, ZeRO-1", "layers": args.layers,
                          "placement": args.placement, "world_src_shrink": shrink.world_src,
                          "n_gpus": world, "grow_balance_fanout": args.balance, "multicast": args.multicast, "dedup": args.dedup, "dedup_early": args.dedup_early,
                          "results": results}), flush=True)
    dist.barrier()
    edm.close()  # the new worlds' NCCL communicators before the process group
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
