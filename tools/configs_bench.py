"""BASELINE's other configurations through the same fused executor (SURVEY §8d
"Other configs"), one direction each, bit-exact verified, timed max over ranks, with
the §8d roofline T_roof = max_g max(out_g / NVLink, in_g / NVLink, HBM_g / B_HBM).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/configs_bench.py [--config 4 --layers 48]

Prints one JSON line per configuration (rank 0). Config 5 (Llama-3-70B) needs 247 GB of
old + new state per GPU at N=8; on fewer GPUs pass --layers to scale its depth.
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
from paper_2605_18815_b200.api import RoutingPlan  # noqa: E402
from paper_2605_18815_b200.runtime import Transition, device_barrier, dist_env, run_stages, shared_arena  # noqa: E402

NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("hbm_gbs", 6558.0))
    except (OSError, ValueError):
        return 6558.0


def scenario(cfg: int, layers: int):
    if cfg == 1:
        return S.config1()
    if cfg == 2:
        return S.config2(layers or 32)
    if cfg == 3:
        return S.config3(layers or 32)[1]
    if cfg == 4:
        return S.config4(layers or 48)
    if cfg == 5:
        return S.config5(layers or 80)
    raise SystemExit(f"unknown config {cfg}")


def run_one(sc, rank, world, local, reps, arena_cap=0.0, host_barriers=False, level=None, placement="contiguous"):
    plan = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    colocated = None
    if placement == "balanced" and 1 < world < len(plan.traffic()) and sc.world_src is None and sc.world_dst is None \
            and sc.src.world() == sc.dst.world():
        # which devices share a GPU, from the plan's traffic matrix (bench.py's default)
        import dataclasses

        from paper_2605_18815_b200.runtime import colocated_world, colocation
        colocated = colocation(plan.traffic(), world)
        w = colocated_world(colocated)
        sc = dataclasses.replace(sc, world_src=w, world_dst=w)
        plan = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    arena = None
    if arena_cap:
        # old + new state do not fit: the memory-aware arena under a per-GPU cap, stages
        # with a barrier between them (runtime.run_stages)
        arena, cuts = shared_arena(plan, None, rank, world, local, cap_bytes=int(arena_cap * 1e9),
                                   tag=f"{os.environ.get('MASTER_PORT', '0')}-{sc.name}-{level}-{int(host_barriers)}",
                                   level=level)
        tr = Transition(plan, world, rank, local, alloc=False)
        arena.bind(tr.ex, None, cuts)
        tr.ex.prepare()
        # stage boundaries: the device-side SynchronizeAll (no host round trip), or host
        # synchronize + dist.barrier with --host-barriers
        dbar = None if host_barriers else device_barrier(rank, world, local)
        tr.run = lambda stream=0: run_stages(tr.ex, stream, world, barrier=dbar)
    else:
        tr = Transition(plan, world, rank, local)
        tr.connect()
    ex = tr.ex
    seed = 0x5EED5
    ex.fill(A.SIDE_SRC, seed)
    # a dedicated stream: transitions under 1 GiB per GPU replay from a CUDA graph from
    # their second run on, and the legacy default stream cannot be captured
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tr.run(stream.cuda_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    bad = ex.verify(A.SIDE_DST, seed)[0]
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tr.run(stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = torch.tensor([min(ts), float(bad)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, bad = t.tolist()
    pl = [plan.placement(world, g) for g in range(world)]
    link = max(max(p.out_bytes, p.in_bytes) for p in pl)
    hbm = max(2 * p.local_bytes + p.out_bytes + p.in_bytes for p in pl)
    hbm_gbs = peaks()
    t_roof = max(link / (NVLINK_GBS * 1e9), hbm / (hbm_gbs * 1e9))
    out = {"config": sc.name, "n_gpus": world, "plan_bytes": plan.bytes_moved(), "retained_bytes": plan.bytes_retained(),
           "colocation": colocated or placement,
           "transfers": plan.num_transfers(), "ms": round(ms, 3), "mismatches": int(bad),
           "gbs_per_gpu": round(plan.bytes_moved() / (ms / 1e3) / 1e9 / world, 1),
           "roofline": {"bound": "nvlink" if link / NVLINK_GBS > hbm / hbm_gbs else "hbm",
                        "t_roof_ms": round(t_roof * 1e3, 3), "frac": round(t_roof * 1e3 / ms, 4),
                        "max_link_gb": round(link / 1e9, 2), "max_hbm_gb": round(hbm / 1e9, 2),
                        "peaks": {"nvlink_gbs": NVLINK_GBS, "hbm_gbs": hbm_gbs}}}
    if arena is not None:
        st = arena.stats()
        out["arena"] = {"cap_gb": arena_cap, "physical_gb": round(st.physical_bytes / 1e9, 2),
                        "stage_barriers": "host" if host_barriers else "device",
                        "old_gb": round(st.a_bytes / 1e9, 2), "new_gb": round(st.b_bytes / 1e9, 2),
                        "aliased_gb": round(st.aliased_bytes / 1e9, 2), "bands": st.bands, "stages": ex.num_stages(),
                        "level": level if level is not None else "fastest fitting"}
    del tr, ex, arena
    torch.cuda.synchronize()
    return out


def barrier_probe(rank, world, local, n):
    """SynchronizeAll latency: n device barriers enqueued back to back on one stream, timed
    with events (max over ranks); the per-barrier cost a memory-aware stage boundary adds."""
    dbar = device_barrier(rank, world, local)
    stream = torch.cuda.Stream()
    for _ in range(10):
        dbar(stream.cuda_stream)
    torch.cuda.synchronize()
    out = {"what": "device barrier (SynchronizeAll) latency", "n_gpus": world, "barriers": n}
    for label, k in (("per_barrier_us", n),):
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            dbar(stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e3 / k], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[label] = round(t.item(), 2)
    out["timed_out"] = dbar.timed_out()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, action="append")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--arena-cap", type=float, default=0.0,
                    help="GB per GPU: run under the memory-aware arena (old + new need not fit)")
    ap.add_argument("--host-barriers", action="store_true",
                    help="arena stages separated by host synchronize + dist.barrier instead of the device barrier")
    ap.add_argument("--level", type=int, action="append",
                    help="with --arena-cap: force this schedule ladder level (repeatable); default: the fastest that fits")
    ap.add_argument("--both-barriers", action="store_true", help="run every arena case with device and host barriers")
    ap.add_argument("--placement", default="contiguous", choices=["balanced", "contiguous"],
                    help="which of the scenario's devices share a GPU when there are fewer GPUs (runtime.colocation)")
    ap.add_argument("--barrier-probe", type=int, default=0,
                    help="time N back-to-back device barriers (SynchronizeAll latency) and exit")
    args = ap.parse_args()
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.barrier_probe:
        res = barrier_probe(rank, world, local, args.barrier_probe)
        if rank == 0:
            print(json.dumps(res), flush=True)
    else:
        for cfg in args.config or [1, 4]:
            for lv in (args.level or [None]):
                for hb in ((False, True) if args.both_barriers else (args.host_barriers,)):
                    res = run_one(scenario(cfg, args.layers), rank, world, local, args.reps, args.arena_cap, hb, lv,
                                  args.placement)
                    if rank == 0:
                        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
