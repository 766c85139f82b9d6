"""The fused push across GPUs driven from ONE process (so ncu can attach): each GPU's
executor stores its peer-bound tiles straight into the other GPU's memory (peer access,
no cudaIpc). The north star's forward transition split over 2 (--gpus) GPUs, bit-exact,
with per-GPU NVLink GB/s from CUDA events.

    python tools/p2p_profile.py [--layers 4] [--reps 3]
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,... \\
        -k regex:copy_tiles python tools/p2p_profile.py --reps 1
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Executor, RoutingPlan, enable_peer_access  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--ctas", type=int, default=0, help="CTAs per SM of the copy kernels (0: default)")
    ap.add_argument("--tile-bytes", type=int, default=0, help="tile size (0: default 512 KiB)")
    ap.add_argument("--placement", default="contiguous", choices=["balanced", "contiguous"],
                    help="which devices share a GPU (balanced: bench.py's default co-location)")
    ap.add_argument("--same-device", action="store_true",
                    help="place every executor's GPU on device 0 (one-GPU boxes: the one-process multi-executor path)")
    args = ap.parse_args()
    G = args.gpus
    dev = (lambda g: 0) if args.same_device else (lambda g: g)
    if not args.same_device and torch.cuda.device_count() < G:
        print(json.dumps({"skipped": f"needs {G} GPUs"}))
        return
    for a in range(G):
        for b in range(G):
            if dev(a) != dev(b):
                enable_peer_access(dev(a), dev(b))
    sc = S.config2(args.layers)
    if args.placement == "balanced" and 1 < G < 8:  # the bench's co-location (runtime.colocation)
        import dataclasses

        from paper_2605_18815_b200.runtime import colocated_world, colocation
        w = colocated_world(colocation(RoutingPlan.from_scenario(sc).traffic(), G))
        sc = dataclasses.replace(sc, world_src=w, world_dst=w)
    plan = RoutingPlan.from_scenario(sc)
    ex = [Executor(plan, n_gpus=G, gpu=g, device=dev(g), ctas_per_sm=args.ctas, tile_bytes=args.tile_bytes)
          for g in range(G)]
    keep = []
    for side in (A.SIDE_SRC, A.SIDE_DST):
        n = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
        for r in range(n):
            for b in range(6):
                _, nbytes, g = ex[0].buffer(side, r, b)
                if not nbytes:
                    continue
                t = torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{dev(g)}")
                keep.append(t)
                for e in ex:  # every executor sees every buffer (peer pointers for the other GPU's)
                    e.bind(side, r, b, t.data_ptr(), nbytes)
    seed = 0xD00D
    streams = []
    for g, e in enumerate(ex):
        torch.cuda.set_device(dev(g))
        e.prepare()
        e.fill(A.SIDE_SRC, seed)
        streams.append(torch.cuda.Stream(device=dev(g)))
    for g in range(G):
        torch.cuda.synchronize(dev(g))

    def step():
        evs = []
        for g, e in enumerate(ex):
            with torch.cuda.device(dev(g)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(streams[g])
                e.run(streams[g].cuda_stream)
                e1.record(streams[g])
                evs.append((e0, e1))
        for g in range(G):
            torch.cuda.synchronize(dev(g))
        return [a.elapsed_time(b) for a, b in evs]

    step()
    best = None
    for _ in range(args.reps):
        ts = step()
        best = ts if best is None or max(ts) < max(best) else best
    bad = sum(e.verify(A.SIDE_DST, seed)[0] for e in ex)
    st = [e.stats() for e in ex]
    out = {"workload": f"llama3-8b (L={args.layers}) tp8->dp2xtp4 zero1 forward, {G} GPUs from one process (peer access)",
           "placement": args.placement, "world": list(sc.world_src) if sc.world_src is not None else None,
           "ctas_per_sm": args.ctas, "tile_bytes": args.tile_bytes,
           "ms_per_gpu": [round(t, 3) for t in best],
           "remote_gb_per_gpu": [round(s.remote_bytes / 1e9, 3) for s in st],
           "local_gb_per_gpu": [round(s.local_bytes / 1e9, 3) for s in st],
           "nvlink_out_gbs_per_gpu": [round(s.remote_bytes / (t / 1e3) / 1e9, 1) for s, t in zip(st, best)],
           "verified_mismatches": int(bad)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
