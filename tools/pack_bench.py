"""Pack / unpack kernels of the staged (Algorithm 1 buffered) path on ONE GPU, so ncu can
profile them: both halves of a 2-GPU placement live on device 0 — the executor of "GPU 0"
packs every channel it sends to "GPU 1" into contiguous buffers, the executor of "GPU 1"
unpacks them. HBM traffic per channel = 2 x its bytes (gather read + contiguous write, or
contiguous read + scatter write).

    python tools/pack_bench.py [--layers 16] [--reps 5]

Prints one JSON line: pack / unpack GB/s of HBM traffic against the measured copy peak,
bit-exact check of the unpacked destinations.
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
from paper_2605_18815_b200.api import Executor, RoutingPlan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    plan = RoutingPlan.from_scenario(S.config2(args.layers))
    ex = [Executor(plan, n_gpus=2, gpu=g, device=0) for g in range(2)]
    keep = []
    for side in (A.SIDE_SRC, A.SIDE_DST):
        n = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
        for r in range(n):
            for b in range(6):
                _, nbytes, g = ex[0].buffer(side, r, b)
                if not nbytes:
                    continue
                t = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
                keep.append(t)
                for e in ex:  # both halves see every buffer (all on device 0)
                    e.bind(side, r, b, t.data_ptr(), nbytes)
    for e in ex:
        e.prepare_staged()
    seed = 0xFACADE
    ex[0].fill(A.SIDE_SRC, seed)
    ex[1].fill(A.SIDE_SRC, seed)
    n = plan.summary.num_participants
    per = (n + 1) // 2  # contiguous-block placement (executor.cu gpu_of_phys)

    def gpu_of(p):
        return p // per

    chans = [(p, q) for p in range(n) for q in range(n)
             if ex[0].channel_bytes(p, q) and gpu_of(p) == 0 and gpu_of(q) == 1]
    bufs = {c: torch.empty(ex[0].channel_bytes(*c), dtype=torch.uint8, device="cuda") for c in chans}
    total = sum(b.numel() for b in bufs.values())
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def timed(fn):
        best = 1e30
        for _ in range(args.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def pack():
        for c, b in bufs.items():
            ex[0].pack(c[0], c[1], b.data_ptr(), sp)

    def unpack():
        for c, b in bufs.items():
            ex[1].unpack(c[0], c[1], b.data_ptr(), sp)

    pack_ms = timed(pack)
    unpack_ms = timed(unpack)
    # the rest of the transition: GPU 0's and GPU 1's own same-GPU moves, then the other
    # direction's channels, so every destination is complete for the check
    ex[0].run(sp)
    ex[1].run(sp)
    back = [(p, q) for p in range(n) for q in range(n)
            if ex[0].channel_bytes(p, q) and gpu_of(p) == 1 and gpu_of(q) == 0]
    for c in back:
        b = torch.empty(ex[0].channel_bytes(*c), dtype=torch.uint8, device="cuda")
        ex[1].pack(c[0], c[1], b.data_ptr(), sp)
        ex[0].unpack(c[0], c[1], b.data_ptr(), sp)
    torch.cuda.synchronize()
    bad = ex[0].verify(A.SIDE_DST, seed)[0] + ex[1].verify(A.SIDE_DST, seed)[0]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        peak = 6558.0
    pk, uk = 2 * total / (pack_ms / 1e3) / 1e9, 2 * total / (unpack_ms / 1e3) / 1e9
    print(json.dumps({"workload": f"llama3-8b (L={args.layers}) tp8->dp2xtp4 zero1, channels GPU0->GPU1 of a 2-GPU "
                                  "placement, both halves on one B200",
                      "channels": len(chans), "channel_bytes": total,
                      "pack_ms": round(pack_ms, 3), "pack_hbm_gbs": round(pk, 1), "pack_frac": round(pk / peak, 4),
                      "unpack_ms": round(unpack_ms, 3), "unpack_hbm_gbs": round(uk, 1), "unpack_frac": round(uk / peak, 4),
                      "peak_hbm_gbs": peak, "peak_source": "MEASURED_PEAKS.json (copy, read+write)",
                      "verified_mismatches": int(bad)}), flush=True)


if __name__ == "__main__":
    main()
