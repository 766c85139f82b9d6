"""Multi-GPU memory-aware arena (run under torchrun): old and new layouts of every GPU's
virtual ranks in VMM with eager-free aliasing, shared with the peers through POSIX
descriptors, memory-aware stages with a global barrier between them. Round trips must
stay bit-exact and each GPU must use less physical HBM than old + new.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_arena_check.py [layers]
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Arena, RoutingPlan  # noqa: E402
from paper_2605_18815_b200.runtime import (Transition, device_barrier, exchange_arena, global_stage_cuts, init_dist,  # noqa: E402
                                           run_stages, shared_arena)


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rank, world, local, shared = init_dist()
    seed = 0xA7E4
    fails = 0
    dev_barrier = device_barrier(rank, world, local)
    # groups 0: one group per stage (most aliasing); 2: the stage order in two halves
    # groups < 0: the schedule ladder under a per-GPU cap (config 5 depth-scaled: old + new
    # state does not fit, the arena has to rebuild it in layer bands; the analogue of the
    # full 70B model on 8 GPUs under 180 GB)
    # ranks sharing one device (a 1-GPU box): config 5 at L=4, caps summing to < 150 GB
    c5cap = ({2: 62e9, 4: 36e9} if shared else {2: 86e9, 4: 45e9}).get(world)
    c5layers = 4 if shared else 8
    cases = [(S.config2(layers), 0), (S.config2(layers), 2), (S.config3(2)[0], 0)]
    if c5cap:
        cases.append((S.config5(c5layers), "cap"))
        cases.append((S.config5(c5layers), "rounds"))
    for sc, groups in cases:
        ab = RoutingPlan.from_scenario(sc, allow_oversourced=True)
        ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
        tag = f"{os.environ.get('MASTER_PORT', '0')}-{sc.name}-{groups}"
        if groups == "cap":
            arena, cuts = shared_arena(ab, ba, rank, world, local, cap_bytes=int(c5cap), tag=tag, chunk_bytes=64 << 20)
        elif groups == "rounds":  # one unit per GPU per group, 4 layer bands
            arena = Arena.multi(ab, ba, world, rank, local, chunk_bytes=64 << 20, groups=-1, bands=4)
            exchange_arena(arena, rank, world, tag=tag)
            cuts = global_stage_cuts(arena, world)
        else:
            arena = Arena.multi(ab, ba, world, rank, local, chunk_bytes=64 << 20, groups=groups or 64)
            exchange_arena(arena, rank, world, tag=tag)
            cuts = global_stage_cuts(arena, world)
        fwd = Transition(ab, world, rank, local, alloc=False)
        bwd = Transition(ba, world, rank, local, alloc=False)
        arena.bind(fwd.ex, bwd.ex, cuts)
        fwd.ex.prepare()
        bwd.ex.prepare()
        fwd.ex.fill(A.SIDE_SRC, seed)
        torch.cuda.synchronize()
        dist.barrier()
        bad = []
        import time
        ms = []
        # stage boundaries as host barriers, then as the device-side SynchronizeAll
        for dbar in (None, None, dev_barrier, dev_barrier):
            sp = torch.cuda.current_stream().cuda_stream
            t0 = time.perf_counter()
            run_stages(fwd.ex, sp, world, barrier=dbar)
            torch.cuda.synchronize()
            dist.barrier()
            ms.append(round(1e3 * (time.perf_counter() - t0), 1))
            bad.append(fwd.ex.verify(A.SIDE_DST, seed)[0])
            run_stages(bwd.ex, sp, world, barrier=dbar)
            torch.cuda.synchronize()
            dist.barrier()
            bad.append(bwd.ex.verify(A.SIDE_DST, seed)[0])
        if dev_barrier.timed_out():
            bad.append(-1)
        st = arena.stats()
        print(f"[rank {rank}] {sc.name} groups={groups} bands={st.bands}: stages {fwd.ex.num_stages()}/{bwd.ex.num_stages()}, mismatches {bad}, forward {ms} ms (host, host, device, device barriers), physical {st.physical_bytes/1e9:.2f} GB "
              f"(old {st.a_bytes/1e9:.2f} + new {st.b_bytes/1e9:.2f}, aliased {st.aliased_bytes/1e9:.2f})", flush=True)
        fails += sum(1 for b in bad if b)
        del fwd, bwd, arena
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([fails], device="cpu" if shared else "cuda")
    dist.all_reduce(t)
    dist.destroy_process_group()
    if rank == 0:
        print("ARENA_OK" if t.item() == 0 else f"ARENA_FAIL {t.item()}", flush=True)
    sys.exit(0 if t.item() == 0 else 1)


if __name__ == "__main__":
    main()
