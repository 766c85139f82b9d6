"""Multi-GPU correctness (run under torchrun, one process per GPU, NCCL plumbing):
push-model transition over cudaIpc-mapped peer HBM, bit-exact on every GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_check.py [layers]
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import RoutingPlan  # noqa: E402
from paper_2605_18815_b200.runtime import Transition, init_dist  # noqa: E402


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    staged = "--staged" in sys.argv
    vmm = "--vmm" in sys.argv  # shareable VMM buffers mapped by descriptor instead of cudaIpc
    dedup = "--dedup" in sys.argv  # replica dedup: one NVLink crossing per destination GPU
    early = "--dedup-early" in sys.argv  # ... with the copies overlapping the non-replica pushes
    # --random K: only K random toy MoE models (the generator of tests/test_spec_kats.py)
    n_random = int(sys.argv[sys.argv.index("--random") + 1]) if "--random" in sys.argv else 0
    dedup = dedup or early
    # --oracle: every local buffer compared byte for byte with the oracle's CPU executor
    # (forward destinations, and the source layout the way back rebuilds)
    check_oracle = "--oracle" in sys.argv
    # more ranks than GPUs (e.g. 8 ranks on a 4-GPU box, or 2/4 on a 1-GPU box) exercise
    # the N>1 placement: ranks sharing a device still exchange cudaIpc handles / VMM
    # descriptors and push through them (gloo plumbing, runtime.init_dist)
    rank, world, local, shared = init_dist()
    seed = 0xBEEF
    failures = 0
    ctrl = dist.new_group(backend="gloo") if early else None
    side = torch.cuda.Stream() if early else None
    scenarios = [S.config2(layers), S.config4(1), S.config3(2)[0], S.config3(2)[1]]
    scenarios += [sc for sc in S.edge_scenarios() if sc.grads == "drop"]  # ragged, identity, join/leave
    if n_random:
        import random
        scenarios = []
        for k in range(n_random):
            rng = random.Random(1000 + k)
            m = S.toy_model(rng, max_layers=4, max_per_layer=4, experts=4)
            src = S.random_cfg(rng, m, max_world=8)
            dst = S.random_cfg(rng, m, max_world=8, zero=src.zero)
            scenarios.append(S.Scenario(m, src, dst, world_src=list(range(src.world())),
                                        world_dst=list(range(dst.world())), name=f"random-moe-{k}"))
    if "--colocate" in sys.argv:
        # bench.py's balanced co-location: devices grouped onto GPUs from the plan's traffic
        # matrix, applied by relabelling identity world maps (same-size worlds only)
        import dataclasses

        from paper_2605_18815_b200.runtime import colocated_world, colocation
        out = []
        for sc in scenarios:
            identity = sc.world_src in (None, list(range(sc.src.world()))) and \
                sc.world_dst in (None, list(range(sc.dst.world())))
            if identity and sc.src.world() == sc.dst.world() and 1 < world < sc.src.world():
                w = colocated_world(colocation(RoutingPlan.from_scenario(sc, allow_oversourced=True).traffic(), world))
                sc = dataclasses.replace(sc, world_src=w, world_dst=w, name=sc.name + ".colocated")
            out.append(sc)
        scenarios = out
        if rank == 0:
            print(f"COLOCATED {sum(sc.name.endswith('.colocated') for sc in scenarios)}", flush=True)
    for sc in scenarios:
        ab = RoutingPlan.from_scenario(sc, allow_oversourced=True)
        ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
        fwd = Transition(ab, world, rank, local, alloc=False)
        bwd = Transition(ba, world, rank, local, alloc=False)
        keep = []
        mine = {}  # (side of the forward plan, rank, buf) -> this rank's tensor
        if vmm:
            from paper_2605_18815_b200.runtime import share_buffers
            tag = f"{os.environ.get('MASTER_PORT', '0')}-{sc.name}"
            keep.append(share_buffers(fwd, rank, world, local, tag=tag + "-f"))
            keep.append(share_buffers(bwd, rank, world, local, tag=tag + "-b",
                                      adopt={(1 - k[0], k[1], k[2]): v for k, v in keep[0].items()
                                             if k[0] in (A.SIDE_SRC, A.SIDE_DST)}))
        for side_ab in ((A.SIDE_SRC, A.SIDE_DST) if not vmm else ()):
            nr = ab.summary.src_world if side_ab == A.SIDE_SRC else ab.summary.dst_world
            for r in range(nr):
                for b in range(6):
                    _, n, g = fwd.ex.buffer(side_ab, r, b)
                    if n and g == rank:
                        t = torch.zeros(n, dtype=torch.uint8, device="cuda")
                        keep.append(t)
                        mine[(side_ab, r, b)] = t
                        fwd.ex.bind(side_ab, r, b, t.data_ptr(), n)
                        bwd.ex.bind(1 - side_ab, r, b, t.data_ptr(), n)
        if dedup:
            fwd.ex.set_replica_dedup(True, early=early)
            bwd.ex.set_replica_dedup(True, early=early)
        if vmm:
            fwd.ex.prepare()
            bwd.ex.prepare()
            fwd_run, bwd_run = fwd.run, bwd.run
        elif staged:
            from paper_2605_18815_b200.runtime import StagedTransition
            mode = sys.argv[sys.argv.index("--mode") + 1] if "--mode" in sys.argv else "async"
            fwd_run = StagedTransition(ab, fwd.ex, world, rank, mode=mode).run
            bwd_run = StagedTransition(ba, bwd.ex, world, rank, mode=mode).run
        else:
            fwd.connect()
            bwd.connect()
            fwd_run, bwd_run = fwd.run, bwd.run
        if early:
            from paper_2605_18815_b200.runtime import run_dedup_early

            def with_dup(tr):
                def run():
                    run_dedup_early(tr.ex, torch.cuda.current_stream(), side, ctrl)
                return run
            fwd_run, bwd_run = with_dup(fwd), with_dup(bwd)
        elif dedup:
            def with_dup(tr):
                def run():
                    tr.run()
                    torch.cuda.synchronize()
                    dist.barrier()
                    tr.ex.run_dup()
                return run
            fwd_run, bwd_run = with_dup(fwd), with_dup(bwd)
        fwd.ex.fill(A.SIDE_SRC, seed)
        torch.cuda.synchronize()
        dist.barrier()
        fwd_run()
        torch.cuda.synchronize()
        dist.barrier()
        bad_b = fwd.ex.verify(A.SIDE_DST, seed)[0]
        ora = 0
        # the oracle holds every rank's old and new state in host memory, in every rank
        # process: only scenarios whose state is small (a few GB) are compared byte for byte
        small = 2 * (ab.bytes_moved() + ab.bytes_retained()) < 8e9
        oracle_now = check_oracle and mine and small
        if oracle_now:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import pyoracle as O
            osc = O.OScenario(sc.text())
            osrc = O.OState(osc, 0)
            osrc.load(seed)
            odst = O.OState(osc, 1)
            O.execute(O.OPlan(osc, True), osrc, odst, nthreads=4)
            for (side, r, b), t in mine.items():
                if side == A.SIDE_DST and t.cpu().numpy().tobytes() != odst.buffer(r, b):
                    ora += 1
        bwd_run()
        torch.cuda.synchronize()
        dist.barrier()
        bad_a = bwd.ex.verify(A.SIDE_DST, seed)[0]
        if oracle_now:
            for (side, r, b), t in mine.items():
                if side == A.SIDE_SRC and t.cpu().numpy().tobytes() != osrc.buffer(r, b):
                    ora += 1
            bad_b += ora
        st = fwd.ex.stats()
        print(f"[rank {rank}] {'oracle-checked ' if oracle_now else ''}{'staged' if staged else 'vmm' if vmm else 'fused'}{'+dedup' if dedup else ''}{'(early)' if early else ''} {sc.name}: dst mismatches {bad_b}, round-trip mismatches {bad_a}, "
              f"local {st.local_bytes/1e9:.2f} GB, remote {st.remote_bytes/1e9:.2f} GB", flush=True)
        failures += int(bad_a != 0) + int(bad_b != 0)
        del fwd, bwd, keep
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([failures], device="cpu" if shared else "cuda")
    dist.all_reduce(t)
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_OK" if t.item() == 0 else f"MGPU_FAIL {t.item()}", flush=True)
    sys.exit(0 if t.item() == 0 else 1)


if __name__ == "__main__":
    main()
