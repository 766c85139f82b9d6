"""Promoted Scatter / Gather executed as primitives (optimize_primitives, SPEC.md:282-290;
PAPER.md:719-740), 4 rank processes (torchrun; ranks may share a GPU):

  forward  TP1 -> TP4: every sharded tensor leaves device 0 as a Scatter (root pushes)
  way back TP4 -> TP1: every sharded tensor returns as a Gather, which the root PULLS over
                       NVLink from the three sources' mapped buffers

Both directions bit-exact against canon on every rank; the root's executor reports
exactly the schedule's Scatter / Gather bytes; the schedule dump shows the promotion.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tests/mgpu_collectives_check.py
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import RoutingPlan, Schedule  # noqa: E402
from paper_2605_18815_b200.runtime import Transition, device_barrier, init_dist  # noqa: E402


def model(scale: int) -> S.Model:
    h = 256 * scale
    return S.Model("coll", [S.Tensor("emb", (16 * h, h), 0, tp=0), S.Tensor("l0.norm", (h,), 0),
                            S.Tensor("l0.w1", (4 * h, h), 0, tp=0), S.Tensor("l0.w2", (h, 4 * h), 0, tp=1),
                            S.Tensor("head", (8 * h, h), 0, tp=0)])


def collective_bytes(plan, kind):
    sch = Schedule(plan, [1 << 60] * plan.summary.num_participants, promote=True)
    lines = [l for l in sch.dump().splitlines() if l.startswith(f"collective {kind} ")]
    return sum(int(l.rsplit("bytes=", 1)[1]) for l in lines), len(lines)


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    rank, world, local, shared = init_dist()
    assert world == 4, "run with 4 rank processes"
    fwd_sc = S.Scenario(model(scale), S.Cfg(dp=1), S.Cfg(tp=4), world_src=[0], world_dst=[0, 1, 2, 3],
                        name="coll.tp1-to-tp4")
    ab = RoutingPlan.from_scenario(fwd_sc)
    ba = RoutingPlan.from_scenario(fwd_sc.reversed())
    scatter_b, n_scatter = collective_bytes(ab, "scatter")
    gather_b, n_gather = collective_bytes(ba, "gather")
    fwd = Transition(ab, world, rank, local, alloc=False)
    bwd = Transition(ba, world, rank, local, alloc=False)
    keep = []
    for side in (A.SIDE_SRC, A.SIDE_DST):
        nr = ab.summary.src_world if side == A.SIDE_SRC else ab.summary.dst_world
        for r in range(nr):
            for b in range(6):
                _, n, g = fwd.ex.buffer(side, r, b)
                if n and g == rank:
                    t = torch.zeros(n, dtype=torch.uint8, device="cuda")
                    keep.append(t)
                    fwd.ex.bind(side, r, b, t.data_ptr(), n)
                    bwd.ex.bind(1 - side, r, b, t.data_ptr(), n)
    for tr in (fwd, bwd):
        tr.ex.set_collectives(True)  # before the ipc exchange: the Gather root maps the sources
        tr.connect()
    dbar = device_barrier(rank, world, local)
    sp = torch.cuda.current_stream().cuda_stream
    seed = 0xC011
    fwd.ex.fill(A.SIDE_SRC, seed)
    torch.cuda.synchronize()
    dist.barrier()
    fails = 0
    for rep in range(2):
        fwd.run(sp)
        dbar(sp)
        torch.cuda.synchronize()
        bad_f = fwd.ex.verify(A.SIDE_DST, seed)[0]
        bwd.run(sp)
        dbar(sp)
        torch.cuda.synchronize()
        bad_b = bwd.ex.verify(A.SIDE_DST, seed)[0]
        fails += int(bad_f != 0) + int(bad_b != 0)
    sf, sb = fwd.ex.stats(), bwd.ex.stats()
    print(f"[rank {rank}] scatter: {n_scatter} collectives {scatter_b} B, pushed as root {sf.scatter_bytes} B; "
          f"gather: {n_gather} collectives {gather_b} B, pulled as root {sb.gather_bytes} B; mismatches {fails}",
          flush=True)
    if rank == 0:
        fails += int(n_scatter == 0 or sf.scatter_bytes != scatter_b)
        fails += int(n_gather == 0 or sb.gather_bytes != gather_b)
    else:
        fails += int(sf.scatter_bytes != 0 or sb.gather_bytes != 0)
    if dbar.timed_out():
        fails += 1
    t = torch.tensor([fails], device="cpu" if shared else "cuda")
    dist.all_reduce(t)
    dist.destroy_process_group()
    if rank == 0:
        print("COLL_OK" if t.item() == 0 else f"COLL_FAIL {t.item()}", flush=True)
    sys.exit(0 if t.item() == 0 else 1)


if __name__ == "__main__":
    main()
