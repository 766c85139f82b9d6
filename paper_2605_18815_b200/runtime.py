"""Host orchestration for one process = one GPU (torch.distributed for plumbing).

`Transition` wires a RoutingPlan to an Executor on this process's GPU: allocate
(or bind) the state buffers of the virtual ranks placed here, exchange cudaIpc
handles of destination buffers with the other ranks (all_gather_object), build
descriptors, then run. torch is used only for device selection, streams and the
process group — all data movement is libreshard_b200.so.
"""
from __future__ import annotations

import os
from typing import List, Optional

from . import _capi as A
from .api import Executor, RoutingPlan


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class Transition:
    """One direction of a reshard on this GPU (push model)."""

    def __init__(self, plan: RoutingPlan, n_gpus: int, gpu: int, device: int, with_grads: bool = False,
                 alloc: bool = True, tile_bytes: int = 0, ctas_per_sm: int = 0):
        self.plan = plan
        self.ex = Executor(plan, n_gpus=n_gpus, gpu=gpu, device=device, with_grads=with_grads,
                           tile_bytes=tile_bytes, ctas_per_sm=ctas_per_sm)
        if alloc:
            self.ex.alloc()
        self.n_gpus = n_gpus

    def connect(self, group=None) -> None:
        """Exchange destination-buffer IPC handles (no-op on one GPU), then build tiles."""
        if self.n_gpus > 1:
            import torch.distributed as dist
            blob = self.ex.ipc_export()
            blobs: List[Optional[bytes]] = [None] * dist.get_world_size(group)
            dist.all_gather_object(blobs, blob, group=group)
            for b in blobs:
                self.ex.ipc_import(b)
        self.ex.prepare()

    def run(self, stream: int = 0) -> int:
        return self.ex.run(stream)


class StagedTransition:
    """Algorithm 1 buffered execution (ExecuteSwitch) over NCCL: the
    measured comparison for the fused push path. Per stage of the memory-aware
    schedule: PackData into one contiguous buffer per (device -> peer) channel,
    AsyncSend/AsyncRecv as one NCCL group (batch_isend_irecv), then UnpackData.
    Channels are enumerated in the global (step, device) order on every rank, so
    NCCL's per-pair FIFO matching pairs them without metadata."""

    def __init__(self, plan: RoutingPlan, ex: Executor, n_gpus: int, gpu: int, mem_avail=None, group=None):
        from .api import Schedule, xor_peer
        self.plan, self.ex, self.n_gpus, self.gpu, self.group = plan, ex, n_gpus, gpu, group
        n = plan.summary.num_participants
        self.sched = Schedule(plan, mem_avail or [1 << 62] * n, promote=False)
        ex.prepare_staged()
        self.phys = list(range(n))  # device index -> phys (identity world maps in the benches)
        span = (max(self.phys) + 1 + n_gpus - 1) // n_gpus
        self.gpu_of = [p // span for p in self.phys]
        self.plan_stages = []
        for k, (steps, _) in enumerate(self.sched.stages()):
            chans = []
            for s in steps:
                for i in range(n):
                    p = xor_peer(i, s, n)
                    if p < 0 or self.gpu_of[i] == self.gpu_of[p]:
                        continue
                    nbytes = ex.channel_bytes(self.phys[i], self.phys[p])
                    if nbytes:
                        chans.append((self.phys[i], self.phys[p], self.gpu_of[i], self.gpu_of[p], nbytes))
            self.plan_stages.append(chans)
        # channels outside the plan's transfer list (the scalar broadcast, routing.hpp:341-353)
        # may fall in steps the schedule elided: one final phase in the same global order
        done = {(c[0], c[1]) for st in self.plan_stages for c in st}
        rest = []
        steps_all = range(1, 1 << max(1, (n - 1).bit_length()))
        for s in steps_all:
            for i in range(n):
                p = xor_peer(i, s, n)
                if p < 0 or self.gpu_of[i] == self.gpu_of[p] or (self.phys[i], self.phys[p]) in done:
                    continue
                nbytes = ex.channel_bytes(self.phys[i], self.phys[p])
                if nbytes:
                    rest.append((self.phys[i], self.phys[p], self.gpu_of[i], self.gpu_of[p], nbytes))
        if rest:
            self.plan_stages.append(rest)

    def run(self, stream: int = 0) -> None:
        import torch
        import torch.distributed as dist
        self.ex.run(stream)  # same-GPU moves, fused
        for chans in self.plan_stages:
            ops, unpacks, keep = [], [], []
            for src, dst, gs, gd, nbytes in chans:
                if gs == self.gpu:
                    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                    self.ex.pack(src, dst, buf.data_ptr(), stream)
                    ops.append(dist.P2POp(dist.isend, buf, gd, group=self.group))
                    keep.append(buf)
                elif gd == self.gpu:
                    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                    ops.append(dist.P2POp(dist.irecv, buf, gs, group=self.group))
                    unpacks.append((src, dst, buf))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            for src, dst, buf in unpacks:
                self.ex.unpack(src, dst, buf.data_ptr(), stream)


def local_ranks(plan: RoutingPlan, ex: Executor, side: int) -> List[int]:
    n = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
    return [r for r in range(n) if ex.buffer(side, r, A.BUF_PARAM)[2] == ex.gpu]
