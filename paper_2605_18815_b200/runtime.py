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


def local_ranks(plan: RoutingPlan, ex: Executor, side: int) -> List[int]:
    n = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
    return [r for r in range(n) if ex.buffer(side, r, A.BUF_PARAM)[2] == ex.gpu]
