"""Elastic Device Manager, B200 edition.

What the EDM builds for a new configuration, off the critical path:
  * its communicator groups (get_or_create_groups, cached per ParallelConfig;
    rank lists derived in C++ by rs_config_groups, torch process groups optional),
  * the transition itself: plan (C++ planner), executor, destination buffers,
    cudaIpc peer mappings (exchanged over a dedicated gloo control group so the side
    thread never touches the NCCL group the training loop uses) and the device
    descriptors (uploaded on a private non-blocking stream).
All of that runs on a side host thread while the old layout keeps training
(overlapped mode). switch() then only waits for the preparation and runs the
transition kernels, and reports the SPEC accounting:
    exposed = switch + max(0, init - overlapped_window)
    ratio   = overlapped / (overlapped + exposed)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading
import time
from typing import Callable, Dict, List, Optional, Tuple

from . import _capi as A
from .scenarios import Cfg, Scenario

DIMS = {"dp": 0, "tp": 1, "pp": 2, "ep": 3, "edp": 4}


def config_groups(cfg: Cfg, dim: str) -> List[List[int]]:
    """Communicator groups of cfg along `dim` (pure derivation)."""
    order = cfg.order.encode()
    c = A.Cfg_t(cfg.dp, cfg.tp, cfg.pp, cfg.ep, int(cfg.zero), order)
    out = (C.c_int * max(1, cfg.world()))()
    ng, gs = C.c_int(), C.c_int()
    A.check(A.lib().rs_config_groups(C.byref(c), DIMS[dim], out, cfg.world(), C.byref(ng), C.byref(gs)))
    return [list(out[g * gs.value:(g + 1) * gs.value]) for g in range(ng.value)]


@dataclasses.dataclass
class GroupSet:
    """Per-dimension communicator groups of one configuration."""
    cfg: Cfg
    groups: Dict[str, List[List[int]]]
    handles: Dict[str, object] = dataclasses.field(default_factory=dict)  # torch groups, if created


def overlap_accounting(init_s: float, switch_s: float, window_s: Optional[float] = None,
                       train_step_s: Optional[float] = None, mode: str = "overlapped") -> dict:
    """simulate_scale_event accounting. With a measured window the
    overlapped part is min(init, window); with a step cost, training continues for
    floor(init / step) whole steps."""
    if mode == "in-place":
        init_s = 0.0
    if mode == "blocking" or init_s == 0.0:
        overlapped = 0.0
    elif window_s is not None:
        overlapped = min(init_s, window_s)
    else:
        steps = int(init_s // train_step_s) if train_step_s else 0
        overlapped = steps * train_step_s if train_step_s else 0.0
    exposed = switch_s + max(0.0, init_s - overlapped)
    ratio = overlapped / (overlapped + exposed) if (overlapped + exposed) > 0 else None
    return {"mode": mode, "init_s": init_s, "overlapped_s": overlapped, "switch_s": switch_s, "exposed_s": exposed,
            "overlap_ratio": ratio}


class ElasticDeviceManager:
    def __init__(self, create_torch_groups: bool = False):
        self.cache: Dict[Tuple, GroupSet] = {}
        self.create_torch_groups = create_torch_groups
        self.ctrl = None
        self._thread: Optional[threading.Thread] = None
        self._result = None
        self._error: Optional[BaseException] = None
        self.creation_cost_s = 0.0

    @staticmethod
    def _key(cfg: Cfg) -> Tuple:
        return (cfg.dp, cfg.tp, cfg.pp, cfg.ep, cfg.zero, cfg.order)

    def get_or_create_groups(self, cfg: Cfg) -> GroupSet:
        """Cache hit: stored GroupSet at zero cost; miss: derive, store, return."""
        k = self._key(cfg)
        if k in self.cache:
            return self.cache[k]
        t0 = time.perf_counter()
        gs = GroupSet(cfg, {d: config_groups(cfg, d) for d in DIMS})
        if self.create_torch_groups:
            import torch.distributed as dist
            for d, groups in gs.groups.items():
                gs.handles[d] = [dist.new_group(g) for g in groups]
        self.creation_cost_s += time.perf_counter() - t0
        self.cache[k] = gs
        return gs

    def control_group(self):
        """gloo group for side-thread control traffic (IPC handle exchange)."""
        if self.ctrl is None:
            import torch.distributed as dist
            if dist.is_initialized() and dist.get_world_size() > 1:
                self.ctrl = dist.new_group(backend="gloo")
        return self.ctrl

    def prepare_async(self, build: Callable[[object], object]) -> None:
        """Run build(ctrl_group) on a side thread (the new world's groups, plan,
        executor, buffers, peer mappings); training continues meanwhile."""
        ctrl = self.control_group()
        self._result, self._error = None, None

        def work():
            t0 = time.perf_counter()
            try:
                self._result = build(ctrl)
            except BaseException as e:  # surfaced by wait()
                self._error = e
            self.init_s = time.perf_counter() - t0

        self._thread = threading.Thread(target=work, name="edm-prepare", daemon=True)
        self._thread.start()

    def ready(self) -> bool:
        return self._thread is not None and not self._thread.is_alive()

    def wait(self):
        if self._thread is not None:
            self._thread.join()
        if self._error is not None:
            raise self._error
        res, self._result = self._result, None  # the caller owns the prepared state now
        return res
