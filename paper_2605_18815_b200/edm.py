"""Elastic Device Manager, B200 edition. The core
(group cache, side thread, accounting) is native: csrc/edm.cpp behind rs_edm_*.

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
import time
from typing import Callable, Dict, List, Optional, Tuple

from . import _capi as A
from .scenarios import Cfg

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


class _Accounting(C.Structure):
    _fields_ = [("init_s", C.c_double), ("overlapped_s", C.c_double), ("switch_s", C.c_double),
                ("exposed_s", C.c_double), ("ratio", C.c_double)]


_BUILD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
_MODES = {"blocking": 0, "overlapped": 1, "in-place": 2}


def _bind(L):
    if getattr(L, "_edm_bound", False):
        return L
    vp, P = C.c_void_p, C.POINTER
    for name, args in (
        ("rs_edm_create", [P(vp)]),
        ("rs_edm_groups", [vp, P(A.Cfg_t), C.c_int, P(C.c_int), C.c_int, P(C.c_int), P(C.c_int), P(C.c_int)]),
        ("rs_edm_cache_stats", [vp, P(C.c_int64), P(C.c_int64), P(C.c_double)]),
        ("rs_edm_prepare_async", [vp, _BUILD_FN, vp]),
        ("rs_edm_ready", [vp, P(C.c_int)]),
        ("rs_edm_wait", [vp, P(C.c_double), P(C.c_int)]),
        ("rs_edm_accounting", [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, P(_Accounting)]),
    ):
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.rs_edm_destroy.argtypes = [vp]
    L.rs_edm_destroy.restype = None
    L._edm_bound = True
    return L


def overlap_accounting(init_s: float, switch_s: float, window_s: Optional[float] = None,
                       train_step_s: Optional[float] = None, mode: str = "overlapped") -> dict:
    """simulate_scale_event accounting, computed by the native EDM
    (rs_edm_accounting). With a measured window the overlapped part is min(init, window);
    with a step cost, training continues for floor(init / step) whole steps."""
    out = _Accounting()
    A.check(_bind(A.lib()).rs_edm_accounting(init_s, switch_s, -1.0 if window_s is None else window_s,
                                             train_step_s or 0.0, _MODES[mode], C.byref(out)))
    return {"mode": mode, "init_s": out.init_s, "overlapped_s": out.overlapped_s, "switch_s": out.switch_s,
            "exposed_s": out.exposed_s, "overlap_ratio": None if out.ratio < 0 else out.ratio}


class ElasticDeviceManager:
    """Python face of the native EDM (rs_edm_*): the group cache and the side thread live
    in C++; this class adds the optional torch process groups and carries the Python
    build callable's result / exception across the thread."""

    def __init__(self, create_torch_groups: bool = False):
        self._lib = _bind(A.lib())
        h = C.c_void_p()
        A.check(self._lib.rs_edm_create(C.byref(h)))
        self.h = h.value
        self.cache: Dict[Tuple, GroupSet] = {}
        self.create_torch_groups = create_torch_groups
        self.ctrl = None
        self._cb = None
        self._result = None
        self._error: Optional[BaseException] = None
        self._torch_cost_s = 0.0
        self.init_s = 0.0

    def __del__(self):
        if getattr(self, "h", None) and A is not None and A._lib is not None:
            A.lib().rs_edm_destroy(self.h)
            self.h = None

    @staticmethod
    def _key(cfg: Cfg) -> Tuple:
        return (cfg.dp, cfg.tp, cfg.pp, cfg.ep, cfg.zero, cfg.order)

    @property
    def creation_cost_s(self) -> float:
        hits, misses, cost = C.c_int64(), C.c_int64(), C.c_double()
        A.check(self._lib.rs_edm_cache_stats(self.h, C.byref(hits), C.byref(misses), C.byref(cost)))
        return cost.value + self._torch_cost_s

    def get_or_create_groups(self, cfg: Cfg) -> GroupSet:
        """Cache hit: stored GroupSet at zero cost; miss: derive (native cache), store, return."""
        k = self._key(cfg)
        if k in self.cache:
            for d in DIMS:  # keeps the native hit counters truthful
                self._groups(cfg, d)
            return self.cache[k]
        gs = GroupSet(cfg, {d: self._groups(cfg, d) for d in DIMS})
        if self.create_torch_groups:
            import torch.distributed as dist
            t0 = time.perf_counter()
            for d, groups in gs.groups.items():
                gs.handles[d] = [dist.new_group(g) for g in groups]
            self._torch_cost_s += time.perf_counter() - t0
        self.cache[k] = gs
        return gs

    def _groups(self, cfg: Cfg, dim: str) -> List[List[int]]:
        order = cfg.order.encode()
        c = A.Cfg_t(cfg.dp, cfg.tp, cfg.pp, cfg.ep, int(cfg.zero), order)
        out = (C.c_int * max(1, cfg.world()))()
        ng, gs, hit = C.c_int(), C.c_int(), C.c_int()
        A.check(self._lib.rs_edm_groups(self.h, C.byref(c), DIMS[dim], out, cfg.world(), C.byref(ng), C.byref(gs),
                                        C.byref(hit)))
        return [list(out[g * gs.value:(g + 1) * gs.value]) for g in range(ng.value)]

    def control_group(self):
        """gloo group for side-thread control traffic (IPC handle exchange)."""
        if self.ctrl is None:
            import torch.distributed as dist
            if dist.is_initialized() and dist.get_world_size() > 1:
                self.ctrl = dist.new_group(backend="gloo")
        return self.ctrl

    def prepare_async(self, build: Callable[[object], object]) -> None:
        """Run build(ctrl_group) on the native side thread (the new world's groups, plan,
        executor, buffers, peer mappings); training continues meanwhile."""
        ctrl = self.control_group()
        self._result, self._error = None, None

        def work(_arg):
            try:
                self._result = build(ctrl)
                return 0
            except BaseException as e:  # surfaced by wait()
                self._error = e
                return 1

        self._cb = _BUILD_FN(work)  # kept alive until wait()
        A.check(self._lib.rs_edm_prepare_async(self.h, self._cb, None))

    def ready(self) -> bool:
        r = C.c_int()
        A.check(self._lib.rs_edm_ready(self.h, C.byref(r)))
        return bool(r.value)

    def wait(self):
        init, rc = C.c_double(), C.c_int()
        A.check(self._lib.rs_edm_wait(self.h, C.byref(init), C.byref(rc)))
        self.init_s = init.value
        self._cb = None
        if self._error is not None:
            err, self._error = self._error, None
            raise err
        res, self._result = self._result, None  # the caller owns the prepared state now
        return res
