"""Elastic Device Manager, B200 edition. The core
(group cache, side thread, accounting) is native: csrc/edm.cpp behind rs_edm_*.

What the EDM builds for a new configuration, off the critical path:
  * its communicator groups (get_or_create_groups, cached per ParallelConfig;
    rank lists derived in C++ by rs_config_groups) and its NCCL communicators, built
    natively and non-blocking (create_nccl_comms: world ncclCommInitRankConfig with
    blocking = 0, one ncclCommSplit per dimension; torch process groups optional),
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
        ("rs_nccl_unique_id", [vp, C.c_size_t]),
        ("rs_nccl_version", [C.c_char_p, C.c_size_t]),
        ("rs_edm_comm_create", [vp, P(A.Cfg_t), vp, C.c_int, C.c_int, C.c_int, P(C.c_int), P(C.c_int),
                                P(C.c_double), P(C.c_double)]),
        ("rs_edm_comm_get", [vp, P(A.Cfg_t), C.c_int, P(vp)]),
        ("rs_edm_comm_check", [vp, P(A.Cfg_t), C.c_int, vp, P(C.c_float)]),
        ("rs_edm_comm_destroy", [vp, P(A.Cfg_t)]),
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


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId of the libnccl in this process (128 bytes)."""
    buf = C.create_string_buffer(128)
    A.check(_bind(A.lib()).rs_nccl_unique_id(buf, 128))
    return buf.raw


def nccl_version() -> str:
    buf = C.create_string_buffer(32)
    A.check(_bind(A.lib()).rs_nccl_version(buf, 32))
    return buf.value.decode()


def _cfg_t(cfg: Cfg):
    return A.Cfg_t(cfg.dp, cfg.tp, cfg.pp, cfg.ep, int(cfg.zero), cfg.order.encode())


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

    def close(self) -> None:
        """Join the side thread and destroy the cached NCCL communicators now (before the
        process group and the CUDA context go away)."""
        if getattr(self, "h", None) and A is not None and A._lib is not None:
            A.lib().rs_edm_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

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

    def create_nccl_comms(self, cfg: Cfg, rank: int, nranks: int, device: int, member_rank: int, group=None) -> dict:
        """The new world's NCCL communicators, built natively and non-blocking:
        rank 0 draws a unique id, broadcast over `group` (the gloo control group: the side
        thread never touches the training loop's NCCL group); then the world communicator
        and one split per dimension, polled to completion on this (side) thread. Process
        `rank` joins, per dimension, the group of virtual rank `member_rank` of `cfg` (its
        first hosted rank: with one rank per GPU these are exactly cfg's groups). Cached per
        configuration; returns {"cache_hit", "init_s", "split_s"}."""
        import torch.distributed as dist
        uid = [nccl_unique_id() if rank == 0 else None]
        if nranks > 1:
            dist.broadcast_object_list(uid, src=0 if group is None else dist.get_global_rank(group, 0), group=group)
        colors = (C.c_int * 5)()
        for d, i in DIMS.items():
            groups = self.get_or_create_groups(cfg).groups[d]
            colors[i] = next(g for g, members in enumerate(groups) if member_rank in members)
        hit, t_init, t_split = C.c_int(), C.c_double(), C.c_double()
        c = _cfg_t(cfg)
        A.check(self._lib.rs_edm_comm_create(self.h, C.byref(c), uid[0], nranks, rank, device, colors, C.byref(hit),
                                             C.byref(t_init), C.byref(t_split)))
        return {"cache_hit": bool(hit.value), "init_s": t_init.value, "split_s": t_split.value}

    def nccl_comm(self, cfg: Cfg, dim: Optional[str] = None) -> int:
        """The ncclComm_t (as an address) of `cfg`'s world (dim None) or dimension, or 0."""
        p = C.c_void_p()
        c = _cfg_t(cfg)
        A.check(self._lib.rs_edm_comm_get(self.h, C.byref(c), -1 if dim is None else DIMS[dim], C.byref(p)))
        return p.value or 0

    def check_nccl_comm(self, cfg: Cfg, dim: Optional[str] = None, stream: int = 0) -> float:
        """All-reduce (sum) of 1.0 over that communicator: returns its size."""
        out = C.c_float()
        c = _cfg_t(cfg)
        A.check(self._lib.rs_edm_comm_check(self.h, C.byref(c), -1 if dim is None else DIMS[dim], C.c_void_p(stream),
                                            C.byref(out)))
        return out.value

    def destroy_nccl_comms(self, cfg: Cfg) -> None:
        c = _cfg_t(cfg)
        A.check(self._lib.rs_edm_comm_destroy(self.h, C.byref(c)))

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
