"""Python mirror of the reference's resharding interface, over the C ABI.

Same names and argument meaning as namespace reshard (routing.hpp / project.hpp):
a ModelSpec + two ParallelConfigs (+ WorldMap, Topology, PlanOptions) give a
RoutingPlan with bytes_moved() / bytes_retained() / transfers / dump; errors raise
ConfigError where the reference throws ConfigError. The Executor runs a plan on
B200s (push over NVLink); it has no CPU path and raises CudaError without a GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

from . import _capi as A
from ._capi import ConfigError, CudaError, ReshardError, VerificationError  # noqa: F401
from .scenarios import Cfg, Model, Scenario


def _cfg_t(c: Cfg, keep: list) -> A.Cfg_t:
    order = c.order.encode()
    keep.append(order)
    return A.Cfg_t(c.dp, c.tp, c.pp, c.ep, int(c.zero), order)


def _alive() -> bool:
    """The library is still loaded (destructors may run during interpreter shutdown)."""
    return A is not None and A._lib is not None


class RoutingPlan:
    """plan_parameters + plan_optimizer + plan_scalars + resolve_peers (routing.hpp:231-396)."""

    def __init__(self, handle: int, model: Optional["ModelSpace"] = None):
        self.h = handle
        self._model = model  # keeps the model alive (the plan references it)
        s = A.PlanSummary_t()
        A.check(A.lib().rs_plan_summary(self.h, C.byref(s)))
        self.summary = s

    @classmethod
    def from_scenario(cls, sc, allow_oversourced: bool = False) -> "RoutingPlan":
        text = sc.text() if isinstance(sc, Scenario) else sc
        h = C.c_void_p()
        A.check(A.lib().rs_plan_from_scenario(text.encode(), int(allow_oversourced), C.byref(h)))
        return cls(h.value)

    def __del__(self):
        if getattr(self, "h", None) and _alive():
            A.lib().rs_plan_destroy(self.h)
            self.h = None

    def bytes_moved(self) -> int:
        return self.summary.bytes_moved

    def bytes_retained(self) -> int:
        return self.summary.bytes_retained

    def num_transfers(self) -> int:
        return self.summary.num_transfers

    def dump(self, device: int = -1) -> str:
        """format_transfer lines in canonical order; device>=0 runs the GPU planner."""
        p, n = C.c_void_p(), C.c_size_t()
        A.check(A.lib().rs_plan_dump(self.h, device, C.byref(p), C.byref(n)))
        return A.take_string(p, n)

    def dump_rows_host(self) -> str:
        p, n = C.c_void_p(), C.c_size_t()
        A.check(A.lib().rs_plan_dump_rows_host(self.h, C.byref(p), C.byref(n)))
        return A.take_string(p, n)

    def regions(self, side: int) -> str:
        p, n = C.c_void_p(), C.c_size_t()
        A.check(A.lib().rs_plan_regions(self.h, side, C.byref(p), C.byref(n)))
        return A.take_string(p, n)

    def placement(self, n_gpus: int, gpu: int) -> A.PlacementStats_t:
        """Bytes GPU `gpu` copies locally / pushes to peers / receives (host-side)."""
        s = A.PlacementStats_t()
        A.check(A.lib().rs_plan_placement(self.h, n_gpus, gpu, C.byref(s)))
        return s

    def traffic(self) -> List[List[int]]:
        """Copy bytes between physical devices, m[s][d] (rs_plan_traffic): off-diagonal
        entries sum to bytes_moved, the diagonal holds on-device copies."""
        n = C.c_int()
        A.check(A.lib().rs_plan_traffic(self.h, None, 0, C.byref(n)))
        buf = (C.c_int64 * max(1, n.value * n.value))()
        A.check(A.lib().rs_plan_traffic(self.h, buf, n.value * n.value, C.byref(n)))
        return [list(buf[i * n.value:(i + 1) * n.value]) for i in range(n.value)]

    def participants(self) -> List[int]:
        """Participating physical devices, ascending (WorldMap::participants)."""
        n = C.c_int()
        A.check(A.lib().rs_plan_participants(self.h, None, 0, C.byref(n)))
        arr = (C.c_int * max(1, n.value))()
        A.check(A.lib().rs_plan_participants(self.h, arr, n.value, C.byref(n)))
        return list(arr[: n.value])

    def transfers(self, device: int = -1) -> List[A.Transfer_t]:
        p, n = C.c_void_p(), C.c_int64()
        A.check(A.lib().rs_plan_transfers(self.h, device, C.byref(p), C.byref(n)))
        arr = C.cast(p, C.POINTER(A.Transfer_t))
        out = [A.Transfer_t.from_buffer_copy(arr[i]) for i in range(n.value)]
        A.lib().rs_free(p)
        return out

    def expand_timed(self, device: int = 0):
        """(milliseconds, runs) of expanding the ZeRO transfer list: GPU planner or host."""
        ms, n = C.c_double(), C.c_int64()
        A.check(A.lib().rs_plan_expand_timed(self.h, device, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def box_routes_timed(self, device: int = 0):
        """(kernel ms, box transfers, equal to the host plan) of the GPU box planner."""
        ms, n, eq = C.c_double(), C.c_int64(), C.c_int()
        A.check(A.lib().rs_plan_box_routes_timed(self.h, device, C.byref(ms), C.byref(n), C.byref(eq)))
        return ms.value, n.value, bool(eq.value)

    def validate(self, drop: int = -1) -> List[str]:
        """validate_plan: violation lines, empty on success."""
        p, n, k = C.c_void_p(), C.c_size_t(), C.c_int64()
        A.check(A.lib().rs_plan_validate(self.h, drop, C.byref(p), C.byref(n), C.byref(k)))
        return [x for x in A.take_string(p, n).splitlines() if x]


class ModelSpace:
    """build_model_space (model.hpp:127-144)."""

    def __init__(self, model: Model):
        arr = (A.Tensor_t * max(1, len(model.tensors)))()
        self._ids = []
        for i, t in enumerate(model.tensors):
            b = t.id.encode()
            self._ids.append(b)
            shape = (C.c_int64 * 4)(*(list(t.shape) + [0] * (4 - len(t.shape))))
            arr[i] = A.Tensor_t(b, len(t.shape), shape, t.layer, -1 if t.tp is None else t.tp,
                                -1 if t.expert is None else t.expert, t.dtype)
        h = C.c_void_p()
        A.check(A.lib().rs_model_create(arr, len(model.tensors), model.layers, model.experts, C.byref(h)))
        self.h = h.value
        self.model = model

    def __del__(self):
        if getattr(self, "h", None) and _alive():
            A.lib().rs_model_destroy(self.h)
            self.h = None


def plan_transition(space: ModelSpace, src: Cfg, dst: Cfg, world_src: Optional[Sequence[int]] = None,
                    world_dst: Optional[Sequence[int]] = None, nodes: int = 1, rpn: int = 8,
                    migrate_grads: bool = False, balance_fanout: bool = False, scalar_words: int = 8,
                    allow_oversourced: bool = False) -> RoutingPlan:
    keep: list = []
    s, d = _cfg_t(src, keep), _cfg_t(dst, keep)
    wm = None
    if world_src is not None or world_dst is not None:
        ws = list(world_src if world_src is not None else range(src.world()))
        wd = list(world_dst if world_dst is not None else range(dst.world()))
        a, b = (C.c_int * max(1, len(ws)))(*ws), (C.c_int * max(1, len(wd)))(*wd)
        keep += [a, b]
        wm = A.WorldMap_t(len(ws), a, len(wd), b)
    topo = A.Topo_t(nodes, rpn)
    opts = A.Options_t(int(migrate_grads), int(balance_fanout), scalar_words, int(allow_oversourced))
    h = C.c_void_p()
    A.check(A.lib().rs_plan_create(space.h, C.byref(s), C.byref(d), C.byref(wm) if wm else None, C.byref(topo),
                                   C.byref(opts), C.byref(h)))
    return RoutingPlan(h.value, space)


class Executor:
    """Per-GPU executor (Algorithm 1 ExecuteSwitch; push model)."""

    def __init__(self, plan: RoutingPlan, n_gpus: int = 1, gpu: int = 0, device: int = 0,
                 with_grads: bool = False, tile_bytes: int = 0, ctas_per_sm: int = 0):
        self.plan = plan
        o = A.ExecOpts_t(n_gpus, gpu, device, int(with_grads), tile_bytes, ctas_per_sm)
        h = C.c_void_p()
        A.check(A.lib().rs_exec_create(plan.h, C.byref(o), C.byref(h)))
        self.h = h.value
        self.n_gpus, self.gpu, self.device = n_gpus, gpu, device

    def __del__(self):
        if getattr(self, "h", None) and _alive():
            A.lib().rs_exec_destroy(self.h)
            self.h = None

    # ---- buffers
    def alloc(self) -> None:
        A.check(A.lib().rs_exec_alloc(self.h))

    def bind(self, side: int, rank: int, buf: int, ptr: int, nbytes: int) -> None:
        A.check(A.lib().rs_exec_bind(self.h, side, rank, buf, C.c_void_p(ptr), nbytes))

    def buffer(self, side: int, rank: int, buf: int):
        p, n, g = C.c_void_p(), C.c_int64(), C.c_int()
        A.check(A.lib().rs_exec_buffer(self.h, side, rank, buf, C.byref(p), C.byref(n), C.byref(g)))
        return p.value or 0, n.value, g.value

    def set_plan(self, plan: RoutingPlan) -> None:
        """Drive the bound buffers with a re-computed plan of the same transition (same
        configs, world map, model, buffer geometry); the next prepare() builds from it."""
        A.check(A.lib().rs_exec_set_plan(self.h, plan.h))
        self.plan = plan

    def set_collectives(self, on: bool = True) -> None:
        """Execute optimize_primitives' Scatter (root pushes) and Gather (root pulls over
        NVLink) as their own primitives; call before ipc_export on every rank (a Gather's
        root maps the source buffers too). Takes effect at the next prepare()."""
        A.check(A.lib().rs_exec_set_collectives(self.h, int(on)))

    def gpu_of_phys(self, phys: int) -> int:
        """GPU index this executor places physical device `phys` on."""
        g = C.c_int()
        A.check(A.lib().rs_exec_gpu_of_phys(self.h, phys, C.byref(g)))
        return g.value

    def ipc_export(self) -> bytes:
        n = C.c_size_t()
        A.check(A.lib().rs_exec_ipc_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(1, n.value))
        A.check(A.lib().rs_exec_ipc_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def ipc_import(self, blob: bytes) -> None:
        A.check(A.lib().rs_exec_ipc_import(self.h, blob, len(blob)))

    def read(self, side: int, rank: int, buf: int, offset: int, nbytes: int, stream: int = 0) -> bytes:
        """Read `nbytes` of a buffer back to the host (synchronous on `stream`)."""
        out = C.create_string_buffer(nbytes)
        A.check(A.lib().rs_exec_read(self.h, side, rank, buf, offset, out, nbytes, C.c_void_p(stream)))
        return out.raw

    # ---- fused push
    def prepare(self) -> None:
        A.check(A.lib().rs_exec_prepare(self.h))

    def run(self, stream: int = 0) -> int:
        n = C.c_int()
        A.check(A.lib().rs_exec_run(self.h, C.c_void_p(stream), C.byref(n)))
        return n.value

    def run_graph(self, stream: int = 0) -> int:
        """run() replayed from a CUDA graph (captured once per prepare and stream)."""
        n = C.c_int()
        A.check(A.lib().rs_exec_run_graph(self.h, C.c_void_p(stream), C.byref(n)))
        return n.value

    def set_stages(self, dst_order) -> None:
        arr = (C.c_int * max(1, len(dst_order)))(*dst_order)
        A.check(A.lib().rs_exec_set_stages(self.h, arr, len(dst_order)))

    def num_stages(self) -> int:
        n = C.c_int()
        A.check(A.lib().rs_exec_num_stages(self.h, C.byref(n)))
        return n.value

    def run_stage(self, stage: int, stream: int = 0) -> int:
        n = C.c_int()
        A.check(A.lib().rs_exec_run_stage(self.h, stage, C.c_void_p(stream), C.byref(n)))
        return n.value

    # ---- staged (Algorithm 1 buffered) channels
    def prepare_staged(self) -> None:
        A.check(A.lib().rs_exec_prepare_staged(self.h))

    def channel_bytes(self, src_phys: int, dst_phys: int) -> int:
        n = C.c_int64()
        A.check(A.lib().rs_exec_channel_bytes(self.h, src_phys, dst_phys, C.byref(n)))
        return n.value

    def pack(self, src_phys: int, dst_phys: int, ptr: int, stream: int = 0) -> None:
        A.check(A.lib().rs_exec_pack(self.h, src_phys, dst_phys, C.c_void_p(ptr), C.c_void_p(stream)))

    def unpack(self, src_phys: int, dst_phys: int, ptr: int, stream: int = 0) -> None:
        A.check(A.lib().rs_exec_unpack(self.h, src_phys, dst_phys, C.c_void_p(ptr), C.c_void_p(stream)))

    # ---- broadcast promotion (NVLS multicast)
    def bcast_groups(self) -> List[A.BcastGroup_t]:
        """Broadcast groups of this plan and placement (identical on every rank)."""
        n = C.c_int()
        A.check(A.lib().rs_exec_bcast_groups(self.h, None, 0, C.byref(n)))
        arr = (A.BcastGroup_t * max(1, n.value))()
        A.check(A.lib().rs_exec_bcast_groups(self.h, arr, n.value, C.byref(n)))
        return list(arr[: n.value])

    def set_multicast(self, group_id: int, mc_va: int) -> None:
        A.check(A.lib().rs_exec_set_multicast(self.h, group_id, C.c_void_p(mc_va or None)))

    def set_replica_dedup(self, on: bool = True, early: bool = False) -> None:
        """A region bound for several replica ranks on one GPU crosses NVLink once; call
        run_dup() on every GPU after run() and a cross-GPU barrier. early: stage 1 is a
        tail of the other pushes sized to hide the copies, stage 0 the rest incl. the
        primaries (num_stages() = 2), so run_dup can follow a
        barrier on stage 0 and overlap stage 1 (runtime.run_dedup_early)."""
        A.check(A.lib().rs_exec_set_replica_dedup(self.h, 2 if (on and early) else int(on)))

    def run_dup(self, stream: int = 0) -> int:
        n = C.c_int()
        A.check(A.lib().rs_exec_run_dup(self.h, C.c_void_p(stream), C.byref(n)))
        return n.value

    # ---- synthetic state
    def fill(self, side: int, seed: int, stream: int = 0) -> None:
        A.check(A.lib().rs_exec_fill(self.h, side, seed, C.c_void_p(stream)))

    def verify(self, side: int, seed: int, stream: int = 0):
        bad, first = C.c_int64(), C.c_int64()
        rc = A.lib().rs_exec_verify(self.h, side, seed, C.c_void_p(stream), C.byref(bad), C.byref(first))
        if rc not in (A.RS_OK, A.RS_ERR_VIOLATION):
            A.check(rc)
        return bad.value, first.value

    def stats(self) -> A.ExecStats_t:
        s = A.ExecStats_t()
        A.check(A.lib().rs_exec_stats(self.h, C.byref(s)))
        return s


def execute(plan: RoutingPlan, buffers, n_gpus: int = 1, gpu: int = 0, device: int = 0, stream: int = 0,
            with_grads: bool = False) -> int:
    """SPEC execute in one call (rs_execute): `buffers` = [(side, rank, buf, ptr, nbytes)]
    for every buffer this GPU reads or writes; prepares, runs the push and waits."""
    arr = (A.StateBuffer_t * max(1, len(buffers)))(*[A.StateBuffer_t(s, r, b, C.c_void_p(p), n) for s, r, b, p, n in buffers])
    o = A.ExecOpts_t(n_gpus, gpu, device, int(with_grads), 0, 0)
    n = C.c_int()
    A.check(A.lib().rs_execute(plan.h, C.byref(o), arr, len(buffers), C.c_void_p(stream), 0, C.byref(n)))
    return n.value


class Arena:
    """VMM old/new layouts with plan-time eager-free aliasing (arena.hpp): one GPU, or
    (Arena.multi) the buffers one GPU of several hosts, shared by POSIX descriptor."""

    def __init__(self, ab: RoutingPlan, ba: Optional[RoutingPlan] = None, device: int = 0, cap_bytes: int = 0,
                 chunk_bytes: int = 0, with_grads: bool = False):
        h = C.c_void_p()
        A.check(A.lib().rs_arena_create(ab.h, ba.h if ba else None, device, cap_bytes, chunk_bytes,
                                        int(with_grads), C.byref(h)))
        self.h = h.value
        self.ab, self.ba = ab, ba

    @classmethod
    def multi(cls, ab: RoutingPlan, ba: Optional[RoutingPlan], n_gpus: int, gpu: int, device: int,
              cap_bytes: int = 0, chunk_bytes: int = 0, with_grads: bool = False, groups: int = 0,
              bands: int = 1) -> "Arena":
        """groups 0: the cheapest schedule level that fits cap_bytes; -1: rounds."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        A.check(A.lib().rs_arena_create_multi(ab.h, ba.h if ba else None, n_gpus, gpu, device, cap_bytes, chunk_bytes,
                                              int(with_grads), groups, bands, C.byref(h)))
        self.h, self.ab, self.ba = h.value, ab, ba
        return self

    def __del__(self):
        if getattr(self, "h", None) and _alive():
            A.lib().rs_arena_destroy(self.h)
            self.h = None

    def buffer(self, layout: int, rank: int, buf: int):
        p, n = C.c_void_p(), C.c_int64()
        A.check(A.lib().rs_arena_buffer(self.h, layout, rank, buf, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def bind_size(self, layout: int, rank: int, buf: int) -> int:
        """Bytes a multicast object must span to bind that buffer whole."""
        n = C.c_int64()
        A.check(A.lib().rs_arena_bind_size(self.h, layout, rank, buf, C.byref(n)))
        return n.value

    def stage_order(self, direction: int) -> List[int]:
        out = (C.c_int * 65536)()
        n = C.c_int()
        A.check(A.lib().rs_arena_stage_order(self.h, direction, out, 65536, C.byref(n)))
        return list(out[: n.value])

    def stage_cuts(self, direction: int) -> List[int]:
        """1 where a barrier must precede that stage position; the positions in between
        share one stage (run concurrently)."""
        out = (C.c_int * 65536)()
        n = C.c_int()
        A.check(A.lib().rs_arena_stage_cuts(self.h, direction, out, 65536, C.byref(n)))
        return list(out[: n.value])

    def release_through(self, stage: int) -> int:
        """FreeObsoleteBuffers at run time (one-way arenas on one GPU): after stage `stage`
        has completed, unmap the old-layout chunks it made dead and release the physical
        memory the new layout does not reuse. Returns the bytes released."""
        n = C.c_int64()
        A.check(A.lib().rs_arena_release_through(self.h, stage, C.byref(n)))
        return n.value

    def stats(self) -> A.ArenaStats_t:
        s = A.ArenaStats_t()
        A.check(A.lib().rs_arena_stats(self.h, C.byref(s)))
        return s

    def export(self):
        """(descriptors, mapping table) of this GPU's physical allocations (caller closes fds)."""
        p_fds, n, p_t, ln = C.POINTER(C.c_int)(), C.c_int(), C.c_void_p(), C.c_size_t()
        A.check(A.lib().rs_arena_export(self.h, C.byref(p_fds), C.byref(n), C.byref(p_t), C.byref(ln)))
        fds = [p_fds[i] for i in range(n.value)]
        table = C.string_at(p_t.value, ln.value)
        A.lib().rs_free(C.cast(p_fds, C.c_void_p))
        A.lib().rs_free(p_t)
        return fds, table

    def import_peer(self, fds: Sequence[int], table: bytes) -> None:
        """Map a peer's buffers (consumes the descriptors)."""
        arr = (C.c_int * max(1, len(fds)))(*fds)
        A.check(A.lib().rs_arena_import(self.h, arr, len(fds), table, len(table)))

    def bind(self, fwd: "Executor", bwd: Optional["Executor"] = None, cuts=None) -> None:
        """Bind A/B buffers into the forward (A->B) and backward (B->A) executors and
        set their stage orders, grouped by `cuts` (default: this arena's own; with
        several GPUs pass the union over all GPUs, runtime.global_stage_cuts)."""
        for layout, nr in ((0, self.ab.summary.src_world), (1, self.ab.summary.dst_world)):
            for r in range(nr):
                for b in range(6):
                    p, n = self.buffer(layout, r, b)
                    if n:
                        fwd.bind(layout, r, b, p, n)
                        if bwd is not None:
                            bwd.bind(1 - layout, r, b, p, n)
        cuts = cuts or [self.stage_cuts(0), self.stage_cuts(1)]
        for d, ex in ((0, fwd), (1, bwd)):
            if ex is None:
                continue
            order = self.stage_order(d)
            cu = list(cuts[d]) if cuts[d] else [1] * len(order)
            arr_o, arr_c = (C.c_int * len(order))(*order), (C.c_int * len(order))(*cu)
            A.check(A.lib().rs_exec_set_stage_groups(ex.h, arr_o, arr_c, len(order)))


class Schedule:
    """build_schedule over a RoutingPlan."""

    KINDS = {0: "p2p", 1: "broadcast", 2: "scatter", 3: "gather"}

    def __init__(self, plan: RoutingPlan, mem_avail: Optional[Sequence[int]] = None, promote: bool = True):
        h = C.c_void_p()
        av = (C.c_int64 * max(1, len(mem_avail)))(*mem_avail) if mem_avail else None
        A.check(A.lib().rs_schedule_build(plan.h, av, len(mem_avail) if mem_avail else 0, int(promote), C.byref(h)))
        self.h = h.value
        self.plan = plan
        s = A.ScheduleSummary_t()
        A.check(A.lib().rs_schedule_summary(self.h, C.byref(s)))
        self.summary = s

    def __del__(self):
        if getattr(self, "h", None) and _alive():
            A.lib().rs_schedule_destroy(self.h)
            self.h = None

    def stages(self):
        out = []
        for k in range(self.summary.num_stages):
            steps = (C.c_int * 4096)()
            n, cost = C.c_int(), C.c_int64()
            A.check(A.lib().rs_schedule_stage(self.h, k, steps, 4096, C.byref(n), C.byref(cost)))
            out.append((list(steps[: n.value]), cost.value))
        return out

    def peer(self, stage: int, q: int, dev: int):
        p, sb, rb = C.c_int(), C.c_int64(), C.c_int64()
        A.check(A.lib().rs_schedule_peer(self.h, stage, q, dev, C.byref(p), C.byref(sb), C.byref(rb)))
        return p.value, sb.value, rb.value

    def collectives(self):
        out = []
        for c in range(self.summary.num_collectives):
            kind, root, n = C.c_int(), C.c_int(), C.c_int()
            b = C.c_int64()
            parts = (C.c_int * 4096)()
            A.check(A.lib().rs_schedule_collective(self.h, c, C.byref(kind), C.byref(root), C.byref(b), parts, 4096,
                                                   C.byref(n)))
            out.append({"kind": self.KINDS[kind.value], "root": root.value, "bytes": b.value,
                        "participants": list(parts[: n.value])})
        return out

    def dump(self) -> str:
        p, n = C.c_void_p(), C.c_size_t()
        A.check(A.lib().rs_schedule_dump(self.h, C.byref(p), C.byref(n)))
        return A.take_string(p, n)


class Multicast:
    """NVLS multicast object (rs_mc_*): created by the root, imported by the members."""

    def __init__(self, handle: int, nbytes: int):
        self.h, self.nbytes = handle, nbytes

    @classmethod
    def create(cls, nbytes: int, n_devices: int) -> "Multicast":
        h = C.c_void_p()
        A.check(A.lib().rs_mc_create(nbytes, n_devices, C.byref(h)))
        return cls(h.value, nbytes)

    @classmethod
    def import_fd(cls, fd: int, nbytes: int) -> "Multicast":
        h = C.c_void_p()
        A.check(A.lib().rs_mc_import(fd, nbytes, C.byref(h)))
        return cls(h.value, nbytes)

    def export_fd(self) -> int:
        fd = C.c_int()
        A.check(A.lib().rs_mc_export(self.h, C.byref(fd)))
        return fd.value

    def add_device(self, device: int) -> None:
        A.check(A.lib().rs_mc_add_device(self.h, device))

    def bind_arena(self, arena: Arena, layout: int, rank: int, buf: int) -> None:
        A.check(A.lib().rs_mc_bind_arena(self.h, arena.h, layout, rank, buf))

    def bind_vmm(self, buf: "VmmBuffer", mc_offset: int = 0) -> None:
        A.check(A.lib().rs_mc_bind_vmm(self.h, buf.h, mc_offset))

    def map(self, device: int) -> int:
        va = C.c_void_p()
        A.check(A.lib().rs_mc_map(self.h, device, C.byref(va)))
        return va.value

    def close(self) -> None:
        if getattr(self, "h", None) and _alive():
            A.lib().rs_mc_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class DeviceBarrier:
    """SynchronizeAll on the device (rs_sync_*): a cross-GPU flag barrier
    enqueued on a stream. Build with runtime.device_barrier (exchanges the handles)."""

    def __init__(self, rank: int, world: int, device: int):
        h = C.c_void_p()
        A.check(A.lib().rs_sync_create(rank, world, device, C.byref(h)))
        self.h = h.value
        self.rank, self.world, self.device = rank, world, device

    def __del__(self):
        if getattr(self, "h", None) and _alive():
            A.lib().rs_sync_destroy(self.h)
            self.h = None

    def export(self) -> bytes:
        n = C.c_size_t()
        buf = C.create_string_buffer(256)
        A.check(A.lib().rs_sync_export(self.h, buf, 256, C.byref(n)))
        return buf.raw[: n.value]

    def import_peer(self, peer: int, blob: bytes) -> None:
        A.check(A.lib().rs_sync_import(self.h, peer, blob, len(blob)))

    def __call__(self, stream: int = 0) -> None:
        """Enqueue one barrier on `stream` (every rank enqueues the same sequence)."""
        A.check(A.lib().rs_sync_barrier(self.h, C.c_void_p(stream)))

    def timed_out(self) -> bool:
        v = C.c_int()
        A.check(A.lib().rs_sync_status(self.h, C.byref(v)))
        return bool(v.value)


class VmmBuffer:
    """One shareable VMM device buffer (rs_vmm_*): allocated here, or a peer's imported
    from its POSIX descriptor and mapped for this GPU."""

    def __init__(self, handle: int, nbytes: int):
        self.h, self.nbytes = handle, nbytes
        p, n = C.c_void_p(), C.c_int64()
        A.check(A.lib().rs_vmm_ptr(self.h, C.byref(p), C.byref(n)))
        self.ptr, self.mapped_bytes = p.value, n.value

    @classmethod
    def alloc(cls, device: int, nbytes: int) -> "VmmBuffer":
        h = C.c_void_p()
        A.check(A.lib().rs_vmm_alloc(device, nbytes, C.byref(h)))
        return cls(h.value, nbytes)

    @classmethod
    def import_fd(cls, fd: int, nbytes: int, device: int) -> "VmmBuffer":
        h = C.c_void_p()
        A.check(A.lib().rs_vmm_import(fd, nbytes, device, C.byref(h)))
        return cls(h.value, nbytes)

    def export_fd(self) -> int:
        fd = C.c_int()
        A.check(A.lib().rs_vmm_export(self.h, C.byref(fd)))
        return fd.value

    def close(self) -> None:
        if getattr(self, "h", None) and _alive():
            A.lib().rs_vmm_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


# ---- schedule ------------------------------------------------------

def xor_peer(i: int, s: int, n: int) -> int:
    """Peer(i, s) = i XOR s, or -1 when outside the device set."""
    return A.lib().rs_xor_peer(i, s, n)


def memory_aware_chunk(steps: Sequence[int], costs: Sequence[int], mem_avail: Sequence[int]):
    """MemoryAwareChunk: returns (stages as lists of steps, budget)."""
    n = len(steps)
    st = (C.c_int * max(1, n))(*steps)
    co = (C.c_int64 * max(1, n))(*costs)
    av = (C.c_int64 * max(1, len(mem_avail)))(*mem_avail)
    out = (C.c_int * max(1, n))()
    budget = C.c_int64()
    A.check(A.lib().rs_memory_aware_chunk(st, co, n, av, len(mem_avail), out, C.byref(budget)))
    stages: List[List[int]] = []
    for k in range(n):
        g = out[k]
        while len(stages) <= g:
            stages.append([])
        stages[g].append(steps[k])
    return stages, budget.value


# ---- host-only memory plans (arena.hpp) ----------------------------------------------

def memory_plan(ab: RoutingPlan, ba: Optional[RoutingPlan] = None, chunk_bytes: int = 0, with_grads: bool = False,
                n_gpus: int = 1, gpu: int = 0, groups: int = 0, bands: int = 1):
    """Host-only arena plan of the buffers `gpu` hosts: (stats, simulated violations,
    stage orders over units rank * bands + band); `groups` coarsens the unit order
    (0 = one group per unit, -1 = rounds), `bands` splits destination ranks into layer bands."""
    st, viol = A.ArenaStats_t(), C.c_int64()
    oa, ob = (C.c_int * 65536)(), (C.c_int * 65536)()
    A.check(A.lib().rs_memory_plan_ex(ab.h, ba.h if ba else None, chunk_bytes, int(with_grads), n_gpus, gpu, groups,
                                      bands, C.byref(st), C.byref(viol), oa, ob, 65536))
    return st, viol.value, [x for x in oa if x >= 0], [x for x in ob if x >= 0]


def memory_plan_cuts(ab: RoutingPlan, ba: Optional[RoutingPlan] = None, chunk_bytes: int = 0, with_grads: bool = False,
                     n_gpus: int = 1, gpu: int = 0, groups: int = 0, bands: int = 1, direction: int = 0) -> List[int]:
    """The plan's stage cuts (1 = a barrier precedes that unit position)."""
    out, n = (C.c_int * 65536)(), C.c_int()
    A.check(A.lib().rs_memory_plan_cuts(ab.h, ba.h if ba else None, chunk_bytes, int(with_grads), n_gpus, gpu, groups,
                                        bands, direction, out, 65536, C.byref(n)))
    return list(out[: n.value])


def memory_min_groups(ab: RoutingPlan, ba: Optional[RoutingPlan], n_gpus: int, gpu: int, cap_bytes: int,
                      chunk_bytes: int = 0, with_grads: bool = False):
    """(fewest stage groups, one band, whose plan fits cap_bytes on `gpu` or -1, physical bytes)."""
    g, phys = C.c_int(), C.c_int64()
    A.check(A.lib().rs_memory_min_groups(ab.h, ba.h if ba else None, chunk_bytes, int(with_grads), n_gpus, gpu,
                                         cap_bytes, C.byref(g), C.byref(phys)))
    return g.value, phys.value


def memory_schedule(ab: RoutingPlan, ba: Optional[RoutingPlan], n_gpus: int, gpu: int, cap_bytes: int,
                    chunk_bytes: int = 0, with_grads: bool = False):
    """(first schedule level that fits cap_bytes on `gpu` or -1, its physical bytes)."""
    lv, phys = C.c_int(), C.c_int64()
    A.check(A.lib().rs_memory_schedule(ab.h, ba.h if ba else None, chunk_bytes, int(with_grads), n_gpus, gpu, cap_bytes,
                                       C.byref(lv), C.byref(phys)))
    return lv.value, phys.value


def memory_schedule_footprints(ab: RoutingPlan, ba: Optional[RoutingPlan], n_gpus: int, gpu: int,
                               chunk_bytes: int = 0, with_grads: bool = False) -> List[int]:
    """Physical bytes `gpu` needs at every level of the schedule ladder."""
    n = C.c_int()
    out = (C.c_int64 * 4096)()
    A.check(A.lib().rs_memory_schedule_footprints(ab.h, ba.h if ba else None, chunk_bytes, int(with_grads), n_gpus, gpu,
                                                  out, 4096, C.byref(n)))
    return list(out[: n.value])


def memory_schedule_costs(ab: RoutingPlan, ba: Optional[RoutingPlan], n_gpus: int, gpu: int,
                          chunk_bytes: int = 0, with_grads: bool = False):
    """[(physical bytes on `gpu`, modeled seconds)] at every level of the schedule ladder."""
    n = C.c_int()
    b = (C.c_int64 * 4096)()
    t = (C.c_double * 4096)()
    A.check(A.lib().rs_memory_schedule_costs(ab.h, ba.h if ba else None, chunk_bytes, int(with_grads), n_gpus, gpu,
                                             b, t, 4096, C.byref(n)))
    return [(b[i], t[i]) for i in range(n.value)]


def memory_schedule_level(ab: RoutingPlan, level: int, n_gpus: int = 1):
    """(bands, groups) of a schedule level of the n_gpus ladder (groups -1: rounds)."""
    b, g = C.c_int(), C.c_int()
    A.check(A.lib().rs_memory_schedule_level(ab.h, n_gpus, level, C.byref(b), C.byref(g)))
    return b.value, g.value


# ---- process plumbing: descriptor exchange, peer access --------------------------------

def fdx_listen(name: str) -> int:
    s = C.c_int()
    A.check(A.lib().rs_fdx_listen(name.encode(), C.byref(s)))
    return s.value


def fdx_send(peer: str, fds: Sequence[int], payload: bytes) -> None:
    arr = (C.c_int * max(1, len(fds)))(*fds)
    A.check(A.lib().rs_fdx_send(peer.encode(), arr, len(fds), payload, len(payload)))


def fdx_recv(sock: int):
    p_fds, n, p_pl, ln = C.POINTER(C.c_int)(), C.c_int(), C.c_void_p(), C.c_size_t()
    A.check(A.lib().rs_fdx_recv(sock, C.byref(p_fds), C.byref(n), C.byref(p_pl), C.byref(ln)))
    fds = [p_fds[i] for i in range(n.value)]
    payload = C.string_at(p_pl.value, ln.value) if ln.value else b""
    A.lib().rs_free(C.cast(p_fds, C.c_void_p))
    A.lib().rs_free(p_pl)
    return fds, payload


def fdx_close(fd: int) -> None:
    A.lib().rs_fdx_close(fd)


def enable_peer_access(device: int, peer: int) -> None:
    """One process driving several GPUs: direct stores from `device` into `peer`."""
    A.check(A.lib().rs_enable_peer_access(device, peer))
