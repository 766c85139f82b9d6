"""ctypes binding of include/reshard_b200.h (libreshard_b200.so, built in-tree).

The library is the product: no Python or CPU fallback exists for the executor.
If the shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libreshard_b200.so")

RS_OK, RS_ERR_VIOLATION, RS_ERR_CONFIG, RS_ERR_INTERNAL, RS_ERR_CUDA, RS_ERR_NCCL, RS_ERR_BUDGET = range(7)
BUF_PARAM, BUF_MASTER, BUF_M, BUF_V, BUF_GRAD, BUF_SCALARS = range(6)
SIDE_SRC, SIDE_DST = 0, 1

EXPORTED = [
    "rs_last_error", "rs_version", "rs_free", "rs_model_create", "rs_model_destroy", "rs_plan_create",
    "rs_plan_from_scenario", "rs_plan_destroy", "rs_plan_summary", "rs_plan_dump", "rs_plan_transfers",
    "rs_plan_regions", "rs_plan_dump_rows_host", "rs_exec_create", "rs_exec_destroy", "rs_exec_alloc",
    "rs_exec_bind", "rs_exec_buffer", "rs_exec_ipc_export", "rs_exec_ipc_import", "rs_exec_prepare",
    "rs_exec_fill", "rs_exec_run", "rs_exec_verify", "rs_exec_stats", "rs_exec_set_stages",
    "rs_memory_plan", "rs_config_groups", "rs_rank_coord", "rs_exec_prepare_staged", "rs_exec_channel_bytes", "rs_exec_pack", "rs_exec_unpack", "rs_plan_placement", "rs_xor_peer", "rs_memory_aware_chunk", "rs_schedule_build", "rs_schedule_destroy",
    "rs_schedule_summary", "rs_schedule_stage", "rs_schedule_peer", "rs_schedule_collective", "rs_schedule_dump",
    "rs_arena_create", "rs_arena_destroy", "rs_exec_gpu_of_phys", "rs_plan_traffic", "rs_plan_participants", "rs_exec_set_plan", "rs_exec_set_collectives", "rs_arena_release_through", "rs_sync_create", "rs_sync_destroy", "rs_sync_export", "rs_sync_import", "rs_sync_barrier", "rs_sync_status", "rs_arena_buffer", "rs_arena_stage_order", "rs_arena_stats",
]


class Tensor_t(C.Structure):
    _fields_ = [("id", C.c_char_p), ("ndim", C.c_int), ("shape", C.c_int64 * 4), ("layer", C.c_int),
                ("tp_axis", C.c_int), ("expert_axis", C.c_int), ("dtype_bytes", C.c_int)]


class Cfg_t(C.Structure):
    _fields_ = [("dp", C.c_int), ("tp", C.c_int), ("pp", C.c_int), ("ep", C.c_int), ("zero", C.c_int),
                ("order", C.c_char_p)]


class WorldMap_t(C.Structure):
    _fields_ = [("n_src", C.c_int), ("src_phys", C.POINTER(C.c_int)), ("n_dst", C.c_int),
                ("dst_phys", C.POINTER(C.c_int))]


class Topo_t(C.Structure):
    _fields_ = [("num_nodes", C.c_int), ("ranks_per_node", C.c_int)]


class Options_t(C.Structure):
    _fields_ = [("migrate_grads", C.c_int), ("balance_fanout", C.c_int), ("scalar_words", C.c_int64),
                ("allow_oversourced", C.c_int)]


class Transfer_t(C.Structure):
    _fields_ = [("kind", C.c_int), ("tensor", C.c_int), ("flat", C.c_int), ("ndim", C.c_int),
                ("lo", C.c_int64 * 4), ("hi", C.c_int64 * 4), ("src_rank", C.c_int), ("dst_rank", C.c_int),
                ("src_phys", C.c_int), ("dst_phys", C.c_int), ("count", C.c_int64), ("bytes", C.c_int64)]


class PlanSummary_t(C.Structure):
    _fields_ = [("num_transfers", C.c_int64), ("bytes_moved", C.c_int64), ("bytes_retained", C.c_int64),
                ("num_box_transfers", C.c_int64), ("num_flat_transfers", C.c_int64), ("num_triples", C.c_int64),
                ("src_world", C.c_int), ("dst_world", C.c_int), ("num_participants", C.c_int),
                ("total_numel", C.c_int64), ("fingerprint", C.c_uint64)]


class ExecOpts_t(C.Structure):
    _fields_ = [("n_gpus", C.c_int), ("gpu", C.c_int), ("device", C.c_int), ("with_grads", C.c_int),
                ("tile_bytes", C.c_int64), ("ctas_per_sm", C.c_int)]


class ExecStats_t(C.Structure):
    _fields_ = [("local_bytes", C.c_int64), ("remote_bytes", C.c_int64), ("tiles", C.c_int64),
                ("tiles_by_class", C.c_int64 * 5), ("launches", C.c_int64), ("mc_bytes", C.c_int64),
                ("dup_bytes", C.c_int64), ("scatter_bytes", C.c_int64), ("gather_bytes", C.c_int64)]


RS_MAX_MEMBERS = 64


class StateBuffer_t(C.Structure):
    _fields_ = [("side", C.c_int), ("rank", C.c_int), ("buf", C.c_int), ("ptr", C.c_void_p), ("bytes", C.c_int64)]


class BcastGroup_t(C.Structure):
    _fields_ = [("id", C.c_int), ("root_rank", C.c_int), ("root_gpu", C.c_int), ("buf", C.c_int), ("slot", C.c_int),
                ("n_members", C.c_int), ("member_gpu", C.c_int * RS_MAX_MEMBERS),
                ("member_rank", C.c_int * RS_MAX_MEMBERS), ("buffer_bytes", C.c_int64), ("payload_bytes", C.c_int64)]


class PlacementStats_t(C.Structure):
    _fields_ = [("local_bytes", C.c_int64), ("out_bytes", C.c_int64), ("in_bytes", C.c_int64), ("ops", C.c_int64)]


class ScheduleSummary_t(C.Structure):
    _fields_ = [("num_devices", C.c_int), ("num_stages", C.c_int), ("num_collectives", C.c_int), ("num_steps", C.c_int),
                ("budget", C.c_int64), ("p2p_bytes", C.c_int64), ("collective_bytes", C.c_int64),
                ("num_fragments", C.c_int64)]


class ArenaStats_t(C.Structure):
    _fields_ = [("physical_bytes", C.c_int64), ("a_bytes", C.c_int64), ("b_bytes", C.c_int64),
                ("aliased_bytes", C.c_int64), ("chunks", C.c_int64), ("stage_groups", C.c_int64 * 2),
                ("bands", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2605_18815_b200.build` "
                          "(the product has no fallback path)")
    L = C.CDLL(LIB_PATH)
    vp, cp, i64, sz = C.c_void_p, C.c_char_p, C.c_int64, C.c_size_t
    P = C.POINTER
    L.rs_last_error.restype = cp
    L.rs_version.restype = cp
    L.rs_free.argtypes = [vp]
    L.rs_model_create.argtypes = [P(Tensor_t), C.c_int, C.c_int, C.c_int, P(vp)]
    L.rs_model_destroy.argtypes = [vp]
    L.rs_plan_create.argtypes = [vp, P(Cfg_t), P(Cfg_t), P(WorldMap_t), P(Topo_t), P(Options_t), P(vp)]
    L.rs_plan_from_scenario.argtypes = [cp, C.c_int, P(vp)]
    L.rs_plan_destroy.argtypes = [vp]
    L.rs_plan_summary.argtypes = [vp, P(PlanSummary_t)]
    L.rs_plan_dump.argtypes = [vp, C.c_int, P(vp), P(sz)]
    L.rs_plan_dump_rows_host.argtypes = [vp, P(vp), P(sz)]
    L.rs_plan_transfers.argtypes = [vp, C.c_int, P(vp), P(i64)]
    L.rs_plan_regions.argtypes = [vp, C.c_int, P(vp), P(sz)]
    L.rs_exec_create.argtypes = [vp, P(ExecOpts_t), P(vp)]
    L.rs_exec_destroy.argtypes = [vp]
    L.rs_exec_alloc.argtypes = [vp]
    L.rs_exec_bind.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, i64]
    L.rs_exec_buffer.argtypes = [vp, C.c_int, C.c_int, C.c_int, P(vp), P(i64), P(C.c_int)]
    L.rs_exec_ipc_export.argtypes = [vp, vp, sz, P(sz)]
    L.rs_exec_ipc_import.argtypes = [vp, vp, sz]
    L.rs_exec_prepare.argtypes = [vp]
    L.rs_exec_fill.argtypes = [vp, C.c_int, C.c_uint64, vp]
    L.rs_exec_run.argtypes = [vp, vp, P(C.c_int)]
    L.rs_exec_verify.argtypes = [vp, C.c_int, C.c_uint64, vp, P(i64), P(i64)]
    L.rs_exec_stats.argtypes = [vp, P(ExecStats_t)]
    L.rs_exec_set_stages.argtypes = [vp, P(C.c_int), C.c_int]
    L.rs_plan_placement.argtypes = [vp, C.c_int, C.c_int, P(PlacementStats_t)]
    L.rs_memory_plan.argtypes = [vp, vp, i64, C.c_int, P(ArenaStats_t), P(i64), P(C.c_int), P(C.c_int), C.c_int]
    L.rs_config_groups.argtypes = [P(Cfg_t), C.c_int, P(C.c_int), C.c_int, P(C.c_int), P(C.c_int)]
    L.rs_rank_coord.argtypes = [P(Cfg_t), C.c_int, P(C.c_int)]
    L.rs_exec_prepare_staged.argtypes = [vp]
    L.rs_exec_channel_bytes.argtypes = [vp, C.c_int, C.c_int, P(i64)]
    L.rs_exec_gpu_of_phys.argtypes = [vp, C.c_int, P(C.c_int)]
    L.rs_plan_traffic.argtypes = [vp, P(C.c_int64), C.c_int, P(C.c_int)]
    L.rs_exec_set_plan.argtypes = [vp, vp]
    L.rs_exec_set_collectives.argtypes = [vp, C.c_int]
    L.rs_arena_release_through.argtypes = [vp, C.c_int, P(i64)]
    L.rs_sync_create.argtypes = [C.c_int, C.c_int, C.c_int, P(vp)]
    L.rs_sync_destroy.argtypes = [vp]
    L.rs_sync_export.argtypes = [vp, vp, sz, P(sz)]
    L.rs_sync_import.argtypes = [vp, C.c_int, vp, sz]
    L.rs_sync_barrier.argtypes = [vp, vp]
    L.rs_sync_status.argtypes = [vp, P(C.c_int)]
    L.rs_plan_participants.argtypes = [vp, P(C.c_int), C.c_int, P(C.c_int)]
    L.rs_exec_pack.argtypes = [vp, C.c_int, C.c_int, vp, vp]
    L.rs_exec_unpack.argtypes = [vp, C.c_int, C.c_int, vp, vp]
    L.rs_xor_peer.argtypes = [C.c_int, C.c_int, C.c_int]
    L.rs_memory_aware_chunk.argtypes = [P(C.c_int), P(i64), C.c_int, P(i64), C.c_int, P(C.c_int), P(i64)]
    L.rs_schedule_build.argtypes = [vp, P(i64), C.c_int, C.c_int, P(vp)]
    L.rs_schedule_destroy.argtypes = [vp]
    L.rs_schedule_summary.argtypes = [vp, P(ScheduleSummary_t)]
    L.rs_schedule_stage.argtypes = [vp, C.c_int, P(C.c_int), C.c_int, P(C.c_int), P(i64)]
    L.rs_schedule_peer.argtypes = [vp, C.c_int, C.c_int, C.c_int, P(C.c_int), P(i64), P(i64)]
    L.rs_schedule_collective.argtypes = [vp, C.c_int, P(C.c_int), P(C.c_int), P(i64), P(C.c_int), C.c_int, P(C.c_int)]
    L.rs_schedule_dump.argtypes = [vp, P(vp), P(sz)]
    L.rs_arena_create.argtypes = [vp, vp, C.c_int, i64, i64, C.c_int, P(vp)]
    L.rs_arena_destroy.argtypes = [vp]
    L.rs_arena_buffer.argtypes = [vp, C.c_int, C.c_int, C.c_int, P(vp), P(i64)]
    L.rs_arena_stage_order.argtypes = [vp, C.c_int, P(C.c_int), C.c_int, P(C.c_int)]
    L.rs_arena_stats.argtypes = [vp, P(ArenaStats_t)]
    for name in EXPORTED:
        fn = getattr(L, name)
        if fn.restype is None and name not in ("rs_free", "rs_model_destroy", "rs_plan_destroy", "rs_exec_destroy",
                                                      "rs_arena_destroy", "rs_schedule_destroy"):
            fn.restype = C.c_int
    _lib = _late_bindings(L)
    return L


class ReshardError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(ReshardError):
    """Mirror of reshard::ConfigError (common.hpp:30-33)."""


class VerificationError(ReshardError):
    pass


class CudaError(ReshardError):
    pass


def check(rc: int) -> None:
    if rc == RS_OK:
        return
    msg = lib().rs_last_error().decode()
    cls = {RS_ERR_CONFIG: ConfigError, RS_ERR_VIOLATION: VerificationError, RS_ERR_CUDA: CudaError}.get(rc, ReshardError)
    raise cls(rc, msg)


def take_string(ptr: C.c_void_p, n: C.c_size_t) -> str:
    s = C.string_at(ptr.value, n.value).decode() if ptr.value else ""
    lib().rs_free(ptr)
    return s


def _late_bindings(L):
    vp, i64, P = C.c_void_p, C.c_int64, C.POINTER
    for name, args in (
        ("rs_arena_create_multi", [vp, vp, C.c_int, C.c_int, C.c_int, i64, i64, C.c_int, C.c_int, C.c_int, P(vp)]),
        ("rs_memory_schedule", [vp, vp, i64, C.c_int, C.c_int, C.c_int, i64, P(C.c_int), P(i64)]),
        ("rs_memory_schedule_level", [vp, C.c_int, C.c_int, P(C.c_int), P(C.c_int)]),
        ("rs_memory_plan_cuts", [vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_int), C.c_int,
                                 P(C.c_int)]),
        ("rs_memory_schedule_footprints", [vp, vp, i64, C.c_int, C.c_int, C.c_int, P(i64), C.c_int, P(C.c_int)]),
        ("rs_memory_schedule_costs", [vp, vp, i64, C.c_int, C.c_int, C.c_int, P(i64), P(C.c_double), C.c_int,
                                      P(C.c_int)]),
        ("rs_memory_plan_ex", [vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P(ArenaStats_t), P(i64), P(C.c_int),
                               P(C.c_int), C.c_int]),
        ("rs_memory_min_groups", [vp, vp, i64, C.c_int, C.c_int, C.c_int, i64, P(C.c_int), P(i64)]),
        ("rs_arena_export", [vp, P(P(C.c_int)), P(C.c_int), P(vp), P(C.c_size_t)]),
        ("rs_arena_import", [vp, P(C.c_int), C.c_int, vp, C.c_size_t]),
        ("rs_fdx_listen", [C.c_char_p, P(C.c_int)]),
        ("rs_fdx_send", [C.c_char_p, P(C.c_int), C.c_int, vp, C.c_size_t]),
        ("rs_fdx_recv", [C.c_int, P(P(C.c_int)), P(C.c_int), P(vp), P(C.c_size_t)]),
        ("rs_fdx_close", [C.c_int]),
        ("rs_exec_num_stages", [vp, P(C.c_int)]),
        ("rs_exec_run_stage", [vp, C.c_int, vp, P(C.c_int)]),
        ("rs_exec_set_stage_groups", [vp, P(C.c_int), P(C.c_int), C.c_int]),
        ("rs_arena_stage_cuts", [vp, C.c_int, P(C.c_int), C.c_int, P(C.c_int)]),
        ("rs_exec_bcast_groups", [vp, P(BcastGroup_t), C.c_int, P(C.c_int)]),
        ("rs_exec_set_multicast", [vp, C.c_int, vp]),
        ("rs_exec_read", [vp, C.c_int, C.c_int, C.c_int, i64, vp, i64, vp]),
        ("rs_exec_set_replica_dedup", [vp, C.c_int]),
        ("rs_exec_run_graph", [vp, vp, P(C.c_int)]),
        ("rs_execute", [vp, P(ExecOpts_t), P(StateBuffer_t), C.c_int, vp, C.c_int, P(C.c_int)]),
        ("rs_exec_run_dup", [vp, vp, P(C.c_int)]),
        ("rs_enable_peer_access", [C.c_int, C.c_int]),
        ("rs_plan_box_routes_timed", [vp, C.c_int, P(C.c_double), P(i64), P(C.c_int)]),
        ("rs_mc_create", [i64, C.c_int, P(vp)]),
        ("rs_mc_import", [C.c_int, i64, P(vp)]),
        ("rs_mc_export", [vp, P(C.c_int)]),
        ("rs_mc_add_device", [vp, C.c_int]),
        ("rs_mc_bind_arena", [vp, vp, C.c_int, C.c_int, C.c_int]),
        ("rs_mc_map", [vp, C.c_int, P(vp)]),
        ("rs_arena_bind_size", [vp, C.c_int, C.c_int, C.c_int, P(i64)]),
        ("rs_vmm_alloc", [C.c_int, i64, P(vp)]),
        ("rs_vmm_import", [C.c_int, i64, C.c_int, P(vp)]),
        ("rs_vmm_export", [vp, P(C.c_int)]),
        ("rs_vmm_ptr", [vp, P(vp), P(i64)]),
        ("rs_mc_bind_vmm", [vp, vp, i64]),
    ):
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.rs_mc_destroy.argtypes = [vp]
    L.rs_mc_destroy.restype = None
    L.rs_vmm_free.argtypes = [vp]
    L.rs_vmm_free.restype = None
    L.rs_plan_validate.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                   C.POINTER(C.c_int64)]
    L.rs_plan_validate.restype = C.c_int
    L.rs_exec_channel_ops.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_int64,
                                      C.POINTER(C.c_int64)]
    L.rs_exec_channel_ops.restype = C.c_int
    L.rs_plan_expand_timed.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.rs_plan_expand_timed.restype = C.c_int
    return L
