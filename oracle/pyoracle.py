"""ctypes wrapper over oracle/_build/liboracle.so (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
this module. It is the checker, never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_PLAN = os.path.join(HERE, "_ref", "ref_plan")


class Transfer(C.Structure):
    _fields_ = [("kind", C.c_int), ("tensor", C.c_int), ("flat", C.c_int), ("nd", C.c_int),
                ("lo", C.c_int64 * 4), ("hi", C.c_int64 * 4),
                ("src_rank", C.c_int), ("dst_rank", C.c_int), ("src_phys", C.c_int), ("dst_phys", C.c_int),
                ("count", C.c_int64), ("bytes", C.c_int64)]


def build(force: bool = False) -> None:
    if force or not os.path.exists(LIB):
        subprocess.check_call(["make", "-s", "-C", HERE, "all"])


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp, cp, sz, i64 = C.c_void_p, C.c_char_p, C.c_size_t, C.c_int64
        L.or_scenario_parse.restype = vp
        L.or_scenario_parse.argtypes = [cp, cp, sz]
        L.or_scenario_free.argtypes = [vp]
        L.or_scenario_total_numel.restype = i64
        L.or_scenario_total_numel.argtypes = [vp]
        L.or_scenario_fingerprint.restype = C.c_uint64
        L.or_scenario_fingerprint.argtypes = [vp]
        L.or_plan_build.restype = C.c_int
        L.or_plan_build.argtypes = [vp, C.c_int, C.POINTER(vp), cp, sz]
        L.or_plan_free.argtypes = [vp]
        L.or_plan_num_transfers.restype = i64
        L.or_plan_num_transfers.argtypes = [vp]
        L.or_plan_transfers.restype = C.POINTER(Transfer)
        L.or_plan_transfers.argtypes = [vp]
        L.or_plan_bytes_moved.restype = i64
        L.or_plan_bytes_moved.argtypes = [vp]
        L.or_plan_bytes_retained.restype = i64
        L.or_plan_bytes_retained.argtypes = [vp]
        L.or_plan_dump.restype = vp
        L.or_plan_dump.argtypes = [vp]
        L.or_regions_dump.restype = vp
        L.or_regions_dump.argtypes = [vp, C.c_int, cp, sz]
        L.or_free.argtypes = [vp]
        L.or_state_create.restype = vp
        L.or_state_create.argtypes = [vp, C.c_int, C.c_int, cp, sz]
        L.or_state_free.argtypes = [vp]
        L.or_state_num_ranks.restype = C.c_int
        L.or_state_num_ranks.argtypes = [vp]
        L.or_state_buffer.restype = vp
        L.or_state_buffer.argtypes = [vp, C.c_int, C.c_int, C.POINTER(i64)]
        L.or_state_load.argtypes = [vp, C.c_uint64]
        L.or_state_clear.argtypes = [vp]
        L.or_execute.restype = C.c_int
        L.or_execute.argtypes = [vp, vp, vp, C.c_int, cp, sz]
        L.or_verify.restype = i64
        L.or_verify.argtypes = [vp, C.c_uint64, cp, sz]
        L.or_oracle_reshard.restype = C.c_int
        L.or_oracle_reshard.argtypes = [vp, vp, vp, cp, sz]
        L.or_state_equal.restype = C.c_int
        L.or_state_equal.argtypes = [vp, vp]
        L.or_canon.restype = C.c_uint64
        L.or_canon.argtypes = [C.c_uint64, i64, C.c_int]
        _lib = L
    return _lib


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _take_str(ptr) -> str:
    if not ptr:
        return ""
    s = C.string_at(ptr).decode()
    lib().or_free(ptr)
    return s


class OScenario:
    def __init__(self, text: str):
        err = C.create_string_buffer(512)
        self.h = lib().or_scenario_parse(text.encode(), err, 512)
        if not self.h:
            raise OracleError(2, err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_scenario_free(self.h)
            self.h = None

    def total_numel(self) -> int:
        return lib().or_scenario_total_numel(self.h)

    def fingerprint(self) -> int:
        return lib().or_scenario_fingerprint(self.h)

    def regions(self, which: int) -> str:
        err = C.create_string_buffer(512)
        p = lib().or_regions_dump(self.h, which, err, 512)
        if not p:
            raise OracleError(2, err.value.decode())
        return _take_str(p)


class OPlan:
    def __init__(self, scn: OScenario, allow_oversourced: bool = False):
        self.scn = scn
        err = C.create_string_buffer(512)
        h = C.c_void_p()
        rc = lib().or_plan_build(scn.h, int(allow_oversourced), C.byref(h), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_plan_free(self.h)
            self.h = None

    def dump(self) -> str:
        return _take_str(lib().or_plan_dump(self.h))

    def num_transfers(self) -> int:
        return lib().or_plan_num_transfers(self.h)

    def transfers(self):
        n = self.num_transfers()
        arr = lib().or_plan_transfers(self.h)
        return [arr[i] for i in range(n)]

    def bytes_moved(self) -> int:
        return lib().or_plan_bytes_moved(self.h)

    def bytes_retained(self) -> int:
        return lib().or_plan_bytes_retained(self.h)


class OState:
    """Host state of every virtual rank of one side (0 src, 1 dst)."""

    def __init__(self, scn: OScenario, which: int, with_grads: bool = False):
        self.scn = scn
        err = C.create_string_buffer(512)
        self.h = lib().or_state_create(scn.h, which, int(with_grads), err, 512)
        if not self.h:
            raise OracleError(2, err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_state_free(self.h)
            self.h = None

    def num_ranks(self) -> int:
        return lib().or_state_num_ranks(self.h)

    def buffer(self, rank: int, buf: int) -> bytes:
        n = C.c_int64()
        p = lib().or_state_buffer(self.h, rank, buf, C.byref(n))
        # ctypes.string_at takes a C int size: buffers past 2 GiB go through an array view
        return (C.c_char * n.value).from_address(p).raw if n.value else b""

    def buffer_ptr(self, rank: int, buf: int):
        n = C.c_int64()
        p = lib().or_state_buffer(self.h, rank, buf, C.byref(n))
        return p, n.value

    def load(self, seed: int) -> None:
        lib().or_state_load(self.h, seed)

    def clear(self) -> None:
        lib().or_state_clear(self.h)

    def verify(self, seed: int):
        err = C.create_string_buffer(512)
        bad = lib().or_verify(self.h, seed, err, 512)
        return bad, err.value.decode()

    def equal(self, other: "OState") -> bool:
        return bool(lib().or_state_equal(self.h, other.h))


def execute(plan: OPlan, src: OState, dst: OState, nthreads: int = 1) -> None:
    err = C.create_string_buffer(512)
    rc = lib().or_execute(plan.h, src.h, dst.h, nthreads, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())


def oracle_reshard(scn: OScenario, src: OState, dst: OState) -> None:
    err = C.create_string_buffer(512)
    rc = lib().or_oracle_reshard(scn.h, src.h, dst.h, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())


def canon(seed: int, element: int, kind: int) -> int:
    return lib().or_canon(seed, element, kind)


def ref_available() -> bool:
    return os.path.exists(REF_PLAN)


def ref_plan(text: str, cmd: str = "plan", timeout: float = 600) -> tuple:
    """Run the reference headers (oracle/_ref/ref_plan). Returns (rc, stdout)."""
    p = subprocess.run([REF_PLAN, cmd, "-"], input=text.encode(), stdout=subprocess.PIPE, timeout=timeout)
    return p.returncode, p.stdout.decode()
