"""Torch views of one virtual rank's state buffers: the registration boundary a training
job uses to hand its tensors to the transition (Megatron hooks that
register state tensors).

The buffers follow the layout contract: params = the rank's
boxes flattened row-major, dense span then expert span, at dtype_bytes; grads = the same
geometry in fp32; optimizer = [dense shard | expert shard] of the span, SoA fp32
master / m / v (ZeRO) or the whole span (no ZeRO). `RankState` exposes
  - param(id): the rank's box of tensor `id`, box-shaped (a view: writes land in the buffer),
  - grad(id): the same box in fp32,
  - optim_slice(kind, id): the part of the rank's optimizer shard that belongs to `id`,
    as (1-D fp32 view, (a, b)) where [a, b) indexes the row-major enumeration of the
    rank's box of that tensor — i.e. full[box].reshape(-1)[a:b] holds the same values.
A job allocates (or adopts) the buffers, copies or trains into the views, binds them
into an Executor, and after the transition reads the new layout's views.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Mapping, Optional, Tuple

from . import _capi as A

_DTYPES = {1: "uint8", 2: "bfloat16", 4: "float32", 8: "float64"}


class Segment_t(C.Structure):
    _fields_ = [("tensor", C.c_int), ("expert", C.c_int), ("box_lo", C.c_int64 * 4), ("box_hi", C.c_int64 * 4),
                ("local_lo", C.c_int64), ("local_hi", C.c_int64), ("param_byte_off", C.c_int64),
                ("elem_off", C.c_int64)]


class RankGeom_t(C.Structure):
    _fields_ = [("phys", C.c_int), ("n_segments", C.c_int), ("dense_len", C.c_int64), ("expert_len", C.c_int64),
                ("dshard_lo", C.c_int64), ("dshard_hi", C.c_int64), ("eshard_lo", C.c_int64), ("eshard_hi", C.c_int64),
                ("param_bytes", C.c_int64), ("nelem", C.c_int64), ("optim_len", C.c_int64),
                ("scalar_bytes", C.c_int64)]


def _bind(L):
    vp, P = C.c_void_p, C.POINTER
    for name, args in (
        ("rs_plan_rank_geom", [vp, C.c_int, C.c_int, P(RankGeom_t)]),
        ("rs_plan_segments", [vp, C.c_int, C.c_int, P(Segment_t), C.c_int, P(C.c_int)]),
        ("rs_plan_tensor", [vp, C.c_int, C.c_char_p, C.c_int, P(C.c_int64), P(C.c_int), P(C.c_int)]),
        ("rs_plan_num_tensors", [vp, P(C.c_int)]),
    ):
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    return L


_L = None


def _lib():
    global _L
    if _L is None:
        _L = _bind(A.lib())
    return _L


@dataclass(frozen=True)
class TensorInfo:
    index: int
    id: str
    shape: Tuple[int, ...]
    dtype_bytes: int


def model_tensors(plan) -> List[TensorInfo]:
    """The model's tensors in declaration order (model.hpp:30-44)."""
    L = _lib()
    n = C.c_int()
    A.check(L.rs_plan_num_tensors(plan.h, C.byref(n)))
    out = []
    for i in range(n.value):
        buf = C.create_string_buffer(512)
        shape, nd, db = (C.c_int64 * 4)(), C.c_int(), C.c_int()
        A.check(L.rs_plan_tensor(plan.h, i, buf, 512, shape, C.byref(nd), C.byref(db)))
        out.append(TensorInfo(i, buf.value.decode(), tuple(shape[: nd.value]), db.value))
    return out


def buffer_bytes(plan, side: int, rank: int, with_grads: bool = False) -> Dict[int, int]:
    """Bytes of every state buffer of the rank (ops.cpp buffer_sizes)."""
    g = rank_geom(plan, side, rank)
    return {A.BUF_PARAM: g.param_bytes, A.BUF_MASTER: 4 * g.optim_len, A.BUF_M: 4 * g.optim_len,
            A.BUF_V: 4 * g.optim_len, A.BUF_GRAD: 4 * g.nelem if with_grads else 0, A.BUF_SCALARS: g.scalar_bytes}


def rank_geom(plan, side: int, rank: int) -> RankGeom_t:
    g = RankGeom_t()
    A.check(_lib().rs_plan_rank_geom(plan.h, side, rank, C.byref(g)))
    return g


def segments(plan, side: int, rank: int) -> List[Segment_t]:
    L = _lib()
    n = C.c_int()
    A.check(L.rs_plan_segments(plan.h, side, rank, None, 0, C.byref(n)))
    arr = (Segment_t * max(1, n.value))()
    A.check(L.rs_plan_segments(plan.h, side, rank, arr, n.value, C.byref(n)))
    return list(arr[: n.value])


class RankState:
    """Views of one virtual rank's buffers (side RS_SIDE_SRC: the old layout, RS_SIDE_DST:
    the new one). `buffers` maps buffer ids (A.BUF_*) to uint8 torch tensors of at least
    buffer_bytes() each, on any device."""

    def __init__(self, plan, side: int, rank: int, buffers: Mapping[int, "object"]):
        import torch
        self.plan, self.side, self.rank = plan, side, rank
        self.geom = rank_geom(plan, side, rank)
        self.tensors = model_tensors(plan)
        self.by_id = {t.id: t for t in self.tensors}
        self.buffers = dict(buffers)
        need = buffer_bytes(plan, side, rank, with_grads=A.BUF_GRAD in self.buffers)
        for b, t in self.buffers.items():
            if t.dtype != torch.uint8 or t.dim() != 1 or t.numel() < need.get(b, 0):
                raise A.ConfigError(A.RS_ERR_CONFIG, f"buffer {b}: need a 1-D uint8 tensor of >= {need.get(b, 0)} bytes")
        self.seg_of: Dict[str, Segment_t] = {}
        for s in segments(plan, side, rank):
            self.seg_of[self.tensors[s.tensor].id] = s

    @classmethod
    def alloc(cls, plan, side: int, rank: int, device="cuda", with_grads: bool = False) -> "RankState":
        import torch
        bufs = {b: torch.zeros(n, dtype=torch.uint8, device=device)
                for b, n in buffer_bytes(plan, side, rank, with_grads).items() if n}
        return cls(plan, side, rank, bufs)

    def holds(self, tensor_id: str) -> bool:
        return tensor_id in self.seg_of

    def box(self, tensor_id: str) -> Tuple[slice, ...]:
        s = self.seg_of[tensor_id]
        nd = len(self.by_id[tensor_id].shape)
        return tuple(slice(s.box_lo[d], s.box_hi[d]) for d in range(nd))

    def param(self, tensor_id: str):
        """The rank's box of the tensor, box-shaped, in the tensor's dtype (a view)."""
        import torch
        s, info = self.seg_of[tensor_id], self.by_id[tensor_id]
        dt = getattr(torch, _DTYPES[info.dtype_bytes])
        shape = [s.box_hi[d] - s.box_lo[d] for d in range(len(info.shape))]
        n = 1
        for e in shape:
            n *= e
        raw = self.buffers[A.BUF_PARAM][s.param_byte_off: s.param_byte_off + n * info.dtype_bytes]
        return raw.view(dt).view(shape)

    def params(self) -> Dict[str, "object"]:
        return {tid: self.param(tid) for tid in self.seg_of}

    def grad(self, tensor_id: str):
        """The rank's box of the gradient, fp32 (needs the grad buffer)."""
        import torch
        s, info = self.seg_of[tensor_id], self.by_id[tensor_id]
        shape = [s.box_hi[d] - s.box_lo[d] for d in range(len(info.shape))]
        n = 1
        for e in shape:
            n *= e
        return self.buffers[A.BUF_GRAD].view(torch.float32)[s.elem_off: s.elem_off + n].view(shape)

    def optim(self, kind: str):
        """Whole optimizer buffer of `kind` in {'master', 'm', 'v'} (fp32, optim_len)."""
        import torch
        b = {"master": A.BUF_MASTER, "m": A.BUF_M, "v": A.BUF_V}[kind]
        return self.buffers[b].view(torch.float32)[: self.geom.optim_len]

    def optim_slice(self, kind: str, tensor_id: str) -> Tuple[Optional["object"], Tuple[int, int]]:
        """(view, (a, b)): the shard's part of the tensor; [a, b) indexes the row-major
        enumeration of this rank's box of the tensor. (None, (0, 0)) if the shard holds
        none of it."""
        s = self.seg_of[tensor_id]
        g = self.geom
        if s.expert:
            lo, hi, base = g.eshard_lo, g.eshard_hi, g.dshard_hi - g.dshard_lo
        else:
            lo, hi, base = g.dshard_lo, g.dshard_hi, 0
        a, b = max(s.local_lo, lo), min(s.local_hi, hi)
        if a >= b:
            return None, (0, 0)
        full = self.optim(kind)
        return full[base + a - lo: base + b - lo], (a - s.local_lo, b - s.local_lo)

    def bind(self, ex, side: Optional[int] = None) -> None:
        """Bind these buffers into an Executor as its `side` (default: this state's side)."""
        side = self.side if side is None else side
        for b, t in self.buffers.items():
            if t.numel():
                ex.bind(side, self.rank, b, t.data_ptr(), t.numel())
