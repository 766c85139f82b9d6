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


def init_dist():
    """One process per rank: set the device and create the default process group. More
    ranks than GPUs (a 1-GPU box running a 2/4/8-rank placement) share devices round
    robin; NCCL refuses two ranks on one device, so those runs use gloo plumbing (the data
    path needs no collective: pushes go through cudaIpc / VMM mappings either way).
    Returns (rank, world, local device, shared)."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    n = torch.cuda.device_count()
    shared = world > n
    local %= n
    torch.cuda.set_device(local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local, shared


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
    measured comparison for the fused push path, with SPEC execute's three modes
    (SPEC.md:375-383):
      async : per stage of the memory-aware schedule, PackData into one contiguous buffer
              per (device -> peer) channel, all steps' AsyncSend/AsyncRecv as one NCCL
              group (batch_isend_irecv), SynchronizeAll, UnpackData;
      sync  : the same buffers, one XOR step at a time;
      naive : no buffering of messages: one NCCL message per op (fragment group), sent
              and received one after another.
    Channels are enumerated in the global (step, device) order on every rank, so NCCL's
    per-pair FIFO matching pairs them without metadata."""

    MODES = ("async", "sync", "naive")

    def __init__(self, plan: RoutingPlan, ex: Executor, n_gpus: int, gpu: int, mem_avail=None, group=None,
                 mode: str = "async"):
        from .api import Schedule, xor_peer
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {self.MODES}")
        self.plan, self.ex, self.n_gpus, self.gpu, self.group, self.mode = plan, ex, n_gpus, gpu, group, mode
        n = plan.summary.num_participants
        self.sched = Schedule(plan, mem_avail or [1 << 62] * n, promote=False)
        ex.prepare_staged()
        # device index -> phys from the plan's WorldMap (join/leave maps need not be
        # contiguous), GPU placement from the executor
        self.phys = plan.participants()
        assert len(self.phys) == n
        self.gpu_of = [ex.gpu_of_phys(p) for p in self.phys]

        def chan(i, p, s):
            nbytes = ex.channel_bytes(self.phys[i], self.phys[p])
            if not nbytes or self.gpu_of[i] == self.gpu_of[p]:
                return None
            return (self.phys[i], self.phys[p], self.gpu_of[i], self.gpu_of[p], nbytes, s)

        self.plan_stages = []
        for steps, _ in self.sched.stages():
            chans = [c for s in steps for i in range(n) if xor_peer(i, s, n) >= 0
                     for c in [chan(i, xor_peer(i, s, n), s)] if c]
            self.plan_stages.append(chans)
        # channels outside the plan's transfer list (the scalar broadcast, routing.hpp:341-353)
        # may fall in steps the schedule elided: one final phase in the same global order
        done = {(c[0], c[1]) for st in self.plan_stages for c in st}
        rest = [c for s in range(1, 1 << max(1, (n - 1).bit_length())) for i in range(n)
                if xor_peer(i, s, n) >= 0 for c in [chan(i, xor_peer(i, s, n), s)] if c and (c[0], c[1]) not in done]
        if rest:
            self.plan_stages.append(rest)
        # every cross-GPU byte this GPU pushes must be on some enumerated channel
        mine = sum(c[4] for st in self.plan_stages for c in st if c[2] == gpu)
        if mine != ex.stats().remote_bytes:
            raise A.ReshardError(A.RS_ERR_INTERNAL, f"staged channels carry {mine} B, executor pushes "
                                                     f"{ex.stats().remote_bytes} B")

    def _ops(self, src, dst):
        n = A.C.c_int64()
        A.check(A.lib().rs_exec_channel_ops(self.ex.h, src, dst, None, 0, A.C.byref(n)))
        arr = (A.C.c_int64 * max(1, n.value))()
        A.check(A.lib().rs_exec_channel_ops(self.ex.h, src, dst, arr, n.value, A.C.byref(n)))
        return list(arr[: n.value])

    def _exchange(self, chans, stream, per_op=False):
        import torch
        import torch.distributed as dist
        # gloo (ranks sharing one GPU) moves host tensors only: the packed channel
        # buffers bounce through host memory there; NCCL sends them from HBM
        host = dist.get_backend(self.group) == "gloo"
        sends, recvs = [], []
        for src, dst, gs, gd, nbytes, _ in chans:
            if gs == self.gpu:
                buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                self.ex.pack(src, dst, buf.data_ptr(), stream)
                if host:
                    torch.cuda.synchronize()
                    buf = buf.cpu()
                sends.append((buf, gd, src, dst))
            elif gd == self.gpu:
                recvs.append((torch.empty(nbytes, dtype=torch.uint8, device="cpu" if host else "cuda"), gs, src, dst))
        if per_op:  # naive: one blocking message per op, in the global channel order
            for src, dst, gs, gd, nbytes, _ in chans:
                if self.gpu not in (gs, gd):
                    continue
                if gs == self.gpu:
                    buf = next(b for b, _, s, d in sends if (s, d) == (src, dst))
                    peer, fn = gd, dist.send
                else:
                    buf = next(b for b, _, s, d in recvs if (s, d) == (src, dst))
                    peer, fn = gs, dist.recv
                off = 0
                for sz in self._ops(src, dst):
                    fn(buf[off:off + sz], peer, group=self.group)
                    off += sz
        else:
            ops = [dist.P2POp(dist.isend, b, g, group=self.group) for b, g, _, _ in sends]
            ops += [dist.P2POp(dist.irecv, b, g, group=self.group) for b, g, _, _ in recvs]
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        for buf, _, src, dst in recvs:
            if host:
                buf = buf.to("cuda")
                torch.cuda.synchronize()
            self.ex.unpack(src, dst, buf.data_ptr(), stream)
            if host:
                torch.cuda.synchronize()  # the bounce buffer must outlive the unpack

    def run(self, stream: int = 0) -> None:
        self.ex.run(stream)  # same-GPU moves, fused
        for chans in self.plan_stages:
            if self.mode == "async":
                self._exchange(chans, stream)
            elif self.mode == "sync":
                for s in sorted({c[5] for c in chans}, key=lambda x: [c[5] for c in chans].index(x)):
                    self._exchange([c for c in chans if c[5] == s], stream)
            else:
                self._exchange(chans, stream, per_op=True)


def job_token(tag: str = "0", group=None) -> str:
    """A per-job token for the abstract-namespace socket names and payloads: rank 0 draws a
    random nonce and broadcasts it (collective over `group`), so two jobs of the same user
    on one node never connect to each other's listeners, and a payload carrying another
    token is rejected."""
    import secrets

    import torch.distributed as dist
    obj = [secrets.token_hex(8) if dist.get_rank(group) == 0 else None]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(obj, src=src, group=group)
    return f"{tag}-{obj[0]}"


def _split_token(payload: bytes, token: str) -> bytes:
    head, sep, rest = payload.partition(b"\0")
    if not sep or head.decode(errors="replace") != token:
        raise A.ReshardError(A.RS_ERR_INTERNAL, "fdx payload from a different job (token mismatch)")
    return rest


def global_stage_cuts(arena, world: int):
    """A barrier is needed before a stage if ANY GPU's aliasing needs it (each GPU plans
    only the chunks it hosts): element-wise max of the cuts over all ranks."""
    cuts = [arena.stage_cuts(0), arena.stage_cuts(1)]
    if world < 2:
        return cuts
    import torch
    import torch.distributed as dist
    n0 = len(cuts[0])
    t = torch.tensor(cuts[0] + cuts[1], dtype=torch.int32, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    v = t.tolist()
    return [v[:n0], v[n0:]]


def exchange_arena(arena, rank: int, world: int, tag: str) -> None:
    """Share every GPU's arena buffers with every other GPU: POSIX descriptors of the
    VMM allocations over Unix sockets (fdx), mapped by the receiver (import_peer).
    Bind executors afterwards with arena.bind(fwd, bwd, global_stage_cuts(arena, world))."""
    import threading

    import torch.distributed as dist

    from .api import fdx_close, fdx_listen, fdx_recv, fdx_send
    if world < 2:
        return
    tok = job_token(tag)
    sock = fdx_listen(f"reshard-{tok}-{rank}")
    dist.barrier()
    errors = []

    def receive():
        try:
            for _ in range(world - 1):
                fds, table = fdx_recv(sock)
                try:
                    table = _split_token(table, tok)
                except BaseException:
                    for fd in fds:
                        os.close(fd)
                    raise
                arena.import_peer(fds, table)
        except BaseException as e:  # surfaced below
            errors.append(e)

    t = threading.Thread(target=receive, name="arena-import")
    t.start()
    for peer in range(world):
        if peer == rank:
            continue
        fds, table = arena.export()
        try:
            fdx_send(f"reshard-{tok}-{peer}", fds, tok.encode() + b"\0" + table)
        finally:
            for fd in fds:
                os.close(fd)
    t.join()
    fdx_close(sock)
    if errors:
        raise errors[0]
    dist.barrier()


def shared_arena(ab: RoutingPlan, ba: Optional[RoutingPlan], rank: int, world: int, device: int, cap_bytes: int = 0,
                 tag: str = "0", chunk_bytes: int = 0, level: Optional[int] = None):
    """Memory-aware arena over `world` GPUs: every GPU plans the buffers it hosts with the
    same schedule level (layer bands x concurrency groups: the cheapest level that fits
    every GPU's cap, max over ranks; `level` forces one ladder level, which must fit),
    then the buffers are shared (exchange_arena). Returns (arena, global stage cuts)."""
    import torch
    import torch.distributed as dist

    from .api import Arena, memory_schedule_costs, memory_schedule_level
    if cap_bytes <= 0:
        cap_bytes = torch.cuda.mem_get_info(device)[0] - (1 << 30)
    # every rank marks the ladder levels that fit its cap and models each level's time
    # (stage groups in sequence, each bound by its busiest GPU's NVLink or HBM, with the
    # union of every GPU's stage cuts: the same on every rank); the group takes the
    # fastest level feasible on all GPUs
    costs = memory_schedule_costs(ab, ba, world, rank, chunk_bytes)
    need = [b for b, _ in costs]
    ok = torch.tensor([1 if x <= cap_bytes else 0 for x in need], dtype=torch.int32, device="cuda")
    est = torch.tensor([t for _, t in costs], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        dist.all_reduce(est, op=dist.ReduceOp.MAX)
    fits = [i for i, v in enumerate(ok.tolist()) if v]
    if not fits:
        raise A.ReshardError(A.RS_ERR_BUDGET, f"infeasible budget on some GPU (this GPU needs >= {min(need) / 1e9:.2f} GB, "
                                              f"cap {cap_bytes / 1e9:.2f} GB)")
    t = est.tolist()
    if level is not None:
        if level not in fits:
            raise A.ReshardError(A.RS_ERR_BUDGET, f"schedule level {level} does not fit the cap on every GPU")
        lv = level
    else:
        lv = min(fits, key=lambda i: (t[i], i))
    bands, k = memory_schedule_level(ab, lv, world)
    arena = Arena.multi(ab, ba, world, rank, device, cap_bytes=cap_bytes, chunk_bytes=chunk_bytes, groups=k, bands=bands)
    exchange_arena(arena, rank, world, tag)
    return arena, global_stage_cuts(arena, world)


def share_buffers(tr: "Transition", rank: int, world: int, device: int, tag: str = "0", group=None,
                  adopt: Optional[dict] = None) -> dict:
    """Shareable VMM buffers for every buffer of the virtual ranks this GPU hosts (both
    sides); `adopt` maps (side, rank, buf) to VmmBuffers to reuse (the current state as
    the source). Destination buffers are passed to every peer by POSIX descriptor (fdx)
    and mapped there, so the fused push writes into them; everything is bound into
    tr.ex. Collective over `group` (gloo in the EDM side thread). Returns
    {(side, rank, buf): VmmBuffer} for local buffers plus ("peer", side, rank, buf) keys
    for the mapped peers' buffers (keep it alive while the executor runs)."""
    import json
    import threading

    import torch.distributed as dist

    from .api import VmmBuffer, fdx_close, fdx_listen, fdx_recv, fdx_send
    adopt = adopt or {}
    out = {}
    ex = tr.ex
    table = []
    for side in (A.SIDE_SRC, A.SIDE_DST):
        nr = tr.plan.summary.src_world if side == A.SIDE_SRC else tr.plan.summary.dst_world
        for r in range(nr):
            for b in range(6):
                _, n, g = ex.buffer(side, r, b)
                if not n or g != ex.gpu:
                    continue
                buf = adopt.get((side, r, b))
                if buf is None or buf.nbytes < n:
                    buf = VmmBuffer.alloc(device, n)
                out[(side, r, b)] = buf
                ex.bind(side, r, b, buf.ptr, n)
                if side == A.SIDE_DST:
                    table.append((r, b, n))
    if world < 2:
        return out
    tok = job_token(tag, group)
    sock = fdx_listen(f"reshard-vmm-{tok}-{rank}")
    dist.barrier(group=group)
    errors = []
    received = []

    def receive():
        try:
            for _ in range(world - 1):
                fds, payload = fdx_recv(sock)
                try:
                    payload = _split_token(payload, tok)
                except BaseException:
                    for fd in fds:
                        os.close(fd)
                    raise
                rows = json.loads(payload.decode())  # plain data: no code runs on receipt
                for fd, (r, b, n) in zip(fds, rows):
                    received.append((r, b, n, VmmBuffer.import_fd(fd, n, device)))
        except BaseException as e:  # surfaced below
            errors.append(e)

    t = threading.Thread(target=receive, name="vmm-import")
    t.start()
    for peer in range(world):
        if peer == rank:
            continue
        fds = [out[(A.SIDE_DST, r, b)].export_fd() for r, b, _ in table]
        try:
            fdx_send(f"reshard-vmm-{tok}-{peer}", fds, tok.encode() + b"\0" + json.dumps(table).encode())
        finally:
            for fd in fds:
                os.close(fd)
    t.join()
    fdx_close(sock)
    if errors:
        raise errors[0]
    for r, b, n, buf in received:
        out[("peer", A.SIDE_DST, r, b)] = buf
        ex.bind(A.SIDE_DST, r, b, buf.ptr, n)
    dist.barrier(group=group)
    return out


def setup_multicast(source, ex: Executor, rank: int, world: int, device: int, tag: str = "0", min_payload: int = 0,
                    group=None):
    """Broadcast promotion over NVLS multicast for the executor's broadcast groups
    (Executor.bcast_groups): per group the root GPU creates a multicast object and passes
    it to the members (fdx); every member adds its device; after a barrier each binds its
    buffer (root: the source, members: the destination ranks' buffers, equal layouts);
    the root maps it and its executor stores the group once through the multicast address.
    `source` holds the buffers: an Arena (Arena.multi) or the dict of share_buffers().
    Collective over `group`. Returns the objects to keep alive (close() them before the
    buffers go away); call ex.prepare() afterwards."""
    import threading

    import torch.distributed as dist

    from .api import Arena, Multicast, fdx_close, fdx_listen, fdx_recv, fdx_send
    arena = source if isinstance(source, Arena) else None
    gran = 2 << 20
    groups = [g for g in ex.bcast_groups() if g.payload_bytes >= min_payload]
    mcs = {}
    if arena is not None:
        size = {g.id: arena.bind_size(0, g.root_rank, g.buf) for g in groups}
    else:
        size = {g.id: (g.buffer_bytes + gran - 1) // gran * gran for g in groups}

    def bind(mc, side, r, b):
        if arena is not None:
            mc.bind_arena(arena, side, r, b)
        else:
            mc.bind_vmm(source[(side, r, b)])

    expect = sum(1 for g in groups if rank in list(g.member_gpu[: g.n_members]) and g.root_gpu != rank)
    tok = job_token(tag, group)
    sock = fdx_listen(f"reshard-mc-{tok}-{rank}")
    dist.barrier(group=group)
    errors = []

    def receive():
        try:
            for _ in range(expect):
                fds, payload = fdx_recv(sock)
                try:
                    payload = _split_token(payload, tok)
                except BaseException:
                    for fd in fds:
                        os.close(fd)
                    raise
                gid = int(payload.decode())
                mcs[gid] = Multicast.import_fd(fds[0], size[gid])
        except BaseException as e:  # surfaced below
            errors.append(e)

    t = threading.Thread(target=receive, name="mc-import")
    t.start()
    for g in groups:
        if g.root_gpu != rank:
            continue
        members = sorted(set(g.member_gpu[: g.n_members]))
        mc = Multicast.create(size[g.id], len(members) + 1)
        mcs[g.id] = mc
        for peer in members:
            fd = mc.export_fd()
            try:
                fdx_send(f"reshard-mc-{tok}-{peer}", [fd], tok.encode() + b"\0" + str(g.id).encode())
            finally:
                os.close(fd)
    t.join()
    fdx_close(sock)
    if errors:
        raise errors[0]
    for gid in sorted(mcs):
        mcs[gid].add_device(device)
    dist.barrier(group=group)
    by_id = {g.id: g for g in groups}
    for gid in sorted(mcs):
        g = by_id[gid]
        if g.root_gpu == rank:
            bind(mcs[gid], A.SIDE_SRC, g.root_rank, g.buf)
        for k in range(g.n_members):
            if g.member_gpu[k] == rank:
                bind(mcs[gid], A.SIDE_DST, g.member_rank[k], g.buf)
    dist.barrier(group=group)
    for gid in sorted(mcs):
        if by_id[gid].root_gpu == rank:
            ex.set_multicast(gid, mcs[gid].map(device))
    return [mcs[k] for k in sorted(mcs)]


def device_barrier(rank: int, world: int, device: int, group=None):
    """The device-side SynchronizeAll of this rank (api.DeviceBarrier), with every peer's
    flag array mapped (handles exchanged over `group`). Collective."""
    import torch.distributed as dist

    from .api import DeviceBarrier
    b = DeviceBarrier(rank, world, device)
    if world > 1:
        blobs: List[Optional[bytes]] = [None] * world
        dist.all_gather_object(blobs, b.export(), group=group)
        for peer, blob in enumerate(blobs):
            b.import_peer(peer, blob)
    return b


def run_stages(ex: Executor, stream: int, world: int, barrier=None) -> None:
    """Memory-aware stages across GPUs: a stage may write chunks that the previous stage
    read on another GPU, so every stage boundary is a global barrier — on the device
    (`barrier`, a DeviceBarrier: nothing returns to the host between stages) or, without
    one, a host synchronize + dist.barrier."""
    import torch
    import torch.distributed as dist
    for s in range(ex.num_stages()):
        ex.run_stage(s, stream)
        if world > 1:
            if barrier is not None:
                barrier(stream)
            else:
                torch.cuda.synchronize()
                dist.barrier()
    # replica dedup: the copies from each GPU's primary replica, once every stage has landed
    # (a later write than planned never clobbers live data; the primary's chunks are final).
    # Local to each GPU and ordered on its stream: whatever reads them next (a push from
    # this GPU) follows in stream order, so no barrier is needed after.
    ex.run_dup(stream)


def run_releasing(ex: Executor, arena, stream) -> int:
    """A one-way transition on one GPU that hands consumed source memory back while it runs
    (Algorithm 1 FreeObsoleteBuffers): every memory-aware stage is
    enqueued at once with an event after each; the host then waits for stage s and
    releases the old-layout chunks s made dead while the GPU runs stage s+1.
    `stream` is a torch stream. Returns the bytes released."""
    import torch
    evs = []
    for s in range(ex.num_stages()):
        ex.run_stage(s, stream.cuda_stream)
        e = torch.cuda.Event()
        e.record(stream)
        evs.append(e)
    freed = 0
    for s, e in enumerate(evs):
        e.synchronize()
        freed += arena.release_through(s)
    return freed


def run_dedup_early(ex: Executor, stream, side_stream, group=None) -> None:
    """One transition with early replica dedup (Executor.set_replica_dedup(early=True)):
    stage 0 = the pushes of regions other ranks on the destination GPU copy plus most of the
    rest, stage 1 = a tail of this GPU's other pushes sized to hide the copies. The host waits for stage 0 only, meets every rank at a barrier (use a gloo
    `group`: an NCCL barrier kernel would queue behind the stage-1 copy kernel, which holds
    every SM), then runs the replica copies on `side_stream` while stage 1 is still
    pushing. `stream` / `side_stream` are torch streams on this rank's device; on return
    `stream` is ordered after the copies. Call it on EVERY rank."""
    import torch
    import torch.distributed as dist
    if ex.num_stages() != 2:
        raise A.ConfigError(A.RS_ERR_CONFIG, "run_dedup_early needs set_replica_dedup(True, early=True) before prepare")
    done0 = torch.cuda.Event()
    ex.run_stage(0, stream.cuda_stream)
    done0.record(stream)
    ex.run_stage(1, stream.cuda_stream)
    done0.synchronize()
    dist.barrier(group=group)
    side_stream.wait_event(done0)
    ex.run_dup(side_stream.cuda_stream)
    stream.wait_stream(side_stream)


def local_ranks(plan: RoutingPlan, ex: Executor, side: int) -> List[int]:
    n = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
    return [r for r in range(n) if ex.buffer(side, r, A.BUF_PARAM)[2] == ex.gpu]


def colocation(traffic: List[List[int]], n_gpus: int, nvlink_gbs: float = 690.0,
               hbm_gbs: float = 6200.0) -> List[List[int]]:
    """Which physical devices share each GPU when there are fewer GPUs than devices (the
    8-device transitions at N = 2, 4): the equal-size grouping whose busiest GPU is fastest
    under the arena time model's bounds (NVLink out, NVLink in, HBM = on-GPU copies read and
    written + peer traffic), from the plan's device traffic matrix (RoutingPlan.traffic()).
    Ties keep the first grouping in enumeration order, contiguous blocks first, so every
    rank derives the same answer. Returns the groups, GPU by GPU (sorted device ids)."""
    import itertools
    n = len(traffic)
    if n_gpus <= 1 or n_gpus >= n or n % n_gpus:  # one GPU, one device per GPU, or uneven
        per = -(-n // max(1, n_gpus))  # the executor's blocks: device // ceil(n / n_gpus)
        return [list(range(g * per, min(n, (g + 1) * per))) for g in range(n_gpus)]
    contiguous = [list(range(g * (n // n_gpus), (g + 1) * (n // n_gpus))) for g in range(n_gpus)]
    size = n // n_gpus

    def partitions(rest):
        if not rest:
            yield []
            return
        for comb in itertools.combinations(rest[1:], size - 1):
            g = (rest[0],) + comb
            for p in partitions([x for x in rest if x not in g]):
                yield [list(g)] + p

    def seconds(groups):  # the busiest GPU's bound (bytes / (GB/s) -> ns; only compared)
        of = {d: i for i, g in enumerate(groups) for d in g}
        out, inn, loc = [0] * n_gpus, [0] * n_gpus, [0] * n_gpus
        for s in range(n):
            for d in range(n):
                b = traffic[s][d]
                if of[s] == of[d]:
                    loc[of[s]] += b
                else:
                    out[of[s]] += b
                    inn[of[d]] += b
        return max(max(out[g] / nvlink_gbs, inn[g] / nvlink_gbs, (2 * loc[g] + out[g] + inn[g]) / hbm_gbs)
                   for g in range(n_gpus))

    import math
    if math.comb(n - 1, size - 1) ** (n_gpus - 1) > 200000:  # too many groupings to try
        return contiguous
    best, best_t = contiguous, seconds(contiguous)
    for p in partitions(list(range(n))):
        t = seconds(p)
        if t < best_t * (1 - 1e-12):
            best, best_t = p, t
    return best


def colocated_world(groups: List[List[int]]) -> List[int]:
    """Device ids for an identity world map relabelled so the executor's contiguous blocks
    (device // devices-per-GPU) are `groups`: entry r is the device that hosts world rank r
    (old and new configuration alike)."""
    size = len(groups[0])
    new_id = {}
    for g, devs in enumerate(groups):
        for i, d in enumerate(devs):
            new_id[d] = g * size + i
    return [new_id[r] for r in range(len(new_id))]
