"""Multi-process host logic on CPU (gloo, world_size 2): every rank derives the same
plan independently (determinism replaces coordination), and the
per-GPU push partition covers every byte of the transition exactly once."""
import hashlib
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layers, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18815_b200 import scenarios as S
    from paper_2605_18815_b200.api import RoutingPlan
    plan = RoutingPlan.from_scenario(S.config2(layers))
    sha = hashlib.sha256(plan.dump().encode()).hexdigest()
    st = plan.placement(world, rank)
    mine = {"sha": sha, "local": st.local_bytes, "out": st.out_bytes, "in": st.in_bytes,
            "moved": plan.bytes_moved(), "retained": plan.bytes_retained()}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    if rank == 0:
        q.put(allv)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_replicated_plan_and_push_partition(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 2, q)) for r in range(world)]
    for p in procs:
        p.start()
    allv = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len({v["sha"] for v in allv}) == 1
    assert sum(v["out"] for v in allv) == sum(v["in"] for v in allv) > 0
    moved, retained = allv[0]["moved"], allv[0]["retained"]
    total = sum(v["local"] + v["out"] for v in allv)
    # every plan byte and every retained byte is copied exactly once; the scalar blob is
    # counted in bytes_moved for the 7 receivers and copied to all 8 destination ranks
    assert total == moved - 7 * 64 + retained + 8 * 64


def test_placement_single_gpu_is_all_local():
    from paper_2605_18815_b200 import scenarios as S
    from paper_2605_18815_b200.api import RoutingPlan
    plan = RoutingPlan.from_scenario(S.config2(1))
    st = plan.placement(1, 0)
    assert st.out_bytes == 0 and st.in_bytes == 0
    assert st.local_bytes == plan.bytes_moved() - 7 * 64 + plan.bytes_retained() + 8 * 64


def _fdx_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18815_b200.api import fdx_close, fdx_listen, fdx_recv, fdx_send
    sock = fdx_listen(f"reshard-test-{port}-{rank}")
    dist.barrier()
    if rank == 0:
        r, w = os.pipe()
        os.write(w, b"descriptor crossed the process boundary")
        os.close(w)
        fdx_send(f"reshard-test-{port}-1", [r] * 300, b"payload")  # > one SCM_RIGHTS batch
        os.close(r)
    else:
        fds, payload = fdx_recv(sock)
        q.put((len(fds), payload, os.read(fds[0], 100)))
        for fd in fds:
            os.close(fd)
    fdx_close(sock)
    dist.barrier()
    dist.destroy_process_group()


def test_fdx_passes_descriptors_between_processes():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fdx_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    n, payload, data = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert n == 300 and payload == b"payload" and data == b"descriptor crossed the process boundary"


def test_memory_plan_per_gpu_is_safe():
    from paper_2605_18815_b200 import scenarios as S
    from paper_2605_18815_b200.api import RoutingPlan
    import ctypes as C
    from paper_2605_18815_b200 import _capi as A
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    st, viol = A.ArenaStats_t(), C.c_int64()
    A.check(A.lib().rs_memory_plan(ab.h, ba.h, 0, 0, C.byref(st), C.byref(viol), None, None, 0))
    assert viol.value == 0



def test_placement_covers_d2_plan_exactly():
    """The way back (DP2xTP4 -> TP8, D2 extension): the ops cover every plan byte and
    every retained byte once (flagged tensors' runs come from the D2 list)."""
    from paper_2605_18815_b200 import scenarios as S
    from paper_2605_18815_b200.api import RoutingPlan
    for L in (1, 2):
        plan = RoutingPlan.from_scenario(S.config2(L).reversed(), allow_oversourced=True)
        st = plan.placement(1, 0)
        assert st.local_bytes == plan.bytes_moved() - 7 * 64 + plan.bytes_retained() + 8 * 64


def _token_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_18815_b200.api import fdx_close, fdx_listen, fdx_recv, fdx_send
    from paper_2605_18815_b200.runtime import _split_token, job_token
    tok = job_token("t")
    toks = [None] * world
    dist.all_gather_object(toks, tok)
    ok = len(set(toks)) == 1 and tok.startswith("t-") and len(tok) > 10
    # a payload from another job (other token) is rejected; one from this job passes
    sock = fdx_listen(f"reshard-tok-{tok}-{rank}")
    dist.barrier()
    import threading
    got = []

    def receive():  # the runtime receives on a thread too (a send waits for its reader)
        for _ in range(2):
            fds, payload = fdx_recv(sock)
            for fd in fds:
                os.close(fd)
            try:
                got.append(_split_token(payload, tok))
            except Exception:
                got.append(None)

    th = threading.Thread(target=receive)
    th.start()
    peer = (rank + 1) % world
    r, w = os.pipe()
    fdx_send(f"reshard-tok-{tok}-{peer}", [r], tok.encode() + b"\0" + b"hello")
    fdx_send(f"reshard-tok-{tok}-{peer}", [w], b"t-other\0" + b"evil")
    os.close(r)
    os.close(w)
    th.join()
    fdx_close(sock)
    ok = ok and got == [b"hello", None]
    res = [None] * world
    dist.all_gather_object(res, ok)
    if rank == 0:
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_job_token_guards_fd_exchange():
    """Two concurrent jobs never share socket names or accept each other's payloads: rank 0
    draws a per-job token that every rank uses in the socket names, and payloads carrying
    another token are rejected."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_token_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == [True, True]
