"""GPU parity: the sm_100a executor (through the C ABI) against canon payloads and
against the oracle's CPU executor, bit for bit; GPU planner against the reference."""
import hashlib
import os

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import pyoracle as O  # noqa: E402
from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Executor, RoutingPlan  # noqa: E402

SEED = 0xC0FFEE


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def _run_single_gpu(sc, with_grads=False, allow=False, bind_torch=False):
    plan = RoutingPlan.from_scenario(sc, allow_oversourced=allow)
    ex = Executor(plan, with_grads=with_grads)
    tensors = {}
    if bind_torch:  # caller-owned buffers (the framework-registration path)
        for side, n in ((0, plan.summary.src_world), (1, plan.summary.dst_world)):
            for r in range(n):
                for b in range(6):
                    _, nbytes, _ = ex.buffer(side, r, b)
                    if nbytes:
                        # zeroed like the oracle's buffers: the 16-B segment padding stays 0
                        t = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
                        tensors[(side, r, b)] = t
                        ex.bind(side, r, b, t.data_ptr(), nbytes)
    ex.alloc()
    ex.fill(A.SIDE_SRC, SEED)
    bad, _ = ex.verify(A.SIDE_SRC, SEED)
    assert bad == 0
    ex.prepare()
    ex.run()
    torch.cuda.synchronize()
    bad, first = ex.verify(A.SIDE_DST, SEED)
    assert bad == 0, f"{bad} mismatches, first flat index {first}"
    return plan, ex, tensors


def _ranks():
    """Rank processes for the N>1 checks: one per GPU (up to 4); on a 1-GPU box 4 rank
    processes share the device (gloo plumbing, cudaIpc / VMM pushes between processes),
    so the N>1 code paths run on every box the driver leases."""
    n = torch.cuda.device_count()
    return min(n, 4) if n >= 2 else 4


def _oracle_dst(sc, with_grads=False, allow=False):
    s = O.OScenario(sc.text())
    p = O.OPlan(s, allow)
    src = O.OState(s, 0, with_grads)
    src.load(SEED)
    dst = O.OState(s, 1, with_grads)
    O.execute(p, src, dst, nthreads=4)
    return dst


@pytest.mark.parametrize("allow", [False, True])
def test_tiny_gpt_bit_exact_vs_oracle(allow):
    sc = S.config1(zero=allow)
    plan, ex, tensors = _run_single_gpu(sc, allow=allow, bind_torch=True)
    dst = _oracle_dst(sc, allow=allow)
    for r in range(plan.summary.dst_world):
        for b in range(6):
            if (1, r, b) in tensors:
                got = tensors[(1, r, b)].cpu().numpy().tobytes()
                assert got == dst.buffer(r, b), (r, b)


def test_golden_campaign_on_gpu(golden):
    n = 0
    for e in golden:
        if e["rc"] != 0 or e["group"] != "campaign":
            continue
        grads = "grads=migrate" in e["scenario"]
        _run_single_gpu(e["scenario"], with_grads=grads)
        n += 1
    assert n >= 60


def test_llama8b_two_layers_bit_exact():
    """North-star shape at L=2: every destination buffer of all 8 ranks equals the oracle's."""
    sc = S.config2(2)
    plan, ex, tensors = _run_single_gpu(sc, bind_torch=True)
    dst = _oracle_dst(sc)
    n = 0
    for r in range(plan.summary.dst_world):
        for b in range(6):
            if (1, r, b) not in tensors:
                continue
            got = tensors[(1, r, b)].cpu().numpy().tobytes()
            assert hashlib.sha256(got).digest() == hashlib.sha256(dst.buffer(r, b)).digest(), (r, b)
            n += 1
    assert n == 8 * 5


def test_qwen_moe_one_layer():
    _run_single_gpu(S.config4(1))


def test_round_trip_restores_state():
    sc = S.config2(1)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)  # way back hits D2
    e1, e2 = Executor(ab), Executor(ba)
    keep = {}
    for side_ab, side_ba in ((0, 1), (1, 0)):
        n = ab.summary.src_world if side_ab == 0 else ab.summary.dst_world
        for r in range(n):
            for b in range(6):
                _, nbytes, _ = e1.buffer(side_ab, r, b)
                if nbytes:
                    t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                    keep[(side_ab, r, b)] = t
                    e1.bind(side_ab, r, b, t.data_ptr(), nbytes)
                    e2.bind(side_ba, r, b, t.data_ptr(), nbytes)
    e1.fill(0, SEED)
    e1.prepare()
    e2.prepare()
    e1.run()
    torch.cuda.synchronize()
    for (side, r, b), t in keep.items():
        if side == 0:
            t.zero_()
    torch.cuda.synchronize()
    e2.run()
    torch.cuda.synchronize()
    assert e1.verify(1, SEED)[0] == 0
    assert e2.verify(1, SEED)[0] == 0  # A restored bit-exactly


def test_gpu_planner_full_config2(golden):
    """GPU batched planner == host expansion == oracle at full L=32 (1.84M runs)."""
    sc = S.config2(32)
    p = RoutingPlan.from_scenario(sc)
    d_gpu = p.dump(device=0)
    d_host = p.dump(device=-1)
    assert d_gpu == d_host
    o = O.OPlan(O.OScenario(sc.text()))
    assert hashlib.sha256(d_gpu.encode()).digest() == hashlib.sha256(o.dump().encode()).digest()


def test_gpu_planner_golden(golden):
    n = 0
    for e in golden:
        if e["rc"] != 0 or e["ref_seconds"] > 60:
            continue
        p = RoutingPlan.from_scenario(e["scenario"])
        assert hashlib.sha256(p.dump(device=0).encode()).hexdigest() == e["sha256"], e["name"]
        n += 1
    assert n >= 90


def test_no_gpu_no_fallback_message():
    # the executor refuses to run without its CUDA library; here we only check the
    # error path for an invalid placement is a clean ConfigError
    plan = RoutingPlan.from_scenario(S.config1())
    with pytest.raises(A.ConfigError):
        Executor(plan, n_gpus=2, gpu=5)


def test_arena_round_trip_aliased():
    """Memory-aware arena: new-layout chunks alias dead old-layout chunks; a round
    trip through stages is still bit-exact."""
    from paper_2605_18815_b200.api import Arena
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    # cap = the most-aliased plan's footprint: the arena must pick one group per stage
    # (with room to spare it would run everything as one stage and alias nothing)
    from paper_2605_18815_b200.api import memory_plan
    most, viol, _, _ = memory_plan(ab, ba, chunk_bytes=2 << 20, groups=0)
    assert viol == 0
    arena = Arena(ab, ba, chunk_bytes=2 << 20, cap_bytes=most.physical_bytes)
    st = arena.stats()
    assert st.aliased_bytes > 0 and st.physical_bytes == most.physical_bytes
    assert list(st.stage_groups) == list(most.stage_groups)
    assert st.physical_bytes < st.a_bytes + st.b_bytes
    e1, e2 = Executor(ab), Executor(ba)
    arena.bind(e1, e2)
    assert e1.num_stages() == st.stage_groups[0] and e2.num_stages() == st.stage_groups[1]
    e1.fill(0, SEED)
    e1.prepare()
    e2.prepare()
    for _ in range(2):
        e1.run()
        torch.cuda.synchronize()
        assert e1.verify(1, SEED)[0] == 0
        e2.run()
        torch.cuda.synchronize()
        assert e2.verify(1, SEED)[0] == 0


@pytest.mark.parametrize("colocate", [[], ["--colocate"]])
def test_multi_gpu_push_over_nvlink(colocate):
    """N>1 (one process per GPU; on a 1-GPU box the rank processes share it), every local
    buffer byte-compared with the oracle; with --colocate the 8-device scenarios are grouped
    onto the GPUs as bench.py does (runtime.colocation, relabelled world maps)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", "29531" if not colocate else "29532",
                        os.path.join(root, "tests", "mgpu_check.py"), "2", "--oracle"] + colocate,
                       capture_output=True, text=True, timeout=900)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    if colocate:
        assert "COLOCATED 0" not in r.stdout and "COLOCATED" in r.stdout, r.stdout[-3000:]


@pytest.mark.parametrize("dedup", [[], ["--dedup"]])
def test_multi_gpu_random_moe_models(dedup):
    """The random toy MoE models of test_random_moe_models_vs_oracle_buffers pushed across
    GPUs (one process per GPU, cudaIpc peer stores), forward and back, bit-exact."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", "29537",
                        os.path.join(root, "tests", "mgpu_check.py"), "1", "--random", "16", "--oracle"] + dedup,
                       capture_output=True, text=True, timeout=900)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_multi_gpu_arena_stages():
    """N>1 memory-aware arena: VMM buffers shared across processes by POSIX descriptors,
    eager-free aliasing, one global barrier per stage; skipped on a 1-GPU box."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(root, "tests", "mgpu_arena_check.py"), "2"],
                       capture_output=True, text=True, timeout=900)
    assert "ARENA_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_multicast_broadcast_grow():
    """Broadcast promotion over NVLS multicast (config 3 grow DP4 -> DP8): the joiners'
    parameters leave the root once through a multicast object; bit-exact against canon.
    Needs >= 3 GPUs (a broadcast group spans >= 2 GPUs besides the root)."""
    import json
    import subprocess
    import sys
    n = torch.cuda.device_count()
    if n < 4:
        pytest.skip("needs 4 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
                        "--master-addr", "127.0.0.1", "--master-port", "29535",
                        os.path.join(root, "tools", "bcast_bench.py"), "--layers", "2", "--reps", "2"],
                       capture_output=True, text=True, timeout=900)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads(line[-1])
    assert d["push"]["mismatches"] == 0
    assert d["bcast_groups"] and d["multicast"]["mismatches"] == 0
    assert d["multicast"]["mc_gb_rank0"] > 0
    # replica dedup alone and with multicast: fewer NVLink bytes from the root, same state
    assert d["dedup"]["mismatches"] == 0 and d["dedup_multicast"]["mismatches"] == 0
    assert d["dedup"]["remote_gb_rank0"] < d["push"]["remote_gb_rank0"]


def test_broadcast_groups_need_two_remote_gpus():
    """Broadcast detection (one GPU is enough to list the groups): config 3
    grow at 4 GPUs yields the two per-slot parameter groups rooted at rank 0; at 2 GPUs
    every joiner sits on one GPU and nothing is promoted."""
    from paper_2605_18815_b200 import scenarios as S
    from paper_2605_18815_b200.api import Executor, RoutingPlan
    _, grow = S.config3(2)
    plan = RoutingPlan.from_scenario(grow)
    ex4 = Executor(plan, n_gpus=4, gpu=0, device=0)
    g4 = [g for g in ex4.bcast_groups() if g.payload_bytes > 1 << 20]
    assert [(g.root_rank, g.slot, list(g.member_rank[: g.n_members])) for g in g4] == [(0, 0, [4, 6]), (0, 1, [5, 7])]
    assert all(g.payload_bytes == g4[0].payload_bytes for g in g4)
    ex2 = Executor(plan, n_gpus=2, gpu=0, device=0)
    assert not [g for g in ex2.bcast_groups() if g.payload_bytes > 1 << 20]


def test_multi_gpu_vmm_shared_buffers():
    """N>1 with shareable VMM state buffers mapped by POSIX descriptor (share_buffers)
    instead of cudaIpc; the way back adopts the forward's buffers. Skipped on one GPU."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", "29537",
                        os.path.join(root, "tests", "mgpu_check.py"), "2", "--vmm"],
                       capture_output=True, text=True, timeout=900)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_pack_unpack_single_gpu_staged_channels():
    """Staged (Algorithm 1 buffered) channels packed and unpacked on one GPU: the
    destinations are bit-exact and both kernels move their bytes."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "pack_bench.py"), "--layers", "2", "--reps", "1"],
                       capture_output=True, text=True, timeout=600)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, r.stdout[-2000:] + r.stderr[-2000:]
    d = json.loads(line[-1])
    assert d["verified_mismatches"] == 0 and d["channels"] > 0 and d["channel_bytes"] > 0


def test_single_process_peer_push():
    """One process drives 2 GPUs (peer access, no cudaIpc): the fused push is bit-exact.
    On a one-GPU box both executors sit on device 0 (the one-process multi-executor path)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    extra = [] if torch.cuda.device_count() >= 2 else ["--same-device"]
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "p2p_profile.py"), "--layers", "1", "--reps", "1"] + extra,
                       capture_output=True, text=True, timeout=600)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, r.stdout[-2000:] + r.stderr[-2000:]
    assert json.loads(line[-1])["verified_mismatches"] == 0


def test_gpu_box_planner_equals_host():
    """The batched (dst rank, tensor, src rank) box intersections on the GPU give exactly
    the host plan's box transfers (params, grads, replicated optimizer) — the golden test
    above compares the GPU planner's whole dump with the reference's."""
    for sc in [S.config2(32), S.config4(4), S.config5(8), S.config1(), S.config3(4)[1]] + S.edge_scenarios():
        p = RoutingPlan.from_scenario(sc, allow_oversourced=True)
        ms, n, eq = p.box_routes_timed(0)
        assert eq, sc.name


def test_multi_gpu_replica_dedup():
    """N>1 with replica dedup (one NVLink crossing per destination GPU, local copies after a
    barrier): every scenario's round trip bit-exact. Skipped on one GPU."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", "29539",
                        os.path.join(root, "tests", "mgpu_check.py"), "2", "--dedup"],
                       capture_output=True, text=True, timeout=600)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_multi_gpu_replica_dedup_early():
    """Early replica dedup: the primaries' pushes first, a barrier on them, then the replica
    copies on a second stream while the other pushes continue; round trips bit-exact."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", "29543",
                        os.path.join(root, "tests", "mgpu_check.py"), "2", "--dedup-early"],
                       capture_output=True, text=True, timeout=600)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_cuda_graph_replay_small_transition():
    """The tiny-GPT transition (launch-bound) replayed from a CUDA graph: bit-exact, and
    re-captured after a re-prepare."""
    plan = RoutingPlan.from_scenario(S.config1())
    ex = Executor(plan)
    ex.alloc()
    ex.fill(A.SIDE_SRC, SEED)
    ex.prepare()
    st = torch.cuda.Stream()
    for _ in range(3):
        ex.run_graph(st.cuda_stream)
    st.synchronize()
    assert ex.verify(A.SIDE_DST, SEED)[0] == 0
    ex.prepare()
    ex.run_graph(st.cuda_stream)
    st.synchronize()
    assert ex.verify(A.SIDE_DST, SEED)[0] == 0


def test_execute_one_call():
    """rs_execute: the SPEC execute shape (buffers in, state moved) in one C call."""
    from paper_2605_18815_b200.api import execute
    plan = RoutingPlan.from_scenario(S.config1())
    ex = Executor(plan)  # only to size the buffers and fill / verify the canon payloads
    bufs, keep = [], []
    for side, n in ((0, plan.summary.src_world), (1, plan.summary.dst_world)):
        for r in range(n):
            for b in range(6):
                _, nbytes, _ = ex.buffer(side, r, b)
                if nbytes:
                    t = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
                    keep.append(t)
                    ex.bind(side, r, b, t.data_ptr(), nbytes)
                    bufs.append((side, r, b, t.data_ptr(), nbytes))
    ex.fill(A.SIDE_SRC, SEED)
    torch.cuda.synchronize()
    assert execute(plan, bufs) >= 1
    assert ex.verify(A.SIDE_DST, SEED)[0] == 0


def test_eight_rank_placement_oversubscribed():
    """The N=8 placement (one virtual rank per rank process) with 8 processes on the GPUs
    this box has (ranks share devices; gloo plumbing): every scenario bit-exact."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
                        "--master-addr", "127.0.0.1", "--master-port", "29541",
                        os.path.join(root, "tests", "mgpu_check.py"), "2"],
                       capture_output=True, text=True, timeout=900)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def _oracle_canon_samples(plan, ex, seed, side, per_rank=24, rng_seed=5):
    """Independent spot check of a full-size state against the ORACLE's canon (oracle.c,
    not the product's common.hpp / verify kernel): random elements of random segments of
    every rank of `side`, param bytes and (inside the ZeRO shard) master / m / v, read
    back from HBM. Returns (elements checked, mismatches)."""
    import random
    import struct
    from paper_2605_18815_b200.state import model_tensors, rank_geom, segments
    rng = random.Random(rng_seed)
    tens = model_tensors(plan)
    off, acc = [], 0
    for t in tens:
        off.append(acc)
        n = 1
        for d in t.shape:
            n *= d
        acc += n
    nranks = plan.summary.src_world if side == A.SIDE_SRC else plan.summary.dst_world
    checked = bad = 0
    for r in range(nranks):
        g = rank_geom(plan, side, r)
        segs = segments(plan, side, r)
        for _ in range(per_rank):
            sg = rng.choice(segs)
            t = tens[sg.tensor]
            nd = len(t.shape)
            ext = [sg.box_hi[d] - sg.box_lo[d] for d in range(nd)]
            coord = [sg.box_lo[d] + rng.randrange(ext[d]) for d in range(nd)]
            idx = 0  # row-major index inside the segment's box
            gk = 0   # row-major index inside the whole tensor
            for d in range(nd):
                idx = idx * ext[d] + (coord[d] - sg.box_lo[d])
                gk = gk * t.shape[d] + coord[d]
            k = off[sg.tensor] + gk
            w = t.dtype_bytes
            got = ex.read(side, r, A.BUF_PARAM, sg.param_byte_off + idx * w, w)
            want = (O.canon(seed, k, 0) & ((1 << (8 * w)) - 1)).to_bytes(w, "little")
            checked += 1
            bad += got != want
            li = sg.local_lo + idx
            lo, hi = (g.eshard_lo, g.eshard_hi) if sg.expert else (g.dshard_lo, g.dshard_hi)
            if lo <= li < hi:
                oi = li - lo + ((g.dshard_hi - g.dshard_lo) if sg.expert else 0)
                c1, c2 = O.canon(seed, k, 1), O.canon(seed ^ 0x5EED, k, 1)
                for b, val in ((A.BUF_MASTER, c1 & 0xFFFFFFFF), (A.BUF_M, c1 >> 32), (A.BUF_V, c2 & 0xFFFFFFFF)):
                    checked += 1
                    bad += ex.read(side, r, b, 4 * oi, 4) != struct.pack("<I", val)
    return checked, bad


def test_north_star_full_size_round_trip():
    """BASELINE config 2 at full size (Llama-3-8B, L=32, 112.42 GB of plan bytes; 240.9 GB
    of old + new state) on one B200 through the memory-aware arena. Size-independent
    properties: every destination element equals its canon value after the forward
    transition, and the way back restores every source element bit for bit."""
    import gc
    from paper_2605_18815_b200.api import Arena
    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' cached blocks would shrink the free-HBM cap
    sc = S.config2(32)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    assert ab.bytes_moved() == 112_419_930_560
    arena = Arena(ab, ba, device=0, cap_bytes=0)  # cap 0: free HBM - 1 GiB
    st = arena.stats()
    assert st.a_bytes + st.b_bytes > torch.cuda.get_device_properties(0).total_memory
    assert st.aliased_bytes > 0
    e1, e2 = Executor(ab), Executor(ba)
    arena.bind(e1, e2)
    e1.fill(0, SEED)
    e1.prepare()
    e2.prepare()
    e1.run()
    torch.cuda.synchronize()
    bad, first = e1.verify(1, SEED)
    assert bad == 0, f"forward: {bad} mismatches, first flat index {first}"
    checked, bad = _oracle_canon_samples(ab, e1, SEED, A.SIDE_DST)
    assert checked > 400 and bad == 0, f"forward: {bad} of {checked} sampled elements differ from the oracle's canon"
    e2.run()
    torch.cuda.synchronize()
    bad, first = e2.verify(1, SEED)
    assert bad == 0, f"way back: {bad} mismatches, first flat index {first}"
    checked, bad = _oracle_canon_samples(ba, e2, SEED, A.SIDE_DST)
    assert checked > 400 and bad == 0, f"way back: {bad} of {checked} sampled elements differ from the oracle's canon"


@pytest.mark.parametrize("flags", [[], ["--dedup-early"]])
def test_edm_scale_events_bit_exact(flags):
    """The EDM end to end (BASELINE config 3 at L=2): DP8 -> DP4 -> DP8 on the side thread
    while GEMM steps run, blocking and overlapped; every switch verified against canon."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = "29545" if not flags else "29547"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", port,
                        os.path.join(root, "tools", "edm_bench.py"), "--layers", "2", "--gemm", "2048"] + flags,
                       capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])["results"]
    assert len(res) == 2
    for name, modes in res.items():
        for mode in ("blocking", "overlapped"):
            assert modes[mode]["verified_mismatches"] == 0, (name, mode)
            assert modes[mode]["bytes_moved"] > 0


@pytest.mark.parametrize("seed", range(16))
def test_random_moe_models_vs_oracle_buffers(seed):
    """Random toy MoE models (EP, rank orders, world-size changes; the CPU audits in
    test_spec_kats.py use the same generator) executed on the GPU and compared byte for
    byte with the oracle's CPU executor on every destination buffer."""
    import random
    rng = random.Random(1000 + seed)
    m = S.toy_model(rng, max_layers=4, max_per_layer=4, experts=4)
    src = S.random_cfg(rng, m, max_world=8)
    dst = S.random_cfg(rng, m, max_world=8, zero=src.zero)
    sc = S.Scenario(m, src, dst, world_src=list(range(src.world())), world_dst=list(range(dst.world())))
    plan, ex, tensors = _run_single_gpu(sc, allow=src.zero, bind_torch=True)
    ref = _oracle_dst(sc, allow=src.zero)
    n = 0
    for r in range(plan.summary.dst_world):
        for b in range(6):
            if (1, r, b) in tensors:
                assert tensors[(1, r, b)].cpu().numpy().tobytes() == ref.buffer(r, b), (r, b)
                n += 1
    assert n > 0


def test_promoted_scatter_gather_executed():
    """optimize_primitives' Scatter (TP1 -> TP4, root pushes) and Gather (TP4 -> TP1, root
    pulls over NVLink) executed as primitives across 4 rank processes: bit-exact, and the
    root moves exactly the schedule's promoted bytes (tests/mgpu_collectives_check.py)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
                        "--master-addr", "127.0.0.1", "--master-port", "29549",
                        os.path.join(root, "tests", "mgpu_collectives_check.py"), "4"],
                       capture_output=True, text=True, timeout=600)
    assert "COLL_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("mode", ["async", "naive"])
def test_staged_schedule_transport(mode):
    """Algorithm 1's buffered execution driven by the transition schedule (memory-aware
    stages of XOR steps, per-peer packed channels): NCCL send/recv between GPUs, or on a
    one-GPU box gloo between rank processes sharing the device; every scenario's round
    trip bit-exact (tests/mgpu_check.py --staged)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = "29551" if mode == "async" else "29553"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={_ranks()}",
                        "--master-addr", "127.0.0.1", "--master-port", port,
                        os.path.join(root, "tests", "mgpu_check.py"), "1", "--random", "6", "--staged", "--mode", mode,
                        "--oracle"],
                       capture_output=True, text=True, timeout=900)
    assert "MGPU_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
