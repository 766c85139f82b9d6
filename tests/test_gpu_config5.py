"""BASELINE config 5 (Llama-3-70B TP4xPP2 -> TP8 + ZeRO-1 under a 180 GB/GPU HBM cap) and
the D2 extension on the GPU.

The reference planner throws on config 5 (D2, routing.hpp:318-331: the TP-replicated norms
are covered by several source ZeRO shards); the plans here use the documented extension
(DESIGN.md §2), so their ROUTING is parity unpinned. The STATE is pinned: every destination
element equals its canon value, and on the toy-width models every destination buffer equals
the oracle's CPU executor's byte for byte (oracle.c restates the same extension)."""
import gc
import random

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import pyoracle as O  # noqa: E402
from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Arena, Executor, RoutingPlan  # noqa: E402

SEED = 0x70B


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def _gpu_vs_oracle(sc):
    plan = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    ex = Executor(plan)
    keep = {}
    for side, n in ((0, plan.summary.src_world), (1, plan.summary.dst_world)):
        for r in range(n):
            for b in range(6):
                _, nbytes, _ = ex.buffer(side, r, b)
                if nbytes:
                    t = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")  # padding stays 0 like the oracle's
                    keep[(side, r, b)] = t
                    ex.bind(side, r, b, t.data_ptr(), nbytes)
    ex.fill(A.SIDE_SRC, SEED)
    ex.prepare()
    ex.run()
    torch.cuda.synchronize()
    bad, first = ex.verify(A.SIDE_DST, SEED)
    assert bad == 0, f"{sc.name}: {bad} mismatches, first {first}"
    s = O.OScenario(sc.text())
    src = O.OState(s, 0)
    src.load(SEED)
    dst = O.OState(s, 1)
    O.execute(O.OPlan(s, True), src, dst, nthreads=4)
    n = 0
    for (side, r, b), t in keep.items():
        if side == 1:
            assert t.cpu().numpy().tobytes() == dst.buffer(r, b), (sc.name, r, b)
            n += 1
    return plan, n


def test_config5_shape_full_depth_vs_oracle_buffers():
    """The 70B tensor list at full depth (80 layers, 723 tensors) and toy width, TP4xPP2 ->
    TP8 + ZeRO-1: the reference throws (D2); the extension's GPU state equals the oracle's."""
    m = S.llama3_70b(80, hidden=64, kv=16, ffn=224, vocab=1000)
    sc = S.Scenario(m, S.Cfg(tp=4, pp=2, zero=True), S.Cfg(tp=8, zero=True), name="llama3-70b-shape.tp4pp2-to-tp8")
    with pytest.raises(A.ConfigError, match="not fully sourced"):
        RoutingPlan.from_scenario(sc)
    plan, n = _gpu_vs_oracle(sc)
    assert n == 8 * 5  # 8 destination ranks x (param, master, m, v, scalars)
    _gpu_vs_oracle(sc.reversed())


@pytest.mark.parametrize("seed", range(12))
def test_d2_extension_random_campaign_vs_oracle_buffers(seed):
    """The CPU D2 campaign (test_plan_parity.py) on the GPU: over-sourced ZeRO intervals
    resolved by the extension, destination buffers byte-equal to the oracle's."""
    rng = random.Random(7000 + seed)
    for _ in range(50):
        m = S.toy_model(rng, experts=rng.choice([1, 1, 2, 4]))
        src = S.random_cfg(rng, m, max_world=8, zero=True)
        dst = S.random_cfg(rng, m, max_world=8, zero=True)
        if src.tp > 1:
            break
    sc = S.Scenario(m, src, dst, balance=bool(seed % 2), rpn=rng.choice([2, 4, 8]), name=f"d2-random-{seed}")
    _gpu_vs_oracle(sc)


def test_config5_one_gpu_under_180gb_cap():
    """Config 5 at the per-GPU pressure of the full model on 8 GPUs: at L=8 on one GPU the
    old + new state is 251.8 GB; the memory-aware arena rebuilds it in layer bands inside
    a 180 GB cap (or the free HBM, whichever is lower). Forward and back, every element
    checked against canon."""
    gc.collect()
    torch.cuda.empty_cache()
    sc = S.config5(8)
    ab = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    cap = min(180_000_000_000, torch.cuda.mem_get_info(0)[0] - (1 << 30))
    arena = Arena(ab, ba, device=0, cap_bytes=cap)
    st = arena.stats()
    print(f"config5 L=8: old {st.a_bytes / 1e9:.1f} GB + new {st.b_bytes / 1e9:.1f} GB, physical "
          f"{st.physical_bytes / 1e9:.1f} GB (cap {cap / 1e9:.1f}), bands {st.bands}, aliased {st.aliased_bytes / 1e9:.1f} GB")
    assert st.a_bytes + st.b_bytes > 250e9
    assert st.physical_bytes <= cap and st.aliased_bytes > 0
    e1, e2 = Executor(ab), Executor(ba)
    arena.bind(e1, e2)
    e1.fill(0, SEED)
    e1.prepare()
    e2.prepare()
    e1.run()
    torch.cuda.synchronize()
    bad, first = e1.verify(1, SEED)
    assert bad == 0, f"forward: {bad} mismatches, first flat index {first}"
    from test_gpu_exec import _oracle_canon_samples  # the oracle's canon, sampled from HBM
    checked, bad = _oracle_canon_samples(ab, e1, SEED, A.SIDE_DST)
    assert checked > 200 and bad == 0, f"forward: {bad} of {checked} sampled elements differ from the oracle"
    e2.run()
    torch.cuda.synchronize()
    bad, first = e2.verify(1, SEED)
    assert bad == 0, f"way back: {bad} mismatches, first flat index {first}"
    checked, bad = _oracle_canon_samples(ba, e2, SEED, A.SIDE_DST)
    assert checked > 200 and bad == 0, f"way back: {bad} of {checked} sampled elements differ from the oracle"
    del e1, e2, arena
    gc.collect()
