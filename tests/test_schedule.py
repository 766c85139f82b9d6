"""Algorithm 1 transition schedule: SPEC KATs (AC5 XOR, AC6
chunking trace, AC7 promotion soundness) and an independent Python restatement of
the schedule checked against the product on the golden campaign."""
import random

import pytest

from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.api import (ReshardError, RoutingPlan, Schedule, memory_aware_chunk,
                                       xor_peer)


# ---------------------------------------------------------------- restatement

def py_steps(n):
    p = 1
    while p < n:
        p <<= 1
    return list(range(1, p))


def py_chunk(steps, cost, avail):
    """PAPER.md:696-717 FChunk, greedy over ascending steps."""
    m = min(avail)
    stages, cur, used = [], [], 0
    for s in steps:
        if cost[s] > m:
            raise ValueError("infeasible budget")
        if used + cost[s] > m and cur:
            stages.append(cur)
            cur, used = [s], cost[s]
        else:
            cur.append(s)
            used += cost[s]
    if cur:
        stages.append(cur)
    return stages, m


# ------------------------------------------------------------------ SPEC KATs

@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8, 12, 16])
def test_xor_properties_and_d4_completeness(n):
    steps = py_steps(n)
    covered = set()
    for s in steps:
        seen = set()
        for i in range(n):
            p = xor_peer(i, s, n)
            if p < 0:
                continue
            assert xor_peer(p, s, n) == i          # Peer(Peer(i,s),s) = i
            assert i not in seen                   # <= 1 active peer per rank per step
            seen.add(i)
            covered.add((min(i, p), max(i, p)))
    assert covered == {(i, j) for i in range(n) for j in range(i + 1, n)}  # every pair gets a step
    # N=4 table; N=5, rank 3 at s=6 -> 5 >= N -> skipped
    if n == 4:
        assert [(i, xor_peer(i, 1, 4)) for i in (0, 2)] == [(0, 1), (2, 3)]
        assert [(i, xor_peer(i, 3, 4)) for i in (0, 1)] == [(0, 3), (1, 2)]
    if n == 5:
        assert xor_peer(3, 6, 5) == -1


def test_chunk_trace_paper():
    # M_avail=[10,8,12], costs [5,4,3] -> min 8 -> [{s1},{s2,s3}]
    stages, m = memory_aware_chunk([1, 2, 3], [5, 4, 3], [10, 8, 12])
    assert m == 8 and stages == [[1], [2, 3]]
    # budget >= total -> one stage; budget == max single -> one step per stage
    assert memory_aware_chunk([1, 2, 3], [5, 4, 3], [100])[0] == [[1, 2, 3]]
    assert memory_aware_chunk([1, 2, 3], [5, 5, 5], [5])[0] == [[1], [2], [3]]
    with pytest.raises(ReshardError, match="infeasible budget"):
        memory_aware_chunk([1, 2], [5, 9], [8])


def _promoted(sc):
    return Schedule(RoutingPlan.from_scenario(sc)).collectives()


def test_forced_collectives():
    W = S.Model("m", [S.Tensor("W", (8, 4), tp=0)])
    # dp 1 -> 4 replication: 1 src, 3 identical dst slices -> Broadcast
    c = _promoted(S.Scenario(W, S.Cfg(dp=1), S.Cfg(dp=4)))
    # (one per logical tensor: the param and its replicated, non-ZeRO optimizer state)
    assert [x["kind"] for x in c] == ["broadcast"] * 2 and c[0]["root"] == 0 and c[0]["participants"] == [0, 1, 2, 3]
    # tp 1 -> 4 split along axis 0: contiguous distinct slices -> Scatter
    c = _promoted(S.Scenario(W, S.Cfg(tp=1), S.Cfg(tp=4)))
    assert [x["kind"] for x in c] == ["scatter"] * 2
    # tp 4 -> 1 merge -> Gather
    c = _promoted(S.Scenario(W, S.Cfg(tp=4), S.Cfg(tp=1)))
    assert [x["kind"] for x in c] == ["gather"] * 2 and c[0]["root"] == 0


# ------------------------------------------------- schedule vs restatement

def _restated(plan, avail, promote=True):
    """Stage structure from an independent restatement over the plan's transfers."""
    tr = plan.transfers()
    parts = sorted({t.src_phys for t in tr} | {t.dst_phys for t in tr} | set(range(0)))
    # participants = WorldMap::participants(): ranks of both worlds (identity maps here)
    n = plan.summary.num_participants
    dev = {p: i for i, p in enumerate(range(n))}
    groups = {}
    for k, t in enumerate(tr):
        groups.setdefault((t.kind, t.tensor), []).append(k)
    promoted = set()
    kinds = []
    for key, idx in sorted(groups.items()):
        if not promote:
            break
        srcs = {dev[tr[k].src_phys] for k in idx}
        dsts = {dev[tr[k].dst_phys] for k in idx}
        regs = [tuple(zip(tr[k].lo[:tr[k].ndim], tr[k].hi[:tr[k].ndim])) for k in idx]
        ident = all(r == regs[0] for r in regs)
        one = len(dsts) == len(idx)

        def contig(rs):
            rs = sorted(rs)
            axis = None
            for a, b in zip(rs, rs[1:]):
                diff = [d for d in range(len(a)) if a[d] != b[d]]
                if len(diff) != 1:
                    return False
                if axis is not None and diff[0] != axis:
                    return False
                axis = diff[0]
                if a[axis][1] != b[axis][0]:
                    return False
            return True
        if len(srcs) == 1 and len(dsts) > 1 and one and ident:
            kinds.append("broadcast")
        elif len(srcs) == 1 and len(dsts) > 1 and one and contig(regs):
            kinds.append("scatter")
        elif len(srcs) > 1 and len(dsts) == 1 and len(srcs) == len(idx) and contig(regs):
            kinds.append("gather")
        else:
            continue
        promoted.update(idx)
        if sum(tr[k].bytes for k in idx) > min(avail):  # collective buffers share the budget
            raise ValueError("infeasible budget")
    pair = {}
    for k, t in enumerate(tr):
        if k in promoted:
            continue
        i, j = dev[t.src_phys], dev[t.dst_phys]
        pair[(i, j)] = pair.get((i, j), 0) + t.bytes
    cost = {}
    for s in py_steps(n):
        cost[s] = max([pair.get((i, i ^ s), 0) + pair.get((i ^ s, i), 0) for i in range(n) if (i ^ s) < n] + [0])
    steps = [s for s in py_steps(n) if cost[s] > 0]
    stages, m = py_chunk(steps, cost, avail)
    return sorted(kinds), stages, m, sum(pair.values())


def test_schedule_matches_restatement_on_campaign(golden):
    rng = random.Random(7)
    n = 0
    for e in golden:
        if e["rc"] != 0 or e["group"] != "campaign" or "world " in e["scenario"]:
            continue
        plan = RoutingPlan.from_scenario(e["scenario"])
        if plan.num_transfers() == 0:
            continue
        nd = plan.summary.num_participants
        tot = max(1, plan.bytes_moved())
        avail = [rng.randint(tot // 4 + 1, tot) for _ in range(nd)]
        try:
            kinds, stages, m, p2p = _restated(plan, avail)
        except ValueError:
            with pytest.raises(ReshardError, match="infeasible"):
                Schedule(plan, avail)
            continue
        sch = Schedule(plan, avail)
        assert sorted(c["kind"] for c in sch.collectives()) == kinds, e["name"]
        assert [st for st, _ in sch.stages()] == stages, e["name"]
        assert sch.summary.budget == m
        assert sch.summary.p2p_bytes == p2p
        # memory bound + layout agreement (send of i->p == recv of p<-i)
        for k, (steps, cost) in enumerate(sch.stages()):
            assert cost <= m
            for q, s in enumerate(steps):
                for i in range(nd):
                    p, sb, rb = sch.peer(k, q, i)
                    if p >= 0:
                        p2, sb2, rb2 = sch.peer(k, q, p)
                        assert p2 == i and sb == rb2 and rb == sb2
        n += 1
    assert n >= 40


def test_schedule_completeness_north_star():
    plan = RoutingPlan.from_scenario(S.config2(2))
    sch = Schedule(plan, [8 << 30] * 8)
    assert sch.summary.p2p_bytes + sch.summary.collective_bytes == plan.bytes_moved() - 7 * 64
    assert sch.summary.num_fragments == plan.num_transfers()
    d = sch.dump()
    lines = [l for l in d.splitlines() if l.startswith("stage ") or l.startswith("  ")]
    assert len(lines) == plan.num_transfers()  # every transfer exactly once
