"""Co-location of the 8-device transitions on fewer GPUs (bench.py at N = 2, 4): the plan's
device traffic matrix, the grouping search, and the relabelled world map that applies it
without changing the plan."""
import dataclasses
import random

from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.api import RoutingPlan
from paper_2605_18815_b200.runtime import colocated_world, colocation


def _cut(m, groups):
    of = {d: i for i, g in enumerate(groups) for d in g}
    out = [0] * len(groups)
    inn = [0] * len(groups)
    for s in range(len(m)):
        for d in range(len(m)):
            if of[s] != of[d]:
                out[of[s]] += m[s][d]
                inn[of[d]] += m[s][d]
    return max(max(out), max(inn))


def test_traffic_matrix_off_diagonal_is_bytes_moved():
    rng = random.Random(77)
    cases = [S.config1(), S.config2(2), S.config4(1), S.config5(2)]
    for _ in range(6):
        m = S.toy_model(rng, experts=rng.choice([1, 2, 4]))
        src = S.random_cfg(rng, m, max_world=8)
        cases.append(S.Scenario(m, src, S.random_cfg(rng, m, max_world=8, zero=src.zero)))
    for sc in cases:
        p = RoutingPlan.from_scenario(sc, allow_oversourced=True)
        t = p.traffic()
        off = sum(t[s][d] for s in range(len(t)) for d in range(len(t)) if s != d)
        assert off == p.bytes_moved(), sc.name


def test_north_star_colocation_halves_the_busiest_gpu_at_n2():
    """TP8 -> DP2xTP4: contiguous blocks put 32.12 GB on the busiest GPU's NVLink at N=2 and
    N=4; the balanced grouping 16.06 GB at N=2 and 24.09 GB at N=4. At N=8 nothing moves."""
    ab = RoutingPlan.from_scenario(S.config2(32))
    t = ab.traffic()
    contiguous = {2: [[0, 1, 2, 3], [4, 5, 6, 7]], 4: [[0, 1], [2, 3], [4, 5], [6, 7]]}
    expect = {2: 16_059_990_016, 4: 24_089_985_024}
    for n in (2, 4):
        g = colocation(t, n)
        assert sorted(d for grp in g for d in grp) == list(range(8))
        assert all(len(grp) == 8 // n for grp in g)
        assert abs(_cut(t, contiguous[n]) - 32_119_980_032) < 1e6
        assert abs(_cut(t, g) - expect[n]) < 1e6, (n, g, _cut(t, g))
    assert colocation(t, 8) == [[d] for d in range(8)]
    assert colocation(t, 1) == [list(range(8))]


def test_relabelled_world_map_keeps_the_plan():
    """The relabelling moves devices between GPUs only: both directions' dumps are
    identical to the identity plan's, and the executor's contiguous blocks become the
    chosen groups."""
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    for n in (2, 4):
        groups = colocation(ab.traffic(), n)
        w = colocated_world(groups)
        assert sorted(w) == list(range(8))
        for g, grp in enumerate(groups):
            assert sorted(w[r] // (8 // n) for r in grp) == [g] * len(grp)
        sc2 = dataclasses.replace(sc, world_src=w, world_dst=w)
        assert RoutingPlan.from_scenario(sc2).dump() == ab.dump()
        back = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
        back2 = RoutingPlan.from_scenario(sc2.reversed(), allow_oversourced=True)
        assert back2.dump() == back.dump()
        # the placement the executor and the roofline see
        pl = [RoutingPlan.from_scenario(sc2).placement(n, g) for g in range(n)]
        assert max(max(p.out_bytes, p.in_bytes) for p in pl) == _cut(ab.traffic(), groups)


def test_traffic_matrix_follows_the_relabelling():
    """Relabelling devices permutes the traffic matrix and nothing else: entry (s, d) of
    the identity plan is entry (w[s], w[d]) of the relabelled one, for random permutations
    of config 2, config 5 and config 3's two events."""
    rng = random.Random(5)
    shrink, grow = S.config3(2)
    for sc in (S.config2(2), S.config5(2)):
        t = RoutingPlan.from_scenario(sc, allow_oversourced=True).traffic()
        for _ in range(3):
            w = list(range(8))
            rng.shuffle(w)
            t2 = RoutingPlan.from_scenario(dataclasses.replace(sc, world_src=w, world_dst=w),
                                           allow_oversourced=True).traffic()
            assert all(t2[w[s]][w[d]] == t[s][d] for s in range(8) for d in range(8))
    w = list(range(8))
    rng.shuffle(w)
    for sc, ws, wd in ((shrink, w, w[:4]), (grow, w[:4], w)):
        t = RoutingPlan.from_scenario(sc).traffic()
        t2 = RoutingPlan.from_scenario(dataclasses.replace(sc, world_src=ws, world_dst=wd)).traffic()
        assert all(t2[w[s]][w[d]] == t[s][d] for s in range(8) for d in range(8))
