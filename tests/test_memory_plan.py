"""Memory-aware arena plan on the host (no GPU): the plan-time eager-free aliasing is
checked by an independent chunk-level replay of the staged execution."""
import pytest

from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.api import RoutingPlan, memory_plan


def test_north_star_fits_one_gpu_and_is_safe():
    sc = S.config2(32)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    st, viol, oa, ob = memory_plan(ab, ba)
    assert viol == 0
    assert st.physical_bytes < 180e9 < st.a_bytes + st.b_bytes  # 240.9 GB old+new -> fits one B200
    assert sorted(oa) == list(range(8)) and sorted(ob) == list(range(8))


@pytest.mark.parametrize("chunk", [2 << 20, 32 << 20, 256 << 20])
def test_replay_safe_across_chunk_sizes(chunk):
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    st, viol, _, _ = memory_plan(ab, ba, chunk_bytes=chunk)
    assert viol == 0 and st.aliased_bytes > 0


def test_replay_safe_on_campaign(golden):
    n = 0
    for e in golden:
        if e["rc"] != 0 or e["group"] != "campaign" or "world " in e["scenario"]:
            continue
        ab = RoutingPlan.from_scenario(e["scenario"])
        # one-way plans on tiny chunks exercise partial-buffer lifetimes
        st, viol, _, _ = memory_plan(ab, None, chunk_bytes=4096)
        assert viol == 0, e["name"]
        n += 1
    assert n >= 40


@pytest.mark.parametrize("n_gpus", [1, 2, 4])
@pytest.mark.parametrize("groups", [0, 1, 2, 3])
def test_grouped_plans_per_gpu_are_safe(n_gpus, groups):
    """Every GPU's share of the arena, with the stage order coarsened into concurrency
    groups, replays without reading clobbered data; fewer groups never alias more."""
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    for g in range(n_gpus):
        st, viol, _, _ = memory_plan(ab, ba, chunk_bytes=8 << 20, n_gpus=n_gpus, gpu=g, groups=groups)
        assert viol == 0
        if groups == 1:
            assert st.aliased_bytes == 0 and list(st.stage_groups) == [1, 1]
        assert 1 <= st.stage_groups[0] <= 8


def test_min_groups_fits_cap():
    from paper_2605_18815_b200.api import memory_min_groups
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    full, _, _, _ = memory_plan(ab, ba, groups=1)
    most, _, _, _ = memory_plan(ab, ba, groups=0)
    assert memory_min_groups(ab, ba, 1, 0, full.physical_bytes)[0] == 1
    k, need = memory_min_groups(ab, ba, 1, 0, most.physical_bytes)
    assert k > 1 and need <= most.physical_bytes
    assert memory_min_groups(ab, ba, 1, 0, most.physical_bytes - 1)[0] == -1


def test_ladder_is_monotone_within_a_band_count():
    """Group counts nest (1, 2, 4, ...), so within one band count more groups never need
    more memory; the ladder starts with the no-aliasing plan."""
    from paper_2605_18815_b200.api import memory_schedule_footprints, memory_schedule_level
    sc = S.config2(2)
    ab = RoutingPlan.from_scenario(sc)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    for n_gpus, gpu in ((1, 0), (2, 1)):
        f = memory_schedule_footprints(ab, ba, n_gpus, gpu, chunk_bytes=8 << 20)
        levels = [memory_schedule_level(ab, i, n_gpus) for i in range(len(f))]
        assert levels[0] == (1, 1)
        assert any(g == -1 for _, g in levels) == (n_gpus > 1)  # rounds only across GPUs
        nested = [(lv, x) for lv, x in zip(levels, f) if lv[1] > 0]
        for (a, fa), (b, fb) in zip(nested, nested[1:]):
            if a[0] == b[0]:
                assert fb <= fa, (a, b, fa, fb)


def test_config5_full_fits_eight_gpus_under_the_cap():
    """BASELINE config 5 (Llama-3-70B TP4xPP2 -> TP8, ZeRO-1): 247 GB of old + new state
    per GPU on 8 GPUs. Rebuilding each new rank in layer bands inside the memory its old
    layout frees brings every GPU under 180 GB; the plan replays without clobbering."""
    from paper_2605_18815_b200.api import memory_schedule_footprints, memory_schedule_level
    sc = S.config5(80)
    ab = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    cap = 179 * 10**9
    f = [memory_schedule_footprints(ab, None, 8, g) for g in range(8)]
    assert min(f[g][0] for g in range(8)) > 240e9  # no aliasing: does not fit
    fits = [i for i in range(len(f[0])) if all(f[g][i] <= cap for g in range(8))]
    assert fits
    bands, groups = memory_schedule_level(ab, fits[0], 8)
    assert bands > 1
    for g in range(8):
        st, viol, _, _ = memory_plan(ab, None, n_gpus=8, gpu=g, groups=groups, bands=bands)
        assert viol == 0 and st.physical_bytes <= cap and st.bands == bands


def test_cuts_snap_to_group_starts_so_gpus_agree():
    """With coarse groups (here: rounds) every GPU's cuts fall on group starts, so the
    barriers all GPUs share stay at most one per group."""
    from paper_2605_18815_b200.api import memory_plan_cuts
    sc = S.config4(8)
    ab = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    n_gpus, bands = 4, 2
    cuts = [memory_plan_cuts(ab, None, n_gpus=n_gpus, gpu=g, groups=-1, bands=bands) for g in range(n_gpus)]
    units = len(cuts[0])
    rounds = -(-units // n_gpus)
    group_of = [x * rounds // units for x in range(units)]
    union = [max(c[i] for c in cuts) for i in range(units)]
    for i, u in enumerate(union):
        if u:
            assert i == 0 or group_of[i - 1] != group_of[i], (i, union)
    assert sum(union) <= rounds


def test_band_interleaved_level_is_the_fastest_that_fits():
    """Config 5 at N=4, L=40 (the full model's per-GPU state at N=8) under 180 GB: the
    band-interleaved order (groups = bands / src pp: each group takes one band of every
    source pipeline stage, all destination ranks of it) fits on every GPU, replays clean,
    and models faster than every other level that fits — the level shared_arena picks."""
    from paper_2605_18815_b200.api import memory_plan, memory_schedule_costs, memory_schedule_level
    ab = RoutingPlan.from_scenario(S.config5(40), allow_oversourced=True)
    costs = [memory_schedule_costs(ab, None, 4, g) for g in range(4)]
    n = len(costs[0])
    fits = [i for i in range(n) if all(costs[g][i][0] <= 180e9 for g in range(4))]
    t = [max(costs[g][i][1] for g in range(4)) for i in range(n)]
    best = min(fits, key=lambda i: (t[i], i))
    bands, groups = memory_schedule_level(ab, best, 4)
    assert groups == -2 and bands >= 8
    first_fit = fits[0]
    assert t[best] < 0.75 * t[first_fit]
    for g in range(4):
        st, viol, _, _ = memory_plan(ab, None, n_gpus=4, gpu=g, groups=-2, bands=bands)
        assert viol == 0 and st.physical_bytes <= 180e9


def test_time_model_uses_the_union_of_every_gpus_cuts():
    """The run barriers wherever any GPU's aliasing needs a cut, so every GPU models a level
    with the same (union) stage structure: identical modeled times on every GPU, and a
    level's time never drops below its one-stage time. Calibration on B200s (N=4 north
    star, profiles/r02_stage_levels_n4.jsonl): 8x8 modeled 62.6 ms / measured 62.3, 32x8
    53.3 / 53.5, 16x16 67.6 / 65.6."""
    from paper_2605_18815_b200.api import memory_schedule_costs
    ab = RoutingPlan.from_scenario(S.config2(32))
    costs = [memory_schedule_costs(ab, None, 4, g) for g in range(4)]
    for i in range(len(costs[0])):
        ts = {round(costs[g][i][1], 12) for g in range(4)}
        assert len(ts) == 1, (i, ts)
        assert costs[0][i][1] >= costs[0][0][1] - 1e-9
