"""Every level of the memory-aware schedule ladder (layer bands x concurrency groups) on
one GPU: the arena aliases new-layout chunks onto dead old-layout chunks in a different
pattern at each level, so each level is its own correctness case. Forward and back are
checked on every destination element (canon), the stage count matches the level, and the
mapped footprint matches the level's planned bytes."""
import pytest

torch = pytest.importorskip("torch")

from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import (Arena, Executor, RoutingPlan, memory_schedule_costs,  # noqa: E402
                                       memory_schedule_level)

pytestmark = pytest.mark.gpu

SEED = 0xA11A5


@pytest.mark.parametrize("name", ["llama8b_L4", "qwen_moe_L2"])
def test_every_schedule_level_round_trip(name):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    sc = S.config2(4) if name == "llama8b_L4" else S.config4(2)
    ab = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
    costs = memory_schedule_costs(ab, ba, 1, 0)
    assert len(costs) >= 8
    free = torch.cuda.mem_get_info()[0]
    seen = set()
    for lv, (need, _) in enumerate(costs):
        bands, groups = memory_schedule_level(ab, lv, 1)
        if need > free - (4 << 30):
            continue
        arena = Arena.multi(ab, ba, 1, 0, 0, cap_bytes=need, groups=groups, bands=bands)
        st = arena.stats()
        assert st.physical_bytes <= need, (lv, st.physical_bytes, need)
        fwd, bwd = Executor(ab), Executor(ba)
        arena.bind(fwd, bwd)
        fwd.fill(0, SEED)
        fwd.prepare()
        bwd.prepare()
        for _ in range(2):  # the second trip starts from the restored layout
            fwd.run()
            torch.cuda.synchronize()
            bad, first = fwd.verify(1, SEED)
            assert bad == 0, f"level {lv} ({bands} bands x {groups} groups) forward: {bad} mismatches at {first}"
            bwd.run()
            torch.cuda.synchronize()
            bad, first = bwd.verify(1, SEED)
            assert bad == 0, f"level {lv} ({bands} bands x {groups} groups) back: {bad} mismatches at {first}"
        seen.add((fwd.num_stages(), bwd.num_stages(), st.physical_bytes))
        del fwd, bwd, arena
        torch.cuda.synchronize()
    # the ladder really exercised different stage structures and footprints
    assert len(seen) >= 4, seen
