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
