"""Product planner (C ABI, libreshard_b200.so) vs the reference (golden plans
generated from the reference headers) and vs the oracle, on CPU."""
import hashlib

import pytest

import pyoracle as O
from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.api import ConfigError, ModelSpace, RoutingPlan, plan_transition


def _sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def test_golden_plans(golden):
    n = 0
    for e in golden:
        if e["ref_seconds"] > 30:
            continue
        try:
            p = RoutingPlan.from_scenario(e["scenario"])
        except ConfigError as err:
            assert e["rc"] == 2, (e["name"], str(err))
            assert e["error"] == "# error: " + str(err), e["name"]
            n += 1
            continue
        assert e["rc"] == 0, (e["name"], e.get("error"))
        d = p.dump()
        if "dump" in e and d != e["dump"]:
            a, b = d.splitlines(), e["dump"].splitlines()
            for i, (x, y) in enumerate(zip(a, b)):
                assert x == y, (e["name"], i, x, y)
            assert len(a) == len(b), (e["name"], len(a), len(b))
        assert _sha(d) == e["sha256"], e["name"]
        assert p.num_transfers() == e["transfers"], e["name"]
        assert p.bytes_moved() == e["bytes_moved"], e["name"]
        assert p.bytes_retained() == e["bytes_retained"], e["name"]
        # GPU planner's row algorithm, evaluated on the host, agrees too
        assert p.dump_rows_host() == d, e["name"]
        n += 1
    assert n >= 100


def test_golden_regions(golden):
    n = 0
    for e in golden:
        if "regions_src" not in e:
            continue
        p = RoutingPlan.from_scenario(e["scenario"])
        assert p.regions(0) == e["regions_src"], e["name"]
        assert p.regions(1) == e["regions_dst"], e["name"]
        n += 1
    assert n >= 10


@pytest.mark.parametrize("name", ["llama3-8b-L1.tp8-to-dp2tp4-zero1", "llama3-8b-L2.tp8-to-dp2tp4-zero1",
                                  "qwen3-30b-a3b-L1.ep8-to-ep4tp2", "llama3-70b-L2.tp4pp2-to-tp8",
                                  "llama3-8b.dp8-to-dp4", "llama3-8b.dp4-to-dp8"])
def test_golden_big(golden, name):
    e = next(x for x in golden if x["name"] == name)
    try:
        p = RoutingPlan.from_scenario(e["scenario"])
    except ConfigError as err:
        assert e["rc"] == 2 and e["error"] == "# error: " + str(err)
        return
    assert (p.num_transfers(), p.bytes_moved(), p.bytes_retained()) == (e["transfers"], e["bytes_moved"], e["bytes_retained"])
    assert _sha(p.dump()) == e["sha256"]


def test_full_config2_vs_oracle():
    """North-star plan at full L=32 (the reference itself would take hours: D3)."""
    sc = S.config2(32)
    p = RoutingPlan.from_scenario(sc)
    assert p.bytes_moved() == 112_419_930_560
    assert p.summary.num_box_transfers == 3164 and p.summary.num_flat_transfers == 1_836_142
    o = O.OPlan(O.OScenario(sc.text()))
    assert p.bytes_retained() == o.bytes_retained()
    assert _sha(p.dump()) == _sha(o.dump())


def test_d2_extension_matches_oracle():
    for sc in [S.config1(True)] + [S.Scenario(S.tiny_gpt(), S.Cfg(tp=2, pp=2, zero=True), S.Cfg(tp=4, zero=True))]:
        with pytest.raises(ConfigError):
            RoutingPlan.from_scenario(sc)
        p = RoutingPlan.from_scenario(sc, allow_oversourced=True)
        o = O.OPlan(O.OScenario(sc.text()), True)
        assert p.dump() == o.dump()
        assert p.bytes_moved() == o.bytes_moved()


def test_pod_api_matches_scenario_path():
    sc = S.config1(False)
    space = ModelSpace(sc.model)
    p = plan_transition(space, sc.src, sc.dst, rpn=4)
    q = RoutingPlan.from_scenario(sc)
    assert p.dump() == q.dump()
    tr = p.transfers()
    assert len(tr) == q.num_transfers() == 68
    assert sum(t.bytes for t in tr) + 3 * 64 == p.bytes_moved()


def test_config_errors_mirror_reference():
    m = S.Model("m", [S.Tensor("W", (4, 4), tp=0)])
    with pytest.raises(ConfigError, match="does not divide"):
        plan_transition(ModelSpace(m), S.Cfg(tp=3), S.Cfg(tp=2))
    with pytest.raises(ConfigError, match="duplicate tensor_id"):
        ModelSpace(S.Model("m", [S.Tensor("W", (4,)), S.Tensor("W", (4,))]))


def test_d2_extension_north_star_way_back_matches_oracle():
    """The bench's way back (DP2xTP4 -> TP8, over-sourced norms): the whole dump, with the
    proximity rule and with balance_fanout (the extension's cursor order)."""
    import dataclasses
    for sc in (S.config2(2).reversed(), dataclasses.replace(S.config2(2).reversed(), balance=True)):
        p = RoutingPlan.from_scenario(sc, allow_oversourced=True)
        o = O.OPlan(O.OScenario(sc.text()), True)
        assert p.dump() == o.dump()
        assert p.bytes_moved() == o.bytes_moved() and p.bytes_retained() == o.bytes_retained()


@pytest.mark.parametrize("seed", range(24))
def test_d2_extension_random_campaign_matches_oracle(seed):
    """Random toy models with replicated tensors, ZeRO on both sides, src tp > 1 (where the
    reference throws, D2): the extension's dump equals the oracle's, with and without
    balance_fanout, identity and shuffled join/leave world maps."""
    import random
    rng = random.Random(7000 + seed)
    for _ in range(50):
        m = S.toy_model(rng, experts=rng.choice([1, 1, 2, 4]))
        src = S.random_cfg(rng, m, max_world=8, zero=True)
        dst = S.random_cfg(rng, m, max_world=8, zero=True)
        if src.tp > 1:
            break
    sc = S.Scenario(m, src, dst, balance=bool(seed % 2), rpn=rng.choice([2, 4, 8]))
    if seed % 3 == 2:  # joiners / leavers on a shuffled set of physical devices
        phys = list(range(src.world() + dst.world()))
        rng.shuffle(phys)
        sc.world_src = sorted(phys[: src.world()])
        sc.world_dst = sorted(phys[src.world() - min(src.world(), dst.world()) // 2:][: dst.world()])
    o = O.OPlan(O.OScenario(sc.text()), True)
    p = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    assert p.dump() == o.dump()
    assert p.dump(device=-1) == p.dump_rows_host()
    assert p.bytes_moved() == o.bytes_moved()
    assert p.validate() == []
