"""validate_plan: zero violations on valid plans, the constructed
fault (one recv fragment deleted) is reported as an uncovered destination region."""
from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.api import RoutingPlan


def test_valid_plans_have_no_violations(golden):
    n = 0
    for e in golden:
        if e["rc"] != 0 or e["ref_seconds"] > 5:
            continue
        assert RoutingPlan.from_scenario(e["scenario"]).validate() == [], e["name"]
        n += 1
    assert n >= 85


def test_d2_extension_plans_are_valid():
    for sc in (S.config1(True), S.config2(2).reversed(), S.table4(8)):
        assert RoutingPlan.from_scenario(sc, allow_oversourced=True).validate() == []


def test_north_star_full_scale_valid():
    assert RoutingPlan.from_scenario(S.config2(32)).validate() == []


def test_deleted_fragment_is_reported():
    p = RoutingPlan.from_scenario(S.config1(False))
    v = p.validate(drop=3)
    assert len(v) == 1 and v[0].startswith("uncovered destination region: rank ")
    p = RoutingPlan.from_scenario(S.config2(1))
    v = p.validate(drop=p.summary.num_box_transfers + 17)  # a ZeRO optimizer run
    assert len(v) == 1 and " optim [" in v[0] and v[0].startswith("uncovered destination region")
