"""Elastic Device Manager host logic: group derivation, cache,
overlap accounting (Table 2 ratios), side-thread preparation."""
import random
import time

import pytest

from paper_2605_18815_b200 import scenarios as S
from paper_2605_18815_b200.edm import ElasticDeviceManager, config_groups, overlap_accounting


def test_tp_groups_spec_kat():
    # cfg (dp=2,tp=2,pp=2): tp groups {0,1},{2,3},{4,5},{6,7} under pp-dp-tp
    assert config_groups(S.Cfg(dp=2, tp=2, pp=2), "tp") == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert config_groups(S.Cfg(dp=2, tp=2, pp=2), "dp") == [[0, 2], [1, 3], [4, 6], [5, 7]]
    assert config_groups(S.Cfg(dp=2, tp=2, pp=2), "pp") == [[0, 4], [1, 5], [2, 6], [3, 7]]


def test_groups_partition_random_configs():
    # for every dimension, groups partition {0..N-1}
    rng = random.Random(3)
    for _ in range(200):
        ep = rng.choice([1, 2, 4])
        dp = ep * rng.choice([1, 2, 3])
        cfg = S.Cfg(dp=dp, tp=rng.choice([1, 2, 4]), pp=rng.choice([1, 2]), ep=ep,
                    order=rng.choice(["pp-dp-tp", "tp-dp-pp", "dp-pp-tp"]))
        for dim, size in (("dp", cfg.dp), ("tp", cfg.tp), ("pp", cfg.pp), ("ep", cfg.ep), ("edp", cfg.dp // cfg.ep)):
            g = config_groups(cfg, dim)
            flat = sorted(r for grp in g for r in grp)
            assert flat == list(range(cfg.world())), (cfg, dim)
            assert all(len(grp) == size for grp in g), (cfg, dim)


def test_cache_idempotent_zero_cost():
    edm = ElasticDeviceManager()
    a = edm.get_or_create_groups(S.Cfg(dp=2, tp=4))
    cost = edm.creation_cost_s
    b = edm.get_or_create_groups(S.Cfg(dp=2, tp=4))
    assert a is b and edm.creation_cost_s == cost  # second request: cache hit, zero cost


def test_overlap_ratios_table2():
    # exposed 1.91 s with 40.98 s overlapped -> 95.6 %; 3.05 / 40.32 -> 93.0 %
    for exposed, overlapped, ratio in ((1.91, 40.98, 0.956), (3.05, 40.32, 0.930)):
        r = overlap_accounting(init_s=overlapped, switch_s=exposed, window_s=overlapped)
        assert abs(r["exposed_s"] - exposed) < 1e-9
        assert abs(r["overlap_ratio"] - ratio) < 0.001
    # init_cost 0 -> overlapped and blocking expose the same
    assert overlap_accounting(0.0, 2.0, window_s=10)["exposed_s"] == overlap_accounting(0.0, 2.0, mode="blocking")["exposed_s"]
    # overlap dominance
    for init, win, sw in ((5, 3, 1), (5, 10, 1), (0.5, 0, 2)):
        assert overlap_accounting(init, sw, window_s=win)["exposed_s"] <= overlap_accounting(init, sw, mode="blocking")["exposed_s"]
    # whole training steps only
    assert overlap_accounting(init_s=10.0, switch_s=1.0, train_step_s=3.0)["overlapped_s"] == 9.0


def test_prepare_async_overlaps_host_work():
    from paper_2605_18815_b200.api import RoutingPlan
    edm = ElasticDeviceManager()

    def build(ctrl):
        return RoutingPlan.from_scenario(S.config2(4))

    edm.prepare_async(build)
    spins = 0
    while not edm.ready():
        spins += 1
        time.sleep(0.001)
    plan = edm.wait()
    assert plan.bytes_moved() > 0 and edm.init_s > 0


def test_native_cache_counts_and_errors():
    """The native EDM's cache counts hits/misses; a failing build surfaces at wait()."""
    import ctypes as C

    from paper_2605_18815_b200 import _capi as A
    edm = ElasticDeviceManager()
    cfg = S.Cfg(dp=4, tp=2)
    edm.get_or_create_groups(cfg)
    edm.get_or_create_groups(cfg)
    hits, misses, cost = C.c_int64(), C.c_int64(), C.c_double()
    A.check(edm._lib.rs_edm_cache_stats(edm.h, C.byref(hits), C.byref(misses), C.byref(cost)))
    assert misses.value == 5 and hits.value == 5  # five dimensions, derived once, then served

    def boom(ctrl):
        raise ValueError("build failed")

    edm.prepare_async(boom)
    with pytest.raises(ValueError):
        edm.wait()
    edm.prepare_async(lambda ctrl: 42)  # the manager is reusable after a failure
    while not edm.ready():
        time.sleep(0.001)
    assert edm.wait() == 42


def test_accounting_modes():
    r = overlap_accounting(init_s=4.0, switch_s=1.0, mode="in-place")
    assert r["init_s"] == 0.0 and r["exposed_s"] == 1.0
    r = overlap_accounting(init_s=4.0, switch_s=1.0, window_s=10.0, mode="blocking")
    assert r["overlapped_s"] == 0.0 and r["exposed_s"] == 5.0 and r["overlap_ratio"] == 0.0
    assert overlap_accounting(0.0, 0.0)["overlap_ratio"] is None


@pytest.mark.gpu
def test_native_nccl_communicators_single_rank():
    """The EDM's native, non-blocking NCCL communicator build (world + one split per
    dimension) on a one-rank world: cached per configuration, and an all-reduce over each
    communicator sums to its size. (Multi-rank worlds run in tools/edm_bench.py.)"""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_18815_b200.edm import ElasticDeviceManager, nccl_version
    from paper_2605_18815_b200.scenarios import Cfg
    assert nccl_version().startswith("2.")
    edm = ElasticDeviceManager()
    cfg = Cfg(dp=1, zero=True)
    info = edm.create_nccl_comms(cfg, rank=0, nranks=1, device=0, member_rank=0)
    assert not info["cache_hit"] and info["init_s"] > 0
    assert edm.nccl_comm(cfg) != 0 and edm.nccl_comm(cfg, "dp") != 0
    s = torch.cuda.Stream()
    assert edm.check_nccl_comm(cfg, None, s.cuda_stream) == 1.0
    assert edm.check_nccl_comm(cfg, "tp", s.cuda_stream) == 1.0
    assert edm.create_nccl_comms(cfg, rank=0, nranks=1, device=0, member_rank=0)["cache_hit"]
    edm.destroy_nccl_comms(cfg)
    assert edm.nccl_comm(cfg) == 0
