"""Oracle executor (SPEC.md:365-403 restated): load -> execute -> verify, oracle
equivalence and round trip, on the reference-pinned golden scenarios."""
import pytest

import pyoracle as O

M64 = (1 << 64) - 1


def _mix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def py_canon(seed, k, kind):
    """common.hpp:77-80 restated in Python (independent of oracle.c)."""
    return _mix64(_mix64(seed ^ ((k * 0xD6E8FEB86659FD93) & M64)) ^ (((kind + 1) * 0xA5A5A5A5A5A5A5A5) & M64))


def test_canon_matches_python_restatement():
    for seed in (0, 1, 0xC0FFEE):
        for k in (0, 1, 7, 123456789, 8030261247):
            for kind in range(4):
                assert O.canon(seed, k, kind) == py_canon(seed, k, kind)


def _exec_case(text, seed=0xC0FFEE, with_grads=False, allow=False):
    s = O.OScenario(text)
    p = O.OPlan(s, allow)
    src = O.OState(s, 0, with_grads)
    src.load(seed)
    dst = O.OState(s, 1, with_grads)
    O.execute(p, src, dst, nthreads=2)
    bad, msg = dst.verify(seed)
    assert bad == 0, msg
    ref = O.OState(s, 1, with_grads)
    O.oracle_reshard(s, src, ref)
    assert dst.equal(ref)
    return s, src, dst


def test_exec_golden_campaign(golden):
    n = 0
    for e in golden:
        if e["rc"] != 0 or e["ref_seconds"] > 5 or e["group"] == "baseline" and "llama" in e["name"]:
            continue
        _exec_case(e["scenario"], with_grads="grads=migrate" in e["scenario"])
        n += 1
    assert n >= 60


def test_exec_tiny_gpt():
    from paper_2605_18815_b200 import scenarios as S
    _exec_case(S.config1(False).text())


def test_round_trip():
    from paper_2605_18815_b200 import scenarios as S
    sc = S.config1(False)
    seed = 7
    s = O.OScenario(sc.text())
    src = O.OState(s, 0)
    src.load(seed)
    mid = O.OState(s, 1)
    O.execute(O.OPlan(s), src, mid)
    r = O.OScenario(sc.reversed().text())
    back = O.OState(r, 1)
    O.execute(O.OPlan(r), mid, back)
    assert back.verify(seed)[0] == 0
    for rank in range(src.num_ranks()):
        for b in range(6):
            assert back.buffer(rank, b) == src.buffer(rank, b)


def test_fault_injection_single_violation():
    # one corrupted element -> exactly one violation
    import ctypes
    from paper_2605_18815_b200 import scenarios as S
    s, src, dst = _exec_case(S.config1(False).text())
    ptr, n = dst.buffer_ptr(1, 1)
    b = (ctypes.c_uint8 * n).from_address(ptr)
    b[40] ^= 0x01
    bad, msg = dst.verify(0xC0FFEE)
    assert bad == 1 and "optim" in msg


def test_d2_extension_executes():
    from paper_2605_18815_b200 import scenarios as S
    with pytest.raises(O.OracleError):
        O.OPlan(O.OScenario(S.config1(True).text()))
    _exec_case(S.config1(True).text(), allow=True)
