"""Edge cases of the executor on the B200, each bit-exact against canon payloads and, for
the small ones, byte-identical to the oracle's CPU executor: the identity transition
(everything retained), ragged byte widths that force every alignment class (1/2/4/8/16-B
vectors), ZeRO shard boundaries at odd element offsets, a single-tensor model, scalar-only
words, join/leave world maps, and gradients migrated with the state."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import pyoracle as O  # noqa: E402
from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200.api import Executor, RoutingPlan  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402

SEED = 0x5EED


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


CASES = {sc.name: sc for sc in S.edge_scenarios()}  # plan parity: tests/golden group "edge"


def _oracle(sc, grads):
    s = O.OScenario(sc.text())
    p = O.OPlan(s, False)
    src = O.OState(s, 0, grads)
    src.load(SEED)
    dst = O.OState(s, 1, grads)
    O.execute(p, src, dst, nthreads=2)
    return dst


@pytest.mark.parametrize("name", sorted(CASES))
def test_edge_case_bit_exact(name):
    sc = CASES[name]
    grads = sc.grads == "migrate"
    plan = RoutingPlan.from_scenario(sc)
    ex = Executor(plan, with_grads=grads)
    tensors = {}
    for side, n in ((0, plan.summary.src_world), (1, plan.summary.dst_world)):
        for r in range(n):
            for b in range(6):
                _, nbytes, _ = ex.buffer(side, r, b)
                if nbytes:
                    # zeroed: alignment padding between segments matches the oracle's
                    t = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
                    tensors[(side, r, b)] = t
                    ex.bind(side, r, b, t.data_ptr(), nbytes)
    ex.fill(A.SIDE_SRC, SEED)
    ex.prepare()
    ex.run()
    torch.cuda.synchronize()
    bad, first = ex.verify(A.SIDE_DST, SEED)
    assert bad == 0, f"{name}: {bad} mismatches, first {first}"
    if "identity" in name:
        assert plan.bytes_moved() <= 8 * 8 * 8  # only the scalar broadcast moves
    dst = _oracle(sc, grads)
    for r in range(plan.summary.dst_world):
        for b in range(6):
            if (1, r, b) in tensors:
                assert tensors[(1, r, b)].cpu().numpy().tobytes() == dst.buffer(r, b), (name, r, b)
    st = ex.stats()
    if "ragged" in name:
        assert sum(1 for c in st.tiles_by_class if c) >= 2  # several alignment classes ran
