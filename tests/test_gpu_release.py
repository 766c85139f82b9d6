"""FreeObsoleteBuffers at run time: a one-way transition on one
GPU hands consumed old-layout memory back to the driver while its later stages run
(`Arena.release_through`, `runtime.run_releasing`). The new layout is bit-exact, the
released bytes show up as free HBM, and the chunks the new layout reuses stay mapped."""
import gc

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Arena, Executor, RoutingPlan  # noqa: E402
from paper_2605_18815_b200.runtime import run_releasing  # noqa: E402

SEED = 0xF4EE


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


def test_release_consumed_source_chunks_while_running():
    gc.collect()
    torch.cuda.empty_cache()
    ab = RoutingPlan.from_scenario(S.config2(4))
    arena = Arena(ab, None, device=0, cap_bytes=45_000_000_000)  # old + new = 58.5 GB: must alias
    st = arena.stats()
    assert st.aliased_bytes > 0 and st.physical_bytes <= 45e9
    ex = Executor(ab)
    arena.bind(ex, None)
    ex.fill(A.SIDE_SRC, SEED)
    ex.prepare()
    assert ex.num_stages() >= 2
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(0)[0]
    s = torch.cuda.Stream()
    freed = run_releasing(ex, arena, s)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(0)[0]
    print(f"released {freed / 1e9:.2f} GB of {st.a_bytes / 1e9:.2f} GB old layout "
          f"({st.aliased_bytes / 1e9:.2f} GB reused by the new layout); free HBM +{(free1 - free0) / 1e9:.2f} GB")
    assert freed > 0 and freed + st.aliased_bytes <= st.a_bytes
    assert free1 - free0 >= 0.95 * freed
    bad, first = ex.verify(A.SIDE_DST, SEED)
    assert bad == 0, f"{bad} mismatches, first {first}"
    with pytest.raises(A.ConfigError):
        Arena(ab, RoutingPlan.from_scenario(S.config2(4).reversed(), allow_oversourced=True), device=0,
              cap_bytes=0).release_through(0)
    del ex, arena
    gc.collect()
