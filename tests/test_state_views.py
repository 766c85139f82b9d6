"""The torch registration boundary (state.py): views of a rank's buffers in the layout
contract. CPU: the views tile the buffers exactly. GPU: real torch tensors (random bf16
weights, fp32 optimizer state) registered in the old layout come out of the CUDA
transition as the right slices of the same tensors in the new layout."""
import pytest

torch = pytest.importorskip("torch")

from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import RoutingPlan  # noqa: E402
from paper_2605_18815_b200.state import RankState, buffer_bytes, model_tensors  # noqa: E402

CASES = [("config1", lambda: S.config1()), ("config1-zero-ext", lambda: S.config1(zero=True)),
         ("config2-L1", lambda: S.config2(1)), ("config4-L1", lambda: S.config4(1)),
         ("ragged-dp2-zero-to-tp2", lambda: [x for x in S.edge_scenarios() if x.name == "edge.ragged-dp2-zero-to-tp2"][0]),
         ("ragged-pp2-to-tp2", lambda: [x for x in S.edge_scenarios() if x.name == "edge.ragged-pp2-to-tp2-grads"][0])]


def _plan(sc):
    return RoutingPlan.from_scenario(sc, allow_oversourced=True)


@pytest.mark.parametrize("name,make", CASES)
def test_views_tile_the_buffers(name, make):
    sc = make()
    plan = _plan(sc)
    tensors = model_tensors(plan)
    assert [t.id for t in tensors] == [t.id for t in sc.model.tensors]
    for side, world in ((A.SIDE_SRC, sc.src.world()), (A.SIDE_DST, sc.dst.world())):
        for r in range(world):
            st = RankState.alloc(plan, side, r, device="meta")
            nbytes = buffer_bytes(plan, side, r)
            pieces, opieces = [], []
            for tid in st.seg_of:
                s = st.seg_of[tid]
                p = st.param(tid)
                assert tuple(p.shape) == tuple(sl.stop - sl.start for sl in st.box(tid))
                pieces.append((s.param_byte_off, p.numel() * p.element_size()))
                v, (a, b) = st.optim_slice("master", tid)
                if v is not None:
                    assert v.numel() == b - a and 0 <= a < b <= p.numel()
                    opieces.append((v.storage_offset(), v.numel()))
            assert _tiles(pieces, nbytes[A.BUF_PARAM], align=16), "param views must tile the buffer"
            assert _tiles(opieces, st.geom.optim_len), "optimizer slices must tile the shard"


def _tiles(pieces, total, align=1):
    """Pieces cover [0, total) in order, each starting at the next `align`-aligned offset."""
    pos = 0
    for off, n in sorted(pieces):
        if off != (pos + align - 1) // align * align:
            return False
        pos = off + n
    return pos == total


def _full_state(sc, seed):
    g = torch.Generator().manual_seed(seed)
    full = {}
    for t in sc.model.tensors:
        if t.dtype == 1:
            param = torch.randint(0, 256, t.shape, generator=g, dtype=torch.uint8)
        else:
            param = torch.randn(t.shape, generator=g).to(torch.bfloat16 if t.dtype == 2 else torch.float32)
        full[t.id] = {"param": param,
                      "master": torch.randn(t.shape, generator=g), "m": torch.randn(t.shape, generator=g),
                      "v": torch.rand(t.shape, generator=g)}
    return full


def _load(st, full):
    for tid in st.seg_of:
        box = st.box(tid)
        st.param(tid).copy_(full[tid]["param"][box])
        for kind in ("master", "m", "v"):
            v, (a, b) = st.optim_slice(kind, tid)
            if v is not None:
                v.copy_(full[tid][kind][box].reshape(-1)[a:b])


def _check(st, full):
    bad = []
    for tid in st.seg_of:
        box = st.box(tid)
        if not torch.equal(st.param(tid).cpu(), full[tid]["param"][box]):
            bad.append((st.rank, tid, "param"))
        for kind in ("master", "m", "v"):
            v, (a, b) = st.optim_slice(kind, tid)
            if v is not None and not torch.equal(v.cpu(), full[tid][kind][box].reshape(-1)[a:b]):
                bad.append((st.rank, tid, kind))
    return bad


@pytest.mark.gpu
@pytest.mark.parametrize("name,make", CASES)
def test_torch_state_survives_transition(name, make):
    """Register real tensors in the old layout, run the CUDA transition, read the new
    layout's views: every box / shard equals the same slice of the original tensors."""
    from paper_2605_18815_b200.api import Executor
    sc = make()
    plan = _plan(sc)
    full = _full_state(sc, 1234)
    grads = sc.grads == "migrate"
    ex = Executor(plan, with_grads=grads)
    src = [RankState.alloc(plan, A.SIDE_SRC, r, with_grads=grads) for r in range(sc.src.world())]
    dst = [RankState.alloc(plan, A.SIDE_DST, r, with_grads=grads) for r in range(sc.dst.world())]
    for st in src + dst:
        st.bind(ex)
    for st in src:
        _load(st, full)
        if grads:
            for tid in st.seg_of:
                st.grad(tid).copy_(full[tid]["master"][st.box(tid)])
    ex.prepare()
    ex.run()
    torch.cuda.synchronize()
    bad = [b for st in dst for b in _check(st, full)]
    if grads:
        bad += [(st.rank, tid, "grad") for st in dst for tid in st.seg_of
                if not torch.equal(st.grad(tid).cpu(), full[tid]["master"][st.box(tid)])]
    assert not bad, bad[:10]
