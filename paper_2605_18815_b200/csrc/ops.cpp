// CopyOp construction: every element movement of a transition (plan transfers,
// retained regions, scalar broadcast) as 2-D strided byte copies between the
// physical buffers of DESIGN.md §3. Pure host code; GPU-independent.
#include <algorithm>
#include <thread>

#include "reshard/executor.hpp"
#include "reshard/pool.hpp"

namespace reshard {
namespace exec {

namespace {

using core::PlanCore;
using core::RankGeom;
using core::Seg;

struct LBox {
    int np;
    std::int64_t plo[2], pext[2], rlo, rows, clo, cols;
};

LBox lift_seg(const TensorSpec& t, const std::int64_t* lo, const std::int64_t* hi) {
    LBox b{};
    const int nd = static_cast<int>(t.shape.size());
    std::int64_t l[4], h[4];
    int n = 0;
    if (nd == 1) l[n] = 0, h[n] = 1, ++n;
    for (int d = 0; d < nd; ++d) l[n] = lo[d], h[n] = hi[d], ++n;
    b.np = n - 2;
    for (int i = 0; i < b.np; ++i) b.plo[i] = l[i], b.pext[i] = h[i] - l[i];
    b.rlo = l[b.np];
    b.rows = h[b.np] - l[b.np];
    b.clo = l[b.np + 1];
    b.cols = h[b.np + 1] - l[b.np + 1];
    return b;
}

/// element index of (p, r, c) in the row-major enumeration of box B
std::int64_t elem_in(const LBox& B, const std::int64_t* p, std::int64_t r, std::int64_t c) {
    std::int64_t q = 0;
    for (int i = 0; i < B.np; ++i) q = q * B.pext[i] + (p[i] - B.plo[i]);
    return (q * B.rows + (r - B.rlo)) * B.cols + (c - B.clo);
}

struct Emitter {
    const PlanCore& P;
    std::vector<CopyOp>& out;

    const Seg& seg(int side, int rank, int t) const {
        const RankGeom& g = (side == 0 ? P.src : P.dst).ranks[static_cast<size_t>(rank)];
        return g.segs[static_cast<size_t>(g.seg_of[static_cast<size_t>(t)])];
    }
    const RankGeom& geom(int side, int rank) const { return (side == 0 ? P.src : P.dst).ranks[static_cast<size_t>(rank)]; }

    /// rectangle (plane p, rows [r0,r1), cols [c0,c1)) of tensor t, kind, src k -> dst j
    void rect(int kind, int t, int k, int j, const std::int64_t* p, std::int64_t r0, std::int64_t r1,
              std::int64_t c0, std::int64_t c1) {
        const TensorSpec& ts = P.space->entries()[static_cast<size_t>(t)].spec;
        const Seg& S = seg(0, k, t);
        const Seg& D = seg(1, j, t);
        const LBox Bs = lift_seg(ts, S.blo, S.bhi), Bd = lift_seg(ts, D.blo, D.bhi);
        const std::int64_t es = elem_in(Bs, p, r0, c0), ed = elem_in(Bd, p, r0, c0);
        const std::int64_t rows = r1 - r0, w = c1 - c0;
        const size_t first = out.size();
        emit(kind, ts, S, D, Bs, Bd, k, j, es, ed, rows, w);
        for (size_t i = first; i < out.size(); ++i) out[i].tensor = t;
    }

    void emit(int kind, const TensorSpec& ts, const Seg& S, const Seg& D, const LBox& Bs, const LBox& Bd, int k, int j,
              std::int64_t es, std::int64_t ed, std::int64_t rows, std::int64_t w) {
        if (kind == 0) {
            const int dt = ts.dtype_bytes;
            out.push_back(CopyOp{k, kParam, j, kParam, S.param_byte_off + es * dt, D.param_byte_off + ed * dt, rows, w * dt,
                                 Bs.cols * dt, Bd.cols * dt});
        } else if (kind == 2) {
            out.push_back(CopyOp{k, kGrad, j, kGrad, (S.elem_off + es) * 4, (D.elem_off + ed) * 4, rows, w * 4,
                                 Bs.cols * 4, Bd.cols * 4});
        } else {
            const std::int64_t os = geom(0, k).optim_index(S.expert, S.local_lo + es);
            const std::int64_t od = geom(1, j).optim_index(D.expert, D.local_lo + ed);
            if (os < 0 || od < 0) throw std::logic_error("optimizer move outside the shard");
            for (int b = kMaster; b <= kV; ++b)
                out.push_back(CopyOp{k, b, j, b, os * 4, od * 4, rows, w * 4, Bs.cols * 4, Bd.cols * 4});
        }
    }

    /// box X (tensor coordinates) of kind from src k to dst j, one rect per plane
    void box(int kind, int t, int k, int j, const std::int64_t* lo, const std::int64_t* hi) {
        const TensorSpec& ts = P.space->entries()[static_cast<size_t>(t)].spec;
        const LBox X = lift_seg(ts, lo, hi);
        std::int64_t p[2] = {0, 0};
        const std::int64_t e0 = X.np > 0 ? X.pext[0] : 1, e1 = X.np > 1 ? X.pext[1] : 1;
        for (std::int64_t a = 0; a < e0; ++a)
            for (std::int64_t b = 0; b < e1; ++b) {
                if (X.np > 0) p[0] = X.plo[0] + a;
                if (X.np > 1) p[1] = X.plo[1] + b;
                rect(kind, t, k, j, p, X.rlo, X.rlo + X.rows, X.clo, X.clo + X.cols);
            }
    }

    void triple(const stair::Triple& T) {
        core::for_each_band(T, [&](const std::int64_t* p, std::int64_t u, std::int64_t v, const stair::Iv* cols, int n) {
            for (int i = 0; i < n; ++i) rect(1, T.tensor, T.src, T.dst, p, u, v, cols[i].lo, cols[i].hi);
        });
    }

    /// flat run [lo,hi) of optimizer state (D2 override), split at tensor rows
    void flat_run(const core::FlatXfer& f) {
        const auto& ents = P.space->entries();
        std::int64_t x = f.lo;
        while (x < f.hi) {
            auto it = std::upper_bound(ents.begin(), ents.end(), x,
                                       [](std::int64_t v, const ModelSpace::Entry& e) { return v < e.offset; });
            const int t = static_cast<int>(it - ents.begin()) - 1;
            const auto& e = ents[static_cast<size_t>(t)];
            const std::int64_t zero[4] = {0, 0, 0, 0};
            std::int64_t full[4];
            for (size_t d = 0; d < e.spec.shape.size(); ++d) full[d] = e.spec.shape[d];
            const LBox Tb = lift_seg(e.spec, zero, full);
            const std::int64_t rel = x - e.offset;
            const std::int64_t grow = rel / Tb.cols, c = rel % Tb.cols;
            std::int64_t p[2] = {0, 0}, g = grow / Tb.rows;
            const std::int64_t r = grow % Tb.rows;
            for (int i = Tb.np - 1; i >= 0; --i) p[i] = g % Tb.pext[i], g /= Tb.pext[i];
            const std::int64_t end = std::min(f.hi, x + (Tb.cols - c));
            rect(1, t, f.src, f.dst, p, r, r + 1, c, c + (end - x));
            x = end;
        }
    }
};

}  // namespace

std::vector<CopyOp> build_ops(const PlanCore& P) {
    std::vector<CopyOp> ops;
    Emitter E{P, ops};
    for (size_t i = 0; i < P.box.size(); ++i) {
        const core::BoxXfer& b = P.box[i];
        const size_t first = ops.size();
        E.box(b.kind, b.tensor, b.src, b.dst, b.lo, b.hi);
        for (size_t k = first; k < ops.size(); ++k) ops[k].box = static_cast<int>(i);
    }
    for (const core::BoxXfer& b : P.box_retain) E.box(b.kind, b.tensor, b.src, b.dst, b.lo, b.hi);
    const int nt = P.ntensors();
    auto overridden = [&](int j, int t) {
        return !P.d2_tensor_dst.empty() && P.d2_tensor_dst[static_cast<size_t>(j) * nt + t];
    };
    {
        // the ZeRO triples (thousands, each a band sweep) on host threads: contiguous
        // slices into their own op lists, appended in slice order (the sequential order)
        std::vector<const stair::Triple*> tv;
        tv.reserve(P.triples.size() + P.retain_triples.size());
        for (const stair::Triple& T : P.triples)
            if (!overridden(T.dst, T.tensor)) tv.push_back(&T);
        for (const stair::Triple& T : P.retain_triples) tv.push_back(&T);
        const size_t nth = std::max<size_t>(1, std::min<size_t>(pool::size(), tv.size() / 64 + 1));
        std::vector<std::vector<CopyOp>> part(nth);
        pool::run(nth, [&](size_t t) {
            Emitter Et{P, part[t]};
            for (size_t i = tv.size() * t / nth; i < tv.size() * (t + 1) / nth; ++i) Et.triple(*tv[i]);
        });
        size_t n = ops.size();
        for (const auto& v : part) n += v.size();
        ops.reserve(n);
        for (auto& v : part) ops.insert(ops.end(), v.begin(), v.end());
    }
    // D2 extension: a tensor of a destination rank holding multi-candidate elements is
    // re-derived from its triples' runs minus the segments another source was chosen for
    // (d2_multi, (dst, lo) order); every other element has exactly one source
    if (!P.d2_tensor_dst.empty()) {
        std::vector<core::FlatXfer> v;
        for (const stair::Triple& T : P.triples) {
            if (!overridden(T.dst, T.tensor)) continue;
            v.clear();
            core::append_runs(T, v);
            auto m0 = std::partition_point(P.d2_multi.begin(), P.d2_multi.end(),
                                           [&](const core::PlanCore::D2Multi& m) { return m.dst < T.dst; });
            for (const core::FlatXfer& f : v) {
                std::int64_t at = f.lo;
                for (auto m = m0; m != P.d2_multi.end() && m->dst == T.dst && m->lo < f.hi; ++m) {
                    if (m->hi <= at || m->chosen == T.src) continue;
                    if (m->lo > at) E.flat_run(core::FlatXfer{at, m->lo, T.src, T.dst});
                    at = std::max(at, m->hi);
                }
                if (at < f.hi) E.flat_run(core::FlatXfer{at, f.hi, T.src, T.dst});
            }
        }
    }
    if (P.has_scalars)
        for (int j = 0; j < P.dst_cfg.world_size(); ++j)
            ops.push_back(CopyOp{0, kScalars, j, kScalars, 0, 0, 1, P.scalar_bytes_per_rank, 0, 0});
    return ops;
}

PlacementStats placement_stats(const PlanCore& P, int n_gpus, int gpu) {
    int max_phys = 0;
    for (const auto& r : P.routes) max_phys = std::max(max_phys, r.phys);
    const int per = (max_phys + 1 + n_gpus - 1) / n_gpus;
    auto gpu_src = [&](int rank) { return P.wm.src_phys[static_cast<size_t>(rank)] / per; };
    auto gpu_dst = [&](int rank) { return P.wm.dst_phys[static_cast<size_t>(rank)] / per; };
    PlacementStats s;
    for (const CopyOp& op : build_ops(P)) {
        const std::int64_t b = op.rows * op.row_bytes;
        const int gs = gpu_src(op.src_side_rank), gd = gpu_dst(op.dst_rank);
        if (gs == gpu) {
            ++s.ops;
            (gd == gpu ? s.local_bytes : s.out_bytes) += b;
        } else if (gd == gpu) {
            s.in_bytes += b;
        }
    }
    return s;
}

void buffer_sizes(const PlanCore& P, int side, int rank, bool with_grads, std::int64_t out[kNumBufs]) {
    const RankGeom& g = (side == 0 ? P.src : P.dst).ranks[static_cast<size_t>(rank)];
    out[kParam] = g.param_bytes;
    out[kMaster] = out[kM] = out[kV] = g.optim_len * 4;
    out[kGrad] = with_grads ? g.nelem * 4 : 0;
    out[kScalars] = P.opts.scalar_words * kScalarWordBytes;
}

}  // namespace exec
}  // namespace reshard

namespace reshard {
namespace exec {

std::vector<std::int64_t> traffic_matrix(const PlanCore& P, int* n_out) {
    int n = 0;
    for (const auto& r : P.routes) n = std::max(n, r.phys + 1);
    std::vector<std::int64_t> m(static_cast<size_t>(n) * static_cast<size_t>(n), 0);
    for (const CopyOp& op : build_ops(P)) {
        const int s = P.wm.src_phys[static_cast<size_t>(op.src_side_rank)];
        const int d = P.wm.dst_phys[static_cast<size_t>(op.dst_rank)];
        m[static_cast<size_t>(s) * static_cast<size_t>(n) + static_cast<size_t>(d)] += op.rows * op.row_bytes;
    }
    if (n_out) *n_out = n;
    return m;
}

}  // namespace exec
}  // namespace reshard
