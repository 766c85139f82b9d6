// Host side of the planner: geometry, box routing (reference candidate and
// proximity rules), ZeRO triples, D2 detection/extension, flat-run expansion and
// the reference dump format.
#include "reshard/plan_core.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>

namespace reshard {
namespace core {

namespace {

struct Lifted {
    int np;
    std::int64_t lo[4], hi[4];  // planes..., row, col
    std::int64_t ext[4];
};

Lifted lift(const TensorSpec& t, const std::int64_t* blo, const std::int64_t* bhi) {
    Lifted L{};
    const int nd = static_cast<int>(t.shape.size());
    int o = 0;
    if (nd == 1) {
        L.lo[0] = 0;
        L.hi[0] = 1;
        L.ext[0] = 1;
        o = 1;
    }
    for (int d = 0; d < nd; ++d) {
        L.lo[o + d] = blo[d];
        L.hi[o + d] = bhi[d];
        L.ext[o + d] = t.shape[static_cast<size_t>(d)];
    }
    L.np = std::max(nd, 2) - 2;
    return L;
}

stair::TensorView view_of(const ModelSpace::Entry& e) {
    std::int64_t z[4] = {0, 0, 0, 0};
    const Lifted L = lift(e.spec, z, z);
    stair::TensorView v{};
    v.np = L.np;
    for (int i = 0; i < L.np; ++i) v.pext[i] = L.ext[i];
    v.rows = L.ext[L.np];
    v.cols = L.ext[L.np + 1];
    v.off = e.offset;
    return v;
}

/// Stair of a segment restricted to the element range [lo,hi) of its span.
bool make_stair(const TensorSpec& t, const Seg& s, Interval range, stair::Stair* out) {
    const std::int64_t a = std::max(range.lo, s.local_lo) - s.local_lo;
    const std::int64_t b = std::min(range.hi, s.local_hi) - s.local_lo;
    if (a >= b) return false;
    const Lifted L = lift(t, s.blo, s.bhi);
    stair::Stair X{};
    for (int i = 0; i < L.np; ++i) {
        X.plo[i] = L.lo[i];
        X.phi[i] = L.hi[i];
    }
    X.rlo = L.lo[L.np];
    X.rhi = L.hi[L.np];
    X.clo = L.lo[L.np + 1];
    X.chi = L.hi[L.np + 1];
    X.a = a;
    X.b = b;
    *out = X;
    return true;
}

const Interval& shard_of(const RankGeom& g, const Seg& s) { return s.expert ? g.eshard : g.dshard; }

/// Triple (J ∩ K) \ I; false if the iteration space is empty.
bool make_triple(const ModelSpace& space, int t, const RankGeom& k, const RankGeom& j, const RankGeom* own,
                 stair::Triple* T) {
    const int sk = k.seg_of[static_cast<size_t>(t)], sj = j.seg_of[static_cast<size_t>(t)];
    if (sk < 0 || sj < 0) return false;
    const auto& e = space.entries()[static_cast<size_t>(t)];
    const Seg& Sk = k.segs[static_cast<size_t>(sk)];
    const Seg& Sj = j.segs[static_cast<size_t>(sj)];
    stair::Triple X{};
    if (!make_stair(e.spec, Sk, shard_of(k, Sk), &X.K)) return false;
    if (!make_stair(e.spec, Sj, shard_of(j, Sj), &X.J)) return false;
    X.t = view_of(e);
    std::int64_t n = 1;
    for (int i = 0; i < X.t.np; ++i) {
        X.plo[i] = std::max(X.K.plo[i], X.J.plo[i]);
        X.phi[i] = std::min(X.K.phi[i], X.J.phi[i]);
        if (X.plo[i] >= X.phi[i]) return false;
        n *= X.phi[i] - X.plo[i];
    }
    X.rlo = std::max(X.K.rlo, X.J.rlo);
    X.rhi = std::min(X.K.rhi, X.J.rhi);
    if (X.rlo >= X.rhi) return false;
    if (std::max(X.K.clo, X.J.clo) >= std::min(X.K.chi, X.J.chi)) return false;
    X.nrows = n * (X.rhi - X.rlo);
    X.has_i = 0;
    if (own) {
        const int si = own->seg_of[static_cast<size_t>(t)];
        if (si >= 0) {
            const Seg& Si = own->segs[static_cast<size_t>(si)];
            if (make_stair(e.spec, Si, shard_of(*own, Si), &X.I)) X.has_i = 1;
        }
    }
    X.src = k.rank;
    X.dst = j.rank;
    X.tensor = t;
    *T = X;
    return true;
}

/// Append runs of a triple (band sweep) with normalize_intervals-style merging.
void append_runs(const stair::Triple& T, std::vector<FlatXfer>& out) {
    for_each_band(T, [&](const std::int64_t* p, std::int64_t u, std::int64_t v, const stair::Iv* cols, int n) {
        const bool full = n == 1 && cols[0].lo == 0 && cols[0].hi == T.t.cols;
        auto push = [&](std::int64_t lo, std::int64_t hi) {
            if (!out.empty() && out.back().src == T.src && out.back().dst == T.dst && out.back().hi == lo)
                out.back().hi = hi;
            else
                out.push_back(FlatXfer{lo, hi, T.src, T.dst});
        };
        if (full) {
            push(stair::flat_of(T.t, p, u, 0), stair::flat_of(T.t, p, v, 0));
            return;
        }
        for (std::int64_t r = u; r < v; ++r)
            for (int i = 0; i < n; ++i) push(stair::flat_of(T.t, p, r, cols[i].lo), stair::flat_of(T.t, p, r, cols[i].hi));
    });
}

std::int64_t triple_count(const stair::Triple& T) {
    std::int64_t n = 0;
    for_each_band(T, [&](const std::int64_t*, std::int64_t u, std::int64_t v, const stair::Iv* cols, int k) {
        for (int i = 0; i < k; ++i) n += (v - u) * (cols[i].hi - cols[i].lo);
    });
    return n;
}

Box box_of(const Seg& s, int nd) {
    Box b;
    b.dims.resize(static_cast<size_t>(nd));
    for (int d = 0; d < nd; ++d) b.dims[static_cast<size_t>(d)] = {s.blo[d], s.bhi[d]};
    return b;
}

struct Pending {
    int kind;
    int tensor;
    Box cell;
    int dst_phys, dst_rank;
    std::vector<int> cands;
};

}  // namespace

int payload_width(const ModelSpace& space, int kind, int tensor) {
    switch (kind) {
        case 0: return space.entries()[static_cast<size_t>(tensor)].spec.dtype_bytes;
        case 1: return kOptimStateBytes;
        case 2: return kGradBytes;
        default: return kScalarWordBytes;
    }
}

bool box_xfer_less(const PlanCore& P, const BoxXfer& a, const BoxXfer& b) {
    if (a.src != b.src) return a.src < b.src;
    if (a.dst != b.dst) return a.dst < b.dst;
    if (a.kind != b.kind) return a.kind < b.kind;
    if (a.tensor != b.tensor) return P.id_rank[static_cast<size_t>(a.tensor)] < P.id_rank[static_cast<size_t>(b.tensor)];
    const int nd = static_cast<int>(P.space->entries()[static_cast<size_t>(a.tensor)].spec.shape.size());
    for (int d = 0; d < nd; ++d) {
        if (a.lo[d] != b.lo[d]) return a.lo[d] < b.lo[d];
        if (a.hi[d] != b.hi[d]) return a.hi[d] < b.hi[d];
    }
    return false;
}

Side build_side(const ModelSpace& space, const ParallelConfig& cfg) {
    Side S;
    S.cfg = cfg;
    const int nt = static_cast<int>(space.entries().size());
    S.ranks.resize(static_cast<size_t>(cfg.world_size()));
    for (int r = 0; r < cfg.world_size(); ++r) {
        RankGeom& g = S.ranks[static_cast<size_t>(r)];
        g.rank = r;
        g.coord = rank_coord(cfg, r);
        g.seg_of.assign(static_cast<size_t>(nt), -1);
        std::vector<Seg> dense, expert;
        for (int t = 0; t < nt; ++t) {
            const TensorSpec& ts = space.entries()[static_cast<size_t>(t)].spec;
            const Box b = rank_box(space, cfg, g.coord, ts);
            if (b.dims.empty()) continue;
            Seg s;
            s.tensor = t;
            s.expert = ts.is_expert;
            for (size_t d = 0; d < b.dims.size(); ++d) {
                s.blo[d] = b.dims[d].lo;
                s.bhi[d] = b.dims[d].hi;
            }
            const std::int64_t n = b.numel();
            std::int64_t& len = ts.is_expert ? g.expert_len : g.dense_len;
            s.local_lo = len;
            s.local_hi = len + n;
            len += n;
            (ts.is_expert ? expert : dense).push_back(s);
        }
        std::int64_t bytes = 0, elems = 0;
        for (std::vector<Seg>* list : {&dense, &expert})
            for (Seg& s : *list) {
                // every segment starts 16-B aligned: natural alignment for any dtype and
                // full 16-B vectors for the copy kernels (no padding at these models' shapes)
                bytes = (bytes + 15) / 16 * 16;
                s.param_byte_off = bytes;
                s.elem_off = elems;
                bytes += (s.local_hi - s.local_lo) * space.entries()[static_cast<size_t>(s.tensor)].spec.dtype_bytes;
                elems += s.local_hi - s.local_lo;
                g.seg_of[static_cast<size_t>(s.tensor)] = static_cast<int>(g.segs.size());
                g.segs.push_back(s);
            }
        g.param_bytes = bytes;
        g.nelem = elems;
        if (cfg.zero_enabled) {
            g.dshard = detail::shard_range(g.dense_len, cfg.dp, g.coord.dp_rank);
            g.eshard = detail::shard_range(g.expert_len, cfg.dp / cfg.ep, g.coord.edp_rank);
        } else {
            g.dshard = {0, g.dense_len};
            g.eshard = {0, g.expert_len};
        }
        g.optim_len = g.dshard.length() + g.eshard.length();
    }
    return S;
}

namespace {

/// D2 handling for one destination rank: full runs from every source, merged to
/// the reference's recv intervals (maximal runs of D_j \ S_own), over-coverage
/// detection, and (allow mode) uniform-candidate re-splitting of over-sourced ivs.
struct D2Result {
    bool over = false;
    Interval first_bad_iv{0, 0};
    std::vector<FlatXfer> final_runs;  // allow mode: the route's final runs, (src, lo) order
    std::vector<int> flagged_tensors;
};

D2Result d2_route(const PlanCore& P, int j, const std::vector<const stair::Triple*>& trip, bool build_final,
                  std::int64_t* cursor) {
    D2Result R;
    struct Piece {
        std::int64_t lo, hi;
        int src;
    };
    std::vector<Piece> pieces;
    for (const stair::Triple* T : trip) {
        std::vector<FlatXfer> v;
        append_runs(*T, v);
        for (const FlatXfer& f : v) pieces.push_back({f.lo, f.hi, f.src});
    }
    (void)j;
    std::sort(pieces.begin(), pieces.end(), [](const Piece& a, const Piece& b) {
        return a.lo != b.lo ? a.lo < b.lo : (a.hi != b.hi ? a.hi < b.hi : a.src < b.src);
    });
    // recv ivs = union of pieces (every recv element is covered by >= 1 source)
    std::vector<Interval> ivs, multi;
    for (const Piece& p : pieces) {
        if (!ivs.empty() && p.lo <= ivs.back().hi) ivs.back().hi = std::max(ivs.back().hi, p.hi);
        else ivs.push_back({p.lo, p.hi});
    }
    // over-coverage per iv: total piece length vs iv length
    size_t pi = 0;
    std::vector<std::int64_t> bounds;
    for (const Interval& iv : ivs) {
        size_t first = pi;
        std::int64_t total = 0;
        while (pi < pieces.size() && pieces[pi].lo < iv.hi) total += pieces[pi].hi - pieces[pi].lo, ++pi;
        const bool bad = total != iv.length();
        if (bad && !R.over) {
            R.over = true;
            R.first_bad_iv = iv;
        }
        if (!build_final) continue;
        if (!bad) {
            // pieces partition the iv; consecutive pieces of one source abut -> one run
            for (size_t q = first; q < pi; ++q) {
                if (q > first && R.final_runs.back().src == pieces[q].src && R.final_runs.back().hi == pieces[q].lo)
                    R.final_runs.back().hi = pieces[q].hi;
                else
                    R.final_runs.push_back({pieces[q].lo, pieces[q].hi, pieces[q].src, -1});
            }
            continue;
        }
        // uniform-candidate runs (oracle.c plan_optimizer D2 extension)
        bounds.clear();
        bounds.push_back(iv.lo);
        bounds.push_back(iv.hi);
        for (size_t q = first; q < pi; ++q) bounds.push_back(pieces[q].lo), bounds.push_back(pieces[q].hi);
        std::sort(bounds.begin(), bounds.end());
        bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
        std::int64_t run_lo = -1, run_hi = -1;
        std::vector<int> run_c, cs;
        auto flush = [&]() {
            if (run_c.empty()) return;
            int chosen;
            if (P.opts.balance_fanout && run_c.size() > 1) {
                chosen = run_c[static_cast<size_t>((*cursor)++) % run_c.size()];
            } else {
                chosen = -1;
                const int dphys = P.wm.dst_phys[static_cast<size_t>(j)];
                for (int c : run_c)
                    if (P.topo.same_node(P.wm.src_phys[static_cast<size_t>(c)], dphys)) {
                        chosen = c;
                        break;
                    }
                if (chosen < 0) chosen = run_c.front();
            }
            R.final_runs.push_back({run_lo, run_hi, chosen, -1});
            if (run_c.size() > 1) multi.push_back({run_lo, run_hi});
        };
        for (size_t b = 0; b + 1 < bounds.size(); ++b) {
            const std::int64_t lo = bounds[b], hi = bounds[b + 1];
            cs.clear();
            for (size_t q = first; q < pi; ++q)
                if (pieces[q].lo <= lo && hi <= pieces[q].hi) cs.push_back(pieces[q].src);
            std::sort(cs.begin(), cs.end());
            cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
            if (!run_c.empty() && run_hi == lo && cs == run_c) {
                run_hi = hi;
            } else {
                flush();
                run_lo = lo;
                run_hi = hi;
                run_c = cs;
            }
        }
        flush();
    }
    // tensors holding over-sourced elements: the executor takes their optimizer moves from
    // the resolved runs (a choice among replicas); elsewhere every element has a single
    // source, exactly as in the triples
    for (const stair::Triple* T : trip) {
        const std::int64_t tlo = T->t.off;
        const std::int64_t thi = tlo + P.space->entries()[static_cast<size_t>(T->tensor)].spec.numel();
        for (const Interval& m : multi)
            if (m.lo < thi && tlo < m.hi) {
                R.flagged_tensors.push_back(T->tensor);
                break;
            }
    }
    return R;
}

}  // namespace

PlanCore build_plan(const ModelSpace& space, const ParallelConfig& srcc, const ParallelConfig& dstc,
                    const WorldMap* wmp, const Topology& topo, const PlanOptions& opts, bool allow_oversourced) {
    // CLI order: validate both configs, then the routing passes.
    ModelSpec ms;
    ms.num_layers = space.num_layers();
    ms.num_experts = space.num_experts();
    for (const auto& e : space.entries()) ms.tensors.push_back(e.spec);
    validate_config(srcc, ms);
    validate_config(dstc, ms);

    PlanCore P;
    P.space = &space;
    P.src_cfg = srcc;
    P.dst_cfg = dstc;
    P.topo = topo;
    P.opts = opts;
    P.allow_oversourced = allow_oversourced;
    P.wm = wmp ? *wmp : WorldMap::identity(srcc.world_size(), dstc.world_size());
    P.wm.validate();
    if (P.wm.src_world_size() != srcc.world_size()) throw ConfigError("world map src size does not match src config");
    if (P.wm.dst_world_size() != dstc.world_size()) throw ConfigError("world map dst size does not match dst config");

    const int nt = static_cast<int>(space.entries().size());
    P.by_id.resize(static_cast<size_t>(nt));
    std::iota(P.by_id.begin(), P.by_id.end(), 0);
    std::sort(P.by_id.begin(), P.by_id.end(), [&](int a, int b) {
        return space.entries()[static_cast<size_t>(a)].spec.tensor_id < space.entries()[static_cast<size_t>(b)].spec.tensor_id;
    });
    P.id_rank.resize(static_cast<size_t>(nt));
    for (int i = 0; i < nt; ++i) P.id_rank[static_cast<size_t>(P.by_id[static_cast<size_t>(i)])] = i;

    P.src = build_side(space, srcc);
    P.dst = build_side(space, dstc);
    for (int i = 0; i < srcc.world_size(); ++i) P.src.ranks[static_cast<size_t>(i)].phys = P.wm.src_phys[static_cast<size_t>(i)];
    for (int j = 0; j < dstc.world_size(); ++j) P.dst.ranks[static_cast<size_t>(j)].phys = P.wm.dst_phys[static_cast<size_t>(j)];
    for (int phys : P.wm.participants()) P.routes.push_back({phys, P.wm.src_rank_of(phys), P.wm.dst_rank_of(phys)});

    // ---- box routing: recv cells with candidates, in the reference's pending order
    // (routing.hpp:205-222, :253-265; cells per route, tensors in id order).
    std::vector<Pending> pend;
    std::vector<size_t> route_begin, route_end;
    const int ns = srcc.world_size();
    for (const RouteInfo& r : P.routes) {
        route_begin.push_back(pend.size());
        if (r.dst_rank >= 0) {
            const RankGeom& D = P.dst.ranks[static_cast<size_t>(r.dst_rank)];
            const RankGeom* own = r.src_rank >= 0 ? &P.src.ranks[static_cast<size_t>(r.src_rank)] : nullptr;
            for (int oi = 0; oi < nt; ++oi) {
                const int t = P.by_id[static_cast<size_t>(oi)];
                const int sd = D.seg_of[static_cast<size_t>(t)];
                if (sd < 0) continue;
                const TensorSpec& ts = space.entries()[static_cast<size_t>(t)].spec;
                const int nd = static_cast<int>(ts.shape.size());
                const Box dbox = box_of(D.segs[static_cast<size_t>(sd)], nd);
                std::vector<Box> recv;
                const int so = own ? own->seg_of[static_cast<size_t>(t)] : -1;
                if (so >= 0) recv = detail::boxes_diff({dbox}, {box_of(own->segs[static_cast<size_t>(so)], nd)});
                else recv = {dbox};
                for (const Box& rb : recv) {
                    for (Box& cell : split_by_projection_grid(space, srcc, ts.tensor_id, rb)) {
                        std::vector<int> cands;
                        for (int k = 0; k < ns; ++k) {
                            const RankGeom& K = P.src.ranks[static_cast<size_t>(k)];
                            const int sk = K.seg_of[static_cast<size_t>(t)];
                            if (sk >= 0 && box_of(K.segs[static_cast<size_t>(sk)], nd).contains(cell)) cands.push_back(k);
                        }
                        if (cands.empty())
                            throw ConfigError(strfmt("unreachable state: no source holds %s %s needed by device %d",
                                                     ts.tensor_id.c_str(), format_box(cell).c_str(), r.phys));
                        pend.push_back(Pending{0, t, std::move(cell), r.phys, r.dst_rank, std::move(cands)});
                    }
                }
            }
        }
        route_end.push_back(pend.size());
    }
    const size_t n_param = pend.size();
    if (opts.gradients == GradientPolicy::Migrate)
        for (size_t i = 0; i < n_param; ++i) {
            Pending g = pend[i];
            g.kind = 2;
            pend.push_back(std::move(g));
        }
    if (srcc.zero_enabled != dstc.zero_enabled) throw ConfigError("transitions toggling zero_enabled are unsupported");
    if (!srcc.zero_enabled)
        for (size_t ri = 0; ri < P.routes.size(); ++ri)
            for (size_t i = route_begin[ri]; i < route_end[ri]; ++i) {
                Pending o = pend[i];
                o.kind = 1;
                pend.push_back(std::move(o));
            }

    // ---- resolve_peers for box pendings (routing.hpp:360-396)
    std::int64_t cursor = 0;
    P.box.reserve(pend.size());
    for (const Pending& p : pend) {
        int chosen;
        if (opts.balance_fanout && p.cands.size() > 1) {
            chosen = p.cands[static_cast<size_t>(cursor++) % p.cands.size()];
        } else {
            chosen = -1;
            for (int c : p.cands)
                if (topo.same_node(P.wm.src_phys[static_cast<size_t>(c)], p.dst_phys)) {
                    chosen = c;
                    break;
                }
            if (chosen < 0) chosen = p.cands.front();
        }
        BoxXfer x;
        x.kind = p.kind;
        x.tensor = p.tensor;
        for (size_t d = 0; d < p.cell.dims.size(); ++d) {
            x.lo[d] = p.cell.dims[d].lo;
            x.hi[d] = p.cell.dims[d].hi;
        }
        x.src = chosen;
        x.dst = p.dst_rank;
        x.count = p.cell.numel();
        x.bytes = x.count * payload_width(space, p.kind, p.tensor);
        P.box.push_back(x);
    }
    std::sort(P.box.begin(), P.box.end(), [&](const BoxXfer& a, const BoxXfer& b) { return box_xfer_less(P, a, b); });

    // ---- retained boxes (routing.hpp:98 retain = R_src ∩ R_dst), same device
    std::int64_t retained = 0;
    for (const RouteInfo& r : P.routes) {
        if (r.src_rank < 0 || r.dst_rank < 0) continue;
        const RankGeom& S = P.src.ranks[static_cast<size_t>(r.src_rank)];
        const RankGeom& D = P.dst.ranks[static_cast<size_t>(r.dst_rank)];
        for (int t = 0; t < nt; ++t) {
            const int ss = S.seg_of[static_cast<size_t>(t)], sd = D.seg_of[static_cast<size_t>(t)];
            if (ss < 0 || sd < 0) continue;
            const TensorSpec& ts = space.entries()[static_cast<size_t>(t)].spec;
            const int nd = static_cast<int>(ts.shape.size());
            const Box x = intersect(box_of(S.segs[static_cast<size_t>(ss)], nd), box_of(D.segs[static_cast<size_t>(sd)], nd));
            if (x.empty()) continue;
            BoxXfer b;
            b.tensor = t;
            for (int d = 0; d < nd; ++d) {
                b.lo[d] = x.dims[static_cast<size_t>(d)].lo;
                b.hi[d] = x.dims[static_cast<size_t>(d)].hi;
            }
            b.src = r.src_rank;
            b.dst = r.dst_rank;
            b.count = x.numel();
            retained += b.count * ts.dtype_bytes;
            if (!srcc.zero_enabled) retained += b.count * kOptimStateBytes;
            const int kinds[3] = {0, 2, 1};
            for (int kind : kinds) {
                if (kind == 2 && opts.gradients != GradientPolicy::Migrate) continue;
                if (kind == 1 && srcc.zero_enabled) continue;
                b.kind = kind;
                b.bytes = b.count * payload_width(space, kind, t);
                P.box_retain.push_back(b);
            }
        }
    }

    // ---- ZeRO optimizer routing (routing.hpp:305-336) in closed form
    std::int64_t flat_elems = 0;
    if (srcc.zero_enabled) {
        const int ndst = dstc.world_size();
        std::vector<std::vector<const stair::Triple*>> by_dst(static_cast<size_t>(ndst));
        for (int k = 0; k < ns; ++k)
            for (int j = 0; j < ndst; ++j) {
                const RankGeom& J = P.dst.ranks[static_cast<size_t>(j)];
                const int own = P.wm.src_rank_of(J.phys);
                if (own == k) continue;  // R_j ∩ S_own = ∅
                const RankGeom* O = own >= 0 ? &P.src.ranks[static_cast<size_t>(own)] : nullptr;
                for (int t = 0; t < nt; ++t) {
                    stair::Triple T;
                    if (make_triple(space, t, P.src.ranks[static_cast<size_t>(k)], J, O, &T)) P.triples.push_back(T);
                }
            }
        for (const stair::Triple& T : P.triples) by_dst[static_cast<size_t>(T.dst)].push_back(&T);
        for (const RouteInfo& r : P.routes) {
            if (r.src_rank < 0 || r.dst_rank < 0) continue;
            for (int t = 0; t < nt; ++t) {
                stair::Triple T;
                if (make_triple(space, t, P.src.ranks[static_cast<size_t>(r.src_rank)],
                                P.dst.ranks[static_cast<size_t>(r.dst_rank)], nullptr, &T))
                    P.retain_triples.push_back(T);
            }
        }
        for (const stair::Triple& T : P.retain_triples) retained += triple_count(T) * kOptimStateBytes;

        // D2: only tensors replicated across src TP ranks can be covered by two shards.
        bool d2_possible = false;
        if (srcc.tp > 1)
            for (const auto& e : space.entries()) d2_possible |= !e.spec.tp_shard_axis.has_value();
        std::vector<char> d2_dst(static_cast<size_t>(ndst), 0);
        if (d2_possible) {
            // cursor position after box pendings (params, grads) for the extension
            std::int64_t cur = cursor;
            for (const RouteInfo& r : P.routes) {
                if (r.dst_rank < 0) continue;
                const int j = r.dst_rank;
                std::vector<const stair::Triple*> rep;
                for (const stair::Triple* T : by_dst[static_cast<size_t>(j)])
                    if (!space.entries()[static_cast<size_t>(T->tensor)].spec.tp_shard_axis) rep.push_back(T);
                if (rep.empty()) continue;
                // quick over-coverage test on replicated tensors only
                std::vector<FlatXfer> v;
                for (const stair::Triple* T : rep) append_runs(*T, v);
                std::sort(v.begin(), v.end(), [](const FlatXfer& a, const FlatXfer& b) { return a.lo < b.lo; });
                bool over = false;
                std::int64_t reach = v.empty() ? 0 : v[0].hi;
                for (size_t i = 1; i < v.size() && !over; ++i) {
                    over = v[i].lo < reach;
                    reach = std::max(reach, v[i].hi);
                }
                if (!over) continue;
                D2Result R = d2_route(P, j, by_dst[static_cast<size_t>(j)], allow_oversourced, &cur);
                if (!R.over) continue;
                if (!allow_oversourced)
                    throw ConfigError(strfmt("unreachable state: optimizer interval [%lld:%lld] for device %d not fully sourced",
                                             static_cast<long long>(R.first_bad_iv.lo),
                                             static_cast<long long>(R.first_bad_iv.hi), r.phys));
                d2_dst[static_cast<size_t>(j)] = 1;
                if (P.d2_tensor_dst.empty()) P.d2_tensor_dst.assign(static_cast<size_t>(ndst) * nt, 0);
                for (int t : R.flagged_tensors) P.d2_tensor_dst[static_cast<size_t>(j) * nt + t] = 1;
                for (FlatXfer& f : R.final_runs) {
                    f.dst = j;
                    P.d2_runs.push_back(f);
                }
            }
            std::stable_sort(P.d2_runs.begin(), P.d2_runs.end(), [](const FlatXfer& a, const FlatXfer& b) {
                if (a.src != b.src) return a.src < b.src;
                if (a.dst != b.dst) return a.dst < b.dst;
                return a.lo < b.lo;
            });
            // merge abutting runs of the same (src,dst) only where the reference would:
            // D2 runs are kept as produced (uniform pieces are separate pendings).
        }
        // transfer count + bytes: non-D2 routes from triples, D2 routes from final runs
        std::vector<FlatXfer> tmp;
        for (const stair::Triple& T : P.triples) {
            if (d2_dst[static_cast<size_t>(T.dst)]) continue;
            flat_elems += triple_count(T);
        }
        for (const FlatXfer& f : P.d2_runs) flat_elems += f.hi - f.lo;
        P.n_flat = -1;  // resolved lazily by expand_* (count needs merging)
        {
            // count transfers exactly: merged runs per (src,dst) group
            std::int64_t cnt = 0;
            int cs = -1, cd = -1;
            std::int64_t last_hi = -1;
            for (const stair::Triple& T : P.triples) {
                if (d2_dst[static_cast<size_t>(T.dst)]) continue;
                tmp.clear();
                append_runs(T, tmp);
                for (const FlatXfer& f : tmp) {
                    if (f.src == cs && f.dst == cd && f.lo == last_hi) {
                        last_hi = f.hi;
                        continue;
                    }
                    ++cnt;
                    cs = f.src;
                    cd = f.dst;
                    last_hi = f.hi;
                }
            }
            P.n_flat = cnt + static_cast<std::int64_t>(P.d2_runs.size());
        }
    }

    // ---- scalars (routing.hpp:341-353)
    if (P.wm.src_world_size() > 0) {
        P.has_scalars = true;
        P.scalar_root_phys = P.wm.src_phys[0];
        P.scalar_bytes_per_rank = opts.scalar_words * kScalarWordBytes;
        for (int phys : P.wm.dst_phys)
            if (phys != P.scalar_root_phys) P.scalar_recv_phys.push_back(phys);
        std::sort(P.scalar_recv_phys.begin(), P.scalar_recv_phys.end());
    }

    std::int64_t moved = 0;
    for (const BoxXfer& b : P.box) moved += b.bytes;
    moved += flat_elems * kOptimStateBytes;
    if (P.has_scalars) moved += P.scalar_bytes_per_rank * static_cast<std::int64_t>(P.scalar_recv_phys.size());
    P.bytes_moved = moved;
    P.bytes_retained = retained;
    return P;
}

namespace {
bool is_d2(const PlanCore& P, int dst) {
    for (const FlatXfer& f : P.d2_runs)
        if (f.dst == dst) return true;
    return false;
}

std::vector<FlatXfer> merge_with_d2(const PlanCore& P, std::vector<FlatXfer> base) {
    if (P.d2_runs.empty()) return base;
    std::vector<FlatXfer> out;
    out.reserve(base.size() + P.d2_runs.size());
    std::merge(base.begin(), base.end(), P.d2_runs.begin(), P.d2_runs.end(), std::back_inserter(out),
               [](const FlatXfer& a, const FlatXfer& b) {
                   if (a.src != b.src) return a.src < b.src;
                   if (a.dst != b.dst) return a.dst < b.dst;
                   return a.lo < b.lo;
               });
    return out;
}
}  // namespace

std::vector<FlatXfer> expand_flat_host(const PlanCore& P) {
    std::vector<FlatXfer> out;
    std::vector<char> skip(static_cast<size_t>(P.dst_cfg.world_size()), 0);
    for (int j = 0; j < P.dst_cfg.world_size(); ++j) skip[static_cast<size_t>(j)] = is_d2(P, j);
    for (const stair::Triple& T : P.triples)
        if (!skip[static_cast<size_t>(T.dst)]) append_runs(T, out);
    return merge_with_d2(P, std::move(out));
}

std::vector<FlatXfer> expand_flat_rows_host(const PlanCore& P) {
    std::vector<FlatXfer> out;
    std::vector<char> skip(static_cast<size_t>(P.dst_cfg.world_size()), 0);
    for (int j = 0; j < P.dst_cfg.world_size(); ++j) skip[static_cast<size_t>(j)] = is_d2(P, j);
    for (const stair::Triple& T : P.triples) {
        if (skip[static_cast<size_t>(T.dst)]) continue;
        for (std::int64_t q = 0; q < T.nrows; ++q) {
            stair::Iv r[2];
            const int n = stair::triple_row_runs(T, q, r);
            for (int i = 0; i < n; ++i) {
                if (!out.empty() && out.back().src == T.src && out.back().dst == T.dst && out.back().hi == r[i].lo)
                    out.back().hi = r[i].hi;
                else
                    out.push_back({r[i].lo, r[i].hi, T.src, T.dst});
            }
        }
    }
    return merge_with_d2(P, std::move(out));
}

std::string dump(const PlanCore& P, const std::vector<FlatXfer>& flat) { return dump(P, P.box, flat); }

std::string dump(const PlanCore& P, const std::vector<BoxXfer>& boxes, const std::vector<FlatXfer>& flat) {
    const ModelSpace& space = *P.space;
    std::string out;
    out.reserve(static_cast<size_t>(boxes.size() + flat.size()) * 56);
    char line[1024];
    auto box_line = [&](const BoxXfer& b) {
        const TensorSpec& ts = space.entries()[static_cast<size_t>(b.tensor)].spec;
        int n = std::snprintf(line, sizeof line, "%s %s [", to_string(static_cast<StateKind>(b.kind)), ts.tensor_id.c_str());
        for (size_t d = 0; d < ts.shape.size(); ++d)
            n += std::snprintf(line + n, sizeof line - static_cast<size_t>(n), d ? ",%lld:%lld" : "%lld:%lld",
                               static_cast<long long>(b.lo[d]), static_cast<long long>(b.hi[d]));
        n += std::snprintf(line + n, sizeof line - static_cast<size_t>(n), "] src=%d dst=%d bytes=%lld\n", b.src, b.dst,
                           static_cast<long long>(b.bytes));
        out.append(line, static_cast<size_t>(n));
    };
    auto flat_line = [&](const FlatXfer& f) {
        const int n = std::snprintf(line, sizeof line, "optim - [%lld:%lld] src=%d dst=%d bytes=%lld\n",
                                    static_cast<long long>(f.lo), static_cast<long long>(f.hi), f.src, f.dst,
                                    static_cast<long long>((f.hi - f.lo) * kOptimStateBytes));
        out.append(line, static_cast<size_t>(n));
    };
    // canonical merge: (src, dst, kind, ...); flat runs are kind Optim with id "".
    size_t bi = 0, fi = 0;
    auto key_less = [](int s1, int d1, int k1, int s2, int d2, int k2) {
        if (s1 != s2) return s1 < s2;
        if (d1 != d2) return d1 < d2;
        return k1 < k2;
    };
    while (bi < boxes.size() || fi < flat.size()) {
        bool take_box;
        if (bi == boxes.size()) take_box = false;
        else if (fi == flat.size()) take_box = true;
        else {
            const BoxXfer& b = boxes[bi];
            const FlatXfer& f = flat[fi];
            // for equal (src,dst,kind=optim) flat ("" id) sorts before any box id
            take_box = key_less(b.src, b.dst, b.kind, f.src, f.dst, 1);
        }
        if (take_box) box_line(boxes[bi++]);
        else flat_line(flat[fi++]);
    }
    return out;
}

}  // namespace core
}  // namespace reshard
