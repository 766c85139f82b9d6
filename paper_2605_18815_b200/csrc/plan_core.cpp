// Host side of the planner: geometry, box routing (reference candidate and
// proximity rules), ZeRO triples, D2 detection/extension, flat-run expansion and
// the reference dump format.
#include "reshard/plan_core.hpp"
#include "reshard/pool.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <thread>

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

/// Stairs of every (rank, tensor) of one side, built once per plan (a triple needs three
/// of them; the (src, dst, tensor) loop would otherwise rebuild each one many times)
struct StairTable {
    std::vector<std::vector<char>> ok;            // [rank][tensor]
    std::vector<std::vector<stair::Stair>> st;    // [rank][tensor]
};

StairTable stair_table(const ModelSpace& space, const Side& side) {
    StairTable T;
    const int nt = static_cast<int>(space.entries().size());
    T.ok.assign(side.ranks.size(), std::vector<char>(static_cast<size_t>(nt), 0));
    T.st.assign(side.ranks.size(), std::vector<stair::Stair>(static_cast<size_t>(nt)));
    for (size_t r = 0; r < side.ranks.size(); ++r) {
        const RankGeom& g = side.ranks[r];
        for (int t = 0; t < nt; ++t) {
            const int sg = g.seg_of[static_cast<size_t>(t)];
            if (sg < 0) continue;
            const Seg& S = g.segs[static_cast<size_t>(sg)];
            T.ok[r][static_cast<size_t>(t)] =
                make_stair(space.entries()[static_cast<size_t>(t)].spec, S, shard_of(g, S), &T.st[r][static_cast<size_t>(t)]);
        }
    }
    return T;
}

/// Triple (J ∩ K) \ I from precomputed stairs (own < 0: no I); false if the iteration
/// space is empty
bool make_triple_cached(const ModelSpace& space, int t, const StairTable& src, const StairTable& dst, int k, int j,
                        int own, const std::vector<stair::TensorView>& views, stair::Triple* T) {
    const size_t tt = static_cast<size_t>(t);
    if (!src.ok[static_cast<size_t>(k)][tt] || !dst.ok[static_cast<size_t>(j)][tt]) return false;
    (void)space;
    // reject on the references first: most (src, dst, tensor) combinations do not meet
    const stair::Stair& K = src.st[static_cast<size_t>(k)][tt];
    const stair::Stair& J = dst.st[static_cast<size_t>(j)][tt];
    const stair::TensorView& V = views[tt];
    std::int64_t plo[2] = {0, 0}, phi[2] = {0, 0}, n = 1;
    for (int i = 0; i < V.np; ++i) {
        plo[i] = std::max(K.plo[i], J.plo[i]);
        phi[i] = std::min(K.phi[i], J.phi[i]);
        if (plo[i] >= phi[i]) return false;
        n *= phi[i] - plo[i];
    }
    const std::int64_t rlo = std::max(K.rlo, J.rlo), rhi = std::min(K.rhi, J.rhi);
    if (rlo >= rhi) return false;
    if (std::max(K.clo, J.clo) >= std::min(K.chi, J.chi)) return false;
    stair::Triple X{};
    X.K = K;
    X.J = J;
    X.t = V;
    for (int i = 0; i < 2; ++i) X.plo[i] = plo[i], X.phi[i] = phi[i];
    X.rlo = rlo;
    X.rhi = rhi;
    X.nrows = n * (rhi - rlo);
    X.has_i = 0;
    if (own >= 0 && src.ok[static_cast<size_t>(own)][tt]) {
        X.I = src.st[static_cast<size_t>(own)][tt];
        X.has_i = 1;
    }
    X.src = k;
    X.dst = j;
    X.tensor = t;
    *T = X;
    return true;
}

}  // namespace

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

namespace {

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

/// the planner's per-route / per-rank-pair loops on the host worker pool (contiguous
/// slices; results are merged in order by the callers)
template <class F>
void parallel_for(size_t n, F&& fn) {
    pool::parallel_for(n, std::forward<F>(fn));
}

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

/// D2 handling for one destination rank. Only tensors replicated across source TP ranks
/// can be covered by two source shards, so over-sourced recv intervals are found from
/// the overlaps of their runs and grown to the reference's maximal recv intervals
/// (normalize_intervals: connected under lo <= hi) through the runs of every source.
/// Inside them (allow mode) the elements are re-split into maximal runs with a uniform
/// candidate set and one source is chosen per run (proximity rule or balance cursor).
struct D2Route {
    std::vector<Interval> bad;       // over-sourced recv intervals, ascending
    std::vector<FlatXfer> patch;     // allow mode: the runs inside them, lo order
    std::vector<PlanCore::D2Multi> multi;
    std::int64_t regular_runs = 0, regular_elems = 0;  // the triples' runs inside `bad`
    std::int64_t patch_elems = 0;
    std::vector<int> flagged_tensors;
};

D2Route d2_route(const PlanCore& P, int j, const std::vector<const stair::Triple*>& trip, bool resolve,
                 std::int64_t* cursor) {
    D2Route R;
    const auto& ents = P.space->entries();
    const int nt = static_cast<int>(ents.size());
    // runs of a triple, expanded on first use: only the triples around over-sourced
    // intervals are ever expanded (a handful of the route's ~2,000)
    std::vector<std::vector<FlatXfer>> cache(trip.size());
    std::vector<char> done(trip.size(), 0);
    auto runs = [&](int ti) -> const std::vector<FlatXfer>& {
        if (!done[static_cast<size_t>(ti)]) {
            append_runs(*trip[static_cast<size_t>(ti)], cache[static_cast<size_t>(ti)]);
            done[static_cast<size_t>(ti)] = 1;
        }
        return cache[static_cast<size_t>(ti)];
    };
    // overlapping runs of the replicated tensors seed the over-sourced intervals
    std::vector<FlatXfer> rep;
    std::vector<int> slot;                      // src rank -> slot
    std::vector<int> slot_src;                  // slot -> src rank
    std::vector<std::vector<int>> tri;          // [slot][tensor] -> index in trip or -1
    for (size_t ti = 0; ti < trip.size(); ++ti) {
        const stair::Triple* T = trip[ti];
        if (T->src >= static_cast<int>(slot.size())) slot.resize(static_cast<size_t>(T->src) + 1, -1);
        int& k = slot[static_cast<size_t>(T->src)];
        if (k < 0) {
            k = static_cast<int>(tri.size());
            tri.emplace_back(static_cast<size_t>(nt), -1);
            slot_src.push_back(T->src);
        }
        tri[static_cast<size_t>(k)][static_cast<size_t>(T->tensor)] = static_cast<int>(ti);
        if (!ents[static_cast<size_t>(T->tensor)].spec.tp_shard_axis) {
            const auto& v = runs(static_cast<int>(ti));
            rep.insert(rep.end(), v.begin(), v.end());
        }
    }
    std::sort(rep.begin(), rep.end(), [](const FlatXfer& a, const FlatXfer& b) { return a.lo < b.lo; });
    std::vector<Interval> seeds;
    for (size_t i = 0; i < rep.size();) {
        std::int64_t reach = rep[i].hi;
        bool over = false;
        size_t e = i + 1;
        for (; e < rep.size() && rep[e].lo <= reach; ++e) {
            over = over || rep[e].lo < reach;
            reach = std::max(reach, rep[e].hi);
        }
        if (over) seeds.push_back({rep[i].lo, reach});
        i = e;
    }
    if (seeds.empty()) return R;
    const std::int64_t space_end = ents.back().offset + ents.back().spec.numel();
    auto tensor_at = [&](std::int64_t x) {
        auto it = std::upper_bound(ents.begin(), ents.end(), x, [](std::int64_t v, const ModelSpace::Entry& e) { return v < e.offset; });
        return static_cast<int>(it - ents.begin()) - 1;
    };
    // grow each seed to its recv interval (normalize_intervals: connected under lo <= hi)
    for (const Interval& sd : seeds) {
        if (!R.bad.empty() && sd.lo <= R.bad.back().hi) continue;  // already inside
        Interval iv = sd;
        for (bool changed = true; changed;) {
            changed = false;
            for (size_t k = 0; k < tri.size(); ++k) {
                for (std::int64_t x : {iv.hi - 1, iv.hi}) {  // a run with lo <= hi < its hi
                    if (x < 0 || x >= space_end) continue;
                    const int ti = tri[k][static_cast<size_t>(tensor_at(x))];
                    if (ti < 0) continue;
                    const auto& l = runs(ti);
                    auto it = std::upper_bound(l.begin(), l.end(), iv.hi, [](std::int64_t y, const FlatXfer& f) { return y < f.lo; });
                    if (it != l.begin() && std::prev(it)->hi > iv.hi) iv.hi = std::prev(it)->hi, changed = true;
                }
                if (iv.lo > 0) {  // a run with lo < lo_iv <= its hi
                    const int ti = tri[k][static_cast<size_t>(tensor_at(iv.lo - 1))];
                    if (ti < 0) continue;
                    const auto& l = runs(ti);
                    auto jt = std::lower_bound(l.begin(), l.end(), iv.lo, [](const FlatXfer& f, std::int64_t y) { return f.hi < y; });
                    if (jt != l.end() && jt->lo < iv.lo) iv.lo = jt->lo, changed = true;
                }
            }
        }
        if (!R.bad.empty() && iv.lo <= R.bad.back().hi) R.bad.back().hi = std::max(R.bad.back().hi, iv.hi);
        else R.bad.push_back(iv);
    }
    // every triple run inside an interval (per source, ascending)
    auto for_runs_in = [&](const Interval& iv, auto&& fn) {
        const int t0 = tensor_at(iv.lo), t1 = tensor_at(iv.hi - 1);
        for (size_t k = 0; k < tri.size(); ++k)
            for (int t = t0; t <= t1; ++t) {
                const int ti = tri[k][static_cast<size_t>(t)];
                if (ti < 0) continue;
                const auto& l = runs(ti);
                auto it = std::lower_bound(l.begin(), l.end(), iv.lo, [](const FlatXfer& f, std::int64_t y) { return f.hi <= y; });
                for (; it != l.end() && it->lo < iv.hi; ++it) fn(static_cast<int>(k), *it);
            }
    };
    struct Ev {
        std::int64_t pos;
        int src, d;
    };
    std::vector<Ev> events;
    std::vector<std::int64_t> bounds;
    std::vector<int> cover(slot.size(), 0), cs, run_c;
    std::vector<Interval> multi;
    std::vector<std::int64_t> prev_hi(tri.size());
    for (const Interval& iv : R.bad) {
        events.clear();
        bounds.clear();
        bounds.push_back(iv.lo);
        bounds.push_back(iv.hi);
        std::fill(prev_hi.begin(), prev_hi.end(), -1);
        for_runs_in(iv, [&](int k, const FlatXfer& f) {
            // the plan's runs merge abutting runs of one source across tensors
            if (f.lo != prev_hi[static_cast<size_t>(k)]) ++R.regular_runs;
            prev_hi[static_cast<size_t>(k)] = f.hi;
            R.regular_elems += f.hi - f.lo;
            events.push_back({f.lo, f.src, +1});
            events.push_back({f.hi, f.src, -1});
            bounds.push_back(f.lo);
            bounds.push_back(f.hi);
        });
        if (!resolve) continue;
        std::sort(bounds.begin(), bounds.end());
        bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
        std::sort(events.begin(), events.end(), [](const Ev& a, const Ev& b) { return a.pos < b.pos; });
        std::fill(cover.begin(), cover.end(), 0);
        std::int64_t run_lo = -1, run_hi = -1;
        run_c.clear();
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
            R.patch.push_back({run_lo, run_hi, chosen, j});
            R.patch_elems += run_hi - run_lo;
            if (run_c.size() > 1) {
                multi.push_back({run_lo, run_hi});
                R.multi.push_back({run_lo, run_hi, j, chosen});
            }
        };
        size_t ei = 0;
        for (size_t b = 0; b + 1 < bounds.size(); ++b) {
            const std::int64_t lo = bounds[b], hi = bounds[b + 1];
            for (; ei < events.size() && events[ei].pos <= lo; ++ei) cover[static_cast<size_t>(events[ei].src)] += events[ei].d;
            cs.clear();
            for (size_t c = 0; c < cover.size(); ++c)
                if (cover[c] > 0) cs.push_back(static_cast<int>(c));
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
    // tensors holding multi-candidate elements: the executor re-derives their moves
    for (const stair::Triple* T : trip) {
        const std::int64_t tlo = T->t.off;
        const std::int64_t thi = tlo + ents[static_cast<size_t>(T->tensor)].spec.numel();
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
    const pool::Warm warm;  // several short parallel loops follow: keep the workers hot
    // RS_TIMING=1: per-phase wall time on stderr
    static const bool timing = std::getenv("RS_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    std::string phases;
    auto phase = [&](const char* name) {
        if (!timing) return;
        const auto t = std::chrono::steady_clock::now();
        phases += strfmt(" %s %.2f", name, std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
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

    pool::run(2, [&](size_t w) {
        if (w == 0) P.src = build_side(space, srcc);
        else P.dst = build_side(space, dstc);
    });
    for (int i = 0; i < srcc.world_size(); ++i) P.src.ranks[static_cast<size_t>(i)].phys = P.wm.src_phys[static_cast<size_t>(i)];
    for (int j = 0; j < dstc.world_size(); ++j) P.dst.ranks[static_cast<size_t>(j)].phys = P.wm.dst_phys[static_cast<size_t>(j)];
    for (int phys : P.wm.participants()) P.routes.push_back({phys, P.wm.src_rank_of(phys), P.wm.dst_rank_of(phys)});

    phase("sides");
    // ---- box routing: recv cells with candidates, in the reference's pending order
    // (routing.hpp:205-222, :253-265; cells per route, tensors in id order).
    std::vector<Pending> pend;
    std::vector<size_t> route_begin, route_end;
    const int ns = srcc.world_size();
    std::vector<std::vector<Pending>> per_route(P.routes.size());
    parallel_for(P.routes.size(), [&](size_t ri) {
        const RouteInfo& r = P.routes[ri];
        std::vector<Pending>& out = per_route[ri];
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
                            // containment straight on the segment's box (no Box built per test)
                            const RankGeom& K = P.src.ranks[static_cast<size_t>(k)];
                            const int sk = K.seg_of[static_cast<size_t>(t)];
                            if (sk < 0) continue;
                            const Seg& g = K.segs[static_cast<size_t>(sk)];
                            bool in = true;
                            for (int d = 0; d < nd && in; ++d)
                                in = g.blo[d] <= cell.dims[static_cast<size_t>(d)].lo &&
                                     cell.dims[static_cast<size_t>(d)].hi <= g.bhi[d];
                            if (in) cands.push_back(k);
                        }
                        if (cands.empty())
                            throw ConfigError(strfmt("unreachable state: no source holds %s %s needed by device %d",
                                                     ts.tensor_id.c_str(), format_box(cell).c_str(), r.phys));
                        out.push_back(Pending{0, t, std::move(cell), r.phys, r.dst_rank, std::move(cands)});
                    }
                }
            }
        }
    });
    for (auto& v : per_route) {
        route_begin.push_back(pend.size());
        for (Pending& x : v) pend.push_back(std::move(x));
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

    phase("box-pending");
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

    phase("box-resolve");
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

    phase("retain");
    // ---- ZeRO optimizer routing (routing.hpp:305-336) in closed form
    std::int64_t flat_elems = 0;
    if (srcc.zero_enabled) {
        const int ndst = dstc.world_size();
        std::vector<std::vector<const stair::Triple*>> by_dst(static_cast<size_t>(ndst));
        StairTable src_st, dst_st;
        pool::run(2, [&](size_t w) {
            if (w == 0) src_st = stair_table(space, P.src);
            else dst_st = stair_table(space, P.dst);
        });
        phase("stairs");
        std::vector<stair::TensorView> views;
        views.reserve(static_cast<size_t>(nt));
        for (int t = 0; t < nt; ++t) views.push_back(view_of(space.entries()[static_cast<size_t>(t)]));
        std::vector<std::vector<stair::Triple>> per_pair(static_cast<size_t>(ns) * ndst);
        parallel_for(per_pair.size(), [&](size_t kj) {
            const int k = static_cast<int>(kj) / ndst, j = static_cast<int>(kj) % ndst;
            const RankGeom& J = P.dst.ranks[static_cast<size_t>(j)];
            const int own = P.wm.src_rank_of(J.phys);
            if (own == k) return;  // R_j ∩ S_own = ∅
            for (int t = 0; t < nt; ++t) {
                stair::Triple T;
                if (make_triple_cached(space, t, src_st, dst_st, k, j, own, views, &T)) per_pair[kj].push_back(T);
            }
        });
        for (const auto& v : per_pair) P.triples.insert(P.triples.end(), v.begin(), v.end());
        for (const stair::Triple& T : P.triples) by_dst[static_cast<size_t>(T.dst)].push_back(&T);
        phase("triples-pairs");
        std::vector<std::vector<stair::Triple>> per_route_retain(P.routes.size());
        parallel_for(P.routes.size(), [&](size_t ri) {
            const RouteInfo& r = P.routes[ri];
            if (r.src_rank < 0 || r.dst_rank < 0) return;
            for (int t = 0; t < nt; ++t) {  // (J ∩ K) of the device's own old and new rank
                stair::Triple T;
                if (make_triple_cached(space, t, src_st, dst_st, r.src_rank, r.dst_rank, -1, views, &T))
                    per_route_retain[ri].push_back(T);
            }
        });
        for (const auto& v : per_route_retain) P.retain_triples.insert(P.retain_triples.end(), v.begin(), v.end());
        for (const stair::Triple& T : P.retain_triples) retained += triple_count(T) * kOptimStateBytes;

        phase("triples");
        // D2: only tensors replicated across src TP ranks can be covered by two shards.
        bool d2_possible = false;
        if (srcc.tp > 1)
            for (const auto& e : space.entries()) d2_possible |= !e.spec.tp_shard_axis.has_value();
        std::int64_t d2_regular_runs = 0, d2_regular_elems = 0, d2_patch_elems = 0;
        if (d2_possible) {
            // cursor position after box pendings (params, grads) for the extension
            std::int64_t cur = cursor;
            std::vector<D2Route> per_route(P.routes.size());
            auto route_d2 = [&](size_t ri, std::int64_t* c) {
                const RouteInfo& r = P.routes[ri];
                if (r.dst_rank >= 0)
                    per_route[ri] = d2_route(P, r.dst_rank, by_dst[static_cast<size_t>(r.dst_rank)], allow_oversourced, c);
            };
            if (opts.balance_fanout) {  // the cursor threads through the routes in order
                for (size_t ri = 0; ri < P.routes.size(); ++ri) route_d2(ri, &cur);
            } else {  // proximity rule: routes are independent
                parallel_for(P.routes.size(), [&](size_t ri) {
                    std::int64_t unused = 0;
                    route_d2(ri, &unused);
                });
            }
            for (size_t ri = 0; ri < P.routes.size(); ++ri) {
                const RouteInfo& r = P.routes[ri];
                if (r.dst_rank < 0) continue;
                const int j = r.dst_rank;
                D2Route& R = per_route[ri];
                if (R.bad.empty()) continue;
                if (!allow_oversourced)
                    throw ConfigError(strfmt("unreachable state: optimizer interval [%lld:%lld] for device %d not fully sourced",
                                             static_cast<long long>(R.bad.front().lo),
                                             static_cast<long long>(R.bad.front().hi), r.phys));
                if (P.d2_bad.empty()) P.d2_bad.resize(static_cast<size_t>(ndst));
                P.d2_bad[static_cast<size_t>(j)] = std::move(R.bad);
                if (P.d2_tensor_dst.empty()) P.d2_tensor_dst.assign(static_cast<size_t>(ndst) * nt, 0);
                for (int t : R.flagged_tensors) P.d2_tensor_dst[static_cast<size_t>(j) * nt + t] = 1;
                P.d2_runs.insert(P.d2_runs.end(), R.patch.begin(), R.patch.end());
                P.d2_multi.insert(P.d2_multi.end(), R.multi.begin(), R.multi.end());
                d2_regular_runs += R.regular_runs;
                d2_regular_elems += R.regular_elems;
                d2_patch_elems += R.patch_elems;
            }
            std::sort(P.d2_multi.begin(), P.d2_multi.end(), [](const PlanCore::D2Multi& a, const PlanCore::D2Multi& b) {
                return a.dst != b.dst ? a.dst < b.dst : a.lo < b.lo;
            });
            // uniform pieces are separate pendings: D2 runs are kept as produced
            std::stable_sort(P.d2_runs.begin(), P.d2_runs.end(), [](const FlatXfer& a, const FlatXfer& b) {
                if (a.src != b.src) return a.src < b.src;
                if (a.dst != b.dst) return a.dst < b.dst;
                return a.lo < b.lo;
            });
        }
        phase("d2");
        // transfer count + bytes: the triples' runs, minus those inside over-sourced
        // intervals, plus the D2 runs that replace them
        // (src, dst) groups of consecutive triples are independent: count them in parallel
        std::vector<size_t> gstart;
        for (size_t i = 0; i < P.triples.size(); ++i)
            if (i == 0 || P.triples[i].src != P.triples[i - 1].src || P.triples[i].dst != P.triples[i - 1].dst)
                gstart.push_back(i);
        gstart.push_back(P.triples.size());
        std::vector<std::int64_t> g_elems(gstart.size(), 0), g_runs(gstart.size(), 0);
        parallel_for(gstart.size() - 1, [&](size_t g) {
            std::int64_t cnt = 0, el = 0, last_hi = -1;
            for (size_t i = gstart[g]; i < gstart[g + 1]; ++i) {
                const stair::Triple& T = P.triples[i];
                el += triple_count(T);
                // per band in O(1): rows x pieces, minus row-to-row merges when the pattern
                // wraps (first piece at column 0, last at the row end), minus a merge with the
                // previous band / triple of the same (src, dst) when they abut
                for_each_band(T, [&](const std::int64_t* p, std::int64_t u, std::int64_t v, const stair::Iv* cols, int n) {
                    const std::int64_t first_lo = stair::flat_of(T.t, p, u, cols[0].lo);
                    const bool wrap = cols[0].lo == 0 && cols[n - 1].hi == T.t.cols;
                    cnt += (v - u) * n - (wrap ? v - u - 1 : 0) - (first_lo == last_hi ? 1 : 0);
                    last_hi = stair::flat_of(T.t, p, v - 1, cols[n - 1].hi);
                });
            }
            g_runs[g] = cnt;
            g_elems[g] = el;
        });
        for (size_t g = 0; g + 1 < gstart.size(); ++g) flat_elems += g_elems[g];
        flat_elems += d2_patch_elems - d2_regular_elems;
        std::int64_t total_runs = 0;
        for (size_t g = 0; g + 1 < gstart.size(); ++g) total_runs += g_runs[g];
        P.n_flat = total_runs - d2_regular_runs + static_cast<std::int64_t>(P.d2_runs.size());
    }

    phase("count");
    if (timing) std::fprintf(stderr, "[reshard] build_plan (ms):%s\n", phases.c_str());
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

std::vector<FlatXfer> apply_d2(const PlanCore& P, std::vector<FlatXfer> base) {
    if (P.d2_bad.empty()) return base;
    auto less = [](const FlatXfer& a, const FlatXfer& b) {
        if (a.src != b.src) return a.src < b.src;
        if (a.dst != b.dst) return a.dst < b.dst;
        return a.lo < b.lo;
    };
    // a triple run lies inside or outside each recv interval (intervals are maximal under
    // abutting), so testing its start suffices; base is (src, dst, lo)-sorted: one pointer
    // into the destination's sorted bad list per (src, dst) group
    std::vector<FlatXfer> kept;
    kept.reserve(base.size());
    int gs = -1, gd = -1;
    size_t q = 0;
    const std::vector<Interval>* bad = nullptr;
    for (const FlatXfer& f : base) {
        if (f.src != gs || f.dst != gd) {
            gs = f.src, gd = f.dst, q = 0;
            bad = static_cast<size_t>(f.dst) < P.d2_bad.size() ? &P.d2_bad[static_cast<size_t>(f.dst)] : nullptr;
        }
        if (bad && !bad->empty()) {
            while (q < bad->size() && (*bad)[q].hi <= f.lo) ++q;
            if (q < bad->size() && (*bad)[q].lo <= f.lo) continue;
        }
        kept.push_back(f);
    }
    std::vector<FlatXfer> out;
    out.reserve(kept.size() + P.d2_runs.size());
    std::merge(kept.begin(), kept.end(), P.d2_runs.begin(), P.d2_runs.end(), std::back_inserter(out), less);
    return out;
}

std::vector<FlatXfer> expand_flat_host(const PlanCore& P) {
    std::vector<FlatXfer> out;
    for (const stair::Triple& T : P.triples) append_runs(T, out);
    return apply_d2(P, std::move(out));
}

std::vector<FlatXfer> expand_flat_rows_host(const PlanCore& P) {
    std::vector<FlatXfer> out;
    for (const stair::Triple& T : P.triples) {
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
    return apply_d2(P, std::move(out));
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
