// validate_plan: the RoutingPlan invariants plus destination
// coverage, returned (not thrown) as violation lines.
//   * every destination element is retained or received exactly once
//     (retain ∪ recv == R_dst, pairwise disjoint: the single-source property);
//   * every transfer lies inside the sender's region and the receiver's region;
//   * sender and receiver are different devices.
#include <algorithm>
#include <map>

#include "reshard/plan_core.hpp"
#include "reshard/validate.hpp"

namespace reshard {
namespace core {

namespace {

Box box_from(const std::int64_t* lo, const std::int64_t* hi, int nd) {
    Box b;
    b.dims.resize(static_cast<size_t>(nd));
    for (int d = 0; d < nd; ++d) b.dims[static_cast<size_t>(d)] = {lo[d], hi[d]};
    return b;
}

Box seg_box(const Seg& s, int nd) { return box_from(s.blo, s.bhi, nd); }

/// optimizer element set of a rank as global flat runs (ZeRO) — project_optimizer
std::vector<Interval> zero_runs(const PlanCore& P, const ParallelConfig& cfg, int rank) {
    return project_optimizer(*P.space, cfg, rank).flat;
}

}  // namespace

std::vector<std::string> validate_plan(const PlanCore& P, const std::vector<FlatXfer>& flat, std::int64_t drop) {
    const ModelSpace& space = *P.space;
    std::vector<std::string> out;
    const int nt = P.ntensors();
    // transfer list (box + flat), optionally with one fragment removed (fault injection)
    std::vector<BoxXfer> box = P.box;
    std::vector<FlatXfer> fl = flat;
    if (drop >= 0) {
        if (drop < static_cast<std::int64_t>(box.size())) box.erase(box.begin() + drop);
        else if (drop - static_cast<std::int64_t>(box.size()) < static_cast<std::int64_t>(fl.size()))
            fl.erase(fl.begin() + (drop - static_cast<std::int64_t>(box.size())));
    }
    // ---- box kinds (params, grads, replicated optimizer): per (dst rank, kind, tensor)
    std::map<std::tuple<int, int, int>, std::vector<Box>> recv;
    for (const BoxXfer& b : box) {
        const int nd = static_cast<int>(space.entries()[static_cast<size_t>(b.tensor)].spec.shape.size());
        const Box x = box_from(b.lo, b.hi, nd);
        const RankGeom& S = P.src.ranks[static_cast<size_t>(b.src)];
        const RankGeom& D = P.dst.ranks[static_cast<size_t>(b.dst)];
        const int ss = S.seg_of[static_cast<size_t>(b.tensor)], sd = D.seg_of[static_cast<size_t>(b.tensor)];
        const std::string id = space.entries()[static_cast<size_t>(b.tensor)].spec.tensor_id;
        if (ss < 0 || !seg_box(S.segs[static_cast<size_t>(ss)], nd).contains(x))
            out.push_back(strfmt("transfer outside source region: %s %s %s src=%d", to_string(static_cast<StateKind>(b.kind)),
                                 id.c_str(), format_box(x).c_str(), b.src));
        if (sd < 0 || !seg_box(D.segs[static_cast<size_t>(sd)], nd).contains(x))
            out.push_back(strfmt("transfer outside destination region: %s %s %s dst=%d", to_string(static_cast<StateKind>(b.kind)),
                                 id.c_str(), format_box(x).c_str(), b.dst));
        if (P.wm.src_phys[static_cast<size_t>(b.src)] == P.wm.dst_phys[static_cast<size_t>(b.dst)])
            out.push_back(strfmt("transfer to the same device: %s %s src=%d dst=%d", id.c_str(), format_box(x).c_str(), b.src, b.dst));
        recv[{b.dst, b.kind, b.tensor}].push_back(x);
    }
    std::vector<int> kinds = {0};
    if (P.opts.gradients == GradientPolicy::Migrate) kinds.push_back(2);
    if (!P.src_cfg.zero_enabled) kinds.push_back(1);
    for (int j = 0; j < P.dst_cfg.world_size(); ++j) {
        const RankGeom& D = P.dst.ranks[static_cast<size_t>(j)];
        const int own = P.wm.src_rank_of(D.phys);
        for (int t = 0; t < nt; ++t) {
            const int sd = D.seg_of[static_cast<size_t>(t)];
            if (sd < 0) continue;
            const TensorSpec& ts = space.entries()[static_cast<size_t>(t)].spec;
            const int nd = static_cast<int>(ts.shape.size());
            const Box need = seg_box(D.segs[static_cast<size_t>(sd)], nd);
            std::vector<Box> have;
            if (own >= 0) {
                const RankGeom& O = P.src.ranks[static_cast<size_t>(own)];
                const int so = O.seg_of[static_cast<size_t>(t)];
                if (so >= 0) {
                    const Box r = intersect(need, seg_box(O.segs[static_cast<size_t>(so)], nd));
                    if (!r.empty()) have.push_back(r);
                }
            }
            for (int kind : kinds) {
                std::vector<Box> pieces = have;
                auto it = recv.find({j, kind, t});
                if (it != recv.end()) pieces.insert(pieces.end(), it->second.begin(), it->second.end());
                std::int64_t total = 0;
                for (const Box& b : pieces) total += b.numel();
                const std::vector<Box> missing = detail::boxes_diff({need}, pieces);
                for (const Box& m : missing)
                    out.push_back(strfmt("uncovered destination region: rank %d %s %s %s", j,
                                         to_string(static_cast<StateKind>(kind)), ts.tensor_id.c_str(), format_box(m).c_str()));
                if (missing.empty() && total != need.numel())
                    out.push_back(strfmt("doubly sourced destination region: rank %d %s %s", j,
                                         to_string(static_cast<StateKind>(kind)), ts.tensor_id.c_str()));
            }
        }
    }
    // ---- ZeRO optimizer (flat runs)
    if (P.src_cfg.zero_enabled) {
        std::vector<std::vector<Interval>> recv_runs(static_cast<size_t>(P.dst_cfg.world_size()));
        std::vector<std::vector<Interval>> src_runs(static_cast<size_t>(P.src_cfg.world_size()));
        for (int i = 0; i < P.src_cfg.world_size(); ++i) src_runs[static_cast<size_t>(i)] = zero_runs(P, P.src_cfg, i);
        for (const FlatXfer& f : fl) {
            recv_runs[static_cast<size_t>(f.dst)].push_back({f.lo, f.hi});
            // source runs are normalized (maximal, disjoint): the run must sit inside one
            const auto& sr = src_runs[static_cast<size_t>(f.src)];
            auto it = std::upper_bound(sr.begin(), sr.end(), f.lo, [](std::int64_t v, const Interval& r) { return v < r.hi; });
            if (it == sr.end() || it->lo > f.lo || it->hi < f.hi)
                out.push_back(strfmt("transfer outside source region: optim - [%lld:%lld] src=%d",
                                     static_cast<long long>(f.lo), static_cast<long long>(f.hi), f.src));
        }
        for (int j = 0; j < P.dst_cfg.world_size(); ++j) {
            const std::vector<Interval> need = zero_runs(P, P.dst_cfg, j);
            const int own = P.wm.src_rank_of(P.dst.ranks[static_cast<size_t>(j)].phys);
            std::vector<Interval> pieces = recv_runs[static_cast<size_t>(j)];
            if (own >= 0) {
                const std::vector<Interval> keep = intervals_intersect(need, src_runs[static_cast<size_t>(own)]);
                pieces.insert(pieces.end(), keep.begin(), keep.end());
            }
            std::sort(pieces.begin(), pieces.end());
            for (size_t k = 1; k < pieces.size(); ++k)
                if (pieces[k].lo < pieces[k - 1].hi) {
                    out.push_back(strfmt("doubly sourced destination region: rank %d optim [%lld:%lld]", j,
                                         static_cast<long long>(pieces[k].lo),
                                         static_cast<long long>(std::min(pieces[k].hi, pieces[k - 1].hi))));
                    break;
                }
            const std::vector<Interval> got = normalize_intervals(pieces);
            for (const Interval& m : intervals_diff(need, got))
                out.push_back(strfmt("uncovered destination region: rank %d optim [%lld:%lld]", j,
                                     static_cast<long long>(m.lo), static_cast<long long>(m.hi)));
            for (const Interval& m : intervals_diff(got, need))
                out.push_back(strfmt("transfer outside destination region: rank %d optim [%lld:%lld]", j,
                                     static_cast<long long>(m.lo), static_cast<long long>(m.hi)));
        }
    }
    return out;
}

}  // namespace core
}  // namespace reshard
