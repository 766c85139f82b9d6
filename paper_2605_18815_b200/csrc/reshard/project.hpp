// Projection F_P(VPS, rank) and the physical local layout. API mirrors the
// reference project.hpp (full_region :27-38, project :44-74, LocalSegment/
// LocalLayout/local_layout :77-112, shard_range :118-124, project_optimizer
// :146-159, state_region :164-168, split_by_projection_grid :174-196).
#pragma once

#include <string>
#include <vector>

#include "reshard/model.hpp"
#include "reshard/parallel.hpp"
#include "reshard/region.hpp"

namespace reshard {

inline RegionSet full_region(const ModelSpace& space) {
    RegionSet r;
    r.space_fp = space.fingerprint();
    for (const auto& e : space.entries()) {
        Box b;
        for (std::int64_t ext : e.spec.shape) b.dims.push_back({0, ext});
        r.add_box(e.spec.tensor_id, std::move(b));
    }
    r.add_flat({0, space.total_numel()});
    r.normalize();
    return r;
}

/// The box a rank holds of one tensor, or an empty box when the tensor's layer is
/// outside the rank's pipeline stage. (One box per tensor: the closed form the
/// planner and the executor both build on.)
inline Box rank_box(const ModelSpace& space, const ParallelConfig& cfg, const RankCoord& c, const TensorSpec& t) {
    const auto [lo, hi] = stage_layer_range(space.num_layers(), cfg.pp, c.pp_rank);
    Box b;
    if (t.layer < lo || t.layer >= hi) return b;
    b.dims.reserve(t.shape.size());
    for (std::int64_t ext : t.shape) b.dims.push_back({0, ext});
    if (t.tp_shard_axis) {
        const std::int64_t ext = t.shape[*t.tp_shard_axis];
        if (ext % cfg.tp)
            throw ConfigError(strfmt("tp=%d does not divide extent %lld of tensor '%s'", cfg.tp,
                                     static_cast<long long>(ext), t.tensor_id.c_str()));
        const std::int64_t w = ext / cfg.tp;
        b.dims[*t.tp_shard_axis] = {c.tp_rank * w, (c.tp_rank + 1) * w};
    }
    if (t.expert_axis) {
        if (space.num_experts() % cfg.ep)
            throw ConfigError(strfmt("ep=%d does not divide num_experts=%d", cfg.ep, space.num_experts()));
        const std::int64_t w = space.num_experts() / cfg.ep;
        b.dims[*t.expert_axis] = {c.ep_rank * w, (c.ep_rank + 1) * w};
    }
    return b;
}

inline RegionSet project(const ModelSpace& space, const ParallelConfig& cfg, int rank) {
    const RankCoord c = rank_coord(cfg, rank);
    RegionSet r;
    r.space_fp = space.fingerprint();
    for (const auto& e : space.entries()) {
        Box b = rank_box(space, cfg, c, e.spec);
        if (!b.dims.empty()) r.add_box(e.spec.tensor_id, std::move(b));
    }
    return r;  // one non-empty box per visible tensor is already normalized
}

struct LocalSegment {
    std::string tensor_id;
    Box box;
    std::int64_t local_lo;
    std::int64_t local_hi;
};

struct LocalLayout {
    std::vector<LocalSegment> dense;
    std::vector<LocalSegment> expert;
    std::int64_t dense_len = 0;
    std::int64_t expert_len = 0;
};

/// Visible boxes flattened row-major in declaration order; dense and expert spans
/// are indexed separately (they shard over different replica groups).
inline LocalLayout local_layout(const ModelSpace& space, const ParallelConfig& cfg, int rank) {
    const RankCoord c = rank_coord(cfg, rank);
    LocalLayout L;
    for (const auto& e : space.entries()) {
        Box b = rank_box(space, cfg, c, e.spec);
        if (b.dims.empty()) continue;
        const std::int64_t n = b.numel();
        auto& list = e.spec.is_expert ? L.expert : L.dense;
        auto& len = e.spec.is_expert ? L.expert_len : L.dense_len;
        list.push_back(LocalSegment{e.spec.tensor_id, std::move(b), len, len + n});
        len += n;
    }
    return L;
}

namespace detail {

/// ceil-rule contiguous shard of [0,len) over `parts` owners (last one truncated).
inline Interval shard_range(std::int64_t len, int parts, int index) {
    if (len == 0) return {0, 0};
    const std::int64_t chunk = (len + parts - 1) / parts;
    const std::int64_t lo = std::min<std::int64_t>(static_cast<std::int64_t>(index) * chunk, len);
    return {lo, std::min<std::int64_t>(lo + chunk, len)};
}

inline void invert_segments(const ModelSpace& space, const std::vector<LocalSegment>& segs, const Interval& shard,
                            RegionSet& out) {
    for (const LocalSegment& s : segs) {
        const Interval ov = intersect({s.local_lo, s.local_hi}, shard);
        if (ov.empty()) continue;
        for (const Interval& run :
             box_subrange_flat_runs(space, s.tensor_id, s.box, ov.lo - s.local_lo, ov.hi - s.local_lo))
            out.add_flat(run);
    }
}

}  // namespace detail

/// The rank's ZeRO-1 shard (dense over dp, expert over dp/ep) as global flat runs.
inline RegionSet project_optimizer(const ModelSpace& space, const ParallelConfig& cfg, int rank) {
    if (!cfg.zero_enabled) throw ConfigError("no sharded optimizer: zero_enabled is false");
    const RankCoord c = rank_coord(cfg, rank);
    const LocalLayout L = local_layout(space, cfg, rank);
    RegionSet out;
    out.space_fp = space.fingerprint();
    detail::invert_segments(space, L.dense, detail::shard_range(L.dense_len, cfg.dp, c.dp_rank), out);
    detail::invert_segments(space, L.expert, detail::shard_range(L.expert_len, cfg.dp / cfg.ep, c.edp_rank), out);
    out.flat = normalize_intervals(std::move(out.flat));
    return out;
}

inline RegionSet state_region(const ModelSpace& space, const ParallelConfig& cfg, int rank, StateKind kind) {
    return (kind == StateKind::Optim && cfg.zero_enabled) ? project_optimizer(space, cfg, rank)
                                                          : project(space, cfg, rank);
}

/// Cut `box` at the TP-slice and expert-block boundaries of `cfg` (TP axis first),
/// so each cell has a uniform set of candidate source ranks.
inline std::vector<Box> split_by_projection_grid(const ModelSpace& space, const ParallelConfig& cfg,
                                                 const std::string& tensor_id, const Box& box) {
    const TensorSpec& t = space.entry(tensor_id).spec;
    std::vector<Box> cells{box};
    auto cut_axis = [&cells](int axis, std::int64_t width) {
        std::vector<Box> next;
        for (const Box& c : cells) {
            const Interval span = c.dims[axis];
            for (std::int64_t lo = span.lo - span.lo % width; lo < span.hi; lo += width) {
                const Interval piece = intersect(span, {lo, lo + width});
                if (piece.empty()) continue;
                next.push_back(c);
                next.back().dims[axis] = piece;
            }
        }
        cells.swap(next);
    };
    if (t.tp_shard_axis) cut_axis(*t.tp_shard_axis, t.shape[*t.tp_shard_axis] / cfg.tp);
    if (t.expert_axis) cut_axis(*t.expert_axis, space.num_experts() / cfg.ep);
    return cells;
}

}  // namespace reshard
