// The reference's routing passes by name (reshard/routing.hpp), over the linear-sweep
// region algebra of region.hpp.
#include "reshard/routing.hpp"

#include <algorithm>

namespace reshard {

namespace detail {

CategorySet decompose(const RegionSet& src, const RegionSet& dst) {
    CategorySet c;
    c.src = src;
    c.dst = dst;
    c.send = region_diff(src, dst);
    c.recv = region_diff(dst, src);
    c.retain = region_intersect(src, dst);
    return c;
}

}  // namespace detail

namespace {

RegionSet empty_region(const ModelSpace& space) {
    RegionSet r;
    r.space_fp = space.fingerprint();
    return r;
}

/// Recv cells of one device's box category, cut at the source projection grid so each
/// cell has one candidate set: every source rank whose region contains it
/// (reference routing.hpp:197-222).
void queue_cells(const ModelSpace& space, const ParallelConfig& src_cfg, const std::vector<RegionSet>& src_regions,
                 StateKind kind, const RankRoute& route, const RegionSet& recv, std::vector<detail::PendingRecv>& out) {
    for (const auto& [id, boxes] : recv.boxes)
        for (const Box& b : boxes)
            for (Box& cell : split_by_projection_grid(space, src_cfg, id, b)) {
                detail::PendingRecv p;
                for (int j = 0; j < static_cast<int>(src_regions.size()); ++j)
                    if (region_contains_box(src_regions[static_cast<size_t>(j)], id, cell)) p.candidates.push_back(j);
                if (p.candidates.empty())
                    throw ConfigError(strfmt("unreachable state: no source holds %s %s needed by device %d", id.c_str(),
                                             format_box(cell).c_str(), route.phys));
                p.kind = kind;
                p.tensor_id = id;
                p.box = std::move(cell);
                p.dst_phys = route.phys;
                p.dst_rank = route.dst_rank;
                out.push_back(std::move(p));
            }
}

std::vector<RegionSet> project_all(const ModelSpace& space, const ParallelConfig& cfg, bool optimizer) {
    std::vector<RegionSet> v(static_cast<size_t>(cfg.world_size()));
    for (int i = 0; i < cfg.world_size(); ++i)
        v[static_cast<size_t>(i)] = optimizer ? project_optimizer(space, cfg, i) : project(space, cfg, i);
    return v;
}

/// ZeRO recv intervals of one device cut at source-shard boundaries (reference
/// routing.hpp:317-335): per interval, the pieces of source 0, then source 1, ...; each
/// piece has its owner as sole candidate. Over-covered intervals (D2) throw the
/// reference's ConfigError, or with `allow` become maximal runs with a uniform candidate
/// set (the extension the closed-form planner and oracle.c implement).
void queue_flat(const std::vector<RegionSet>& shards, const RankRoute& route, bool allow,
                std::vector<detail::PendingRecv>& out) {
    const std::vector<Interval>& recv = route.optim.recv.flat;
    if (recv.empty()) return;
    struct Piece {
        std::int64_t lo, hi;
        int src;
    };
    // two-pointer sweep of every source's shard against the recv list: pieces per interval
    std::vector<std::vector<Piece>> per_iv(recv.size());
    for (int j = 0; j < static_cast<int>(shards.size()); ++j) {
        const std::vector<Interval>& s = shards[static_cast<size_t>(j)].flat;
        size_t a = 0, b = 0;
        while (a < recv.size() && b < s.size()) {
            const std::int64_t lo = std::max(recv[a].lo, s[b].lo), hi = std::min(recv[a].hi, s[b].hi);
            if (lo < hi) per_iv[a].push_back({lo, hi, j});
            if (recv[a].hi < s[b].hi) ++a;
            else ++b;
        }
    }
    std::vector<std::int64_t> bounds;
    std::vector<int> cands, run;
    for (size_t i = 0; i < recv.size(); ++i) {
        const Interval& iv = recv[i];
        std::int64_t covered = 0;
        for (const Piece& p : per_iv[i]) covered += p.hi - p.lo;
        auto emit = [&](std::int64_t lo, std::int64_t hi, std::vector<int> c) {
            detail::PendingRecv p;
            p.kind = StateKind::Optim;
            p.flat_payload = true;
            p.flat = {lo, hi};
            p.dst_phys = route.phys;
            p.dst_rank = route.dst_rank;
            p.candidates = std::move(c);
            out.push_back(std::move(p));
        };
        if (covered == iv.length()) {
            for (const Piece& p : per_iv[i]) emit(p.lo, p.hi, {p.src});  // source order, then lo
            continue;
        }
        if (!allow)
            throw ConfigError(strfmt("unreachable state: optimizer interval %s for device %d not fully sourced",
                                     format_interval(iv).c_str(), route.phys));
        // D2 extension: elementary segments between piece ends, merged while the
        // candidate set stays the same
        bounds.assign({iv.lo, iv.hi});
        for (const Piece& p : per_iv[i]) bounds.push_back(p.lo), bounds.push_back(p.hi);
        std::sort(bounds.begin(), bounds.end());
        bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
        std::int64_t run_lo = 0, run_hi = 0;
        run.clear();
        for (size_t k = 0; k + 1 < bounds.size(); ++k) {
            cands.clear();
            for (const Piece& p : per_iv[i])
                if (p.lo <= bounds[k] && bounds[k + 1] <= p.hi) cands.push_back(p.src);
            std::sort(cands.begin(), cands.end());
            cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
            if (!run.empty() && run_hi == bounds[k] && cands == run) {
                run_hi = bounds[k + 1];
                continue;
            }
            if (!run.empty()) emit(run_lo, run_hi, run);
            run_lo = bounds[k];
            run_hi = bounds[k + 1];
            run = cands;
        }
        if (!run.empty()) emit(run_lo, run_hi, run);
    }
}

void plan_optimizer_impl(const ModelSpace& space, RoutingPlan& plan, bool allow) {
    if (space.fingerprint() != plan.space_fp) throw ConfigError("plan_optimizer: model space does not match the plan");
    const ParallelConfig& src = plan.src_cfg;
    const ParallelConfig& dst = plan.dst_cfg;
    if (src.zero_enabled != dst.zero_enabled) throw ConfigError("transitions toggling zero_enabled are unsupported");
    if (!src.zero_enabled) {
        // replicated optimizer: parameter geometry, routed like parameters
        const std::vector<RegionSet> src_regions = project_all(space, src, false);
        for (RankRoute& r : plan.routes) {
            r.optim = r.params;
            if (r.dst_rank >= 0) queue_cells(space, src, src_regions, StateKind::Optim, r, r.optim.recv, plan.pending);
        }
        return;
    }
    const std::vector<RegionSet> src_shards = project_all(space, src, true);
    const std::vector<RegionSet> dst_shards = project_all(space, dst, true);
    const RegionSet none = empty_region(space);
    for (RankRoute& r : plan.routes) {
        r.optim = detail::decompose(r.src_rank >= 0 ? src_shards[static_cast<size_t>(r.src_rank)] : none,
                                    r.dst_rank >= 0 ? dst_shards[static_cast<size_t>(r.dst_rank)] : none);
        queue_flat(src_shards, r, allow, plan.pending);
    }
}

}  // namespace

ByteCount RoutingPlan::bytes_retained(const ModelSpace& space) const {
    ByteCount n = 0;
    for (const RankRoute& r : routes) {
        for (const auto& [id, boxes] : r.params.retain.boxes) {
            const int w = space.entry(id).spec.dtype_bytes;
            for (const Box& b : boxes) n += b.numel() * w;
        }
        n += r.optim.retain.flat_numel() * kOptimStateBytes;
        for (const auto& kv : r.optim.retain.boxes)
            for (const Box& b : kv.second) n += b.numel() * kOptimStateBytes;
    }
    return n;
}

RoutingPlan plan_parameters(const ModelSpace& space, const ParallelConfig& src, const ParallelConfig& dst,
                            const WorldMap& world, const PlanOptions& opts) {
    ModelSpec ms;
    ms.num_layers = space.num_layers();
    ms.num_experts = space.num_experts();
    for (const auto& e : space.entries()) ms.tensors.push_back(e.spec);
    validate_config(src, ms);  // both configs are validated before routing
    validate_config(dst, ms);
    world.validate();
    if (world.src_world_size() != src.world_size()) throw ConfigError("world map src size does not match src config");
    if (world.dst_world_size() != dst.world_size()) throw ConfigError("world map dst size does not match dst config");
    RoutingPlan p;
    p.space_fp = space.fingerprint();
    p.src_cfg = src;
    p.dst_cfg = dst;
    p.world_map = world;
    p.opts = opts;
    p.space_ = &space;
    const std::vector<RegionSet> src_regions = project_all(space, src, false);
    const std::vector<RegionSet> dst_regions = project_all(space, dst, false);
    const RegionSet none = empty_region(space);
    for (int phys : world.participants()) {
        RankRoute r;
        r.phys = phys;
        r.src_rank = world.src_rank_of(phys);
        r.dst_rank = world.dst_rank_of(phys);
        r.params = detail::decompose(r.src_rank >= 0 ? src_regions[static_cast<size_t>(r.src_rank)] : none,
                                     r.dst_rank >= 0 ? dst_regions[static_cast<size_t>(r.dst_rank)] : none);
        if (r.dst_rank >= 0) queue_cells(space, src, src_regions, StateKind::Param, r, r.params.recv, p.pending);
        p.routes.push_back(std::move(r));
    }
    if (opts.gradients == GradientPolicy::Migrate) {
        // gradients share the parameter geometry: the parameter queue again, as Grad
        const size_t n = p.pending.size();
        for (size_t i = 0; i < n; ++i)
            if (p.pending[i].kind == StateKind::Param) {
                detail::PendingRecv g = p.pending[i];
                g.kind = StateKind::Grad;
                p.pending.push_back(std::move(g));
            }
    }
    return p;
}

void plan_optimizer(const ModelSpace& space, RoutingPlan& plan) { plan_optimizer_impl(space, plan, false); }

void plan_optimizer(const ModelSpace& space, RoutingPlan& plan, bool allow_oversourced) {
    plan_optimizer_impl(space, plan, allow_oversourced);
}

void plan_scalars(RoutingPlan& plan) {
    const WorldMap& wm = plan.world_map;
    if (wm.src_world_size() == 0) return;
    ScalarBroadcast b;
    b.root_src_rank = 0;
    b.root_phys = wm.src_phys[0];
    b.words = plan.opts.scalar_words;
    b.bytes_per_rank = b.words * kScalarWordBytes;
    for (int phys : wm.dst_phys)
        if (phys != b.root_phys) b.recv_phys.push_back(phys);
    std::sort(b.recv_phys.begin(), b.recv_phys.end());
    plan.scalars = std::move(b);
}

void resolve_peers(RoutingPlan& plan, const Topology& topo) {
    if (!plan.space_) throw ConfigError("resolve_peers: plan has no model space (call plan_parameters first)");
    const ModelSpace& space = *plan.space_;
    if (space.fingerprint() != plan.space_fp) throw ConfigError("resolve_peers: model space does not match the plan");
    const WorldMap& wm = plan.world_map;
    std::int64_t cursor = 0;
    plan.transfers.reserve(plan.transfers.size() + plan.pending.size());
    for (detail::PendingRecv& p : plan.pending) {
        if (p.candidates.empty()) throw std::logic_error("pending recv without candidates");
        int chosen = -1;
        if (plan.opts.balance_fanout && p.candidates.size() > 1) {
            chosen = p.candidates[static_cast<size_t>(cursor++) % p.candidates.size()];
        } else {
            // candidates ascend: the first one on the destination's node is the lowest id
            for (int c : p.candidates)
                if (topo.same_node(wm.src_phys[static_cast<size_t>(c)], p.dst_phys)) {
                    chosen = c;
                    break;
                }
            if (chosen < 0) chosen = p.candidates.front();
        }
        SliceTransfer t;
        t.kind = p.kind;
        t.tensor_id = std::move(p.tensor_id);
        t.flat_payload = p.flat_payload;
        t.box = std::move(p.box);
        t.flat = p.flat;
        t.src_rank = chosen;
        t.src_phys = wm.src_phys[static_cast<size_t>(chosen)];
        t.dst_rank = p.dst_rank;
        t.dst_phys = p.dst_phys;
        t.count = t.flat_payload ? t.flat.length() : t.box.numel();
        const int w = t.kind == StateKind::Param ? space.entry(t.tensor_id).spec.dtype_bytes
                      : t.kind == StateKind::Optim ? kOptimStateBytes
                      : t.kind == StateKind::Grad  ? kGradBytes
                                                   : kScalarWordBytes;
        t.bytes = t.count * w;
        plan.transfers.push_back(std::move(t));
    }
    plan.pending.clear();
    // sort by a precomputed key: (src, dst, kind, tensor id rank, region) without string
    // compares in the comparator
    std::vector<std::string> ids;
    for (const auto& e : space.entries()) ids.push_back(e.spec.tensor_id);
    std::sort(ids.begin(), ids.end());
    std::vector<std::uint32_t> idr(plan.transfers.size());
    for (size_t i = 0; i < plan.transfers.size(); ++i) {
        const std::string& id = plan.transfers[i].tensor_id;
        idr[i] = id.empty() ? 0u : static_cast<std::uint32_t>(std::lower_bound(ids.begin(), ids.end(), id) - ids.begin()) + 1u;
    }
    std::vector<std::uint32_t> ord(plan.transfers.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = static_cast<std::uint32_t>(i);
    const auto& T = plan.transfers;
    std::sort(ord.begin(), ord.end(), [&](std::uint32_t a, std::uint32_t b) {
        const SliceTransfer &x = T[a], &y = T[b];
        if (x.src_rank != y.src_rank) return x.src_rank < y.src_rank;
        if (x.dst_rank != y.dst_rank) return x.dst_rank < y.dst_rank;
        if (x.kind != y.kind) return static_cast<int>(x.kind) < static_cast<int>(y.kind);
        if (idr[a] != idr[b]) return idr[a] < idr[b];
        if (x.flat_payload && y.flat_payload)
            return std::make_pair(x.flat.lo, x.flat.hi) < std::make_pair(y.flat.lo, y.flat.hi);
        return x.region_key() < y.region_key();
    });
    std::vector<SliceTransfer> sorted;
    sorted.reserve(T.size());
    for (std::uint32_t i : ord) sorted.push_back(std::move(plan.transfers[i]));
    plan.transfers = std::move(sorted);
    plan.resolved = true;
}

}  // namespace reshard
