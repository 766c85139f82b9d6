// The reference's routing passes by name (routing.hpp) over the closed-form planner.
#include "reshard/routing.hpp"

#include <algorithm>

namespace reshard {

RoutingPlan plan_parameters(const ModelSpace& space, const ParallelConfig& src, const ParallelConfig& dst,
                            const WorldMap& world, const PlanOptions& opts) {
    ModelSpec ms;
    ms.num_layers = space.num_layers();
    ms.num_experts = space.num_experts();
    for (const auto& e : space.entries()) ms.tensors.push_back(e.spec);
    validate_config(src, ms);
    validate_config(dst, ms);
    RoutingPlan p;
    p.space_fp = space.fingerprint();
    p.src_cfg = src;
    p.dst_cfg = dst;
    p.world_map = world;
    p.opts = opts;
    p.space_ = &space;
    return p;
}

void plan_optimizer(const ModelSpace& space, RoutingPlan& plan) {
    if (space.fingerprint() != plan.space_fp) throw ConfigError("plan_optimizer: model space does not match the plan");
    if (plan.src_cfg.zero_enabled != plan.dst_cfg.zero_enabled)
        throw ConfigError("transitions toggling zero_enabled are unsupported");
    plan.optimizer_ = true;
}

void plan_scalars(RoutingPlan& plan) { plan.scalars_ = true; }

void resolve_peers(RoutingPlan& plan, const Topology& topo) {
    if (!plan.space_) throw ConfigError("resolve_peers: plan has no model space (call plan_parameters first)");
    const core::PlanCore P =
        core::build_plan(*plan.space_, plan.src_cfg, plan.dst_cfg, &plan.world_map, topo, plan.opts, plan.allow_oversourced_);
    const auto& ents = plan.space_->entries();
    std::vector<SliceTransfer> out;
    ByteCount moved = 0;
    auto keep_kind = [&](int kind) { return kind != static_cast<int>(StateKind::Optim) || plan.optimizer_; };
    for (const core::BoxXfer& b : P.box) {
        if (!keep_kind(b.kind)) continue;
        SliceTransfer t;
        t.kind = static_cast<StateKind>(b.kind);
        t.tensor_id = ents[static_cast<size_t>(b.tensor)].spec.tensor_id;
        const size_t nd = ents[static_cast<size_t>(b.tensor)].spec.shape.size();
        t.box.dims.resize(nd);
        for (size_t d = 0; d < nd; ++d) t.box.dims[d] = {b.lo[d], b.hi[d]};
        t.src_rank = b.src;
        t.dst_rank = b.dst;
        t.count = b.count;
        t.bytes = b.bytes;
        out.push_back(std::move(t));
    }
    if (plan.optimizer_)
        for (const core::FlatXfer& f : core::expand_flat_host(P)) {
            SliceTransfer t;
            t.kind = StateKind::Optim;
            t.flat_payload = true;
            t.flat = {f.lo, f.hi};
            t.src_rank = f.src;
            t.dst_rank = f.dst;
            t.count = f.hi - f.lo;
            t.bytes = t.count * kOptimStateBytes;
            out.push_back(std::move(t));
        }
    for (SliceTransfer& t : out) {
        t.src_phys = P.wm.src_phys[static_cast<size_t>(t.src_rank)];
        t.dst_phys = P.wm.dst_phys[static_cast<size_t>(t.dst_rank)];
        moved += t.bytes;
    }
    std::sort(out.begin(), out.end(), transfer_order_less);
    if (plan.scalars_ && P.has_scalars)
        moved += P.scalar_bytes_per_rank * static_cast<ByteCount>(P.scalar_recv_phys.size());
    plan.transfers = std::move(out);
    plan.moved_ = moved;
    plan.retained_ = P.bytes_retained;
    plan.resolved = true;
}

}  // namespace reshard
