// The reference's routing API by name (reference routing.hpp:34-396: SliceTransfer,
// transfer_order_less, format_transfer, RoutingPlan, plan_parameters, plan_optimizer,
// plan_scalars, resolve_peers) over PlanCore, so a C++ caller switches only its include
// path. The passes record what the caller asked for; resolve_peers builds the plan in
// closed form (core::build_plan, bit-exact with the reference's) and materializes the
// canonical transfer list. resolve_peers takes the ModelSpace from its plan: the shipped
// reference passes nullptr there and does not compile (D1, routing.hpp:389).
//
// Not mirrored: RoutingPlan::routes (per-device RegionSet categories) and ::pending
// (unresolved candidates) — use project()/local_layout() for geometry.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <tuple>
#include <vector>

#include "reshard/plan_core.hpp"

namespace reshard {

struct SliceTransfer {
    StateKind kind = StateKind::Param;
    std::string tensor_id;  // empty for flat payloads
    bool flat_payload = false;
    Box box;
    Interval flat;
    int src_rank = -1;
    int dst_rank = -1;
    int src_phys = -1;
    int dst_phys = -1;
    std::int64_t count = 0;
    ByteCount bytes = 0;

    std::vector<std::int64_t> region_key() const {
        std::vector<std::int64_t> k;
        if (flat_payload) {
            k = {flat.lo, flat.hi};
        } else {
            for (const auto& d : box.dims) k.insert(k.end(), {d.lo, d.hi});
        }
        return k;
    }
    std::string region_text() const { return flat_payload ? format_interval(flat) : format_box(box); }
};

/// canonical order: (src rank, dst rank, kind, tensor id, region)
inline bool transfer_order_less(const SliceTransfer& a, const SliceTransfer& b) {
    return std::make_tuple(a.src_rank, a.dst_rank, static_cast<int>(a.kind), a.tensor_id, a.region_key()) <
           std::make_tuple(b.src_rank, b.dst_rank, static_cast<int>(b.kind), b.tensor_id, b.region_key());
}

/// "kind id region src=S dst=D bytes=B", the reference's dump line
inline std::string format_transfer(const SliceTransfer& t) {
    return strfmt("%s %s %s src=%d dst=%d bytes=%lld", to_string(t.kind), t.tensor_id.empty() ? "-" : t.tensor_id.c_str(),
                  t.region_text().c_str(), t.src_rank, t.dst_rank, static_cast<long long>(t.bytes));
}

struct RoutingPlan {
    std::uint64_t space_fp = 0;
    ParallelConfig src_cfg, dst_cfg;
    WorldMap world_map;
    PlanOptions opts;
    std::vector<SliceTransfer> transfers;  // filled by resolve_peers, canonical order
    bool resolved = false;

    /// payload bytes of every transfer (and the scalar broadcast once planned)
    ByteCount bytes_moved() const { return moved_; }
    /// bytes that stay on their device (params + optimizer state kept in place)
    ByteCount bytes_retained(const ModelSpace&) const { return retained_; }

    // set by the passes (not part of the reference's public fields)
    const ModelSpace* space_ = nullptr;
    bool optimizer_ = false, scalars_ = false, allow_oversourced_ = false;
    ByteCount moved_ = 0, retained_ = 0;
};

/// Parameter (and, with GradientPolicy::Migrate, gradient) routing; validates both configs.
RoutingPlan plan_parameters(const ModelSpace& space, const ParallelConfig& src, const ParallelConfig& dst,
                            const WorldMap& world, const PlanOptions& opts = {});
/// ZeRO / replicated optimizer routing (throws the reference's ConfigError on toggling
/// zero_enabled and, at resolve time, on over-sourced intervals — D2)
void plan_optimizer(const ModelSpace& space, RoutingPlan& plan);
/// the scalar broadcast from source rank 0
void plan_scalars(RoutingPlan& plan);
/// pick every transfer's source (proximity rule or balance_fanout), byte counts, order
void resolve_peers(RoutingPlan& plan, const Topology& topo);

}  // namespace reshard
