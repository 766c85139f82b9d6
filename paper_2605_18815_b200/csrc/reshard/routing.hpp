// The reference's routing API (reference routing.hpp:34-396) for C++ callers: the same
// value types and public fields — SliceTransfer, CategorySet, RankRoute, ScalarBroadcast,
// detail::PendingRecv, RoutingPlan{routes, pending, transfers, scalars} — and the same
// passes, so a caller switches only its include path and library.
//
//   plan_parameters   routes[*].params (R_src / R_dst / send / recv / retain per device)
//                     and the parameter (and gradient) recv cells with their candidates
//   plan_optimizer    routes[*].optim and the optimizer recv pieces (ZeRO: flat runs cut at
//                     source-shard boundaries, one candidate each)
//   plan_scalars      the scalar broadcast
//   resolve_peers     one source per pending fragment (proximity rule or balance_fanout),
//                     canonical order; consumes `pending`
//
// Region algebra is the linear-sweep one of region.hpp, so these passes are fast at full
// model size (the reference's O(n*m) interval loops need hours at Llama-3-8B L=32, D3).
// The executor and the C ABI do not go through this API: they use the closed-form
// PlanCore (plan_core.hpp), which the golden tests prove transfer-for-transfer equal.
//
// Deviations, all documented: resolve_peers reads payload widths from the ModelSpace
// passed to plan_parameters (the reference passes a null reference and does not compile,
// D1, routing.hpp:389), so that space must outlive the plan's passes; plan_optimizer has an
// overload that resolves over-sourced ZeRO intervals instead of throwing (D2 extension,
// parity unpinned).
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

/// One device's state split into the mutually exclusive categories.
struct CategorySet {
    RegionSet src;     // R_src of the device
    RegionSet dst;     // R_dst of the device
    RegionSet send;    // R_src \ R_dst
    RegionSet recv;    // R_dst \ R_src
    RegionSet retain;  // R_src ∩ R_dst
};

struct RankRoute {
    int phys = -1;
    int src_rank = -1;  // -1: the device joins (empty R_src)
    int dst_rank = -1;  // -1: the device leaves (empty R_dst)
    CategorySet params;
    CategorySet optim;
};

struct ScalarBroadcast {
    int root_phys = -1;
    int root_src_rank = 0;
    std::vector<int> recv_phys;  // ascending, root excluded; empty = nothing to send
    std::int64_t words = 0;
    ByteCount bytes_per_rank = 0;
};

namespace detail {

/// A recv fragment waiting for resolve_peers to pick its source.
struct PendingRecv {
    StateKind kind = StateKind::Param;
    std::string tensor_id;
    bool flat_payload = false;
    Box box;
    Interval flat;
    int dst_phys = -1;
    int dst_rank = -1;
    std::vector<int> candidates;  // src world ranks, ascending
};

/// send = src \ dst, recv = dst \ src, retain = src ∩ dst
CategorySet decompose(const RegionSet& src, const RegionSet& dst);

}  // namespace detail

struct RoutingPlan;
RoutingPlan plan_parameters(const ModelSpace& space, const ParallelConfig& src, const ParallelConfig& dst,
                            const WorldMap& world, const PlanOptions& opts = {});
void plan_optimizer(const ModelSpace& space, RoutingPlan& plan);
void plan_optimizer(const ModelSpace& space, RoutingPlan& plan, bool allow_oversourced);
void plan_scalars(RoutingPlan& plan);
void resolve_peers(RoutingPlan& plan, const Topology& topo);

/// The decomposition of a transition per device and, once resolved, its exact
/// point-to-point transfer list.
struct RoutingPlan {
    std::uint64_t space_fp = 0;
    ParallelConfig src_cfg, dst_cfg;
    WorldMap world_map;
    PlanOptions opts;
    std::vector<RankRoute> routes;  // one per participating device, ascending phys
    std::vector<detail::PendingRecv> pending;
    std::vector<SliceTransfer> transfers;  // canonical order once resolved
    std::optional<ScalarBroadcast> scalars;
    bool resolved = false;

    const RankRoute& route_of(int phys) const {
        for (const auto& r : routes)
            if (r.phys == phys) return r;
        throw std::logic_error("no route for device");
    }

    /// payload bytes of every transfer plus the scalar broadcast
    ByteCount bytes_moved() const {
        ByteCount n = 0;
        for (const auto& t : transfers) n += t.bytes;
        if (scalars) n += scalars->bytes_per_rank * static_cast<ByteCount>(scalars->recv_phys.size());
        return n;
    }
    /// bytes that stay on their device: retained params at their width, retained
    /// optimizer state at 12 B per element
    ByteCount bytes_retained(const ModelSpace& space) const;

private:
    const ModelSpace* space_ = nullptr;  // payload widths for resolve_peers (D1)
    friend RoutingPlan plan_parameters(const ModelSpace&, const ParallelConfig&, const ParallelConfig&,
                                       const WorldMap&, const PlanOptions&);
    friend void resolve_peers(RoutingPlan&, const Topology&);
};

}  // namespace reshard
