// PlanCore: the compact, closed-form transition plan the C ABI, the GPU planner
// and the executor work from.
//
// It carries exactly the information of the reference RoutingPlan after
// plan_parameters + plan_optimizer + plan_scalars + resolve_peers
// (routing.hpp:231-396), but never materializes per-row optimizer intervals unless
// asked: ZeRO optimizer routing is kept as stair::Triple records
// ((dst shard ∩ src shard) \ own shard per tensor), which expand to the
// reference's SliceTransfer list on demand (host: band sweep; GPU: one thread per
// tensor row, gpu_planner.cu). Box transfers (params, grads, non-ZeRO optimizer)
// follow the reference's candidate/proximity rules exactly, including the order
// of pending fragments that the balance_fanout cursor depends on.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "reshard/model.hpp"
#include "reshard/parallel.hpp"
#include "reshard/project.hpp"
#include "reshard/region.hpp"
#include "reshard/stair.hpp"
#include "reshard/topology.hpp"
#include "reshard/worldmap.hpp"

namespace reshard {

enum class GradientPolicy { Drop, Migrate };

struct PlanOptions {
    GradientPolicy gradients = GradientPolicy::Drop;
    bool balance_fanout = false;
    std::int64_t scalar_words = 8;
};

constexpr int kOptimStateBytes = 12;  // fp32 master + Adam m + v
constexpr int kGradBytes = 4;
constexpr int kScalarWordBytes = 8;

namespace core {

/// One segment of a rank's local layout (project.hpp:77-112), lifted box.
struct Seg {
    int tensor = -1;
    bool expert = false;
    std::int64_t blo[4] = {0, 0, 0, 0}, bhi[4] = {0, 0, 0, 0};  // box in tensor coordinates (original nd)
    std::int64_t local_lo = 0, local_hi = 0;                      // element index in its span (dense / expert)
    std::int64_t param_byte_off = 0;                             // byte offset in the param buffer
    std::int64_t elem_off = 0;                                   // element offset in the param-geometry buffers
};

/// A virtual rank under one configuration: its segments and buffer sizes.
/// Buffer contract: param = segments (dense then expert) at
/// dtype_bytes; grad = same at 4 B; optim = [dense shard | expert shard] (ZeRO) or
/// the whole param geometry (no ZeRO), SoA fp32 master/m/v; scalars = words x 8 B.
struct RankGeom {
    int rank = 0, phys = -1;
    RankCoord coord;
    std::vector<int> seg_of;  // tensor -> index in segs or -1
    std::vector<Seg> segs;    // dense segments then expert segments
    std::int64_t dense_len = 0, expert_len = 0;
    Interval dshard{0, 0}, eshard{0, 0};
    std::int64_t param_bytes = 0, nelem = 0, optim_len = 0;

    /// optimizer-buffer index of element `li` of a segment's span, or -1
    std::int64_t optim_index(bool expert, std::int64_t li) const {
        if (!expert) return (li >= dshard.lo && li < dshard.hi) ? li - dshard.lo : -1;
        if (li >= eshard.lo && li < eshard.hi) return (dshard.hi - dshard.lo) + li - eshard.lo;
        return -1;
    }
};

struct Side {
    ParallelConfig cfg;
    std::vector<RankGeom> ranks;
};

/// A resolved box transfer (param, grad or replicated optimizer).
struct BoxXfer {
    int kind = 0;  // StateKind
    int tensor = -1;
    std::int64_t lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    int src = -1, dst = -1;  // world ranks
    std::int64_t count = 0, bytes = 0;
};

/// A resolved ZeRO optimizer flat run.
struct FlatXfer {
    std::int64_t lo = 0, hi = 0;
    int src = -1, dst = -1;
};

struct RouteInfo {
    int phys = -1, src_rank = -1, dst_rank = -1;
};

struct PlanCore {
    const ModelSpace* space = nullptr;
    ParallelConfig src_cfg, dst_cfg;
    WorldMap wm;
    Topology topo;
    PlanOptions opts;
    bool allow_oversourced = false;

    std::vector<int> id_rank;     // tensor -> rank of its id in string order
    std::vector<int> by_id;       // string order -> tensor
    Side src, dst;
    std::vector<RouteInfo> routes;  // participants, ascending phys

    std::vector<BoxXfer> box;         // canonical order
    std::vector<BoxXfer> box_retain;  // same-device copies (executor only)
    std::vector<stair::Triple> triples;         // ZeRO moves, (src, dst, tensor) order
    std::vector<stair::Triple> retain_triples;  // ZeRO same-device copies
    // D2 extension (allow_oversourced, parity unpinned). Over-sourced
    // recv intervals (`d2_bad`, per destination rank, ascending) replace the triples' runs
    // inside them by `d2_runs`: maximal runs with a uniform candidate set, one source
    // chosen per run. Outside them the triples' runs are the plan's runs unchanged. The
    // executor re-derives only tensors holding multi-candidate elements (`d2_tensor_dst`)
    // from their triples minus the segments another source was chosen for (`d2_multi`).
    struct D2Multi {
        std::int64_t lo = 0, hi = 0;
        int dst = -1, chosen = -1;
    };
    std::vector<FlatXfer> d2_runs;                  // canonical (src, dst, lo) order
    std::vector<std::vector<Interval>> d2_bad;      // [dst rank] over-sourced recv ivs
    std::vector<D2Multi> d2_multi;                  // (dst, lo) order
    std::vector<std::uint8_t> d2_tensor_dst;        // [dst_rank * ntensors + t] -> 1 if overridden

    bool has_scalars = false;
    int scalar_root_phys = -1;
    std::vector<int> scalar_recv_phys;
    std::int64_t scalar_bytes_per_rank = 0;

    std::int64_t bytes_moved = 0, bytes_retained = 0;
    std::int64_t n_flat = 0;  // number of ZeRO optimizer transfers (reference SliceTransfers)

    int ntensors() const { return static_cast<int>(space->entries().size()); }
    std::int64_t num_transfers() const { return static_cast<std::int64_t>(box.size()) + n_flat; }
};

/// Build the plan. Throws ConfigError exactly where the reference throws
/// (validate_config, unreachable state, D2 "not fully sourced"), unless
/// allow_oversourced, which enables the D2 extension.
PlanCore build_plan(const ModelSpace& space, const ParallelConfig& src, const ParallelConfig& dst,
                    const WorldMap* wm, const Topology& topo, const PlanOptions& opts, bool allow_oversourced);

/// Geometry of one side (also used by the executor for buffer sizes).
Side build_side(const ModelSpace& space, const ParallelConfig& cfg);

/// Expand every ZeRO triple to reference flat runs on the host (band sweep),
/// merged exactly like normalize_intervals, in canonical (src, dst, lo) order.
/// Applies the D2 override.
std::vector<FlatXfer> expand_flat_host(const PlanCore& P);

/// Runs of the triples (canonical order) -> the plan's runs: drop those inside the D2
/// over-sourced intervals and merge in `d2_runs` (identity without the extension).
std::vector<FlatXfer> apply_d2(const PlanCore& P, std::vector<FlatXfer> base);

/// Append the runs of a triple (band sweep), merging abutting runs of the same
/// (src, dst) with the last element of `out` like normalize_intervals.
void append_runs(const stair::Triple& T, std::vector<FlatXfer>& out);

/// The same expansion evaluated row by row (the GPU planner's algorithm), host side.
std::vector<FlatXfer> expand_flat_rows_host(const PlanCore& P);

/// Reference dump (routing.hpp:86-90 format_transfer lines, canonical order),
/// given the ZeRO runs (from expand_flat_host or the GPU planner).
std::string dump(const PlanCore& P, const std::vector<FlatXfer>& flat);
/// The same with the box transfers given explicitly (e.g. from the GPU planner).
std::string dump(const PlanCore& P, const std::vector<BoxXfer>& boxes, const std::vector<FlatXfer>& flat);

/// bytes per element of a state kind (param: the tensor's dtype_bytes)
int payload_width(const ModelSpace& space, int kind, int tensor);
/// canonical transfer order (routing.hpp:79 transfer_order_less) for box transfers
bool box_xfer_less(const PlanCore& P, const BoxXfer& a, const BoxXfer& b);

/// Visit the band rectangles of a triple: emit(p[2], r_lo, r_hi, cols[2], n).
template <class F>
void for_each_band(const stair::Triple& T, F&& emit);

}  // namespace core
}  // namespace reshard

#include "reshard/plan_core_impl.hpp"
