// Transition engine (Algorithm 1): collective
// promotion, memory-aware chunking of XOR steps under the global-min budget, and
// per-peer contiguous buffer layouts both peers derive without metadata exchange.
//
// Devices are the plan's participants (WorldMap::participants, ascending phys);
// device index i = position in that list, N = count. XOR steps range over
// [1, 2^ceil(log2 N)) — Algorithm 1's {1..N-1} misses pairs with i^j >= N when N is
// not a power of two.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "reshard/plan_core.hpp"

namespace reshard {
namespace sched {

/// One resolved fragment of the plan (a reference SliceTransfer), by device index.
struct Fragment {
    int kind = 0;
    int tensor = -1;  // -1: flat optimizer run
    std::int64_t lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    int src_rank = -1, dst_rank = -1;
    int src_dev = -1, dst_dev = -1;
    std::int64_t bytes = 0;
};

enum class CommKind : int { P2P = 0, Broadcast = 1, Scatter = 2, Gather = 3 };

/// CommOp: a promoted collective over one logical tensor.
struct CommOp {
    CommKind kind = CommKind::P2P;
    int root = -1;                   // device index (src for Broadcast/Scatter, dst for Gather)
    std::vector<int> participants;   // sorted, duplicate-free device indices
    std::vector<std::int64_t> frags; // fragment indices (plan order)
    std::int64_t bytes = 0;          // payload bytes (sum over fragments)
};

/// Per-peer contiguous buffer: fragments in plan order with byte offsets.
struct PeerBuffer {
    int peer = -1;
    std::vector<std::int64_t> frags;
    std::vector<std::int64_t> offsets;
    std::int64_t bytes = 0;
};

struct RankStep {
    int step = 0;
    int peer = -1;  // -1: inactive
    PeerBuffer send, recv;
};

/// Stage: steps, per-device per-step buffer layouts, cost.
struct Stage {
    std::vector<int> steps;
    std::vector<std::vector<RankStep>> ranks;  // [device][k] for steps[k]
    std::int64_t mem_cost = 0;
};

struct TransitionSchedule {
    int N = 0;
    std::vector<int> devices;  // device index -> phys
    std::vector<Fragment> frags;
    std::vector<CommOp> collectives;        // dedicated phase before the p2p stages
    std::vector<Stage> stages;
    std::vector<std::int64_t> step_cost;    // by step s (index s), 0 = unused
    std::int64_t budget = 0;                // M_global_min
    std::vector<std::vector<std::string>> free_list;  // per device: obsolete buffers freed before stage 1
};

/// Peer(i, s) = i XOR s; -1 if outside [0, N).
inline int xor_peer(int i, int s, int N) {
    const int p = i ^ s;
    return (p >= 0 && p < N && p != i) ? p : -1;
}
/// Steps with potential traffic for N devices: [1, 2^ceil(log2 N)) (D4 fix).
std::vector<int> xor_steps(int N);

/// MemoryAwareChunk. Throws BudgetError
/// ("infeasible budget: finer fragmentation required") if one step exceeds the budget.
std::vector<std::vector<int>> memory_aware_chunk(const std::vector<int>& steps, const std::vector<std::int64_t>& cost,
                                                 const std::vector<std::int64_t>& mem_avail, std::int64_t* budget);

/// Fragments of a plan (box transfers + expanded ZeRO runs), plan order.
std::vector<Fragment> plan_fragments(const core::PlanCore& P, const std::vector<core::FlatXfer>& flat);

/// OptimizePrimitives. Returns the collectives;
/// `residual` receives the indices of fragments left as p2p.
std::vector<CommOp> optimize_primitives(const core::PlanCore& P, const std::vector<Fragment>& frags,
                                        std::vector<std::int64_t>* residual, bool promote = true);

/// build_schedule: primitives -> free-list -> step costs ->
/// chunking -> per-stage per-peer buffer layouts.
TransitionSchedule build_schedule(const core::PlanCore& P, const std::vector<core::FlatXfer>& flat,
                                  const std::vector<std::int64_t>& mem_avail, bool promote = true);

/// Schedule dump: collectives, then "stage S step s" annotated transfer lines.
std::string dump_schedule(const core::PlanCore& P, const TransitionSchedule& T);

}  // namespace sched
}  // namespace reshard
