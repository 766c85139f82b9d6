// State-aware memory plan under a per-GPU HBM cap (PAPER.md
// :782-802 "eagerly deallocates source parameters"; Algorithm 1 FreeObsoleteBuffers).
//
// Old and new layouts of one GPU's virtual ranks are laid out in CUDA VMM address
// ranges backed by a pool of physical chunks. A destination chunk may share the
// physical memory of a source chunk whose last read happens in an EARLIER stage
// than the destination chunk's first write — the eager free of Algorithm 1, decided
// once at plan time so the hot path makes no driver calls: the same physical chunk
// is simply mapped at two virtual addresses. For a round trip (A->B then B->A on the
// same buffers) both directions' constraints are enforced jointly; the B->A stage
// order is the reverse of A->B's source-death order, which is what makes the pairs
// compatible.
//
// Stage = one destination virtual rank (all of its buffers). Stages run as
// separate kernel launches on one stream, so a stage starts only after every read of
// the previous stages completed.
#pragma once

#include <cstdint>
#include <vector>

#include "reshard/executor.hpp"
#include "reshard/plan_core.hpp"

namespace reshard {
namespace mem {

struct ArenaConfig {
    int device = 0;
    std::int64_t cap_bytes = 0;             // physical budget; 0 -> free memory minus 1 GiB
    std::int64_t chunk_bytes = 32ll << 20;  // physical chunk (multiple of the VMM granularity)
};

struct ArenaStats {
    std::int64_t physical_bytes = 0;  // physical memory mapped (A + fresh B chunks)
    std::int64_t a_bytes = 0, b_bytes = 0;
    std::int64_t aliased_bytes = 0;   // B bytes living in A's dead chunks
    std::int64_t chunks = 0;
};

/// Stage order of a direction: destination ranks, greedy so sources die early.
std::vector<int> greedy_stage_order(const core::PlanCore& P, const std::vector<exec::CopyOp>& ops);

/// Host-side memory plan (no driver calls; CPU-testable).
struct BufPlan {
    std::int64_t bytes = 0, reserved = 0;
    bool direct = false;     // small buffer: plain allocation, never aliased
    std::vector<int> phys;   // physical chunk per VA chunk
};
struct MemoryPlan {
    std::int64_t chunk = 0;
    std::vector<BufPlan> bufs[2];  // [layout][rank * kNumBufs + buf]
    std::vector<int> order[2];     // stage orders (dst ranks) A->B, B->A
    int nphys = 0;
    ArenaStats stats;
};
MemoryPlan plan_memory(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t chunk, bool with_grads);
/// Replays the staged execution chunk by chunk (A->B, then B->A) tracking which
/// logical chunk each physical chunk holds; counts reads of clobbered data and
/// same-stage read/write races. 0 == the aliasing is safe.
std::int64_t simulate_memory_plan(const MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba);

class Arena {
public:
    /// ab: A->B; ba: B->A on the same buffers (or nullptr for one-way). All virtual
    /// ranks must be placed on this GPU (n_gpus == 1).
    Arena(const core::PlanCore& ab, const core::PlanCore* ba, const ArenaConfig& cfg, bool with_grads);
    ~Arena();
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;

    /// layout 0 = A (src of ab), 1 = B (dst of ab)
    void* ptr(int layout, int rank, int buf) const;
    std::int64_t bytes(int layout, int rank, int buf) const;
    const std::vector<int>& stage_order(int dir) const { return order_[dir]; }
    const ArenaStats& stats() const { return stats_; }

private:
    struct BufMap {
        std::uint64_t va = 0;
        std::int64_t bytes = 0, reserved = 0;
        std::vector<int> phys;  // physical chunk per VA chunk
    };
    std::vector<BufMap> bufs_[2];  // [layout][rank * kNumBufs + buf]
    std::vector<std::uint64_t> handles_;
    std::vector<int> order_[2];
    ArenaConfig cfg_;
    ArenaStats stats_;
    int nranks_[2] = {0, 0};
};

}  // namespace mem
}  // namespace reshard
