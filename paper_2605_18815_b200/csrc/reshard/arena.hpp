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
    int groups = 0;  // concurrency groups of the unit order; 0 -> the cheapest schedule level that fits the cap;
                     // -1 -> rounds (one unit per GPU per group)
    int bands = 1;   // layer bands per destination rank (with groups > 0)
};

struct ArenaStats {
    std::int64_t physical_bytes = 0;  // physical memory mapped (A + fresh B chunks)
    std::int64_t a_bytes = 0, b_bytes = 0;
    std::int64_t aliased_bytes = 0;   // B bytes living in A's dead chunks
    std::int64_t chunks = 0;
};

/// Stage units: (destination rank, layer band), band(t) = layer(t) * bands / num_layers.
/// With bands = 1 a unit is a whole destination rank; finer bands let a GPU rebuild its
/// new layout band by band in the memory its old layout frees (PP-interleaved order,
/// PAPER.md:782-802; config 5 on 8 GPUs needs it).
struct UnitMap {
    int nb = 1, nd = 0;
    std::vector<int> band_of_tensor;
    UnitMap(const core::PlanCore& P, int bands);
    int unit(int rank, int tensor) const { return rank * nb + (tensor < 0 ? 0 : band_of_tensor[static_cast<size_t>(tensor)]); }
    int count() const { return nd * nb; }
};

/// Stage order of a direction over units: greedy on the per-GPU live bytes (old data
/// still to be read + new data written), keeping every GPU under the running peak and
/// freeing the most old bytes first. Deterministic: every rank derives the same order.
std::vector<int> greedy_stage_order(const core::PlanCore& P, const std::vector<exec::CopyOp>& ops, int bands = 1,
                                    int n_gpus = 1);

/// Host-side memory plan (no driver calls; CPU-testable).
struct BufPlan {
    std::int64_t bytes = 0, reserved = 0;
    bool direct = false;     // small buffer: own allocation, never aliased (or hosted elsewhere)
    bool remote = false;     // hosted by another GPU (multi-GPU plans)
    std::vector<int> phys;   // physical chunk per VA chunk
};
struct MemoryPlan {
    std::int64_t chunk = 0;
    int bands = 1;
    int groups = 0;                // concurrency groups of the unit order (0: one per unit)
    std::vector<BufPlan> bufs[2];  // [layout][rank * kNumBufs + buf]
    std::vector<int> order[2];     // stage orders (units) A->B, B->A
    std::vector<int> cut[2];       // per stage position: 1 = a barrier precedes it
    int nphys = 0;
    ArenaStats stats;
};
/// Plan the buffers hosted by `gpu` (contiguous-block placement over n_gpus). Stage
/// orders are global, so with n_gpus > 1 every group boundary is a cross-GPU barrier.
/// `groups` (0 = one per unit) coarsens the unit order into that many concurrency
/// groups: fewer barriers, less aliasing. `bands` splits every destination rank into
/// layer bands.
MemoryPlan plan_memory(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t chunk, bool with_grads,
                       int n_gpus = 1, int gpu = 0, int groups = 0, int bands = 1);
MemoryPlan plan_memory_ops(const core::PlanCore& ab, const core::PlanCore* ba, const std::vector<exec::CopyOp>& ops_ab,
                           const std::vector<exec::CopyOp>& ops_ba, std::int64_t chunk, bool with_grads, int n_gpus,
                           int gpu, int groups, int bands);
/// fewest groups (bands = 1) whose plan fits `cap` bytes on `gpu` (-1: none does); the
/// physical bytes of the last plan tried in *physical
int min_stage_groups(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t chunk, bool with_grads, int n_gpus,
                     int gpu, std::int64_t cap, std::int64_t* physical);
/// The schedule ladder, cheapest first: for bands 1, 2, 4, ... (up to the layer count)
/// group counts from one (no aliasing) to one per unit (most aliasing).
/// groups value of the band-interleaved order: bands ordered so each concurrency group
/// holds one band of every source pipeline stage, all destination ranks of a band
/// together (groups = bands / src pp)
constexpr int kBandInterleaved = -2;
int interleave_stride(const core::PlanCore& P, int nb);
struct ScheduleLevel {
    int bands, groups;  // groups -1: rounds (one unit per GPU per group); -2: band-interleaved
};
std::vector<ScheduleLevel> schedule_levels(const core::PlanCore& ab, int n_gpus = 1);
/// first level of the ladder whose plan fits `cap` on `gpu` (-1: none; *physical = the
/// smallest footprint seen). One GPU; across GPUs use schedule_footprints.
int choose_schedule(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t chunk, bool with_grads, int n_gpus,
                    int gpu, std::int64_t cap, std::int64_t* physical);
/// physical bytes `gpu` needs at every level of the ladder (multi-GPU agreement: every
/// rank marks its feasible levels, the group takes the first level feasible everywhere)
std::vector<std::int64_t> schedule_footprints(const core::PlanCore& ab, const core::PlanCore* ba, std::int64_t chunk,
                                              bool with_grads, int n_gpus, int gpu);
/// Modeled time of a plan's stages (both directions): per concurrency group the busiest
/// GPU's NVLink-out / NVLink-in / HBM bound plus a barrier, groups in sequence. Used to
/// pick, among the schedule levels that fit the cap everywhere, the fastest.
double estimate_seconds(const MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba,
                        const std::vector<exec::CopyOp>& ops_ab, const std::vector<exec::CopyOp>& ops_ba, int n_gpus);
/// (physical bytes on `gpu`, modeled seconds) at every level of the ladder
std::vector<std::pair<std::int64_t, double>> schedule_costs(const core::PlanCore& ab, const core::PlanCore* ba,
                                                            std::int64_t chunk, bool with_grads, int n_gpus, int gpu);
/// Group consecutive stages that may run concurrently (fills mp.cut): a barrier only
/// where a stage overwrites a chunk an earlier stage of the running group still reads.
void plan_stage_cuts(MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba,
                     const std::vector<exec::CopyOp>& ops_ab, const std::vector<exec::CopyOp>& ops_ba);
/// Executed stage (launch group, after the cuts) of the last read of every A chunk, per
/// A buffer (-1: never read)
std::vector<std::vector<int>> last_read_stage(const MemoryPlan& mp, const core::PlanCore& ab,
                                              const std::vector<exec::CopyOp>& ops_ab);
/// Replays the staged execution chunk by chunk (A->B, then B->A) tracking which
/// logical chunk each physical chunk holds; counts reads of clobbered data and
/// same-group read/write races. 0 == the aliasing is safe.
std::int64_t simulate_memory_plan(const MemoryPlan& mp, const core::PlanCore& ab, const core::PlanCore* ba);

class Arena {
public:
    /// ab: A->B; ba: B->A on the same buffers (or nullptr for one-way). With n_gpus > 1
    /// this GPU maps the buffers it hosts; peers' buffers arrive through import_peer().
    Arena(const core::PlanCore& ab, const core::PlanCore* ba, const ArenaConfig& cfg, bool with_grads, int n_gpus = 1,
          int gpu = 0);
    ~Arena();
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;

    /// layout 0 = A (src of ab), 1 = B (dst of ab); remote buffers once imported
    void* ptr(int layout, int rank, int buf) const;
    std::int64_t bytes(int layout, int rank, int buf) const;
    const std::vector<int>& stage_order(int dir) const { return order_[dir]; }
    const std::vector<int>& stage_cuts(int dir) const { return cut_[dir]; }
    int bands() const { return bands_; }
    const ArenaStats& stats() const { return stats_; }

    /// POSIX-FD export of every physical allocation backing this GPU's buffers, with a
    /// table of how the buffers map them (the caller passes both to the peers, fdx).
    void export_local(std::vector<int>* fds, std::vector<std::uint8_t>* table) const;
    /// map a peer's buffers into this process's address space (consumes the fds)
    void import_peer(const std::vector<int>& fds, const std::vector<std::uint8_t>& table);
    /// bind this GPU's buffer (layout, rank, buf) to a multicast object at offset 0,
    /// chunk by chunk (the object then writes through to these physical chunks)
    void bind_multicast(class Multicast& mc, int layout, int rank, int buf) const;
    /// bytes a multicast object must span to bind that buffer whole
    std::int64_t bind_size(int layout, int rank, int buf) const;
    /// FreeObsoleteBuffers at run time (one-way arenas on one GPU): once stage `stage` of
    /// A->B has completed, unmap every old-layout chunk whose last read was in a stage <=
    /// `stage` and return the physical chunks the new layout does not reuse to the driver
    /// (cuMemUnmap + cuMemRelease). Returns the bytes released by this call.
    std::int64_t release_through(int stage);
    std::int64_t released_bytes() const { return released_bytes_; }

private:
    struct BufMap {
        std::uint64_t va = 0;
        std::int64_t bytes = 0, reserved = 0;
        std::vector<int> phys;  // physical chunk per VA chunk (local buffers)
        bool remote = false, mapped_vmm = false, own_handle = false;
        std::uint64_t handle = 0;  // own allocation (small buffers, multi-GPU mode)
    };
    std::vector<BufMap> bufs_[2];  // [layout][rank * kNumBufs + buf]
    std::vector<std::uint64_t> handles_;           // local physical chunks
    std::vector<std::uint64_t> imported_;          // peers' physical allocations
    std::vector<std::pair<std::uint64_t, std::int64_t>> peer_maps_;  // (va, reserved) to unmap
    std::vector<int> order_[2], cut_[2];
    int bands_ = 1;
    ArenaConfig cfg_;
    ArenaStats stats_;
    int nranks_[2] = {0, 0};
    int n_gpus_ = 1;
    bool one_way_ = false;
    std::vector<std::vector<int>> a_last_stage_;     // [A buffer][chunk]
    std::vector<std::vector<char>> a_unmapped_;      // [A buffer][chunk]
    std::vector<char> b_uses_;                       // physical chunk -> mapped by a B chunk
    std::int64_t released_bytes_ = 0;
};

/// One shareable VMM device buffer (POSIX-FD handle): allocated on this process's GPU,
/// or imported from a peer process and mapped for this GPU (P2P over NVLink). State
/// buffers a multicast object can bind and peers can map without cudaIpc.
class VmmBuffer {
public:
    VmmBuffer(int device, std::int64_t bytes);             // allocate + map locally
    VmmBuffer(int fd, std::int64_t bytes, int device);     // import a peer's (consumes fd), map for `device`
    ~VmmBuffer();
    VmmBuffer(const VmmBuffer&) = delete;
    VmmBuffer& operator=(const VmmBuffer&) = delete;

    void* ptr() const { return reinterpret_cast<void*>(va_); }
    std::int64_t bytes() const { return bytes_; }        // requested size
    std::int64_t mapped_bytes() const { return size_; }  // rounded to the VMM granularity
    std::uint64_t handle() const { return handle_; }
    int device() const { return device_; }
    int export_fd() const;

private:
    std::uint64_t handle_ = 0, va_ = 0;
    std::int64_t bytes_ = 0, size_ = 0;
    int device_ = 0;
};

/// NVLS multicast object shared by the processes of its member GPUs (created by the
/// root, passed as a POSIX descriptor). Protocol: create/import -> add_device on every
/// member -> (barrier) -> bind memory -> map (root) -> multimem stores.
class Multicast {
public:
    Multicast(std::int64_t bytes, int n_devices);  // create
    Multicast(int fd, std::int64_t bytes);         // import (consumes fd)
    ~Multicast();
    Multicast(const Multicast&) = delete;
    Multicast& operator=(const Multicast&) = delete;

    int export_fd() const;
    void add_device(int device);
    void bind(int device, std::uint64_t mem_handle, std::int64_t mc_offset, std::int64_t bytes);
    void bind(const VmmBuffer& b, std::int64_t mc_offset) { bind(b.device(), b.handle(), mc_offset, b.mapped_bytes()); }
    void* map(int device);
    std::int64_t bytes() const { return bytes_; }
    std::uint64_t handle() const { return handle_; }

private:
    std::uint64_t handle_ = 0;
    std::int64_t bytes_ = 0;
    std::uint64_t va_ = 0;
    struct Binding {
        int device;
        std::int64_t offset, bytes;
    };
    std::vector<Binding> bindings_;
};

}  // namespace mem
}  // namespace reshard
