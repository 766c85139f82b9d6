// Executor runtime object (per GPU / per process). See executor.hpp.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "reshard/executor.hpp"
#include "reshard/tiles.hpp"

namespace reshard {
namespace exec {

class CudaError : public std::runtime_error {
public:
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

/// Memory-aware schedule infeasible under the HBM cap (C ABI RS_ERR_BUDGET).
class BudgetError : public std::runtime_error {
public:
    explicit BudgetError(const std::string& m) : std::runtime_error(m) {}
};

struct ExecConfig {
    int n_gpus = 1;       // GPUs the physical devices of the plan are placed on
    int gpu = 0;          // this process's GPU index in [0, n_gpus)
    int device = 0;       // CUDA device ordinal
    bool with_grads = false;
    std::int64_t tile_bytes = 0;  // 0 -> 512 KiB
    int ctas_per_sm = 0;          // 0 -> 4
};

struct ExecStats {
    std::int64_t local_bytes = 0;   // bytes this GPU copies into its own HBM
    std::int64_t remote_bytes = 0;  // bytes this GPU stores into peers' HBM
    std::int64_t tiles = 0;
    std::int64_t tiles_by_class[5] = {0, 0, 0, 0, 0};  // 16/8/4/2/1-byte vectors
    std::int64_t launches = 0;                         // kernel launches per run()
    std::int64_t ce_bytes = 0;                         // peer-bound bytes moved by copy engines
    std::int64_t mc_bytes = 0;                         // bytes delivered by multicast stores
    std::int64_t dup_bytes = 0;                        // replica bytes copied on the destination GPU
    std::int64_t scatter_bytes = 0;                    // promoted Scatter bytes pushed as root
    std::int64_t gather_bytes = 0;                     // promoted Gather bytes pulled as root
};

struct RankBufs {
    int gpu = -1;
    void* ptr[kNumBufs] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    std::int64_t bytes[kNumBufs] = {0, 0, 0, 0, 0, 0};
};

/// Pinned host staging for descriptor uploads (reused across prepares).
struct PinnedBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf();
    size_t size() const { return cap; }
    void grow(size_t bytes);
};

/// Device tiles of one launch group set (fused transition, or one channel's
/// pack / unpack); kernels add runtime base addresses so staging buffers can move.
struct TileSet {
    struct Group {
        int cls, begin, count, key;
    };
    /// a recorded 2-D copy (add), cut into tiles at finalize (host) or first launch (GPU)
    using Pending = CopyRec;
    std::vector<Pending> pending;
    bool interleave = false;  // finalize: interleave lanes in proportion to their bytes
    size_t ntiles = 0;
    std::vector<Group> groups;
    void* dev = nullptr;                    // descriptors of the last finalize (dev_buf[cur])
    void* dev_buf[2] = {nullptr, nullptr};  // used in turn by successive finalizes
    size_t dev_bytes[2] = {0, 0};
    int cur = 1;
    // descriptor fences: events recorded after every launch that reads dev_buf[i]; the
    // next finalize into dev_buf[i] makes its upload wait for all of them, so a re-prepare
    // never overwrites descriptors a kernel still in flight reads (any number of runs may
    // be outstanding)
    mutable std::vector<cudaEvent_t> fences[2];
    mutable std::vector<cudaEvent_t> fence_pool;
    // Lazy upload: finalize leaves the descriptors in this set's own pinned buffer; the
    // first launch of each group copies that group's slice on the launch stream right
    // before the kernel, so the uploads of later groups overlap earlier groups' kernels
    // and prepare() never waits for a DMA. hfences guard the pinned buffer's reuse,
    // wait_first holds the previous readers of dev_buf[cur] the first upload must follow.
    PinnedBuf* hbuf[2] = {nullptr, nullptr};
    mutable std::vector<cudaEvent_t> hfences[2];
    mutable std::vector<cudaEvent_t> wait_first;
    mutable std::vector<char> uploaded;
    // GPU cut (default): the pinned slot holds the records and their per-class tile
    // offsets; the first launch uploads them (~76 B per record instead of 40 B per
    // tile) and cut_kernel writes the tiles on the device. RS_HOST_TILES=1 or the
    // tile-level interleave keep the host cut.
    bool gpu_cut = false;
    mutable bool materialized = true;
    size_t nrec_cut = 0;
    void* dev_rec[2] = {nullptr, nullptr};
    size_t rec_bytes[2] = {0, 0};
    void materialize(cudaStream_t stream) const;
    // the stream the descriptors were uploaded (and cut) on, and an event after that:
    // launches of this set on any other stream wait for it
    mutable cudaStream_t mat_stream = nullptr;
    mutable cudaEvent_t mat_ev = nullptr;
    mutable bool mat_pending = false;
    void order_after_upload(cudaStream_t stream) const;
    static bool host_tiles_forced() {
        static const bool v = [] {
            const char* e = std::getenv("RS_HOST_TILES");
            return e && e[0] == '1';
        }();
        return v;
    }
    /// upload every group not uploaded yet on `stream` (before a graph capture)
    void flush_uploads(cudaStream_t stream) const;
    void upload_group(size_t gi, cudaStream_t stream) const;
    cudaEvent_t take_event() const;
    /// record a fence for the current descriptors on `stream` (skipped while capturing:
    /// run_graph fences after the graph launch)
    void fence(cudaStream_t stream) const;
    TileSet() = default;
    TileSet(const TileSet&) = delete;
    TileSet& operator=(const TileSet&) = delete;
    ~TileSet();
    void add(int key, std::uint64_t src, std::uint64_t dst, std::int64_t rows, std::int64_t rb, std::int64_t sp,
             std::int64_t dp, std::int64_t kTile, int lane = 0);
    void finalize(ExecStats* stats, cudaStream_t upload, struct PinnedBuf* staging);
    void cur_buf_flip() { cur ^= 1; }
    /// launch groups in key order; key_mod > 0 restricts to keys with key % key_mod == key_rem
    int launch(cudaStream_t stream, std::uint64_t sbase, std::uint64_t dbase, int sms, int ctas_per_sm, bool bulk,
               int key_mod = 0, int key_rem = 0) const;
};

/// Broadcast promotion (optimize_primitives): one
/// source region pushed to several destination ranks on distinct GPUs, all with the same
/// layout as the source (DP replicas). Executed as one NVLS multicast store stream from
/// the root GPU instead of one push per destination. Slot s of a GPU = its s-th
/// destination rank of the broadcast (one multicast object per slot).
struct BcastGroup {
    int id = 0, root_rank = 0, root_gpu = 0, buf = 0, slot = 0;
    std::vector<int> member_gpus, member_ranks;  // destination GPUs / ranks (root excluded)
    std::int64_t buffer_bytes = 0;              // bytes of buffer `buf` (same on every member)
    std::int64_t payload_bytes = 0;             // bytes the root sends once (per member they arrive)
    std::vector<size_t> ops;                    // build_ops indices covered (every member's copy)
};

class Executor {
public:
    Executor(const core::PlanCore& P, const ExecConfig& cfg);
    ~Executor();
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;

    int gpu_of_phys(int phys) const;
    /// drive the bound buffers with a re-computed plan of the same transition (same
    /// configs, world map, model and buffer geometry); takes effect at the next prepare()
    void set_plan(const core::PlanCore& P);
    /// execute optimize_primitives' Scatter / Gather collectives as primitives: a
    /// Scatter is pushed by its root; a Gather is pulled by its root (destination GPU)
    /// from the peers' source buffers, which export_ipc then shares too. Set on every
    /// rank before export_ipc; takes effect at the next prepare().
    void set_collectives(bool on);
    /// memory-aware stages: destination ranks in execution order, one launch group
    /// per stage (a stage starts after all reads of earlier stages completed)
    void set_stage_order(const std::vector<int>& dst_order, const std::vector<int>& cuts = {});
    /// cudaMalloc every unbound buffer of the virtual ranks placed on this GPU
    void alloc();
    /// use a caller-owned device buffer (side 0 src / 1 dst)
    void bind(int side, int rank, int buf, void* ptr, std::int64_t bytes);
    void* buffer(int side, int rank, int buf, std::int64_t* bytes) const;
    int rank_gpu(int side, int rank) const { return bufs_[side][static_cast<size_t>(rank)].gpu; }

    /// cudaIpc handles of this GPU's destination buffers / map a peer's
    std::vector<std::uint8_t> export_ipc() const;
    void import_ipc(const std::uint8_t* blob, size_t len);

    /// build device tiles for the moves whose source lives here. staged: moves between
    /// GPUs go through per-channel pack/unpack (Algorithm 1 buffered mode) instead of
    /// direct peer stores; only same-GPU moves stay fused.
    void prepare(bool staged = false);
    /// launch the transition (fused part); returns the number of kernel launches
    int run(cudaStream_t stream);
    /// the same launches replayed from a CUDA graph (captured at the first call after
    /// each prepare, per stream): for launch-bound small transitions
    int run_graph(cudaStream_t stream);
    /// memory-aware stages across GPUs: launch one stage; the caller puts a cross-GPU
    /// barrier between stages (a stage's writes may land in chunks freed by the last one)
    int run_stage(int stage, cudaStream_t stream);
    int num_stages() const;
    /// staged mode: bytes of the (src phys -> dst phys) channel, pack into / unpack from
    /// a contiguous buffer (same layout on both sides, derived from the plan)
    std::int64_t channel_bytes(int src_phys, int dst_phys) const;
    int pack(int src_phys, int dst_phys, void* buf, cudaStream_t stream);
    int unpack(int src_phys, int dst_phys, const void* buf, cudaStream_t stream);

    /// broadcast groups of this plan and placement (identical on every rank)
    const std::vector<BcastGroup>& bcast_groups();
    /// root GPU: execute group `id` through the multicast address `mc_va` (its object binds
    /// the root's source buffer and every member's destination buffer at equal offsets);
    /// nullptr reverts to per-destination pushes. Takes effect at the next prepare().
    void set_multicast(int id, void* mc_va);
    /// replica dedup: a source region bound for several replica ranks on one GPU crosses
    /// NVLink once; run_dup() copies it to the others on that GPU — call it on every GPU
    /// after run() and a cross-GPU barrier. Takes effect at the next prepare().
    /// early: stage 1 is a tail of this GPU's non-replica pushes sized to hide the copies,
    /// stage 0 everything else incl. the primaries (num_stages() = 2), so run_dup can
    /// follow a barrier on stage 0 and overlap stage 1
    void set_replica_dedup(bool on, bool early = false);
    int run_dup(cudaStream_t stream);

    void fill(int side, std::uint64_t seed, cudaStream_t stream);
    std::int64_t verify(int side, std::uint64_t seed, cudaStream_t stream, std::int64_t* first_bad);

    const ExecStats& stats() const { return stats_; }
    const core::PlanCore& plan() const { return *P_; }

private:
    std::vector<FillTask> fill_tasks(int side) const;
    void compute_dups(const std::vector<CopyOp>& ops);
    int launch_multicast(cudaStream_t stream) const;
    int run_fused(cudaStream_t stream);
    int run_direct(cudaStream_t stream);
    void upload_tasks(const std::vector<FillTask>& tasks, cudaStream_t stream);

    const core::PlanCore* P_;
    ExecConfig cfg_;
    int per_gpu_ = 1;
    int sms_ = 148;
    std::vector<RankBufs> bufs_[2];
    std::vector<void*> owned_;
    std::vector<void*> ipc_opened_;
    std::map<std::string, void*> ipc_map_;
    struct Channel {
        std::unique_ptr<TileSet> pack, unpack;
        std::int64_t bytes = 0;
        std::vector<std::int64_t> op_bytes;  // packed size of each op, channel order
    };

public:
    /// staged mode: sizes of the channel's ops in packing order (the "naive" mode sends
    /// one message per op)
    std::vector<std::int64_t> channel_ops(int src_phys, int dst_phys) const {
        auto it = channels_.find({src_phys, dst_phys});
        return it == channels_.end() ? std::vector<std::int64_t>{} : it->second.op_bytes;
    }

private:
    std::unique_ptr<TileSet> fused_;
    std::unique_ptr<TileSet> mc_;  // multicast tiles (dst = multicast address)
    std::unique_ptr<TileSet> dup_;  // replica copies on this GPU (run_dup)
    bool dedup_ = false;
    bool collectives_ = false;
    std::vector<std::int8_t> box_coll_;  // per plan box transfer: 0 p2p, 2 Scatter, 3 Gather (sched::CommKind)
    std::vector<int> dup_primary_;  // per op: dst rank holding the primary copy, or -1
    std::vector<char> dup_lead_;    // per op: it carries a region other ranks on its GPU copy
    bool dup_early_ = false;
    std::vector<BcastGroup> bcast_;
    bool bcast_ready_ = false;
    std::map<int, void*> mc_va_;
    std::int64_t mc_src_bytes_ = 0;
    cudaStream_t mc_stream_ = nullptr;
    cudaGraphExec_t graph_exec_ = nullptr;
    cudaStream_t graph_stream_ = nullptr;
    int graph_launches_ = 0;
    bool auto_graph_ = false;  // run() replays a CUDA graph (small, launch-bound transitions)
    int runs_since_prepare_ = 0;
    cudaEvent_t mc_ev_[3] = {nullptr, nullptr, nullptr};
    std::map<std::pair<int, int>, Channel> channels_;
    bool staged_ = false;
    cudaStream_t upload_ = nullptr;
    PinnedBuf staging_;
    cudaStream_t aux_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    bool has_remote_ = false;
    bool remote_bulk_ = false;     // RS_REMOTE_KERNEL=bulk: TMA bulk stores to peers
    bool split_remote_ = false;    // RS_SPLIT_REMOTE=1: peer tiles and local tiles on two streams
    struct CeOp {
        std::uint64_t src, dst;
        std::int64_t bytes;
    };
    std::vector<CeOp> ce_ops_;          // large contiguous peer-bound blocks for the copy engines
    std::vector<cudaStream_t> ce_streams_;  // [0] = aux_
    std::vector<cudaEvent_t> ce_join_;
    std::int64_t ce_min_bytes_ = 4 << 20;  // RS_CE_MIN_BYTES (0 disables)
    int remote_ctas_per_sm_ = 2;   // RS_REMOTE_CTAS_PER_SM
    std::vector<int> stage_of_dst_;  // stage of each unit (dst rank x layer band)
    int stage_bands_ = 1;
    int stage_of(const CopyOp& op) const;
    void* d_fill_ = nullptr;
    size_t fill_bytes_ = 0;
    PinnedBuf fill_staging_;
    void* d_counters_ = nullptr;
    bool prepared_ = false;
    bool use_bulk_ = true;  // TMA bulk pipeline for 16-byte-class tiles (RS_COPY_KERNEL=vector to disable)
    ExecStats stats_;
};

}  // namespace exec
}  // namespace reshard
