// sm_100a executor: copy-tile kernel (local HBM and NVLink peer stores), canon
// fill / verify kernels, per-GPU orchestration and cudaIpc peer mapping.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "reshard/executor.hpp"
#include "reshard/executor_rt.hpp"
#include "reshard/tiles.hpp"
#include "reshard/schedule.hpp"
#include "reshard/pool.hpp"

namespace reshard {
namespace exec {

#define RS_CUDA(x)                                                                                          \
    do {                                                                                                    \
        cudaError_t e_ = (x);                                                                               \
        if (e_ != cudaSuccess) throw CudaError(strfmt("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                                      __FILE__, __LINE__));                                 \
    } while (0)

// ------------------------------------------------------------------ kernels

constexpr int kThreads = 512;
constexpr int kUnroll = 4;
constexpr int kBulkStages = 4;        // smem stages per CTA
constexpr int kBulkStage = 32 << 10;  // bytes per stage
constexpr int kBulkCtasPerSm = 1;

template <int V>
struct VecT;
template <>
struct VecT<16> { using T = uint4; };
template <>
struct VecT<8> { using T = uint2; };
template <>
struct VecT<4> { using T = unsigned int; };
template <>
struct VecT<2> { using T = unsigned short; };
template <>
struct VecT<1> { using T = unsigned char; };

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldg(p); }
template <>
__device__ __forceinline__ uint4 ld_stream<uint4>(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <bool MC, typename T>
__device__ __forceinline__ void st_vec(T* p, const T& v) {
    *p = v;
}
// NVLS multicast store: one 16-B store through the multicast address lands in every
// member GPU's bound memory. .f32 only names the register format: a plain store moves
// the bits unchanged (NaN payloads included; the verify kernel checks every byte).
template <>
__device__ __forceinline__ void st_vec<true, uint4>(uint4* p, const uint4& v) {
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

/// 256-bit vector (sm_100: LDG.E.256 / STG.E.256): half the memory instructions per
/// byte of the 16-byte path, and each peer store carries 32 B of payload per NVLink write
struct alignas(32) V32 {
    unsigned w[8];
};
template <>
__device__ __forceinline__ V32 ld_stream<V32>(const V32* p) {
    V32 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                   "=r"(r.w[7])
                 : "l"(p));
    return r;
}
template <>
__device__ __forceinline__ void st_vec<false, V32>(V32* p, const V32& v) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
                 "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

/// One tile with vectors of type T (the tile's addresses, pitches and row size are
/// multiples of sizeof(T)); the CTA's threads stride over it keeping kUnroll
/// independent loads in flight before storing.
template <typename T, bool MC, int kUnroll = kUnroll>
__device__ __forceinline__ void copy_tile(const Tile& tl) {
    const unsigned vpr = tl.row_bytes / sizeof(T);
    if (tl.rows == 1) {
        const T* __restrict__ s = reinterpret_cast<const T*>(tl.src);
        T* __restrict__ d = reinterpret_cast<T*>(tl.dst);
        unsigned i = threadIdx.x;
        for (; i + (kUnroll - 1) * kThreads < vpr; i += kUnroll * kThreads) {
            T r[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) r[u] = ld_stream(s + i + u * kThreads);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) st_vec<MC>(d + i + u * kThreads, r[u]);
        }
        for (; i < vpr; i += kThreads) st_vec<MC>(d + i, ld_stream(s + i));
    } else {
        const unsigned n = tl.rows * vpr;
        for (unsigned i = threadIdx.x; i < n; i += kUnroll * kThreads) {
            T r[kUnroll];
            unsigned row[kUnroll], col[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const unsigned e = i + u * kThreads;
                row[u] = e / vpr;
                col[u] = e - row[u] * vpr;
                if (e < n) r[u] = ld_stream(reinterpret_cast<const T*>(tl.src + row[u] * tl.src_pitch) + col[u]);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const unsigned e = i + u * kThreads;
                if (e < n) st_vec<MC>(reinterpret_cast<T*>(tl.dst + row[u] * tl.dst_pitch) + col[u], r[u]);
            }
        }
    }
}

/// Copy tiles of alignment class V (all addresses, pitches and row sizes are
/// multiples of V). Persistent grid: CTA b takes tiles b, b+grid, ... MC: the
/// destination is a multicast address (16-B class only). W32: 16-B-class tiles that are
/// also 32-B aligned move as 256-bit vectors.
template <int V, bool MC = false, bool W32 = false>
__global__ void __launch_bounds__(kThreads, W32 ? 2 : 1) copy_tiles_kernel(const Tile* __restrict__ tiles, int ntiles, std::uint64_t sbase,
                                                              std::uint64_t dbase) {
    using T = typename VecT<V>::T;
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        Tile tl = tiles[ti];
        tl.src += sbase;
        tl.dst += dbase;
        if constexpr (W32 && V == 16 && !MC) {
            const std::uint64_t a = tl.src | tl.dst | tl.row_bytes | (tl.rows > 1 ? (tl.src_pitch | tl.dst_pitch) : 0);
            if ((a & 31) == 0) {
                copy_tile<V32, false, 2>(tl);  // 2 x 32 B in flight = the 16-B path's 4 x 16 B
                continue;
            }
        }
        copy_tile<T, MC>(tl);
    }
}

// ---- TMA bulk-copy pipeline (cp.async.bulk global -> smem -> global), 16-B class

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive_expect(std::uint64_t* b, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, std::uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n RS_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra RS_WAIT_%=;\n}" ::"r"(
            smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* s, const void* g, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(s)),
                 "l"(g), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* g, const void* s, std::uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct BulkStage {
    std::uint64_t dst;    // first row's destination
    std::uint64_t pitch;  // destination pitch
    std::uint32_t rows, bytes;
};

/// One warp per CTA streams its tiles through S shared-memory stages of kStage
/// bytes: a stage holds up to kStage/row_bytes rows of one tile (or a piece of one
/// long row). Per iteration c: wait stage c's loads (mbarrier tx count), issue its
/// bulk stores, then refill the slot freed by stage c-1 once those stores have read
/// it (wait_group.read 1), keeping S-1 stages of loads in flight. Every lane commits
/// one bulk group per stage so the per-thread group counts stay in lockstep.
template <int S, int kStage>
__global__ void __launch_bounds__(32) bulk_tiles_kernel(const Tile* __restrict__ tiles, int ntiles, std::uint64_t sbase,
                                                      std::uint64_t dbase) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ std::uint64_t bar[S];
    __shared__ BulkStage rec[S];
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    int t = blockIdx.x;
    std::uint32_t row = 0, off = 0;
    // issue loads for the next stage into slot; false when the CTA has no more work
    auto load_next = [&](int slot) -> bool {
        if (t >= ntiles) return false;
        Tile tl = tiles[t];
        tl.src += sbase;
        tl.dst += dbase;
        std::uint32_t nr, n, r0 = row, o = off;
        if (tl.row_bytes <= static_cast<std::uint32_t>(kStage)) {
            nr = min(static_cast<std::uint32_t>(kStage) / tl.row_bytes, tl.rows - row);
            n = tl.row_bytes;
            row += nr;
        } else {
            nr = 1;
            n = min(static_cast<std::uint32_t>(kStage), tl.row_bytes - off);
            off += n;
            if (off == tl.row_bytes) off = 0, ++row;
        }
        if (row == tl.rows) row = 0, off = 0, t += gridDim.x;
        if (lane == 0) {
            rec[slot] = BulkStage{tl.dst + r0 * tl.dst_pitch + o, tl.dst_pitch, nr, n};
            mbar_arrive_expect(&bar[slot], nr * n);
        }
        __syncwarp();
        unsigned char* buf = smem + slot * kStage;
        for (std::uint32_t r = lane; r < nr; r += 32)
            bulk_load(buf + r * n, reinterpret_cast<const void*>(tl.src + (r0 + r) * tl.src_pitch + o), n, &bar[slot]);
        return true;
    };
    int issued = 0;
    while (issued < S - 1 && load_next(issued % S)) ++issued;
    std::uint32_t parity = 0;  // bit s: parity to wait for on slot s
    for (int c = 0; c < issued; ++c) {
        const int slot = c % S;
        mbar_wait(&bar[slot], (parity >> slot) & 1u);
        parity ^= 1u << slot;
        const BulkStage st = rec[slot];
        const unsigned char* buf = smem + slot * kStage;
        for (std::uint32_t r = lane; r < st.rows; r += 32)
            bulk_store(reinterpret_cast<void*>(st.dst + r * st.pitch), buf + r * st.bytes, st.bytes);
        bulk_commit();
        // slot (c+S-1) % S held stage c-1, whose stores were the previous group
        bulk_wait_read1();
        __syncwarp();
        if (load_next((c + S - 1) % S)) ++issued;
    }
    bulk_wait_all();
}

/// value of element with global flat index k for buffer kind
__device__ __forceinline__ std::uint64_t canon_payload(std::uint64_t seed, std::int64_t k, int kind) {
    switch (kind) {
        case 0: return canon_value(seed, k, StateKind::Param);
        case 1: return canon_value(seed, k, StateKind::Optim) & 0xffffffffull;
        case 2: return canon_value(seed, k, StateKind::Optim) >> 32;
        case 3: return canon_value(seed ^ 0x5eedull, k, StateKind::Optim) & 0xffffffffull;
        default: return canon_value(seed, k, StateKind::Grad) & 0xffffffffull;
    }
}

__device__ __forceinline__ std::int64_t task_flat(const FillTask& f, std::int64_t e) {
    const std::int64_t c = e % f.cols_box;
    std::int64_t q = e / f.cols_box;
    const std::int64_t r = q % f.rows_box;
    q /= f.rows_box;
    std::int64_t p[2] = {0, 0};
    for (int i = f.t.np - 1; i >= 0; --i) {
        p[i] = f.plo[i] + q % f.pext_box[i];
        q /= f.pext_box[i];
    }
    return stair::flat_of(f.t, p, f.rlo + r, f.clo + c);
}

__global__ void fill_kernel(const FillTask* __restrict__ tasks, int ntasks, std::uint64_t seed) {
    for (int ti = blockIdx.y; ti < ntasks; ti += gridDim.y) {
        const FillTask f = tasks[ti];
        const std::int64_t n = f.e_hi - f.e_lo;
        for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < n;
             i += (std::int64_t)gridDim.x * blockDim.x) {
            const std::uint64_t v = canon_payload(seed, task_flat(f, f.e_lo + i), f.kind);
            char* dst = reinterpret_cast<char*>(f.ptr) + i * f.width;
            switch (f.width) {
                case 1: *reinterpret_cast<std::uint8_t*>(dst) = static_cast<std::uint8_t>(v); break;
                case 2: *reinterpret_cast<std::uint16_t*>(dst) = static_cast<std::uint16_t>(v); break;
                case 4: *reinterpret_cast<std::uint32_t*>(dst) = static_cast<std::uint32_t>(v); break;
                default: *reinterpret_cast<std::uint64_t*>(dst) = v; break;
            }
        }
    }
}

__global__ void verify_kernel(const FillTask* __restrict__ tasks, int ntasks, std::uint64_t seed,
                              unsigned long long* __restrict__ bad, long long* __restrict__ first_bad) {
    unsigned long long local_bad = 0;
    for (int ti = blockIdx.y; ti < ntasks; ti += gridDim.y) {
        const FillTask f = tasks[ti];
        const std::int64_t n = f.e_hi - f.e_lo;
        for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < n;
             i += (std::int64_t)gridDim.x * blockDim.x) {
            const std::int64_t k = task_flat(f, f.e_lo + i);
            const std::uint64_t v = canon_payload(seed, k, f.kind);
            const char* src = reinterpret_cast<const char*>(f.ptr) + i * f.width;
            std::uint64_t got;
            std::uint64_t mask;
            switch (f.width) {
                case 1: got = *reinterpret_cast<const std::uint8_t*>(src); mask = 0xffull; break;
                case 2: got = *reinterpret_cast<const std::uint16_t*>(src); mask = 0xffffull; break;
                case 4: got = *reinterpret_cast<const std::uint32_t*>(src); mask = 0xffffffffull; break;
                default: got = *reinterpret_cast<const std::uint64_t*>(src); mask = ~0ull; break;
            }
            if (got != (v & mask)) {
                ++local_bad;
                atomicMin(first_bad, static_cast<long long>(k));
            }
        }
    }
    if (local_bad) atomicAdd(bad, local_bad);
}

__global__ void fill_scalars_kernel(std::uint64_t* p, std::int64_t words, std::uint64_t seed) {
    for (std::int64_t w = threadIdx.x; w < words; w += blockDim.x) p[w] = canon_value(seed, w, StateKind::Scalar);
}

__global__ void verify_scalars_kernel(const std::uint64_t* p, std::int64_t words, std::uint64_t seed,
                                      unsigned long long* bad) {
    for (std::int64_t w = threadIdx.x; w < words; w += blockDim.x)
        if (p[w] != canon_value(seed, w, StateKind::Scalar)) atomicAdd(bad, 1ull);
}

// ------------------------------------------------------------------ host side

namespace {

/// driver API through the runtime's entry-point table (no link-time libcuda
/// dependency, so the library also loads on GPU-less build hosts)
CUresult mem_get_address_range(CUdeviceptr* base, size_t* size, CUdeviceptr p) {
    using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static Fn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
            return CUDA_ERROR_NOT_SUPPORTED;
        fn = reinterpret_cast<Fn>(f);
    }
    return fn(base, size, p);
}


}  // namespace

Executor::Executor(const core::PlanCore& P, const ExecConfig& cfg) : P_(&P), cfg_(cfg) {
    if (cfg_.n_gpus < 1 || cfg_.gpu < 0 || cfg_.gpu >= cfg_.n_gpus) throw ConfigError("bad executor placement");
    int max_phys = 0;
    for (const auto& r : P_->routes) max_phys = std::max(max_phys, r.phys);
    per_gpu_ = (max_phys + 1 + cfg_.n_gpus - 1) / cfg_.n_gpus;
    for (int side = 0; side < 2; ++side) {
        const int n = side == 0 ? P_->src_cfg.world_size() : P_->dst_cfg.world_size();
        bufs_[side].resize(static_cast<size_t>(n));
        for (int r = 0; r < n; ++r) {
            RankBufs& rb = bufs_[side][static_cast<size_t>(r)];
            buffer_sizes(*P_, side, r, cfg_.with_grads, rb.bytes);
            const int phys = side == 0 ? P_->wm.src_phys[static_cast<size_t>(r)] : P_->wm.dst_phys[static_cast<size_t>(r)];
            rb.gpu = gpu_of_phys(phys);
        }
    }
    RS_CUDA(cudaSetDevice(cfg_.device));
}

Executor::~Executor() {
    cudaSetDevice(cfg_.device);
    for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    for (void* p : owned_) cudaFree(p);
    if (d_fill_) cudaFree(d_fill_);
    if (d_counters_) cudaFree(d_counters_);
    if (upload_) cudaStreamDestroy(upload_);
    if (aux_) cudaStreamDestroy(aux_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (mc_stream_) cudaStreamDestroy(mc_stream_);
    for (size_t i = 1; i < ce_streams_.size(); ++i) cudaStreamDestroy(ce_streams_[i]);
    for (cudaEvent_t e : ce_join_) cudaEventDestroy(e);
    for (cudaEvent_t e : mc_ev_)
        if (e) cudaEventDestroy(e);
}

int Executor::gpu_of_phys(int phys) const { return phys / per_gpu_; }

void Executor::set_collectives(bool on) {
    collectives_ = on;
    prepared_ = false;
}

void Executor::set_plan(const core::PlanCore& P) {
    // a re-computed plan of the same transition drives the bound buffers: the layouts
    // (configs, world map, model, buffer sizes) must be identical
    const core::PlanCore& O = *P_;
    auto same_cfg = [](const ParallelConfig& a, const ParallelConfig& b) {
        return a.dp == b.dp && a.tp == b.tp && a.pp == b.pp && a.ep == b.ep && a.zero_enabled == b.zero_enabled &&
               a.rank_order == b.rank_order;
    };
    if (P.space->fingerprint() != O.space->fingerprint() || !same_cfg(P.src_cfg, O.src_cfg) ||
        !same_cfg(P.dst_cfg, O.dst_cfg) || P.wm.src_phys != O.wm.src_phys || P.wm.dst_phys != O.wm.dst_phys ||
        P.opts.scalar_words != O.opts.scalar_words)
        throw ConfigError("set_plan: the plan describes a different transition than the executor's buffers");
    for (int side = 0; side < 2; ++side)
        for (size_t r = 0; r < bufs_[side].size(); ++r) {
            std::int64_t b[kNumBufs];
            buffer_sizes(P, side, static_cast<int>(r), cfg_.with_grads, b);
            for (int k = 0; k < kNumBufs; ++k)
                if (b[k] != bufs_[side][r].bytes[k]) throw ConfigError("set_plan: buffer geometry differs");
        }
    P_ = &P;
    bcast_.clear();
    bcast_ready_ = false;
    prepared_ = false;
}

void Executor::set_stage_order(const std::vector<int>& order, const std::vector<int>& cuts) {
    const int nd = P_->dst_cfg.world_size();
    if (order.empty()) {
        stage_of_dst_.clear();
        stage_bands_ = 1;
        return;
    }
    // units = (destination rank, layer band): order lists every unit once (arena.hpp UnitMap)
    if (order.size() % static_cast<size_t>(nd)) throw ConfigError("stage order must list every unit once");
    const int nb = static_cast<int>(order.size()) / nd;
    if (!cuts.empty() && cuts.size() != order.size()) throw ConfigError("stage cuts must match the stage order");
    std::vector<int> pos(order.size(), -1);
    int group = -1;
    for (size_t s = 0; s < order.size(); ++s) {
        const int u = order[s];
        if (u < 0 || u >= static_cast<int>(order.size()) || pos[static_cast<size_t>(u)] >= 0)
            throw ConfigError("bad stage order");
        // without cuts every position is its own stage; with cuts, positions between two
        // cuts share one stage (they may run concurrently)
        if (cuts.empty() || s == 0 || cuts[s]) ++group;
        pos[static_cast<size_t>(u)] = group;
    }
    stage_of_dst_ = pos;
    stage_bands_ = nb;
    prepared_ = false;
}

int Executor::stage_of(const CopyOp& op) const {
    if (stage_of_dst_.empty()) return 0;
    int band = 0;
    if (stage_bands_ > 1 && op.tensor >= 0) {
        const int L = std::max(1, P_->space->num_layers());
        const int nb = std::min(stage_bands_, L);
        band = P_->space->entries()[static_cast<size_t>(op.tensor)].spec.layer * nb / L;
    }
    return stage_of_dst_[static_cast<size_t>(op.dst_rank * stage_bands_ + band)];
}

void Executor::alloc() {
    RS_CUDA(cudaSetDevice(cfg_.device));
    for (int side = 0; side < 2; ++side)
        for (RankBufs& rb : bufs_[side]) {
            if (rb.gpu != cfg_.gpu) continue;
            for (int b = 0; b < kNumBufs; ++b) {
                if (rb.ptr[b] || rb.bytes[b] == 0) continue;
                void* p = nullptr;
                RS_CUDA(cudaMalloc(&p, static_cast<size_t>(rb.bytes[b])));
                owned_.push_back(p);
                rb.ptr[b] = p;
            }
        }
}

void Executor::bind(int side, int rank, int buf, void* ptr, std::int64_t bytes) {
    if (side < 0 || side > 1 || rank < 0 || rank >= static_cast<int>(bufs_[side].size()) || buf < 0 || buf >= kNumBufs)
        throw ConfigError("bind: bad buffer id");
    RankBufs& rb = bufs_[side][static_cast<size_t>(rank)];
    if (bytes < rb.bytes[buf]) throw ConfigError(strfmt("bind: buffer too small (%lld < %lld)",
                                                         static_cast<long long>(bytes), static_cast<long long>(rb.bytes[buf])));
    rb.ptr[buf] = ptr;
}

void* Executor::buffer(int side, int rank, int buf, std::int64_t* bytes) const {
    const RankBufs& rb = bufs_[side][static_cast<size_t>(rank)];
    *bytes = rb.bytes[buf];
    return rb.ptr[buf];
}

std::vector<std::uint8_t> Executor::export_ipc() const {
    // [int32 count] then per local buffer: int32 rank, int32 buf | (source side << 8),
    // int64 offset, handle. Destination buffers always (peers push into them); source
    // buffers too when collectives are on (a Gather's root pulls from them)
    std::vector<std::uint8_t> out(4, 0);
    int count = 0;
    for (int side = 1; side >= (collectives_ ? 0 : 1); --side)
    for (size_t r = 0; r < bufs_[side].size(); ++r) {
        const RankBufs& rb = bufs_[side][r];
        if (rb.gpu != cfg_.gpu) continue;
        for (int b = 0; b < kNumBufs; ++b) {
            if (!rb.ptr[b]) continue;
            CUdeviceptr base = 0;
            size_t size = 0;
            if (mem_get_address_range(&base, &size, reinterpret_cast<CUdeviceptr>(rb.ptr[b])) != CUDA_SUCCESS)
                throw CudaError("cuMemGetAddressRange failed");
            cudaIpcMemHandle_t h;
            RS_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
            const std::int32_t rr = static_cast<std::int32_t>(r), bb = b | (side == 0 ? 1 << 8 : 0);
            const std::int64_t off = static_cast<std::int64_t>(reinterpret_cast<CUdeviceptr>(rb.ptr[b]) - base);
            const size_t at = out.size();
            out.resize(at + 16 + sizeof h);
            std::memcpy(out.data() + at, &rr, 4);
            std::memcpy(out.data() + at + 4, &bb, 4);
            std::memcpy(out.data() + at + 8, &off, 8);
            std::memcpy(out.data() + at + 16, &h, sizeof h);
            ++count;
        }
    }
    std::memcpy(out.data(), &count, 4);
    return out;
}

void Executor::import_ipc(const std::uint8_t* blob, size_t len) {
    RS_CUDA(cudaSetDevice(cfg_.device));
    if (len < 4) throw ConfigError("ipc blob too short");
    int count;
    std::memcpy(&count, blob, 4);
    size_t at = 4;
    for (int i = 0; i < count; ++i) {
        if (at + 16 + sizeof(cudaIpcMemHandle_t) > len) throw ConfigError("ipc blob truncated");
        std::int32_t r, b;
        std::int64_t off;
        cudaIpcMemHandle_t h;
        std::memcpy(&r, blob + at, 4);
        std::memcpy(&b, blob + at + 4, 4);
        std::memcpy(&off, blob + at + 8, 8);
        std::memcpy(&h, blob + at + 16, sizeof h);
        at += 16 + sizeof h;
        const int side = (b >> 8) & 1 ? 0 : 1;
        b &= 0xff;
        if (b < 0 || b >= kNumBufs) throw ConfigError("ipc blob: bad buffer id");
        RankBufs& rb = bufs_[side].at(static_cast<size_t>(r));
        if (rb.gpu == cfg_.gpu) continue;
        void* base = nullptr;
        auto key = std::string(reinterpret_cast<const char*>(&h), sizeof h);
        auto it = ipc_map_.find(key);
        if (it == ipc_map_.end()) {
            RS_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
            ipc_opened_.push_back(base);
            ipc_map_.emplace(key, base);
        } else {
            base = it->second;
        }
        rb.ptr[b] = static_cast<char*>(base) + off;
    }
}

/// The descriptor cut on the GPU: one thread per recorded copy writes its tiles at the
/// per-(record, alignment class) offsets the host derived from the tile counts.
__global__ void cut_kernel(const CopyRec* __restrict__ recs, const std::int32_t* __restrict__ pos, int n,
                           Tile* __restrict__ out) {
    const int i = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    const std::int32_t* p = pos + 5 * static_cast<size_t>(i);
    int c[5] = {0, 0, 0, 0, 0};
    auto emit = [&](int b, const Tile& t) {
        const int cls = b % 5;
        out[p[cls] + c[cls]++] = t;
    };
    cut_tiles(recs[i], emit);
}

void TileSet::add(int key, std::uint64_t src, std::uint64_t dst, std::int64_t rows, std::int64_t rb, std::int64_t sp,
                  std::int64_t dp, std::int64_t kTile, int lane) {
    // recorded here, cut into tiles by finalize() on host threads
    if (rows <= 0 || rb <= 0) return;
    pending.push_back(Pending{src, dst, rows, rb, sp, dp, kTile, key, lane});
}


void PinnedBuf::grow(size_t bytes) {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
    RS_CUDA(cudaHostAlloc(&ptr, bytes, cudaHostAllocDefault));
    cap = bytes;
}

PinnedBuf::~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
}

namespace {

// Reorder one launch group's tiles so every destination lane (peer GPU, or this GPU's
// HBM) progresses in proportion to its bytes: CTAs walk the tile list front to back, so
// in op order (sorted by destination rank) all senders would converge on the same
// receivers at the same time and leave other links idle.
/// Lane interleave straight into `out`: the tiles arrive as spans (a bucket's per-thread
/// pieces, in order) with their lanes; each step emits the next tile of the lane whose
/// progress fraction after that tile is smallest (lowest lane on ties). Lanes are few
/// (peers + local + pull sources), so a scan beats a heap.
void interleave_into(Tile* out, const std::vector<std::pair<const Tile*, const std::uint8_t*>>& spans,
                     const std::vector<size_t>& lens) {
    int nl = 0;
    size_t n = 0;
    for (size_t k = 0; k < spans.size(); ++k) {
        for (size_t i = 0; i < lens[k]; ++i) nl = std::max(nl, spans[k].second[i] + 1);
        n += lens[k];
    }
    std::vector<std::vector<const Tile*>> q(static_cast<size_t>(nl));
    std::vector<double> total(static_cast<size_t>(nl), 0.0), done(static_cast<size_t>(nl), 0.0);
    auto bytes = [](const Tile& t) { return static_cast<double>(t.rows) * t.row_bytes; };
    for (size_t k = 0; k < spans.size(); ++k)
        for (size_t i = 0; i < lens[k]; ++i) {
            const std::uint8_t l = spans[k].second[i];
            q[l].push_back(spans[k].first + i);
            total[l] += bytes(spans[k].first[i]);
        }
    std::vector<size_t> head(static_cast<size_t>(nl), 0);
    std::vector<double> key(static_cast<size_t>(nl), 0.0);
    auto refresh = [&](int l) {
        const size_t L = static_cast<size_t>(l);
        key[L] = head[L] < q[L].size() ? (done[L] + 0.5 * bytes(*q[L][head[L]])) / total[L] : 1e300;
    };
    for (int l = 0; l < nl; ++l) refresh(l);
    for (size_t o = 0; o < n; ++o) {
        int best = 0;
        for (int l = 1; l < nl; ++l)
            if (key[static_cast<size_t>(l)] < key[static_cast<size_t>(best)]) best = l;
        const size_t B = static_cast<size_t>(best);
        const Tile& t = *q[B][head[B]++];
        done[B] += bytes(t);
        out[o] = t;
        refresh(best);
    }
}

}  // namespace

void TileSet::finalize(ExecStats* stats, cudaStream_t upload, PinnedBuf* staging) {
    // Cut the recorded copies into tiles on host threads, straight into their final
    // places in the pinned staging buffer: pass 1 counts each thread's tiles per bucket
    // (key * 5 + alignment class), a prefix over (bucket, thread) fixes every thread's
    // write offsets, pass 2 writes. Contiguous record slices per thread, so the order is
    // the single-thread order. Buckets with several destination lanes are written to a
    // side array and interleaved into place.
    const auto t_fin0 = std::chrono::steady_clock::now();
    size_t nrec = pending.size();
    // Lane interleave at record granularity (default): within each key the recorded
    // copies are reordered so every destination lane progresses in proportion to its
    // bytes (the tile-level rule applied to whole copies: O(records x lanes), and the
    // tiles then need no reordering). RS_INTERLEAVE_TILES=1: the exact tile-level merge.
    static const bool tile_level = [] {
        const char* v = std::getenv("RS_INTERLEAVE_TILES");
        return v && std::string(v) == "1";
    }();
    bool lanes = false;  // several destination lanes at all (N>1)
    for (size_t i = 1; i < nrec && !lanes; ++i) lanes = pending[i].lane != pending[0].lane;
    if (interleave && !tile_level && lanes) {
        // split large copies at tile boundaries into pieces of ~kPieceTiles tiles (the
        // pieces cut into exactly the tiles of the whole copy), so a multi-GB copy to one
        // peer does not occupy every CTA for its whole length
        std::vector<Pending> split;
        split.reserve(nrec);
        for (const Pending& q0 : pending) split_rec(q0, 16, split);
        pending.swap(split);
        nrec = pending.size();
        std::vector<Pending> out;
        out.reserve(nrec);
        // records grouped by key, recorded order kept within a key (a counting sort: keys
        // are launch-group indices)
        int kmax = 0;
        for (const Pending& q0 : pending) kmax = std::max(kmax, q0.key);
        std::vector<size_t> idx(nrec), kstart(static_cast<size_t>(kmax) + 2, 0);
        for (const Pending& q0 : pending) ++kstart[static_cast<size_t>(q0.key) + 1];
        for (size_t k = 1; k < kstart.size(); ++k) kstart[k] += kstart[k - 1];
        for (size_t i = 0; i < nrec; ++i) idx[kstart[static_cast<size_t>(pending[i].key)]++] = i;
        for (size_t lo = 0; lo < nrec;) {
            size_t hi = lo;
            while (hi < nrec && pending[idx[hi]].key == pending[idx[lo]].key) ++hi;
            int nl = 0;
            for (size_t i = lo; i < hi; ++i) nl = std::max(nl, pending[idx[i]].lane + 1);
            std::vector<std::vector<size_t>> q(static_cast<size_t>(nl));
            std::vector<double> total(static_cast<size_t>(nl), 0.0), done(static_cast<size_t>(nl), 0.0);
            auto bytes = [&](size_t i) { return static_cast<double>(pending[i].rows) * static_cast<double>(pending[i].rb); };
            for (size_t i = lo; i < hi; ++i) {
                q[static_cast<size_t>(pending[idx[i]].lane)].push_back(idx[i]);
                total[static_cast<size_t>(pending[idx[i]].lane)] += bytes(idx[i]);
            }
            std::vector<size_t> head(static_cast<size_t>(nl), 0);
            // each lane's progress key (bytes done + half the next copy, over its total),
            // recomputed only for the lane that advanced; the first lane with the smallest
            // key goes next
            const double kDone = std::numeric_limits<double>::infinity();
            std::vector<double> key(static_cast<size_t>(nl), kDone);
            auto rekey = [&](size_t L) {
                if (head[L] >= q[L].size()) key[L] = kDone;
                else key[L] = total[L] > 0 ? (done[L] + 0.5 * bytes(q[L][head[L]])) / total[L] : 0.0;
            };
            for (size_t L = 0; L < static_cast<size_t>(nl); ++L) rekey(L);
            for (size_t k = lo; k < hi; ++k) {
                size_t B = 0;
                for (size_t L = 1; L < static_cast<size_t>(nl); ++L)
                    if (key[L] < key[B]) B = L;
                const size_t i = q[B][head[B]++];
                done[B] += bytes(i);
                rekey(B);
                out.push_back(pending[i]);
            }
            lo = hi;
        }
        pending.swap(out);
    }
    const size_t nt = std::max<size_t>(1, std::min<size_t>(pool::size(), nrec / 256 + 1));
    int max_key = -1;
    for (const Pending& q : pending) max_key = std::max(max_key, q.key);
    const size_t nb = static_cast<size_t>(max_key + 1) * 5;
    auto parallel = [&](auto&& fn) { pool::run(nt, fn); };
    gpu_cut = !(interleave && tile_level) && !host_tiles_forced();
    std::vector<size_t> begin(nb, 0), bucket_n(nb, 0);
    std::vector<std::array<std::int32_t, 5>> rc;  // GPU cut: tiles per (record, class)
    std::vector<std::vector<size_t>> cnt;         // host cut: tiles per (thread, bucket)
    std::vector<char> multi(nb, 0);
    groups.clear();
    size_t total = 0;
    if (gpu_cut) {
        rc.assign(nrec, {0, 0, 0, 0, 0});
        pool::parallel_for(nrec, [&](size_t i) { count_tiles(pending[i], rc[i].data()); });
        for (size_t i = 0; i < nrec; ++i)
            for (int c = 0; c < 5; ++c) bucket_n[static_cast<size_t>(pending[i].key) * 5 + c] += static_cast<size_t>(rc[i][c]);
    } else {
        cnt.assign(nt, std::vector<size_t>(nb, 0));
        std::vector<std::vector<std::uint8_t>> lane_mask(nt, std::vector<std::uint8_t>(nb, 0));  // bit 0: seen, 1: several
        std::vector<std::vector<std::uint8_t>> lane0(nt, std::vector<std::uint8_t>(nb, 0));
        parallel([&](size_t t) {
            for (size_t i = nrec * t / nt; i < nrec * (t + 1) / nt; ++i) {
                const Pending& q = pending[i];
                auto count = [&](int bi, const Tile&) {
                    const size_t b = static_cast<size_t>(bi);
                    ++cnt[t][b];
                    if (!(lane_mask[t][b] & 1)) lane_mask[t][b] = 1, lane0[t][b] = static_cast<std::uint8_t>(q.lane);
                    else if (lane0[t][b] != q.lane) lane_mask[t][b] |= 2;
                };
                cut_tiles(q, count);
            }
        });
        for (size_t b = 0; b < nb; ++b) {
            int l0 = -1;
            for (size_t t = 0; t < nt; ++t) {
                bucket_n[b] += cnt[t][b];
                if (!(lane_mask[t][b] & 1)) continue;
                if (lane_mask[t][b] & 2) multi[b] = 1;
                if (l0 < 0) l0 = lane0[t][b];
                else if (l0 != lane0[t][b]) multi[b] = 1;
            }
            if (!interleave || !tile_level) multi[b] = 0;
        }
    }
    const auto t_cut = std::chrono::steady_clock::now();
    for (size_t b = 0; b < nb; ++b) {
        begin[b] = total;
        if (!bucket_n[b]) continue;
        const int c = static_cast<int>(b % 5);
        groups.push_back({c, static_cast<int>(total), static_cast<int>(bucket_n[b]), static_cast<int>(b / 5)});
        if (stats) stats->tiles_by_class[c] += static_cast<std::int64_t>(bucket_n[b]);
        total += bucket_n[b];
    }
    (void)staging;
    const size_t host_bytes = gpu_cut ? nrec * (sizeof(CopyRec) + 5 * sizeof(std::int32_t)) : total * sizeof(Tile);
    Tile* out = nullptr;
    if (total) {
        // descriptors alternate between two slots (host pinned + device): this finalize
        // fills slot cur^1 while launches of the previous one may still read slot cur
        cur_buf_flip();
        PinnedBuf*& hb = hbuf[this->cur];
        if (!hb) hb = new PinnedBuf();
        for (cudaEvent_t e : hfences[this->cur]) {  // earlier uploads out of this pinned slot
            RS_CUDA(cudaEventSynchronize(e));
            fence_pool.push_back(e);
        }
        hfences[this->cur].clear();
        if (hb->size() < host_bytes) hb->grow(host_bytes * 5 / 4);
        out = static_cast<Tile*>(hb->ptr);
    }
    if (gpu_cut && total) {
        // records + per-(record, class) tile offsets: the GPU writes the tiles (cut_kernel)
        CopyRec* recs = static_cast<CopyRec*>(hbuf[this->cur]->ptr);
        std::int32_t* pos = reinterpret_cast<std::int32_t*>(recs + nrec);
        std::vector<size_t> run(begin);
        for (size_t i = 0; i < nrec; ++i) {
            recs[i] = pending[i];
            for (int c = 0; c < 5; ++c) {
                const size_t b = static_cast<size_t>(pending[i].key) * 5 + c;
                pos[5 * i + c] = static_cast<std::int32_t>(run[b]);
                run[b] += static_cast<size_t>(rc[i][c]);
            }
        }
        nrec_cut = nrec;
    } else if (total) {
        // side arrays of the multi-lane buckets (tiles + lanes, interleaved afterwards)
        std::vector<std::vector<Tile>> side_t(nb);
        std::vector<std::vector<std::uint8_t>> side_l(nb);
        for (size_t b = 0; b < nb; ++b)
            if (multi[b]) side_t[b].resize(bucket_n[b]), side_l[b].resize(bucket_n[b]);
        // per (thread, bucket) write cursor: the bucket's start + the earlier threads' counts
        std::vector<std::vector<size_t>> cur(nt, std::vector<size_t>(nb, 0));
        for (size_t b = 0; b < nb; ++b) {
            size_t at = multi[b] ? 0 : begin[b];
            for (size_t t = 0; t < nt; ++t) cur[t][b] = at, at += cnt[t][b];
        }
        parallel([&](size_t t) {
            std::vector<size_t>& c = cur[t];
            for (size_t i = nrec * t / nt; i < nrec * (t + 1) / nt; ++i) {
                const Pending& q = pending[i];
                auto write = [&](int bi, const Tile& tile) {
                    const size_t b = static_cast<size_t>(bi);
                    if (multi[b]) {
                        side_l[b][c[b]] = static_cast<std::uint8_t>(q.lane);
                        side_t[b][c[b]++] = tile;
                    } else {
                        out[c[b]++] = tile;
                    }
                };
                cut_tiles(q, write);
            }
        });
        std::vector<size_t> mb;
        for (size_t b = 0; b < nb; ++b)
            if (multi[b] && bucket_n[b]) mb.push_back(b);
        pool::run(mb.size(), [&](size_t k) {
            const size_t b = mb[k];
            const std::vector<std::pair<const Tile*, const std::uint8_t*>> spans{{side_t[b].data(), side_l[b].data()}};
            interleave_into(out + begin[b], spans, {bucket_n[b]});
        });
    }
    pending.clear();
    const auto t_asm = std::chrono::steady_clock::now();
    if (total) {
        // two device descriptor buffers used in turn; both are kept across re-prepares:
        // with peer access enabled every cudaMalloc/cudaFree also edits the peers'
        // mappings (measured: 0.6 s stalls)
        if (total * sizeof(Tile) > dev_bytes[this->cur]) {
            if (dev_buf[this->cur]) cudaFree(dev_buf[this->cur]);
            dev_buf[this->cur] = nullptr;
            dev_bytes[this->cur] = total * sizeof(Tile) * 5 / 4;
            RS_CUDA(cudaMalloc(&dev_buf[this->cur], dev_bytes[this->cur]));
        }
        // the first upload into dev_buf[cur] follows every launch that read it
        for (cudaEvent_t e : wait_first) fence_pool.push_back(e);
        wait_first = std::move(fences[this->cur]);
        fences[this->cur].clear();
        dev = dev_buf[this->cur];
        if (gpu_cut && host_bytes > rec_bytes[this->cur]) {
            if (dev_rec[this->cur]) cudaFree(dev_rec[this->cur]);
            dev_rec[this->cur] = nullptr;
            rec_bytes[this->cur] = host_bytes * 5 / 4;
            RS_CUDA(cudaMalloc(&dev_rec[this->cur], rec_bytes[this->cur]));
        }
        uploaded.assign(groups.size(), 0);
        materialized = false;
    } else {
        uploaded.clear();
        materialized = true;
    }
    (void)upload;
    ntiles = total;
    if (std::getenv("RS_TIMING") && total > 4096) {
        const auto t_up = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[reshard] finalize (%s cut): count %.2f ms (%zu threads), write %.2f ms, rest %.2f ms\n",
                     gpu_cut ? "GPU" : "host",
                     std::chrono::duration<double, std::milli>(t_cut - t_fin0).count(), nt,
                     std::chrono::duration<double, std::milli>(t_asm - t_cut).count(),
                     std::chrono::duration<double, std::milli>(t_up - t_asm).count());
    }
    if (stats) {
        stats->tiles += static_cast<std::int64_t>(total);
        stats->launches += static_cast<std::int64_t>(groups.size());
    }
}

TileSet::~TileSet() {
    for (auto& v : hfences)
        for (cudaEvent_t e : v) cudaEventSynchronize(e), cudaEventDestroy(e);
    for (cudaEvent_t e : wait_first) cudaEventDestroy(e);
    for (PinnedBuf* b : hbuf) delete b;
    for (void* p : dev_buf)
        if (p) cudaFree(p);
    for (void* p : dev_rec)
        if (p) cudaFree(p);
    if (mat_ev) cudaEventDestroy(mat_ev);
    for (auto& v : fences)
        for (cudaEvent_t e : v) cudaEventDestroy(e);
    for (cudaEvent_t e : fence_pool) cudaEventDestroy(e);
}

cudaEvent_t TileSet::take_event() const {
    cudaEvent_t e = nullptr;
    if (!fence_pool.empty()) {
        e = fence_pool.back();
        fence_pool.pop_back();
    } else {
        RS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return e;
}

void TileSet::materialize(cudaStream_t stream) const {
    if (materialized) return;
    for (cudaEvent_t e : wait_first) {
        RS_CUDA(cudaStreamWaitEvent(stream, e, 0));
        fence_pool.push_back(e);
    }
    wait_first.clear();
    const size_t bytes = nrec_cut * (sizeof(CopyRec) + 5 * sizeof(std::int32_t));
    RS_CUDA(cudaMemcpyAsync(dev_rec[cur], hbuf[cur]->ptr, bytes, cudaMemcpyHostToDevice, stream));
    cudaEvent_t e = take_event();
    RS_CUDA(cudaEventRecord(e, stream));
    hfences[cur].push_back(e);
    const CopyRec* recs = static_cast<const CopyRec*>(dev_rec[cur]);
    const std::int32_t* pos = reinterpret_cast<const std::int32_t*>(recs + nrec_cut);
    const int n = static_cast<int>(nrec_cut);
    cut_kernel<<<(n + 127) / 128, 128, 0, stream>>>(recs, pos, n, static_cast<Tile*>(dev));
    RS_CUDA(cudaGetLastError());
    materialized = true;
    if (!mat_ev) RS_CUDA(cudaEventCreateWithFlags(&mat_ev, cudaEventDisableTiming));
    RS_CUDA(cudaEventRecord(mat_ev, stream));
    mat_stream = stream;
}

void TileSet::order_after_upload(cudaStream_t stream) const {
    // descriptors written on another stream: this launch follows them
    if (mat_ev && stream != mat_stream) RS_CUDA(cudaStreamWaitEvent(stream, mat_ev, 0));
}

void TileSet::upload_group(size_t gi, cudaStream_t stream) const {
    if (gpu_cut) {
        if (!materialized) materialize(stream);
        else order_after_upload(stream);
        return;
    }
    if (gi >= uploaded.size() || uploaded[gi]) {
        order_after_upload(stream);
        return;
    }
    for (cudaEvent_t e : wait_first) {
        RS_CUDA(cudaStreamWaitEvent(stream, e, 0));
        fence_pool.push_back(e);
    }
    wait_first.clear();
    const Group& g = groups[gi];
    const Tile* src = static_cast<const Tile*>(hbuf[cur]->ptr) + g.begin;
    RS_CUDA(cudaMemcpyAsync(static_cast<Tile*>(dev) + g.begin, src, static_cast<size_t>(g.count) * sizeof(Tile),
                            cudaMemcpyHostToDevice, stream));
    cudaEvent_t e = take_event();
    RS_CUDA(cudaEventRecord(e, stream));
    hfences[cur].push_back(e);
    uploaded[gi] = 1;
    // later launches on other streams follow every upload done so far on this one
    if (mat_stream && mat_stream != stream) order_after_upload(stream);
    if (!mat_ev) RS_CUDA(cudaEventCreateWithFlags(&mat_ev, cudaEventDisableTiming));
    RS_CUDA(cudaEventRecord(mat_ev, stream));
    mat_stream = stream;
}

void TileSet::flush_uploads(cudaStream_t stream) const {
    if (gpu_cut) {
        materialize(stream);
        return;
    }
    for (size_t gi = 0; gi < uploaded.size(); ++gi) upload_group(gi, stream);
}

void TileSet::fence(cudaStream_t stream) const {
    if (!dev) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    RS_CUDA(cudaStreamIsCapturing(stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) return;
    cudaEvent_t e = nullptr;
    if (!fence_pool.empty()) {
        e = fence_pool.back();
        fence_pool.pop_back();
    } else {
        RS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    RS_CUDA(cudaEventRecord(e, stream));
    fences[cur].push_back(e);
    // bound the list: one event per stream suffices once a later record on the same
    // stream exists, but streams are opaque here, so collapse long lists by waiting
    if (fences[cur].size() > 64) {
        for (size_t i = 0; i + 1 < fences[cur].size(); ++i) {
            RS_CUDA(cudaEventSynchronize(fences[cur][i]));
            fence_pool.push_back(fences[cur][i]);
        }
        fences[cur].erase(fences[cur].begin(), fences[cur].end() - 1);
    }
}

namespace {

/// resident CTAs per SM of a copy kernel (cached): the persistent grid never asks for
/// more CTAs than can be resident at once, so no CTA waits for a whole wave to finish
template <class K>
int resident_ctas(K kernel) {
    static std::mutex mu;
    static std::map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    const void* key = reinterpret_cast<const void*>(kernel);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1) b = 1;
    cache[key] = b;
    return b;
}

bool vec32_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("RS_VEC32");
        return !(v && std::string(v) == "0");
    }();
    return on;
}

}  // namespace

int TileSet::launch(cudaStream_t stream, std::uint64_t sbase, std::uint64_t dbase, int sms, int ctas_per_sm,
                    bool bulk, int key_mod, int key_rem) const {
    int launches = 0;
    const int want = ctas_per_sm > 0 ? ctas_per_sm : 4;
    const Tile* base = static_cast<const Tile*>(dev);
    const bool w32 = vec32_enabled();
    auto grid_of = [&](auto kernel, int n) { return std::min(n, sms * std::min(want, resident_ctas(kernel))); };
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        const Group& g = groups[gi];
        if (key_mod > 0 && g.key % key_mod != key_rem) continue;
        if (key_mod < 0 && g.key != key_rem) continue;  // exact key (one memory-aware stage)
        upload_group(gi, stream);  // first launch after a finalize: this group's descriptors
        const int n = g.count;
        const Tile* t = base + g.begin;
        switch (g.cls) {
            case 0:
                if (bulk) {
                    const int g2 = std::min(n, sms * kBulkCtasPerSm);
                    bulk_tiles_kernel<kBulkStages, kBulkStage><<<g2, 32, kBulkStages * kBulkStage, stream>>>(t, n, sbase, dbase);
                } else if (w32) {
                    auto k = copy_tiles_kernel<16, false, true>;
                    k<<<grid_of(k, n), kThreads, 0, stream>>>(t, n, sbase, dbase);
                } else {
                    auto k = copy_tiles_kernel<16>;
                    k<<<grid_of(k, n), kThreads, 0, stream>>>(t, n, sbase, dbase);
                }
                break;
            case 1: copy_tiles_kernel<8><<<grid_of(copy_tiles_kernel<8>, n), kThreads, 0, stream>>>(t, n, sbase, dbase); break;
            case 2: copy_tiles_kernel<4><<<grid_of(copy_tiles_kernel<4>, n), kThreads, 0, stream>>>(t, n, sbase, dbase); break;
            case 3: copy_tiles_kernel<2><<<grid_of(copy_tiles_kernel<2>, n), kThreads, 0, stream>>>(t, n, sbase, dbase); break;
            default: copy_tiles_kernel<1><<<grid_of(copy_tiles_kernel<1>, n), kThreads, 0, stream>>>(t, n, sbase, dbase); break;
        }
        ++launches;
    }
    RS_CUDA(cudaGetLastError());
    if (launches) fence(stream);
    return launches;
}

void Executor::compute_dups(const std::vector<CopyOp>& ops) {
    // replica dedup: peer-bound ops that bring the same source region to several
    // destination ranks on ONE GPU, at identical destination geometry (DP replicas), cross
    // NVLink once — to the lowest such rank (the primary) — and the others are copied from
    // it on the destination GPU after a cross-GPU barrier (run_dup)
    dup_primary_.assign(ops.size(), -1);
    dup_lead_.assign(ops.size(), 0);
    if (!dedup_) return;
    using Key = std::tuple<int, int, std::int64_t, std::int64_t, std::int64_t, std::int64_t, int, int, std::int64_t,
                           std::int64_t>;
    std::map<Key, std::vector<size_t>> groups;
    for (size_t i = 0; i < ops.size(); ++i) {
        const CopyOp& op = ops[i];
        if (op.rows <= 0 || op.row_bytes <= 0) continue;
        const int sg = bufs_[0][static_cast<size_t>(op.src_side_rank)].gpu, dg = bufs_[1][static_cast<size_t>(op.dst_rank)].gpu;
        if (sg == dg) continue;
        groups[Key{op.src_side_rank, op.src_buf, op.src_off, op.rows, op.row_bytes, op.rows > 1 ? op.src_pitch : 0, dg,
                   op.dst_buf, op.dst_off, op.rows > 1 ? op.dst_pitch : 0}]
            .push_back(i);
    }
    for (auto& kv : groups) {
        auto& v = kv.second;
        if (v.size() < 2) continue;
        std::sort(v.begin(), v.end(), [&](size_t a, size_t b) { return ops[a].dst_rank < ops[b].dst_rank; });
        for (size_t k = 1; k < v.size(); ++k) dup_primary_[v[k]] = ops[v[0]].dst_rank;
        dup_lead_[v[0]] = 1;
    }
}

void Executor::set_replica_dedup(bool on, bool early) {
    dedup_ = on;
    dup_early_ = on && early;
    bcast_ready_ = false;
    mc_va_.clear();
    prepared_ = false;
}

const std::vector<BcastGroup>& Executor::bcast_groups() {
    if (bcast_ready_) return bcast_;
    bcast_.clear();
    const std::vector<CopyOp> ops = build_ops(*P_);
    compute_dups(ops);
    // candidate ops: cross-GPU, destination at the source's own offset in an equally
    // sized buffer (replica layout), 16-B aligned (multimem.st.v4)
    using Key = std::tuple<int, int, std::int64_t, std::int64_t, std::int64_t, std::int64_t>;
    std::map<Key, std::vector<size_t>> by_src;
    for (size_t i = 0; i < ops.size(); ++i) {
        const CopyOp& op = ops[i];
        if (op.rows <= 0 || op.row_bytes <= 0 || dup_primary_[i] >= 0) continue;  // dups never cross NVLink
        const RankBufs& S = bufs_[0][static_cast<size_t>(op.src_side_rank)];
        const RankBufs& D = bufs_[1][static_cast<size_t>(op.dst_rank)];
        if (S.gpu == D.gpu || op.dst_buf != op.src_buf || op.dst_off != op.src_off) continue;
        if (op.rows > 1 && op.dst_pitch != op.src_pitch) continue;
        if ((op.src_off | op.row_bytes | (op.rows > 1 ? op.src_pitch : 0)) % 16 != 0) continue;
        if (S.bytes[op.src_buf] != D.bytes[op.dst_buf]) continue;
        by_src[Key{op.src_side_rank, op.src_buf, op.src_off, op.rows, op.row_bytes, op.rows > 1 ? op.src_pitch : 0}].push_back(i);
    }
    std::map<std::tuple<int, int, int, std::vector<int>>, size_t> index;
    for (const auto& kv : by_src) {
        std::map<int, std::vector<size_t>> per_gpu;  // destination GPU -> ops by dst rank
        for (size_t i : kv.second) per_gpu[bufs_[1][static_cast<size_t>(ops[i].dst_rank)].gpu].push_back(i);
        if (per_gpu.size() < 2) continue;
        size_t slots = 0;
        for (auto& g : per_gpu) {
            std::sort(g.second.begin(), g.second.end(), [&](size_t a, size_t b) { return ops[a].dst_rank < ops[b].dst_rank; });
            slots = std::max(slots, g.second.size());
        }
        const int root = std::get<0>(kv.first), buf = std::get<1>(kv.first);
        for (size_t sl = 0; sl < slots; ++sl) {
            std::vector<int> ranks, gpus;
            std::vector<size_t> sel;
            for (const auto& g : per_gpu)
                if (sl < g.second.size()) {
                    ranks.push_back(ops[g.second[sl]].dst_rank);
                    gpus.push_back(g.first);
                    sel.push_back(g.second[sl]);
                }
            if (ranks.size() < 2) continue;  // a single destination left: plain push
            const auto key = std::make_tuple(root, buf, static_cast<int>(sl), ranks);
            auto it = index.find(key);
            if (it == index.end()) {
                BcastGroup g;
                g.id = static_cast<int>(bcast_.size());
                g.root_rank = root;
                g.root_gpu = bufs_[0][static_cast<size_t>(root)].gpu;
                g.buf = buf;
                g.slot = static_cast<int>(sl);
                g.member_gpus = gpus;
                g.member_ranks = ranks;
                g.buffer_bytes = bufs_[0][static_cast<size_t>(root)].bytes[buf];
                it = index.emplace(key, bcast_.size()).first;
                bcast_.push_back(std::move(g));
            }
            BcastGroup& g = bcast_[it->second];
            const CopyOp& lead = ops[sel[0]];
            g.payload_bytes += lead.rows * lead.row_bytes;
            g.ops.insert(g.ops.end(), sel.begin(), sel.end());
        }
    }
    bcast_ready_ = true;
    return bcast_;
}

void Executor::set_multicast(int id, void* mc_va) {
    bcast_groups();
    if (id < 0 || id >= static_cast<int>(bcast_.size())) throw ConfigError("set_multicast: no such broadcast group");
    if (bcast_[static_cast<size_t>(id)].root_gpu != cfg_.gpu) throw ConfigError("set_multicast: this GPU is not the group's root");
    for (int s : stage_of_dst_)
        if (s != 0) throw ConfigError("set_multicast: needs a single-stage transition (multicast stores span stages)");
    if (mc_va) mc_va_[id] = mc_va;
    else mc_va_.erase(id);
    prepared_ = false;
}

void Executor::prepare(bool staged) {
    const pool::Warm warm;  // op build, tile counts and interleave: short loops back to back
    const auto t_begin = std::chrono::steady_clock::now();
    RS_CUDA(cudaSetDevice(cfg_.device));
    const char* sr = std::getenv("RS_SPLIT_REMOTE");
    split_remote_ = sr && std::string(sr) == "1";
    const std::vector<CopyOp> ops = build_ops(*P_);
    const auto t_ops = std::chrono::steady_clock::now();
    stats_ = ExecStats{};
    staged_ = staged;
    has_remote_ = false;
    ce_ops_.clear();
    const char* ce = std::getenv("RS_CE_MIN_BYTES");
    // off by default: measured slower than SM-only pushes (N=4: 56 ms vs 51 ms) because the
    // copy engines and the SM stores contend for the same links (profiles/r01_nvlink.md)
    ce_min_bytes_ = ce ? std::atoll(ce) : 0;
    channels_.clear();
    if (!fused_) fused_ = std::make_unique<TileSet>();  // reused: keeps its device buffer
    fused_->pending.clear();
    {
        const char* to = std::getenv("RS_TILE_ORDER");
        fused_->interleave = !(to && std::string(to) == "op");
    }
    // tile size: 512 KiB, unless the transition is too small to give every SM a few tiles
    // (then latency-bound: smaller tiles, down to one 32 KiB bulk stage, spread it out)
    std::int64_t kTile = cfg_.tile_bytes > 0 ? cfg_.tile_bytes : (512 << 10);
    std::int64_t here = 0;  // bytes this GPU moves
    bool pushes = false;    // any of them bound for a peer GPU
    for (const CopyOp& op : ops)
        if (bufs_[0][static_cast<size_t>(op.src_side_rank)].gpu == cfg_.gpu) {
            here += op.rows * op.row_bytes;
            pushes = pushes || bufs_[1][static_cast<size_t>(op.dst_rank)].gpu != cfg_.gpu;
        }
    // peer pushes: 256 KiB tiles spread the lanes finer (measured +0.6 % of NVLink rate at
    // N=2, tools/runs/r02_push_sweep.sh); local copies keep 512 KiB
    if (cfg_.tile_bytes <= 0 && pushes) kTile = 256 << 10;
    if (cfg_.tile_bytes <= 0) {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg_.device);
        const std::int64_t want = here / (static_cast<std::int64_t>(nsm) * 4);
        if (want < kTile) kTile = std::max<std::int64_t>(32 << 10, want / 16 * 16);
    }
    if (!mc_) mc_ = std::make_unique<TileSet>();
    if (!dup_) dup_ = std::make_unique<TileSet>();
    dup_->pending.clear();
    compute_dups(ops);
    // promoted collectives (optimize_primitives over the plan's box transfers, the
    // schedule's own rule): Scatter ops are pushed by the root as usual, Gather ops are
    // pulled by the root from the sources' mapped buffers
    box_coll_.clear();
    if (collectives_ && !staged) {
        std::vector<std::int64_t> residual;
        const std::vector<sched::Fragment> frags = sched::plan_fragments(*P_, {});
        box_coll_.assign(P_->box.size(), 0);
        for (const sched::CommOp& c : sched::optimize_primitives(*P_, frags, &residual, true))
            if (c.kind == sched::CommKind::Scatter || c.kind == sched::CommKind::Gather)
                for (std::int64_t f : c.frags) box_coll_[static_cast<size_t>(f)] = static_cast<std::int8_t>(c.kind);
    }
    // early dedup: launch 1 is a tail of this GPU's other peer pushes, long enough to hide the
    // replica copies (HBM, ~4.5x the NVLink push rate; RS_DUP_TAIL_FRAC, default 0.4 of the
    // largest per-GPU replica bytes); everything else, the primaries first, is launch 0
    std::vector<char> tail(ops.size(), 0);
    if (dup_early_ && !staged) {
        std::map<int, std::int64_t> dup_bytes;
        for (size_t oi = 0; oi < ops.size(); ++oi)
            if (dup_primary_[oi] >= 0)
                dup_bytes[bufs_[1][static_cast<size_t>(ops[oi].dst_rank)].gpu] += ops[oi].rows * ops[oi].row_bytes;
        std::int64_t dmax = 0;
        for (const auto& kv : dup_bytes) dmax = std::max(dmax, kv.second);
        double frac = 0.4;
        if (const char* f = std::getenv("RS_DUP_TAIL_FRAC")) frac = std::atof(f);
        std::int64_t budget = static_cast<std::int64_t>(static_cast<double>(dmax) * frac);
        for (size_t oi = ops.size(); oi-- > 0 && budget > 0;) {
            const CopyOp& op = ops[oi];
            if (op.rows <= 0 || op.row_bytes <= 0 || dup_lead_[oi] || dup_primary_[oi] >= 0) continue;
            // peer-bound only: local HBM copies would finish long before the replica copies
            if (bufs_[0][static_cast<size_t>(op.src_side_rank)].gpu != cfg_.gpu ||
                bufs_[1][static_cast<size_t>(op.dst_rank)].gpu == cfg_.gpu)
                continue;
            tail[oi] = 1;
            budget -= op.rows * op.row_bytes;
        }
    }
    mc_src_bytes_ = 0;
    mc_->pending.clear();
    // ops delivered by a multicast store stream: -1 no, else the multicast address; the
    // first op of each source region (lead) emits the tiles, the other members' copies ride along
    std::vector<std::uint64_t> op_mc(ops.size(), 0);
    std::vector<char> op_lead(ops.size(), 0);
    std::vector<int> op_mc_group(ops.size(), 0);  // one launch per multicast object
    if (!staged && !mc_va_.empty()) {
        bcast_groups();
        for (const auto& kv : mc_va_) {
            const BcastGroup& g = bcast_[static_cast<size_t>(kv.first)];
            const size_t members = g.member_ranks.size();
            for (size_t k = 0; k < g.ops.size(); ++k) {
                op_mc[g.ops[k]] = reinterpret_cast<std::uint64_t>(kv.second);
                op_mc_group[g.ops[k]] = kv.first;
                op_lead[g.ops[k]] = (k % members) == 0;
            }
        }
    }
    std::map<std::pair<int, int>, std::int64_t> chan_off;
    for (size_t oi = 0; oi < ops.size(); ++oi) {
        const CopyOp& op = ops[oi];
        const RankBufs& S = bufs_[0][static_cast<size_t>(op.src_side_rank)];
        const RankBufs& D = bufs_[1][static_cast<size_t>(op.dst_rank)];
        if (op.rows <= 0 || op.row_bytes <= 0) continue;
        const bool src_here = S.gpu == cfg_.gpu, dst_here = D.gpu == cfg_.gpu;
        const std::int64_t total = op.rows * op.row_bytes;
        if (staged && S.gpu != D.gpu) {
            // channel between physical devices: ops packed densely in build_ops order,
            // so sender and receiver derive identical offsets without metadata
            const int sp = P_->wm.src_phys[static_cast<size_t>(op.src_side_rank)];
            const int dpp = P_->wm.dst_phys[static_cast<size_t>(op.dst_rank)];
            const auto key = std::make_pair(sp, dpp);
            std::int64_t& off = chan_off[key];
            Channel& ch = channels_[key];
            if (!ch.pack) ch.pack = std::make_unique<TileSet>(), ch.unpack = std::make_unique<TileSet>();
            if (src_here) {
                if (!S.ptr[op.src_buf]) throw ConfigError("prepare: source buffer not bound");
                ch.pack->add(0, reinterpret_cast<std::uint64_t>(S.ptr[op.src_buf]) + static_cast<std::uint64_t>(op.src_off),
                             static_cast<std::uint64_t>(off), op.rows, op.row_bytes, op.src_pitch, op.row_bytes, kTile);
                stats_.remote_bytes += total;
            }
            if (dst_here) {
                if (!D.ptr[op.dst_buf]) throw ConfigError("prepare: destination buffer not bound");
                ch.unpack->add(0, static_cast<std::uint64_t>(off),
                               reinterpret_cast<std::uint64_t>(D.ptr[op.dst_buf]) + static_cast<std::uint64_t>(op.dst_off),
                               op.rows, op.row_bytes, op.row_bytes, op.dst_pitch, kTile);
            }
            off += total;
            ch.bytes = off;
            ch.op_bytes.push_back(total);
            continue;
        }
        if (!staged && dup_primary_[oi] >= 0) {
            // a replica of a region the primary rank on this destination GPU receives:
            // copied there after the cross-GPU barrier (run_dup), never pushed
            if (dst_here) {
                const RankBufs& D0 = bufs_[1][static_cast<size_t>(dup_primary_[oi])];
                if (!D0.ptr[op.dst_buf] || !D.ptr[op.dst_buf]) throw ConfigError("prepare: replica buffer not bound");
                dup_->add(0, reinterpret_cast<std::uint64_t>(D0.ptr[op.dst_buf]) + static_cast<std::uint64_t>(op.dst_off),
                          reinterpret_cast<std::uint64_t>(D.ptr[op.dst_buf]) + static_cast<std::uint64_t>(op.dst_off), op.rows,
                          op.row_bytes, op.dst_pitch, op.dst_pitch, kTile);
                stats_.local_bytes += total;
                stats_.dup_bytes += total;
            }
            continue;
        }
        const int coll = (!box_coll_.empty() && op.box >= 0) ? box_coll_[static_cast<size_t>(op.box)] : 0;
        if (coll == static_cast<int>(sched::CommKind::Gather) && !staged && S.gpu != D.gpu) {
            // Gather: the root (destination GPU) pulls every source's slice over NVLink
            if (!dst_here) continue;
            if (!S.ptr[op.src_buf] || !D.ptr[op.dst_buf])
                throw ConfigError(strfmt("gather pull: source rank %d buffer %d not mapped here (set_collectives on every "
                                         "rank before the ipc exchange)", op.src_side_rank, op.src_buf));
            stats_.gather_bytes += total;
            has_remote_ = true;
            fused_->add(stage_of(op), reinterpret_cast<std::uint64_t>(S.ptr[op.src_buf]) + static_cast<std::uint64_t>(op.src_off),
                        reinterpret_cast<std::uint64_t>(D.ptr[op.dst_buf]) + static_cast<std::uint64_t>(op.dst_off), op.rows,
                        op.row_bytes, op.src_pitch, op.dst_pitch, kTile, cfg_.n_gpus + S.gpu);
            continue;
        }
        if (!src_here) continue;  // pushed by the source's GPU
        if (coll == static_cast<int>(sched::CommKind::Scatter) && !dst_here) stats_.scatter_bytes += total;
        if (op_mc[oi]) {
            if (!S.ptr[op.src_buf]) throw ConfigError("prepare: multicast source buffer not bound");
            if (op_lead[oi]) mc_src_bytes_ += total;
            if (op_lead[oi])
                mc_->add(op_mc_group[oi], reinterpret_cast<std::uint64_t>(S.ptr[op.src_buf]) + static_cast<std::uint64_t>(op.src_off),
                         op_mc[oi] + static_cast<std::uint64_t>(op.dst_off), op.rows, op.row_bytes, op.src_pitch, op.dst_pitch,
                         kTile);
            stats_.remote_bytes += total;
            stats_.mc_bytes += total;
            has_remote_ = true;
            continue;
        }
        if (!S.ptr[op.src_buf] || !D.ptr[op.dst_buf])
            throw ConfigError(strfmt("prepare: buffer not bound (src rank %d buf %d -> dst rank %d buf %d)",
                                     op.src_side_rank, op.src_buf, op.dst_rank, op.dst_buf));
        (dst_here ? stats_.local_bytes : stats_.remote_bytes) += total;
        const int stage = stage_of(op);
        if (!dst_here) has_remote_ = true;
        const bool contiguous = op.rows == 1 || (op.src_pitch == op.row_bytes && op.dst_pitch == op.row_bytes);
        if (!dst_here && ce_min_bytes_ > 0 && contiguous && total >= ce_min_bytes_) {
            // large contiguous peer-bound block: a copy engine moves it (778 GB/s both ways
            // vs ~710 for SM stores, profiles/r01_nvlink.md) concurrently with the kernel
            ce_ops_.push_back({reinterpret_cast<std::uint64_t>(S.ptr[op.src_buf]) + static_cast<std::uint64_t>(op.src_off),
                               reinterpret_cast<std::uint64_t>(D.ptr[op.dst_buf]) + static_cast<std::uint64_t>(op.dst_off),
                               total});
            stats_.ce_bytes += total;
            continue;
        }
        // key = stage * 2 + remote when split_remote_ (peer-bound tiles as their own launch on
        // the caller's stream, local HBM tiles on an aux stream); otherwise one mixed launch
        // early dedup: the primaries' tiles are in launch 0 (run_stage(0)), a tail of the
        // rest is launch 1, so run_dup can start after a barrier on launch 0 and overlap it
        if (dup_early_ && stage != 0) throw ConfigError("early replica dedup needs a single memory stage");
        const int key = split_remote_ ? stage * 2 + (dst_here ? 0 : 1) : dup_early_ ? (tail[oi] ? 1 : 0) : stage;
        fused_->add(key, reinterpret_cast<std::uint64_t>(S.ptr[op.src_buf]) + static_cast<std::uint64_t>(op.src_off),
                    reinterpret_cast<std::uint64_t>(D.ptr[op.dst_buf]) + static_cast<std::uint64_t>(op.dst_off), op.rows,
                    op.row_bytes, op.src_pitch, op.dst_pitch, kTile, D.gpu);
    }
    const auto t_tiles = std::chrono::steady_clock::now();
    if (!upload_) RS_CUDA(cudaStreamCreateWithFlags(&upload_, cudaStreamNonBlocking));
    fused_->finalize(&stats_, upload_, &staging_);
    mc_->finalize(&stats_, upload_, &staging_);
    dup_->finalize(&stats_, upload_, &staging_);
    for (const TileSet::Group& g : mc_->groups)
        if (g.cls != 0) throw ConfigError("prepare: multicast tiles must be 16-byte aligned");
    for (auto& kv : channels_) {
        kv.second.pack->finalize(nullptr, upload_, &staging_);
        kv.second.unpack->finalize(nullptr, upload_, &staging_);
    }
    if (std::getenv("RS_TIMING")) {
        const auto t_end = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[reshard] prepare: ops %.1f ms (%zu), tiles %.1f ms, finalize+upload %.1f ms, %lld tiles\n",
                     std::chrono::duration<double, std::milli>(t_ops - t_begin).count(), ops.size(),
                     std::chrono::duration<double, std::milli>(t_tiles - t_ops).count(),
                     std::chrono::duration<double, std::milli>(t_end - t_tiles).count(),
                     static_cast<long long>(stats_.tiles));
    }
    if (!d_counters_) RS_CUDA(cudaMalloc(&d_counters_, 64));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg_.device);
    sms_ = sms;
    const char* kern = std::getenv("RS_COPY_KERNEL");
    // the TMA bulk pipeline (one warp per SM) wins on large transitions (0.977 of the copy
    // peak); below ~1 GiB its per-SM pipeline ramp dominates and the 512-thread vector
    // kernel is ~2.8x faster (tiny GPT: 17 us vs 47 us for 27 MB, near the HBM roofline)
    use_bulk_ = kern ? std::string(kern) != "vector" : here >= (1ll << 30);
    const char* rk = std::getenv("RS_REMOTE_KERNEL");
    remote_bulk_ = rk && std::string(rk) == "bulk";
    const char* rc = std::getenv("RS_REMOTE_CTAS_PER_SM");
    remote_ctas_per_sm_ = rc ? std::atoi(rc) : 2;
    if (use_bulk_)
        RS_CUDA(cudaFuncSetAttribute(bulk_tiles_kernel<kBulkStages, kBulkStage>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kBulkStages * kBulkStage));
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);  // descriptors changed: recapture
    graph_exec_ = nullptr;
    {
        const char* gr = std::getenv("RS_GRAPH");
        auto_graph_ = !(gr && std::string(gr) == "0") && here < (1ll << 30) && !staged;
        runs_since_prepare_ = 0;
    }
    prepared_ = true;
}

int Executor::launch_multicast(cudaStream_t stream) const {
    if (!mc_ || mc_->groups.empty()) return 0;
    const Tile* base = static_cast<const Tile*>(mc_->dev);
    int n = 0;
    for (size_t gi = 0; gi < mc_->groups.size(); ++gi) {
        const TileSet::Group& g = mc_->groups[gi];
        mc_->upload_group(gi, stream);
        const char* mcc = std::getenv("RS_MC_CTAS_PER_SM");
        const int grid = std::min(g.count, sms_ * (mcc ? std::max(1, std::atoi(mcc)) : 1));
        copy_tiles_kernel<16, true><<<grid, kThreads, 0, stream>>>(base + g.begin, g.count, 0, 0);
        ++n;
    }
    RS_CUDA(cudaGetLastError());
    if (n) mc_->fence(stream);
    return n;
}

int Executor::run_graph(cudaStream_t stream) {
    // the whole launch sequence of run() as one CUDA graph: small transitions are
    // launch-bound (a few kernels of microseconds each); captured once per prepare()
    if (!prepared_) throw ConfigError("run before prepare");
    RS_CUDA(cudaSetDevice(cfg_.device));
    if (!graph_exec_ || graph_stream_ != stream) {
        if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
        // descriptors go up outside the capture (the graph replays kernels only)
        if (fused_) fused_->flush_uploads(stream);
        if (mc_) mc_->flush_uploads(stream);
        cudaGraph_t g = nullptr;
        RS_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        try {
            graph_launches_ = run_direct(stream);
        } catch (...) {
            cudaStreamEndCapture(stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        RS_CUDA(cudaStreamEndCapture(stream, &g));
        const cudaError_t e = cudaGraphInstantiate(&graph_exec_, g, 0);
        cudaGraphDestroy(g);
        RS_CUDA(e);
        graph_stream_ = stream;
    }
    RS_CUDA(cudaGraphLaunch(graph_exec_, stream));
    // descriptor fences for the graph's launches (skipped during capture)
    if (fused_) fused_->fence(stream);
    if (mc_) mc_->fence(stream);
    return graph_launches_;
}

int Executor::run(cudaStream_t stream) {
    if (!prepared_) throw ConfigError("run before prepare");
    // transitions under 1 GiB per GPU are launch-bound: replay them from a CUDA graph
    // (captured per prepare and stream; RS_GRAPH=0 disables)
    // the first run after a prepare goes direct (a one-shot reconfiguration would pay the
    // capture for nothing); repeated runs capture once and replay
    // (the legacy default stream cannot be captured: it always runs direct)
    const bool capturable = stream != nullptr && stream != cudaStreamLegacy && stream != cudaStreamPerThread;
    if (auto_graph_ && capturable && runs_since_prepare_++ > 0) return run_graph(stream);
    return run_direct(stream);
}

int Executor::run_direct(cudaStream_t stream) {
    RS_CUDA(cudaSetDevice(cfg_.device));
    if (!mc_ || mc_->groups.empty()) return run_fused(stream);
    // the multicast stream runs concurrently with the fused pushes (the root's NVLink
    // carries both): one CTA per SM for it, two per SM for the fused kernel
    if (!mc_stream_) {
        RS_CUDA(cudaStreamCreateWithFlags(&mc_stream_, cudaStreamNonBlocking));
        for (auto& e : mc_ev_) RS_CUDA(cudaEventCreate(&e));
    }
    const bool timing = std::getenv("RS_TIMING") != nullptr;
    if (const char* ser = std::getenv("RS_MC_SERIAL"); ser && std::string(ser) == "1") {  // diagnostics
        RS_CUDA(cudaEventRecord(mc_ev_[0], stream));
        const int n0 = launch_multicast(stream);
        RS_CUDA(cudaEventRecord(mc_ev_[1], stream));
        const int n1 = run_fused(stream);
        RS_CUDA(cudaEventRecord(mc_ev_[2], stream));
        if (timing) {
            RS_CUDA(cudaEventSynchronize(mc_ev_[2]));
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, mc_ev_[0], mc_ev_[1]);
            cudaEventElapsedTime(&b, mc_ev_[1], mc_ev_[2]);
            std::fprintf(stderr, "[reshard] gpu %d run: multicast %.3f ms (%.1f GB/s source), then fused %.3f ms\n", cfg_.gpu,
                         a, a > 0 ? mc_src_bytes_ / (a * 1e6) : 0.0, b);
        }
        return n0 + n1;
    }
    RS_CUDA(cudaEventRecord(mc_ev_[0], stream));
    RS_CUDA(cudaStreamWaitEvent(mc_stream_, mc_ev_[0], 0));
    const int n0 = launch_multicast(mc_stream_);
    RS_CUDA(cudaEventRecord(mc_ev_[1], mc_stream_));
    const int saved = cfg_.ctas_per_sm;
    cfg_.ctas_per_sm = 2;
    const int n1 = run_fused(stream);
    cfg_.ctas_per_sm = saved;
    RS_CUDA(cudaEventRecord(mc_ev_[2], stream));
    RS_CUDA(cudaStreamWaitEvent(stream, mc_ev_[1], 0));
    if (timing) {  // diagnostics: both parts timed from the fork
        RS_CUDA(cudaEventSynchronize(mc_ev_[1]));
        RS_CUDA(cudaEventSynchronize(mc_ev_[2]));
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, mc_ev_[0], mc_ev_[1]);
        cudaEventElapsedTime(&b, mc_ev_[0], mc_ev_[2]);
        std::fprintf(stderr, "[reshard] gpu %d run: multicast %.3f ms (%.1f GB/s source), fused %.3f ms (concurrent)\n",
                     cfg_.gpu, a, a > 0 ? mc_src_bytes_ / (a * 1e6) : 0.0, b);
    }
    return n0 + n1;
}

int Executor::run_fused(cudaStream_t stream) {
    if (!has_remote_) return fused_->launch(stream, 0, 0, sms_, cfg_.ctas_per_sm, use_bulk_);
    if (!aux_) {
        RS_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
        RS_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        RS_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    if (!ce_ops_.empty()) {
        // copy-engine part of the push on the aux stream, joined back into the caller's
        RS_CUDA(cudaEventRecord(ev_fork_, stream));
        RS_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
    }
    // measured on B200 (profiles/r01_nvlink.md): with peer-bound tiles, one mixed launch
    // of the 16-B vector kernel keeps NVLink busiest (685 GB/s at N=2, 620 at N=4)
    if (!split_remote_) {
        if (!ce_ops_.empty()) {
            // copy engines first (they start while the kernel launches), round-robin over
            // RS_CE_STREAMS streams so several engines work at once
            if (ce_streams_.empty()) {
                const char* ks = std::getenv("RS_CE_STREAMS");
                const int k = std::max(1, ks ? std::atoi(ks) : 2);
                ce_streams_.push_back(aux_);
                for (int i = 1; i < k; ++i) {
                    cudaStream_t x;
                    RS_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
                    ce_streams_.push_back(x);
                }
                ce_join_.resize(ce_streams_.size());
                for (auto& e : ce_join_) RS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            for (size_t i = 1; i < ce_streams_.size(); ++i) RS_CUDA(cudaStreamWaitEvent(ce_streams_[i], ev_fork_, 0));
            for (size_t i = 0; i < ce_ops_.size(); ++i) {
                const CeOp& c = ce_ops_[i];
                RS_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(c.dst), reinterpret_cast<const void*>(c.src),
                                        static_cast<size_t>(c.bytes), cudaMemcpyDeviceToDevice,
                                        ce_streams_[i % ce_streams_.size()]));
            }
        }
        const int n = fused_->launch(stream, 0, 0, sms_, cfg_.ctas_per_sm, remote_bulk_);
        if (!ce_ops_.empty())
            for (size_t i = 0; i < ce_streams_.size(); ++i) {
                RS_CUDA(cudaEventRecord(ce_join_[i], ce_streams_[i]));
                RS_CUDA(cudaStreamWaitEvent(stream, ce_join_[i], 0));
            }
        return n;
    }
    // NVLink-bound part (vector stores: full 16-B warps to peer HBM) on the caller's
    // stream; local HBM copies (TMA bulk) concurrently on an auxiliary stream
    RS_CUDA(cudaEventRecord(ev_fork_, stream));
    RS_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
    int n = fused_->launch(stream, 0, 0, sms_, remote_ctas_per_sm_, remote_bulk_, 2, 1);
    n += fused_->launch(aux_, 0, 0, sms_, cfg_.ctas_per_sm, use_bulk_, 2, 0);
    for (const CeOp& c : ce_ops_)
        RS_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(c.dst), reinterpret_cast<const void*>(c.src),
                                static_cast<size_t>(c.bytes), cudaMemcpyDeviceToDevice, aux_));
    RS_CUDA(cudaEventRecord(ev_join_, aux_));
    RS_CUDA(cudaStreamWaitEvent(stream, ev_join_, 0));
    return n;
}

int Executor::run_dup(cudaStream_t stream) {
    if (!prepared_) throw ConfigError("run before prepare");
    if (!dup_ || dup_->groups.empty()) return 0;
    RS_CUDA(cudaSetDevice(cfg_.device));
    return dup_->launch(stream, 0, 0, sms_, cfg_.ctas_per_sm, use_bulk_);
}

int Executor::num_stages() const {
    if (dup_early_) return 2;
    return stage_of_dst_.empty() ? 1 : *std::max_element(stage_of_dst_.begin(), stage_of_dst_.end()) + 1;
}

int Executor::run_stage(int stage, cudaStream_t stream) {
    if (!prepared_) throw ConfigError("run before prepare");
    if (split_remote_ || !ce_ops_.empty()) throw ConfigError("run_stage needs the single mixed launch (no CE offload)");
    RS_CUDA(cudaSetDevice(cfg_.device));
    const bool bulk = has_remote_ ? remote_bulk_ : use_bulk_;
    if (stage != 0 || !mc_ || mc_->groups.empty())
        return fused_->launch(stream, 0, 0, sms_, cfg_.ctas_per_sm, bulk, -1, stage);
    // stage 0 carries the multicast stores: concurrent with the fused pushes, as in run()
    if (!mc_stream_) {
        RS_CUDA(cudaStreamCreateWithFlags(&mc_stream_, cudaStreamNonBlocking));
        for (auto& e : mc_ev_) RS_CUDA(cudaEventCreate(&e));
    }
    RS_CUDA(cudaEventRecord(mc_ev_[0], stream));
    RS_CUDA(cudaStreamWaitEvent(mc_stream_, mc_ev_[0], 0));
    const int n0 = launch_multicast(mc_stream_);
    RS_CUDA(cudaEventRecord(mc_ev_[1], mc_stream_));
    const int n1 = fused_->launch(stream, 0, 0, sms_, 2, bulk, -1, stage);
    RS_CUDA(cudaStreamWaitEvent(stream, mc_ev_[1], 0));
    return n0 + n1;
}

std::int64_t Executor::channel_bytes(int src_phys, int dst_phys) const {
    auto it = channels_.find({src_phys, dst_phys});
    return it == channels_.end() ? 0 : it->second.bytes;
}

int Executor::pack(int src_phys, int dst_phys, void* buf, cudaStream_t stream) {
    auto it = channels_.find({src_phys, dst_phys});
    if (it == channels_.end()) return 0;
    RS_CUDA(cudaSetDevice(cfg_.device));
    return it->second.pack->launch(stream, 0, reinterpret_cast<std::uint64_t>(buf), sms_, cfg_.ctas_per_sm, use_bulk_);
}

int Executor::unpack(int src_phys, int dst_phys, const void* buf, cudaStream_t stream) {
    auto it = channels_.find({src_phys, dst_phys});
    if (it == channels_.end()) return 0;
    RS_CUDA(cudaSetDevice(cfg_.device));
    return it->second.unpack->launch(stream, reinterpret_cast<std::uint64_t>(buf), 0, sms_, cfg_.ctas_per_sm, use_bulk_);
}

std::vector<FillTask> Executor::fill_tasks(int side) const {
    std::vector<FillTask> tasks;
    const core::Side& S = side == 0 ? P_->src : P_->dst;
    for (size_t r = 0; r < S.ranks.size(); ++r) {
        const RankBufs& rb = bufs_[side][r];
        if (rb.gpu != cfg_.gpu) continue;
        const core::RankGeom& g = S.ranks[r];
        for (const core::Seg& s : g.segs) {
            const auto& e = P_->space->entries()[static_cast<size_t>(s.tensor)];
            FillTask f{};
            // lifted box
            const int nd = static_cast<int>(e.spec.shape.size());
            std::int64_t l[4], h[4], x[4];
            int n = 0;
            if (nd == 1) l[n] = 0, h[n] = 1, x[n] = 1, ++n;
            for (int d = 0; d < nd; ++d) l[n] = s.blo[d], h[n] = s.bhi[d], x[n] = e.spec.shape[static_cast<size_t>(d)], ++n;
            f.t.np = n - 2;
            for (int i = 0; i < f.t.np; ++i) f.t.pext[i] = x[i], f.plo[i] = l[i], f.pext_box[i] = h[i] - l[i];
            f.t.rows = x[f.t.np];
            f.t.cols = x[f.t.np + 1];
            f.t.off = e.offset;
            f.rlo = l[f.t.np];
            f.rows_box = h[f.t.np] - l[f.t.np];
            f.clo = l[f.t.np + 1];
            f.cols_box = h[f.t.np + 1] - l[f.t.np + 1];
            const std::int64_t n_el = s.local_hi - s.local_lo;
            // params
            if (rb.ptr[kParam]) {
                FillTask p = f;
                p.ptr = reinterpret_cast<std::uint64_t>(rb.ptr[kParam]) + static_cast<std::uint64_t>(s.param_byte_off);
                p.e_lo = 0;
                p.e_hi = n_el;
                p.kind = 0;
                p.width = e.spec.dtype_bytes;
                tasks.push_back(p);
            }
            if (rb.ptr[kGrad]) {
                FillTask p = f;
                p.ptr = reinterpret_cast<std::uint64_t>(rb.ptr[kGrad]) + static_cast<std::uint64_t>(s.elem_off * 4);
                p.e_lo = 0;
                p.e_hi = n_el;
                p.kind = 4;
                p.width = 4;
                tasks.push_back(p);
            }
            const Interval& sh = s.expert ? g.eshard : g.dshard;
            const std::int64_t lo = std::max(sh.lo, s.local_lo), hi = std::min(sh.hi, s.local_hi);
            if (lo < hi)
                for (int b = kMaster; b <= kV; ++b) {
                    if (!rb.ptr[b]) continue;
                    FillTask p = f;
                    const std::int64_t oi = g.optim_index(s.expert, lo);
                    p.ptr = reinterpret_cast<std::uint64_t>(rb.ptr[b]) + static_cast<std::uint64_t>(oi * 4);
                    p.e_lo = lo - s.local_lo;
                    p.e_hi = hi - s.local_lo;
                    p.kind = b;
                    p.width = 4;
                    tasks.push_back(p);
                }
        }
    }
    return tasks;
}

void Executor::upload_tasks(const std::vector<FillTask>& tasks, cudaStream_t stream) {
    // stream-ordered upload through pinned staging on the stream the fill/verify kernel
    // runs on (a pageable cudaMemcpy on the legacy stream is not ordered with a
    // non-blocking caller stream)
    if (tasks.empty()) return;
    const size_t bytes = tasks.size() * sizeof(FillTask);
    RS_CUDA(cudaStreamSynchronize(stream));  // earlier fill/verify kernels may still read d_fill_
    if (bytes > fill_bytes_) {
        if (d_fill_) cudaFree(d_fill_);
        d_fill_ = nullptr;
        fill_bytes_ = 0;
        RS_CUDA(cudaMalloc(&d_fill_, bytes));
        fill_bytes_ = bytes;
    }
    if (fill_staging_.size() < bytes) fill_staging_.grow(bytes);
    std::memcpy(fill_staging_.ptr, tasks.data(), bytes);
    RS_CUDA(cudaMemcpyAsync(d_fill_, fill_staging_.ptr, bytes, cudaMemcpyHostToDevice, stream));
}

void Executor::fill(int side, std::uint64_t seed, cudaStream_t stream) {
    RS_CUDA(cudaSetDevice(cfg_.device));
    const std::vector<FillTask> tasks = fill_tasks(side);
    upload_tasks(tasks, stream);
    if (!tasks.empty()) {
        dim3 grid(static_cast<unsigned>(sms_ * 2), static_cast<unsigned>(std::min<size_t>(tasks.size(), 65535)));
        fill_kernel<<<grid, 256, 0, stream>>>(static_cast<const FillTask*>(d_fill_), static_cast<int>(tasks.size()), seed);
    }
    for (size_t r = 0; r < bufs_[side].size(); ++r) {
        const RankBufs& rb = bufs_[side][r];
        if (rb.gpu == cfg_.gpu && rb.ptr[kScalars])
            fill_scalars_kernel<<<1, 64, 0, stream>>>(static_cast<std::uint64_t*>(rb.ptr[kScalars]),
                                                       rb.bytes[kScalars] / 8, seed);
    }
    RS_CUDA(cudaGetLastError());
    RS_CUDA(cudaStreamSynchronize(stream));
}

std::int64_t Executor::verify(int side, std::uint64_t seed, cudaStream_t stream, std::int64_t* first_bad) {
    RS_CUDA(cudaSetDevice(cfg_.device));
    const std::vector<FillTask> tasks = fill_tasks(side);
    upload_tasks(tasks, stream);
    if (!d_counters_) RS_CUDA(cudaMalloc(&d_counters_, 64));
    unsigned long long* bad = static_cast<unsigned long long*>(d_counters_);
    long long* first = reinterpret_cast<long long*>(static_cast<char*>(d_counters_) + 8);
    const long long big = 0x7fffffffffffffffll;
    RS_CUDA(cudaMemsetAsync(bad, 0, 8, stream));
    RS_CUDA(cudaMemcpyAsync(first, &big, 8, cudaMemcpyHostToDevice, stream));
    if (!tasks.empty()) {
        dim3 grid(static_cast<unsigned>(sms_ * 2), static_cast<unsigned>(std::min<size_t>(tasks.size(), 65535)));
        verify_kernel<<<grid, 256, 0, stream>>>(static_cast<const FillTask*>(d_fill_), static_cast<int>(tasks.size()),
                                                seed, bad, first);
    }
    for (size_t r = 0; r < bufs_[side].size(); ++r) {
        const RankBufs& rb = bufs_[side][r];
        if (rb.gpu == cfg_.gpu && rb.ptr[kScalars])
            verify_scalars_kernel<<<1, 64, 0, stream>>>(static_cast<const std::uint64_t*>(rb.ptr[kScalars]),
                                                         rb.bytes[kScalars] / 8, seed, bad);
    }
    RS_CUDA(cudaGetLastError());
    unsigned long long h_bad = 0;
    long long h_first = 0;
    RS_CUDA(cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, stream));
    RS_CUDA(cudaMemcpyAsync(&h_first, first, 8, cudaMemcpyDeviceToHost, stream));
    RS_CUDA(cudaStreamSynchronize(stream));
    if (first_bad) *first_bad = h_bad ? h_first : -1;
    return static_cast<std::int64_t>(h_bad);
}

}  // namespace exec
}  // namespace reshard
