// Arena: VMM-backed old/new layouts with plan-time eager-free aliasing (arena.hpp).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <map>

#include "reshard/arena.hpp"
#include "reshard/executor_rt.hpp"

namespace reshard {
namespace mem {

namespace {

struct Drv {
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;

    static const Drv& get() {
        static Drv d = [] {
            Drv x;
            auto load = [](const char* name, auto& fn) {
                void* f = nullptr;
                cudaDriverEntryPointQueryResult q;
                if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || !f)
                    throw exec::CudaError(std::string("driver entry point missing: ") + name);
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(f);
            };
            load("cuMemCreate", x.create);
            load("cuMemRelease", x.release);
            load("cuMemAddressReserve", x.reserve);
            load("cuMemAddressFree", x.addr_free);
            load("cuMemMap", x.map);
            load("cuMemUnmap", x.unmap);
            load("cuMemSetAccess", x.set_access);
            load("cuMemGetAllocationGranularity", x.granularity);
            return x;
        }();
        return d;
    }
};

void drv_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw exec::CudaError(strfmt("%s failed (CUresult %d)", what, static_cast<int>(r)));
}

constexpr int kNever = std::numeric_limits<int>::max();

/// [first, last] chunk indices an op touches in its src and dst buffers
struct Extent {
    std::int64_t lo, hi;  // bytes [lo, hi)
};
Extent src_extent(const exec::CopyOp& op) { return {op.src_off, op.src_off + (op.rows - 1) * op.src_pitch + op.row_bytes}; }
Extent dst_extent(const exec::CopyOp& op) { return {op.dst_off, op.dst_off + (op.rows - 1) * op.dst_pitch + op.row_bytes}; }

}  // namespace

std::vector<int> greedy_stage_order(const core::PlanCore& P, const std::vector<exec::CopyOp>& ops) {
    const int ns = P.src_cfg.world_size(), nd = P.dst_cfg.world_size();
    // consumers of each src rank, bytes of each src rank
    std::vector<std::vector<char>> reads(static_cast<size_t>(ns), std::vector<char>(static_cast<size_t>(nd), 0));
    for (const exec::CopyOp& op : ops) reads[static_cast<size_t>(op.src_side_rank)][static_cast<size_t>(op.dst_rank)] = 1;
    std::vector<std::int64_t> sbytes(static_cast<size_t>(ns), 0);
    for (int i = 0; i < ns; ++i) {
        std::int64_t b[exec::kNumBufs];
        exec::buffer_sizes(P, 0, i, false, b);
        for (int k = 0; k < exec::kNumBufs; ++k) sbytes[static_cast<size_t>(i)] += b[k];
    }
    std::vector<char> done(static_cast<size_t>(nd), 0), dead(static_cast<size_t>(ns), 0);
    std::vector<int> order;
    for (int step = 0; step < nd; ++step) {
        int best = -1;
        std::int64_t best_freed = -1;
        for (int j = 0; j < nd; ++j) {
            if (done[static_cast<size_t>(j)]) continue;
            std::int64_t freed = 0;
            for (int i = 0; i < ns; ++i) {
                if (dead[static_cast<size_t>(i)]) continue;
                bool all = true;
                for (int d = 0; d < nd && all; ++d)
                    if (reads[static_cast<size_t>(i)][static_cast<size_t>(d)] && !done[static_cast<size_t>(d)] && d != j) all = false;
                if (all) freed += sbytes[static_cast<size_t>(i)];
            }
            if (freed > best_freed) best = j, best_freed = freed;
        }
        done[static_cast<size_t>(best)] = 1;
        order.push_back(best);
        for (int i = 0; i < ns; ++i) {
            bool all = true;
            for (int d = 0; d < nd && all; ++d)
                if (reads[static_cast<size_t>(i)][static_cast<size_t>(d)] && !done[static_cast<size_t>(d)]) all = false;
            if (all) dead[static_cast<size_t>(i)] = 1;
        }
    }
    return order;
}

Arena::Arena(const core::PlanCore& ab, const core::PlanCore* ba, const ArenaConfig& cfg, bool with_grads) : cfg_(cfg) {
    const Drv& D = Drv::get();
    if (cudaSetDevice(cfg.device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    const std::int64_t C = cfg.chunk_bytes;
    nranks_[0] = ab.src_cfg.world_size();
    nranks_[1] = ab.dst_cfg.world_size();
    for (int l = 0; l < 2; ++l) {
        bufs_[l].resize(static_cast<size_t>(nranks_[l]) * exec::kNumBufs);
        for (int r = 0; r < nranks_[l]; ++r) {
            std::int64_t b[exec::kNumBufs];
            exec::buffer_sizes(ab, l, r, with_grads, b);
            for (int k = 0; k < exec::kNumBufs; ++k) {
                BufMap& m = bufs_[l][static_cast<size_t>(r) * exec::kNumBufs + k];
                m.bytes = b[k];
                m.reserved = (b[k] + C - 1) / C * C;
                m.phys.assign(static_cast<size_t>(m.reserved / C), -1);
            }
        }
    }
    // ---- lifetimes
    const std::vector<exec::CopyOp> ops_ab = exec::build_ops(ab);
    order_[0] = greedy_stage_order(ab, ops_ab);
    std::vector<int> pos_ab(static_cast<size_t>(nranks_[1]));
    for (size_t s = 0; s < order_[0].size(); ++s) pos_ab[static_cast<size_t>(order_[0][s])] = static_cast<int>(s);
    auto chunk_vec = [&](int l) {
        std::vector<std::vector<int>> v(bufs_[l].size());
        for (size_t i = 0; i < bufs_[l].size(); ++i) v[i].assign(bufs_[l][i].phys.size(), -1);
        return v;
    };
    std::vector<std::vector<int>> lr_ab = chunk_vec(0), fw_ab = chunk_vec(1);
    for (auto& v : fw_ab) std::fill(v.begin(), v.end(), kNever);
    auto touch = [&](std::vector<std::vector<int>>& tab, int rank, int buf, Extent e, int stage, bool is_max) {
        auto& v = tab[static_cast<size_t>(rank) * exec::kNumBufs + buf];
        for (std::int64_t c = e.lo / C; c <= (e.hi - 1) / C && c < static_cast<std::int64_t>(v.size()); ++c) {
            int& x = v[static_cast<size_t>(c)];
            x = is_max ? std::max(x, stage) : std::min(x, stage);
        }
    };
    for (const exec::CopyOp& op : ops_ab) {
        const int s = pos_ab[static_cast<size_t>(op.dst_rank)];
        touch(lr_ab, op.src_side_rank, op.src_buf, src_extent(op), s, true);
        touch(fw_ab, op.dst_rank, op.dst_buf, dst_extent(op), s, false);
    }
    std::vector<std::vector<int>> lr_ba = chunk_vec(1), fw_ba = chunk_vec(0);
    for (auto& v : fw_ba) std::fill(v.begin(), v.end(), kNever);
    if (ba) {
        // B->A writes A ranks; A ranks that die last in A->B are rebuilt first
        std::vector<int> death(static_cast<size_t>(nranks_[0]), -1);
        for (int r = 0; r < nranks_[0]; ++r)
            for (int k = 0; k < exec::kNumBufs; ++k)
                for (int x : lr_ab[static_cast<size_t>(r) * exec::kNumBufs + k]) death[static_cast<size_t>(r)] = std::max(death[static_cast<size_t>(r)], x);
        order_[1].resize(static_cast<size_t>(nranks_[0]));
        for (int r = 0; r < nranks_[0]; ++r) order_[1][static_cast<size_t>(r)] = r;
        std::sort(order_[1].begin(), order_[1].end(), [&](int a, int b) {
            return death[static_cast<size_t>(a)] != death[static_cast<size_t>(b)] ? death[static_cast<size_t>(a)] > death[static_cast<size_t>(b)] : a > b;
        });
        std::vector<int> pos_ba(static_cast<size_t>(nranks_[0]));
        for (size_t s = 0; s < order_[1].size(); ++s) pos_ba[static_cast<size_t>(order_[1][s])] = static_cast<int>(s);
        for (const exec::CopyOp& op : exec::build_ops(*ba)) {
            const int s = pos_ba[static_cast<size_t>(op.dst_rank)];
            touch(lr_ba, op.src_side_rank, op.src_buf, src_extent(op), s, true);
            touch(fw_ba, op.dst_rank, op.dst_buf, dst_extent(op), s, false);
        }
    }
    // ---- physical assignment: every A chunk owns one; B chunks alias dead A chunks
    const bool small_direct = true;
    int nphys = 0;
    struct AChunk {
        int lr_ab, fw_ba, phys;
    };
    std::vector<AChunk> achunks;
    for (size_t i = 0; i < bufs_[0].size(); ++i) {
        BufMap& m = bufs_[0][i];
        if (small_direct && m.bytes < C / 4) continue;
        for (size_t c = 0; c < m.phys.size(); ++c) {
            m.phys[c] = nphys++;
            achunks.push_back({lr_ab[i][c], fw_ba[i][c], m.phys[c]});
        }
    }
    stats_.a_bytes = static_cast<std::int64_t>(nphys) * C;
    struct BChunk {
        int fw_ab, lr_ba;
        size_t buf, idx;
    };
    std::vector<BChunk> bchunks;
    for (size_t i = 0; i < bufs_[1].size(); ++i) {
        const BufMap& m = bufs_[1][i];
        if (small_direct && m.bytes < C / 4) continue;
        for (size_t c = 0; c < m.phys.size(); ++c) bchunks.push_back({fw_ab[i][c], lr_ba[i][c], i, c});
    }
    std::stable_sort(bchunks.begin(), bchunks.end(), [](const BChunk& a, const BChunk& b) { return a.fw_ab < b.fw_ab; });
    std::vector<size_t> aorder(achunks.size());
    for (size_t i = 0; i < aorder.size(); ++i) aorder[i] = i;
    std::sort(aorder.begin(), aorder.end(), [&](size_t a, size_t b) { return achunks[a].lr_ab < achunks[b].lr_ab; });
    std::multimap<int, int> avail;  // fw_ba -> physical chunk (dead in A->B, not yet shared)
    size_t ai = 0;
    int fresh = 0;
    for (const BChunk& b : bchunks) {
        while (ai < aorder.size() && achunks[aorder[ai]].lr_ab < b.fw_ab) {
            const AChunk& a = achunks[aorder[ai++]];
            avail.emplace(ba ? a.fw_ba : 0, a.phys);
        }
        int p = -1;
        if (!avail.empty()) {
            auto it = ba ? avail.upper_bound(b.lr_ba) : avail.begin();
            if (it != avail.end()) {
                p = it->second;
                avail.erase(it);
                stats_.aliased_bytes += C;
            }
        }
        if (p < 0) p = nphys + fresh++;
        bufs_[1][b.buf].phys[b.idx] = p;
    }
    nphys += fresh;
    stats_.chunks = nphys;
    stats_.physical_bytes = static_cast<std::int64_t>(nphys) * C;
    std::int64_t cap = cfg.cap_bytes;
    if (cap <= 0) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        cap = static_cast<std::int64_t>(fr) - (1ll << 30);
    }
    if (stats_.physical_bytes > cap)
        throw exec::BudgetError(strfmt("infeasible budget: memory plan needs %.2f GB of HBM, cap %.2f GB",
                                 stats_.physical_bytes / 1e9, cap / 1e9));
    // ---- create and map
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = cfg.device;
    size_t gran = 0;
    drv_check(D.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
    if (C % static_cast<std::int64_t>(gran)) throw ConfigError("arena chunk is not a multiple of the VMM granularity");
    handles_.resize(static_cast<size_t>(nphys));
    for (int i = 0; i < nphys; ++i) {
        CUmemGenericAllocationHandle h;
        drv_check(D.create(&h, static_cast<size_t>(C), &prop, 0), "cuMemCreate");
        handles_[static_cast<size_t>(i)] = h;
    }
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int l = 0; l < 2; ++l)
        for (BufMap& m : bufs_[l]) {
            if (m.bytes == 0) continue;
            if (small_direct && m.bytes < C / 4) {
                void* p = nullptr;
                if (cudaMalloc(&p, static_cast<size_t>(m.bytes)) != cudaSuccess) throw exec::CudaError("cudaMalloc failed");
                m.va = reinterpret_cast<std::uint64_t>(p);
                m.reserved = 0;
                continue;
            }
            CUdeviceptr va = 0;
            drv_check(D.reserve(&va, static_cast<size_t>(m.reserved), static_cast<size_t>(C), 0, 0), "cuMemAddressReserve");
            m.va = va;
            for (size_t c = 0; c < m.phys.size(); ++c)
                drv_check(D.map(va + c * static_cast<std::uint64_t>(C), static_cast<size_t>(C), 0,
                                handles_[static_cast<size_t>(m.phys[c])], 0), "cuMemMap");
            drv_check(D.set_access(va, static_cast<size_t>(m.reserved), &acc, 1), "cuMemSetAccess");
        }
    stats_.b_bytes = 0;
    for (const BufMap& m : bufs_[1]) stats_.b_bytes += m.bytes;
}

Arena::~Arena() {
    const Drv& D = Drv::get();
    cudaSetDevice(cfg_.device);
    cudaDeviceSynchronize();
    for (int l = 0; l < 2; ++l)
        for (BufMap& m : bufs_[l]) {
            if (!m.va) continue;
            if (m.reserved == 0) {
                cudaFree(reinterpret_cast<void*>(m.va));
                continue;
            }
            D.unmap(m.va, static_cast<size_t>(m.reserved));
            D.addr_free(m.va, static_cast<size_t>(m.reserved));
        }
    for (std::uint64_t h : handles_) D.release(h);
}

void* Arena::ptr(int layout, int rank, int buf) const {
    return reinterpret_cast<void*>(bufs_[layout].at(static_cast<size_t>(rank) * exec::kNumBufs + buf).va);
}
std::int64_t Arena::bytes(int layout, int rank, int buf) const {
    return bufs_[layout].at(static_cast<size_t>(rank) * exec::kNumBufs + buf).bytes;
}

}  // namespace mem
}  // namespace reshard
