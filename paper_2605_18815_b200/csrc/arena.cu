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

}  // namespace

Arena::Arena(const core::PlanCore& ab, const core::PlanCore* ba, const ArenaConfig& cfg, bool with_grads) : cfg_(cfg) {
    const Drv& D = Drv::get();
    if (cudaSetDevice(cfg.device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    const std::int64_t C = cfg.chunk_bytes;
    const MemoryPlan mp = plan_memory(ab, ba, C, with_grads);
    order_[0] = mp.order[0];
    order_[1] = mp.order[1];
    stats_ = mp.stats;
    const int nphys = mp.nphys;
    const bool small_direct = true;
    for (int l = 0; l < 2; ++l) {
        nranks_[l] = l == 0 ? ab.src_cfg.world_size() : ab.dst_cfg.world_size();
        bufs_[l].resize(mp.bufs[l].size());
        for (size_t i = 0; i < mp.bufs[l].size(); ++i) {
            bufs_[l][i].bytes = mp.bufs[l][i].bytes;
            bufs_[l][i].reserved = mp.bufs[l][i].reserved;
            bufs_[l][i].phys = mp.bufs[l][i].phys;
        }
    }
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
