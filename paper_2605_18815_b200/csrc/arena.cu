// Arena: VMM-backed old/new layouts with plan-time eager-free aliasing (arena.hpp),
// on one GPU or across GPUs (POSIX-FD export of the physical allocations).
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
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
    CUresult (*export_fd)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
    CUresult (*import_fd)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
    CUresult (*mc_create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*mc_add)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mc_bind)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
    CUresult (*mc_unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*mc_granularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    CUresult (*device_get)(CUdevice*, int) = nullptr;

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
            load("cuMemExportToShareableHandle", x.export_fd);
            load("cuMemImportFromShareableHandle", x.import_fd);
            load("cuMulticastCreate", x.mc_create);
            load("cuMulticastAddDevice", x.mc_add);
            load("cuMulticastBindMem", x.mc_bind);
            load("cuMulticastUnbind", x.mc_unbind);
            load("cuMulticastGetGranularity", x.mc_granularity);
            load("cuDeviceGet", x.device_get);
            return x;
        }();
        return d;
    }
};

void drv_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw exec::CudaError(strfmt("%s failed (CUresult %d)", what, static_cast<int>(r)));
}

CUmemAllocationProp device_prop(int device, bool shareable) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    if (shareable) prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return prop;
}

// export table entry: layout, rank, buf, number of handles, bytes, reserved, piece size
struct Entry {
    std::int32_t layout, rank, buf, nh;
    std::int64_t bytes, reserved, piece;
};

}  // namespace

Arena::Arena(const core::PlanCore& ab, const core::PlanCore* ba, const ArenaConfig& cfg, bool with_grads, int n_gpus,
             int gpu)
    : cfg_(cfg), n_gpus_(n_gpus) {
    const Drv& D = Drv::get();
    if (cudaSetDevice(cfg.device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    const std::int64_t C = cfg.chunk_bytes;
    std::int64_t cap = cfg.cap_bytes;
    if (cap <= 0) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        cap = static_cast<std::int64_t>(fr) - (1ll << 30);
    }
    int groups = cfg.groups, bands = std::max(1, cfg.bands);
    if (groups == 0) {
        std::int64_t need = 0;
        const int level = choose_schedule(ab, ba, C, with_grads, n_gpus, gpu, cap, &need);
        if (level < 0)
            throw exec::BudgetError(strfmt("infeasible budget: memory plan needs %.2f GB of HBM on GPU %d, cap %.2f GB",
                                           need / 1e9, gpu, cap / 1e9));
        const ScheduleLevel L = schedule_levels(ab, n_gpus)[static_cast<size_t>(level)];
        groups = L.groups;
        bands = L.bands;
    }
    const MemoryPlan mp = plan_memory(ab, ba, C, with_grads, n_gpus, gpu, groups, bands);
    // replay the plan chunk by chunk before mapping anything (host-only): a planner
    // regression must fail here, not corrupt state silently
    if (const std::int64_t v = simulate_memory_plan(mp, ab, ba); v != 0)
        throw std::logic_error(strfmt("memory plan: %lld simulated read/write violations on GPU %d",
                                      static_cast<long long>(v), gpu));
    bands_ = mp.bands;
    const bool shareable = n_gpus > 1;
    one_way_ = ba == nullptr && n_gpus == 1;
    if (one_way_) {
        a_last_stage_ = last_read_stage(mp, ab, exec::build_ops(ab));
        a_unmapped_.resize(mp.bufs[0].size());
        for (size_t i = 0; i < mp.bufs[0].size(); ++i) a_unmapped_[i].assign(mp.bufs[0][i].phys.size(), 0);
        b_uses_.assign(static_cast<size_t>(mp.nphys), 0);
        for (const BufPlan& m : mp.bufs[1])
            for (int p : m.phys)
                if (p >= 0) b_uses_[static_cast<size_t>(p)] = 1;
    }
    order_[0] = mp.order[0];
    order_[1] = mp.order[1];
    cut_[0] = mp.cut[0];
    cut_[1] = mp.cut[1];
    stats_ = mp.stats;
    for (int l = 0; l < 2; ++l) {
        nranks_[l] = l == 0 ? ab.src_cfg.world_size() : ab.dst_cfg.world_size();
        bufs_[l].resize(mp.bufs[l].size());
        for (size_t i = 0; i < mp.bufs[l].size(); ++i) {
            bufs_[l][i].bytes = mp.bufs[l][i].bytes;
            bufs_[l][i].reserved = mp.bufs[l][i].reserved;
            bufs_[l][i].phys = mp.bufs[l][i].phys;
            bufs_[l][i].remote = mp.bufs[l][i].remote;
        }
    }
    if (stats_.physical_bytes > cap)
        throw exec::BudgetError(strfmt("infeasible budget: memory plan needs %.2f GB of HBM on GPU %d, cap %.2f GB",
                                       stats_.physical_bytes / 1e9, gpu, cap / 1e9));
    // ---- create and map
    const CUmemAllocationProp prop = device_prop(cfg.device, shareable);
    size_t gran = 0;
    drv_check(D.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
    if (C % static_cast<std::int64_t>(gran)) throw ConfigError("arena chunk is not a multiple of the VMM granularity");
    handles_.resize(static_cast<size_t>(mp.nphys));
    for (int i = 0; i < mp.nphys; ++i) {
        CUmemGenericAllocationHandle h;
        drv_check(D.create(&h, static_cast<size_t>(C), &prop, 0), "cuMemCreate");
        handles_[static_cast<size_t>(i)] = h;
    }
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int l = 0; l < 2; ++l)
        for (BufMap& m : bufs_[l]) {
            if (m.bytes == 0 || m.remote) continue;
            if (m.reserved == 0) {  // small buffer: its own allocation
                if (!shareable) {
                    void* p = nullptr;
                    if (cudaMalloc(&p, static_cast<size_t>(m.bytes)) != cudaSuccess) throw exec::CudaError("cudaMalloc failed");
                    m.va = reinterpret_cast<std::uint64_t>(p);
                    continue;
                }
                const std::int64_t g = static_cast<std::int64_t>(gran);
                const std::int64_t sz = (m.bytes + g - 1) / g * g;
                CUmemGenericAllocationHandle h;
                drv_check(D.create(&h, static_cast<size_t>(sz), &prop, 0), "cuMemCreate");
                CUdeviceptr va = 0;
                drv_check(D.reserve(&va, static_cast<size_t>(sz), gran, 0, 0), "cuMemAddressReserve");
                drv_check(D.map(va, static_cast<size_t>(sz), 0, h, 0), "cuMemMap");
                drv_check(D.set_access(va, static_cast<size_t>(sz), &acc, 1), "cuMemSetAccess");
                m.va = va;
                m.reserved = sz;
                m.own_handle = true;
                m.mapped_vmm = true;
                m.handle = h;
                continue;
            }
            CUdeviceptr va = 0;
            drv_check(D.reserve(&va, static_cast<size_t>(m.reserved), static_cast<size_t>(C), 0, 0), "cuMemAddressReserve");
            m.va = va;
            m.mapped_vmm = true;
            for (size_t c = 0; c < m.phys.size(); ++c)
                drv_check(D.map(va + c * static_cast<std::uint64_t>(C), static_cast<size_t>(C), 0,
                                handles_[static_cast<size_t>(m.phys[c])], 0), "cuMemMap");
            drv_check(D.set_access(va, static_cast<size_t>(m.reserved), &acc, 1), "cuMemSetAccess");
        }
}

void Arena::export_local(std::vector<int>* fds, std::vector<std::uint8_t>* table) const {
    const Drv& D = Drv::get();
    if (n_gpus_ < 2) throw ConfigError("arena export needs a multi-GPU arena");
    fds->clear();
    table->clear();
    // physical chunks first (indices = chunk ids), then the small buffers' own handles
    for (std::uint64_t h : handles_) {
        int fd = -1;
        drv_check(D.export_fd(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
        fds->push_back(fd);
    }
    auto put = [table](const void* p, size_t n) {
        const auto* c = static_cast<const std::uint8_t*>(p);
        table->insert(table->end(), c, c + n);
    };
    const std::int64_t nchunk_handles = static_cast<std::int64_t>(handles_.size());
    put(&nchunk_handles, sizeof nchunk_handles);
    for (int l = 0; l < 2; ++l)
        for (size_t i = 0; i < bufs_[l].size(); ++i) {
            const BufMap& m = bufs_[l][i];
            if (m.remote || m.bytes == 0) continue;
            Entry e{l, static_cast<std::int32_t>(i / exec::kNumBufs), static_cast<std::int32_t>(i % exec::kNumBufs), 0,
                    m.bytes, m.reserved, 0};
            std::vector<std::int32_t> idx;
            if (m.own_handle) {
                int fd = -1;
                drv_check(D.export_fd(&fd, m.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                          "cuMemExportToShareableHandle");
                idx.push_back(static_cast<std::int32_t>(fds->size()));
                fds->push_back(fd);
                e.piece = m.reserved;
            } else {
                for (int p : m.phys) idx.push_back(p);
                e.piece = cfg_.chunk_bytes;
            }
            e.nh = static_cast<std::int32_t>(idx.size());
            put(&e, sizeof e);
            put(idx.data(), idx.size() * sizeof(std::int32_t));
        }
}

void Arena::import_peer(const std::vector<int>& fds, const std::vector<std::uint8_t>& table) {
    const Drv& D = Drv::get();
    if (cudaSetDevice(cfg_.device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    std::vector<CUmemGenericAllocationHandle> hs(fds.size());
    for (size_t i = 0; i < fds.size(); ++i) {
        drv_check(D.import_fd(&hs[i], reinterpret_cast<void*>(static_cast<std::intptr_t>(fds[i])),
                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                  "cuMemImportFromShareableHandle");
        ::close(fds[i]);  // the imported handle keeps the allocation alive
        imported_.push_back(hs[i]);
    }
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = cfg_.device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    size_t at = sizeof(std::int64_t);
    while (at + sizeof(Entry) <= table.size()) {
        Entry e;
        std::memcpy(&e, table.data() + at, sizeof e);
        at += sizeof e;
        // the table comes from another process: validate before using any field
        if (e.layout < 0 || e.layout > 1 || e.buf < 0 || e.buf >= exec::kNumBufs || e.rank < 0 || e.nh < 0 ||
            e.piece <= 0 || e.reserved < 0 || e.bytes < 0 ||
            at + static_cast<size_t>(e.nh) * sizeof(std::int32_t) > table.size() ||
            static_cast<std::int64_t>(e.nh) * e.piece != e.reserved)
            throw ConfigError("arena import: malformed mapping table");
        std::vector<std::int32_t> idx(static_cast<size_t>(e.nh));
        std::memcpy(idx.data(), table.data() + at, idx.size() * sizeof(std::int32_t));
        at += idx.size() * sizeof(std::int32_t);
        BufMap& m = bufs_[e.layout].at(static_cast<size_t>(e.rank) * exec::kNumBufs + e.buf);
        CUdeviceptr va = 0;
        drv_check(D.reserve(&va, static_cast<size_t>(e.reserved), static_cast<size_t>(e.piece), 0, 0), "cuMemAddressReserve");
        for (size_t c = 0; c < idx.size(); ++c)
            drv_check(D.map(va + c * static_cast<std::uint64_t>(e.piece), static_cast<size_t>(e.piece), 0,
                            hs.at(static_cast<size_t>(idx[c])), 0),
                      "cuMemMap");
        drv_check(D.set_access(va, static_cast<size_t>(e.reserved), &acc, 1), "cuMemSetAccess");
        m.va = va;
        m.bytes = e.bytes;
        peer_maps_.push_back({va, e.reserved});
    }
}

std::int64_t Arena::release_through(int stage) {
    if (!one_way_) throw ConfigError("arena release: only one-way arenas on one GPU release old-layout chunks");
    const Drv& D = Drv::get();
    if (cudaSetDevice(cfg_.device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    const std::int64_t C = cfg_.chunk_bytes;
    std::int64_t freed = 0;
    for (size_t i = 0; i < bufs_[0].size(); ++i) {
        BufMap& m = bufs_[0][i];
        if (!m.mapped_vmm || m.own_handle || m.remote || m.phys.empty()) continue;
        for (size_t c = 0; c < m.phys.size(); ++c) {
            if (a_unmapped_[i][c] || a_last_stage_[i][c] > stage) continue;
            drv_check(D.unmap(m.va + c * static_cast<std::uint64_t>(C), static_cast<size_t>(C)), "cuMemUnmap");
            a_unmapped_[i][c] = 1;
            const int p = m.phys[c];
            if (!b_uses_[static_cast<size_t>(p)] && handles_[static_cast<size_t>(p)]) {
                drv_check(D.release(handles_[static_cast<size_t>(p)]), "cuMemRelease");
                handles_[static_cast<size_t>(p)] = 0;
                freed += C;
            }
        }
    }
    released_bytes_ += freed;
    return freed;
}

Arena::~Arena() {
    const Drv& D = Drv::get();
    cudaSetDevice(cfg_.device);
    cudaDeviceSynchronize();
    for (const auto& pm : peer_maps_) {
        D.unmap(pm.first, static_cast<size_t>(pm.second));
        D.addr_free(pm.first, static_cast<size_t>(pm.second));
    }
    for (std::uint64_t h : imported_) D.release(h);
    for (int l = 0; l < 2; ++l)
        for (BufMap& m : bufs_[l]) {
            if (!m.va || m.remote) continue;
            if (!m.mapped_vmm) {
                cudaFree(reinterpret_cast<void*>(m.va));
                continue;
            }
            if (l == 0 && !a_unmapped_.empty()) {  // some chunks already unmapped at run time
                const std::int64_t C = cfg_.chunk_bytes;
                const size_t i = static_cast<size_t>(&m - bufs_[0].data());
                for (size_t c = 0; c < m.phys.size(); ++c)
                    if (!a_unmapped_[i][c]) D.unmap(m.va + c * static_cast<std::uint64_t>(C), static_cast<size_t>(C));
            } else {
                D.unmap(m.va, static_cast<size_t>(m.reserved));
            }
            D.addr_free(m.va, static_cast<size_t>(m.reserved));
            if (m.own_handle) D.release(m.handle);
        }
    for (std::uint64_t h : handles_)
        if (h) D.release(h);
}

void* Arena::ptr(int layout, int rank, int buf) const {
    return reinterpret_cast<void*>(bufs_[layout].at(static_cast<size_t>(rank) * exec::kNumBufs + buf).va);
}
std::int64_t Arena::bytes(int layout, int rank, int buf) const {
    return bufs_[layout].at(static_cast<size_t>(rank) * exec::kNumBufs + buf).bytes;
}

std::int64_t Arena::bind_size(int layout, int rank, int buf) const {
    // from the size alone (plan_memory's rule), so every rank agrees, hosted here or not
    const BufMap& m = bufs_[layout][static_cast<size_t>(rank) * exec::kNumBufs + buf];
    const std::int64_t C = cfg_.chunk_bytes, gran = 2ll << 20;
    return m.bytes < C / 4 ? (m.bytes + gran - 1) / gran * gran : (m.bytes + C - 1) / C * C;
}

namespace {
std::int64_t vmm_round(int device, std::int64_t bytes) {
    const CUmemAllocationProp p = device_prop(device, true);
    size_t gran = 0;
    drv_check(Drv::get().granularity(&gran, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
    const std::int64_t g = static_cast<std::int64_t>(gran);
    return (std::max<std::int64_t>(bytes, 1) + g - 1) / g * g;
}

std::uint64_t vmm_map(std::uint64_t handle, std::int64_t size, int device) {
    const Drv& D = Drv::get();
    CUdeviceptr va = 0;
    drv_check(D.reserve(&va, static_cast<size_t>(size), 0, 0, 0), "cuMemAddressReserve");
    drv_check(D.map(va, static_cast<size_t>(size), 0, handle, 0), "cuMemMap");
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    drv_check(D.set_access(va, static_cast<size_t>(size), &acc, 1), "cuMemSetAccess");
    return va;
}
}  // namespace

VmmBuffer::VmmBuffer(int device, std::int64_t bytes) : bytes_(bytes), device_(device) {
    if (cudaSetDevice(device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    size_ = vmm_round(device, bytes);
    const CUmemAllocationProp p = device_prop(device, true);
    CUmemGenericAllocationHandle h;
    drv_check(Drv::get().create(&h, static_cast<size_t>(size_), &p, 0), "cuMemCreate");
    handle_ = h;
    va_ = vmm_map(handle_, size_, device);
}

VmmBuffer::VmmBuffer(int fd, std::int64_t bytes, int device) : bytes_(bytes), device_(device) {
    if (cudaSetDevice(device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    const Drv& D = Drv::get();
    CUmemGenericAllocationHandle h;
    const CUresult r = D.import_fd(&h, reinterpret_cast<void*>(static_cast<std::intptr_t>(fd)),
                                   CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    ::close(fd);
    drv_check(r, "cuMemImportFromShareableHandle");
    handle_ = h;
    size_ = vmm_round(device, bytes);
    va_ = vmm_map(handle_, size_, device);
}

VmmBuffer::~VmmBuffer() {
    const Drv& D = Drv::get();
    if (va_) {
        D.unmap(va_, static_cast<size_t>(size_));
        D.addr_free(va_, static_cast<size_t>(size_));
    }
    if (handle_) D.release(handle_);
}

int VmmBuffer::export_fd() const {
    int fd = -1;
    drv_check(Drv::get().export_fd(&fd, handle_, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
    return fd;
}

void Arena::bind_multicast(Multicast& mc, int layout, int rank, int buf) const {
    const BufMap& m = bufs_[layout][static_cast<size_t>(rank) * exec::kNumBufs + buf];
    if (m.remote || m.bytes == 0) throw ConfigError("bind_multicast: buffer is not hosted by this GPU");
    if (m.own_handle) {
        const std::int64_t gran = 2ll << 20;
        mc.bind(cfg_.device, m.handle, 0, (m.bytes + gran - 1) / gran * gran);
        return;
    }
    if (!m.mapped_vmm) throw ConfigError("bind_multicast: buffer is not VMM-backed");
    const std::int64_t C = cfg_.chunk_bytes;
    for (size_t c = 0; c < m.phys.size(); ++c)
        mc.bind(cfg_.device, handles_[static_cast<size_t>(m.phys[c])], static_cast<std::int64_t>(c) * C, C);
}

namespace {
CUmulticastObjectProp mc_prop(std::int64_t bytes, int n) {
    CUmulticastObjectProp p = {};
    p.numDevices = static_cast<unsigned>(n);
    p.size = static_cast<size_t>(bytes);
    p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return p;
}
}  // namespace

Multicast::Multicast(std::int64_t bytes, int n_devices) : bytes_(bytes) {
    const Drv& D = Drv::get();
    const CUmulticastObjectProp p = mc_prop(bytes, n_devices);
    size_t gran = 0;
    drv_check(D.mc_granularity(&gran, &p, CU_MULTICAST_GRANULARITY_MINIMUM), "cuMulticastGetGranularity");
    if (bytes % static_cast<std::int64_t>(gran)) throw ConfigError("multicast size is not a multiple of its granularity");
    CUmemGenericAllocationHandle h;
    drv_check(D.mc_create(&h, &p), "cuMulticastCreate");
    handle_ = h;
}

Multicast::Multicast(int fd, std::int64_t bytes) : bytes_(bytes) {
    const Drv& D = Drv::get();
    CUmemGenericAllocationHandle h;
    const CUresult r = D.import_fd(&h, reinterpret_cast<void*>(static_cast<std::intptr_t>(fd)),
                                   CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    ::close(fd);
    drv_check(r, "cuMemImportFromShareableHandle (multicast)");
    handle_ = h;
}

Multicast::~Multicast() {
    const Drv& D = Drv::get();
    if (va_) {
        D.unmap(va_, static_cast<size_t>(bytes_));
        D.addr_free(va_, static_cast<size_t>(bytes_));
    }
    for (const Binding& b : bindings_) {
        CUdevice dev;
        if (D.device_get(&dev, b.device) == CUDA_SUCCESS)
            D.mc_unbind(handle_, dev, static_cast<size_t>(b.offset), static_cast<size_t>(b.bytes));
    }
    if (handle_) D.release(handle_);
}

int Multicast::export_fd() const {
    int fd = -1;
    drv_check(Drv::get().export_fd(&fd, handle_, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
              "cuMemExportToShareableHandle (multicast)");
    return fd;
}

void Multicast::add_device(int device) {
    const Drv& D = Drv::get();
    CUdevice dev;
    drv_check(D.device_get(&dev, device), "cuDeviceGet");
    drv_check(D.mc_add(handle_, dev), "cuMulticastAddDevice");
}

void Multicast::bind(int device, std::uint64_t mem_handle, std::int64_t mc_offset, std::int64_t bytes) {
    if (mc_offset + bytes > bytes_) throw ConfigError("multicast bind beyond the object");
    if (cudaSetDevice(device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    drv_check(Drv::get().mc_bind(handle_, static_cast<size_t>(mc_offset), mem_handle, 0, static_cast<size_t>(bytes), 0),
              "cuMulticastBindMem");
    bindings_.push_back({device, mc_offset, bytes});
}

void* Multicast::map(int device) {
    if (va_) return reinterpret_cast<void*>(va_);
    const Drv& D = Drv::get();
    if (cudaSetDevice(device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    const CUmulticastObjectProp p = mc_prop(bytes_, 1);
    size_t gran = 0;
    drv_check(D.mc_granularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    CUdeviceptr va = 0;
    drv_check(D.reserve(&va, static_cast<size_t>(bytes_), gran, 0, 0), "cuMemAddressReserve (multicast)");
    drv_check(D.map(va, static_cast<size_t>(bytes_), 0, handle_, 0), "cuMemMap (multicast)");
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    drv_check(D.set_access(va, static_cast<size_t>(bytes_), &acc, 1), "cuMemSetAccess (multicast)");
    va_ = va;
    return reinterpret_cast<void*>(va_);
}

}  // namespace mem
}  // namespace reshard
