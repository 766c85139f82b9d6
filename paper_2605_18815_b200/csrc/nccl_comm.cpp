// Non-blocking NCCL communicator construction for the EDM (reshard/nccl_comm.hpp).
#include "reshard/nccl_comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <thread>

#include "reshard/common.hpp"
#include "reshard/executor_rt.hpp"

namespace reshard {
namespace edm {

namespace {

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank_config)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
    ncclResult_t (*split)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*async_error)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*finalize)(ncclComm_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*version)(int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    static const Nccl& get() {
        static Nccl n = [] {
            Nccl x;
            // the NCCL already in the process (torch's) if any, else the system one
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) throw exec::CudaError(std::string("libnccl.so.2 not loadable: ") + dlerror());
            auto sym = [h](const char* name, auto& fn) {
                void* f = dlsym(h, name);
                if (!f) throw exec::CudaError(std::string("NCCL symbol missing: ") + name);
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(f);
            };
            sym("ncclGetUniqueId", x.get_unique_id);
            sym("ncclCommInitRankConfig", x.init_rank_config);
            sym("ncclCommSplit", x.split);
            sym("ncclCommGetAsyncError", x.async_error);
            sym("ncclCommFinalize", x.finalize);
            sym("ncclCommDestroy", x.destroy);
            sym("ncclAllReduce", x.all_reduce);
            sym("ncclGetVersion", x.version);
            sym("ncclGetErrorString", x.error_string);
            return x;
        }();
        return n;
    }
};

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        throw exec::CudaError(strfmt("%s failed: %s", what, Nccl::get().error_string(r)));
}

/// poll a non-blocking communicator until its pending operation completes
void wait_ready(ncclComm_t c, const char* what) {
    const Nccl& N = Nccl::get();
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        ncclResult_t st = ncclSuccess;
        check(N.async_error(c, &st), "ncclCommGetAsyncError");
        if (st == ncclSuccess) return;
        if (st != ncclInProgress) throw exec::CudaError(strfmt("%s: %s", what, N.error_string(st)));
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
            throw exec::CudaError(strfmt("%s: still in progress after 300 s", what));
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

ncclConfig_t nonblocking_config() {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    cfg.splitShare = 1;  // the per-dimension splits share the world communicator's resources
    return cfg;
}

/// non-blocking communicators: finalize (flush), wait, then destroy
void destroy_comm(void* c) {
    if (!c) return;
    const Nccl& N = Nccl::get();
    ncclComm_t comm = static_cast<ncclComm_t>(c);
    if (N.finalize(comm) == ncclInProgress) {
        try {
            wait_ready(comm, "ncclCommFinalize");
        } catch (...) {
        }
    }
    N.destroy(comm);
}

double since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

void nccl_unique_id(std::uint8_t out[kNcclIdBytes]) {
    static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId size");
    ncclUniqueId id;
    check(Nccl::get().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
}

std::string nccl_version() {
    int v = 0;
    check(Nccl::get().version(&v), "ncclGetVersion");
    return strfmt("%d.%d.%d", v / 10000, (v / 100) % 100, v % 100);
}

CommCache::~CommCache() {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& kv : cache_) {
        CommSet& s = *kv.second;
        cudaSetDevice(s.device);
        for (void*& c : s.dims) destroy_comm(c), c = nullptr;
        destroy_comm(s.world);
        s.world = nullptr;
    }
}

const CommSet& CommCache::get_or_create(const std::string& key, const std::uint8_t uid[kNcclIdBytes], int nranks,
                                        int rank, int device, const int colors[kCommDims], bool* hit) {
    {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = cache_.find(key);
        if (it != cache_.end()) {
            if (hit) *hit = true;
            return *it->second;
        }
    }
    if (hit) *hit = false;
    if (nranks < 1 || rank < 0 || rank >= nranks) throw ConfigError("nccl comm: bad rank / size");
    const Nccl& N = Nccl::get();
    if (cudaSetDevice(device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    auto s = std::make_unique<CommSet>();
    s->nranks = nranks;
    s->rank = rank;
    s->device = device;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclConfig_t cfg = nonblocking_config();
    auto t0 = std::chrono::steady_clock::now();
    ncclComm_t world = nullptr;
    check(N.init_rank_config(&world, nranks, id, rank, &cfg), "ncclCommInitRankConfig");
    s->world = world;
    wait_ready(world, "ncclCommInitRankConfig");
    s->init_s = since(t0);
    t0 = std::chrono::steady_clock::now();
    for (int d = 0; d < kCommDims; ++d) {
        if (!colors || colors[d] < 0) continue;
        // config NULL: the child inherits the parent's (non-blocking) configuration. The
        // split is an operation on the parent too: both must be ready before the next one
        // A non-blocking split may publish the child handle only when it completes, so
        // its destination is the heap-resident CommSet slot, read after the parent is ready
        wait_ready(world, "ncclCommSplit (parent)");
        check(N.split(world, colors[d], rank, reinterpret_cast<ncclComm_t*>(&s->dims[d]), nullptr), "ncclCommSplit");
        wait_ready(world, "ncclCommSplit (parent)");
        void* volatile* slot = &s->dims[d];  // written by NCCL's async thread
        for (int spin = 0; !*slot && spin < 100000; ++spin) std::this_thread::sleep_for(std::chrono::microseconds(100));
        if (!s->dims[d]) throw exec::CudaError("ncclCommSplit: no communicator returned");
        wait_ready(static_cast<ncclComm_t>(s->dims[d]), "ncclCommSplit");
    }
    s->split_s = since(t0);
    std::lock_guard<std::mutex> lk(mu_);
    return *cache_.emplace(key, std::move(s)).first->second;
}

const CommSet* CommCache::find(const std::string& key) const {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = cache_.find(key);
    return it == cache_.end() ? nullptr : it->second.get();
}

float CommCache::check_allreduce(const std::string& key, int dim, cudaStream_t stream) {
    const CommSet* s = find(key);
    if (!s) throw ConfigError("nccl comm: configuration not created");
    void* c = dim < 0 ? s->world : (dim < kCommDims ? s->dims[dim] : nullptr);
    if (!c) throw ConfigError("nccl comm: no communicator for that dimension");
    if (cudaSetDevice(s->device) != cudaSuccess) throw exec::CudaError("cudaSetDevice failed");
    float* d = nullptr;
    if (cudaMalloc(&d, sizeof(float)) != cudaSuccess) throw exec::CudaError("cudaMalloc failed");
    const float one = 1.0f;
    float out = 0.0f;
    try {
        if (cudaMemcpyAsync(d, &one, sizeof one, cudaMemcpyHostToDevice, stream) != cudaSuccess)
            throw exec::CudaError("cudaMemcpyAsync failed");
        check(Nccl::get().all_reduce(d, d, 1, ncclFloat32, ncclSum, static_cast<ncclComm_t>(c), stream), "ncclAllReduce");
        wait_ready(static_cast<ncclComm_t>(c), "ncclAllReduce");
        if (cudaMemcpyAsync(&out, d, sizeof out, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
            cudaStreamSynchronize(stream) != cudaSuccess)
            throw exec::CudaError("all-reduce readback failed");
    } catch (...) {
        cudaFree(d);
        throw;
    }
    cudaFree(d);
    return out;
}

void CommCache::destroy(const std::string& key) {
    std::unique_ptr<CommSet> s;
    {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = cache_.find(key);
        if (it == cache_.end()) return;
        s = std::move(it->second);
        cache_.erase(it);
    }
    cudaSetDevice(s->device);
    for (void* c : s->dims) destroy_comm(c);
    destroy_comm(s->world);
}

}  // namespace edm
}  // namespace reshard
