// Device-side SynchronizeAll (reshard/sync.hpp).
#include "reshard/sync.hpp"

#include <cstring>

#include "reshard/common.hpp"
#include "reshard/executor_rt.hpp"

namespace reshard {
namespace sync {

#define RS_CUDA_S(x)                                                                                           \
    do {                                                                                                       \
        cudaError_t e_ = (x);                                                                                  \
        if (e_ != cudaSuccess)                                                                                 \
            throw exec::CudaError(strfmt("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__)); \
    } while (0)

namespace {

__device__ __forceinline__ void st_release_sys(std::uint64_t* p, std::uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ std::uint64_t ld_acquire_sys(const std::uint64_t* p) {
    std::uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ std::uint64_t globaltimer() {
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// one CTA, one thread per rank: signal peer `t`, then wait for peer `t`'s signal
__global__ void barrier_kernel(std::uint64_t* const* peers, const std::uint64_t* own, int rank, int world,
                               std::uint64_t epoch, std::uint64_t timeout_ns, std::uint32_t* status) {
    const int t = threadIdx.x;
    if (t < world && t != rank) {
        __threadfence_system();  // this stream's earlier writes (peer pushes) before the flag
        st_release_sys(peers[t] + rank, epoch);
        const std::uint64_t t0 = globaltimer();
        while (ld_acquire_sys(own + t) < epoch) {
            if (globaltimer() - t0 > timeout_ns) {
                atomicExch(status, 1u);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
    __threadfence_system();
}

}  // namespace

DeviceBarrier::DeviceBarrier(int rank, int world, int device) : rank_(rank), world_(world), device_(device) {
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world) throw ConfigError("device barrier: bad rank/world");
    RS_CUDA_S(cudaSetDevice(device));
    RS_CUDA_S(cudaMalloc(&flags_, kMaxRanks * sizeof(std::uint64_t)));
    RS_CUDA_S(cudaMemset(flags_, 0, kMaxRanks * sizeof(std::uint64_t)));
    RS_CUDA_S(cudaMalloc(&status_, sizeof(std::uint32_t)));
    RS_CUDA_S(cudaMemset(status_, 0, sizeof(std::uint32_t)));
    RS_CUDA_S(cudaMalloc(&d_peers_, kMaxRanks * sizeof(std::uint64_t*)));
    RS_CUDA_S(cudaDeviceSynchronize());
    peers_.assign(static_cast<size_t>(world), nullptr);
    peers_[static_cast<size_t>(rank)] = flags_;
}

DeviceBarrier::~DeviceBarrier() {
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (flags_) cudaFree(flags_);
    if (status_) cudaFree(status_);
    if (d_peers_) cudaFree(d_peers_);
}

std::vector<std::uint8_t> DeviceBarrier::export_handle() const {
    cudaIpcMemHandle_t h;
    RS_CUDA_S(cudaSetDevice(device_));
    RS_CUDA_S(cudaIpcGetMemHandle(&h, flags_));
    std::vector<std::uint8_t> v(sizeof h);
    std::memcpy(v.data(), &h, sizeof h);
    return v;
}

void DeviceBarrier::import_handle(int peer, const std::uint8_t* blob, size_t len) {
    if (peer < 0 || peer >= world_) throw ConfigError("device barrier: bad peer");
    if (peer == rank_) return;
    if (len != sizeof(cudaIpcMemHandle_t)) throw ConfigError("device barrier: bad handle");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, blob, sizeof h);
    RS_CUDA_S(cudaSetDevice(device_));
    void* p = nullptr;
    RS_CUDA_S(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    opened_.push_back(p);
    peers_[static_cast<size_t>(peer)] = static_cast<std::uint64_t*>(p);
    dirty_ = true;
}

void DeviceBarrier::arrive_and_wait(cudaStream_t stream) {
    if (world_ == 1) return;
    for (int i = 0; i < world_; ++i)
        if (!peers_[static_cast<size_t>(i)]) throw ConfigError(strfmt("device barrier: rank %d not mapped", i));
    RS_CUDA_S(cudaSetDevice(device_));
    if (dirty_) {
        RS_CUDA_S(cudaMemcpyAsync(d_peers_, peers_.data(), peers_.size() * sizeof(std::uint64_t*), cudaMemcpyHostToDevice,
                                   stream));
        dirty_ = false;
    }
    ++epoch_;
    barrier_kernel<<<1, 64, 0, stream>>>(d_peers_, flags_, rank_, world_, epoch_, timeout_ns_, status_);
    RS_CUDA_S(cudaGetLastError());
}

int DeviceBarrier::status() {
    std::uint32_t s = 0;
    RS_CUDA_S(cudaSetDevice(device_));
    RS_CUDA_S(cudaMemcpy(&s, status_, sizeof s, cudaMemcpyDeviceToHost));
    if (s) RS_CUDA_S(cudaMemset(status_, 0, sizeof s));
    return static_cast<int>(s);
}

}  // namespace sync
}  // namespace reshard
