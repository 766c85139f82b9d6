// NVLink push bandwidth between 2 B200s (one process, peer access): SM vector
// stores vs TMA bulk stores vs copy engine, uni- and bidirectional, CTA count sweep.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("ERR %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(r)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int T, int U>
__global__ void __launch_bounds__(T) push_vec(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
    size_t stride = (size_t)gridDim.x * T;
    size_t i = blockIdx.x * (size_t)T + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = ldnc(s + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) d[i + u * stride] = r[u];
    }
    for (; i < n; i += stride) d[i] = ldnc(s + i);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int S, int B>
__global__ void __launch_bounds__(32) push_bulk(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar[S];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    size_t nchunks = bytes / B;
    size_t first = blockIdx.x;
    size_t mine = first < nchunks ? (nchunks - first + gridDim.x - 1) / gridDim.x : 0;
    auto load = [&](size_t k) {
        int s = k % S;
        size_t c = first + k * gridDim.x;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(B) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(smem + s * B)), "l"(src + c * B), "r"(B), "r"(smem_u32(&bar[s])) : "memory");
    };
    size_t issued = 0;
    for (; issued < S - 1 && issued < mine; ++issued) load(issued);
    uint32_t par = 0;
    for (size_t k = 0; k < mine; ++k) {
        int s = k % S;
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" :: "r"(smem_u32(&bar[s])), "r"((par >> s) & 1) : "memory");
        par ^= 1u << s;
        size_t c = first + k * gridDim.x;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + c * B), "r"(smem_u32(smem + s * B)), "r"(B) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (issued < mine) load(issued++);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int n = 0;
    CR(cudaGetDeviceCount(&n));
    if (n < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t bytes = 4ull << 30;
    char *src[2], *dst[2];
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    for (int g = 0; g < 2; ++g) {
        CR(cudaSetDevice(g));
        CR(cudaDeviceEnablePeerAccess(1 - g, 0));
        CR(cudaMalloc(&src[g], bytes));
        CR(cudaMalloc(&dst[g], bytes));
        CR(cudaMemset(src[g], g + 1, bytes));
        CR(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
        cudaEventCreate(&e0[g]);
        cudaEventCreate(&e1[g]);
        CR(cudaFuncSetAttribute(push_bulk<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
    }
    // mode: 0 vec, 1 bulk, 2 CE; dirs: 1 = GPU0->1 only, 2 = both
    auto run = [&](int mode, int dirs, int ctas, const char* name) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            for (int g = 0; g < dirs; ++g) {
                CR(cudaSetDevice(g));
                cudaEventRecord(e0[g], st[g]);
                char* remote = dst[1 - g];
                if (mode == 0) push_vec<512, 4><<<ctas, 512, 0, st[g]>>>((const uint4*)src[g], (uint4*)remote, bytes / 16);
                else if (mode == 1) push_bulk<4, 32768><<<ctas, 32, 4 * 32768, st[g]>>>(src[g], remote, bytes);
                else if (mode == 3) push_vec<512, 4><<<ctas, 512, 0, st[g]>>>((const uint4*)src[1 - g], (uint4*)dst[g], bytes / 16);  // pull
                else if (mode == 4) push_vec<512, 8><<<ctas, 512, 0, st[g]>>>((const uint4*)src[1 - g], (uint4*)dst[g], bytes / 16);  // pull, deeper
                else if (mode == 5) push_bulk<4, 32768><<<ctas, 32, 4 * 32768, st[g]>>>(src[1 - g], dst[g], bytes);  // TMA pull
                else cudaMemcpyPeerAsync(remote, 1 - g, src[g], g, bytes, st[g]);
                cudaEventRecord(e1[g], st[g]);
            }
            float worst = 0;
            for (int g = 0; g < dirs; ++g) {
                CR(cudaSetDevice(g));
                cudaEventSynchronize(e1[g]);
                float ms;
                cudaEventElapsedTime(&ms, e0[g], e1[g]);
                worst = ms > worst ? ms : worst;
            }
            if (rep >= 1 && worst < best) best = worst;
        }
        for (int g = 0; g < 2; ++g) { CR(cudaSetDevice(g)); CR(cudaGetLastError()); }
        printf("%-22s dirs=%d ctas=%4d: %.3f ms  %.0f GB/s per direction\n", name, dirs, ctas, best, bytes / best / 1e6);
        return 0;
    };
    for (int dirs = 1; dirs <= 2; ++dirs) {
        for (int ctas : {16, 32, 64, 148, 296, 592}) run(0, dirs, ctas, "SM vec 512x4");
        for (int ctas : {16, 32, 64, 148, 296}) run(1, dirs, ctas, "TMA bulk 4x32K");
        run(2, dirs, 0, "CE cudaMemcpyPeer");
        for (int ctas : {148, 296, 592}) run(3, dirs, ctas, "SM vec PULL 512x4");
        for (int ctas : {148, 296}) run(4, dirs, ctas, "SM vec PULL 512x8");
        for (int ctas : {148, 296}) run(5, dirs, ctas, "TMA bulk PULL 4x32K");
    }
    std::vector<char> h(16);
    CR(cudaSetDevice(1));
    CR(cudaMemcpy(h.data(), dst[1] + bytes - 16, 16, cudaMemcpyDeviceToHost));
    printf("check %d\n", h[3] == 1);
    return 0;
}
