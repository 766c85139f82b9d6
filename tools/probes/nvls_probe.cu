// NVLS multicast probe (single process, N GPUs): is multicast supported, and what
// bandwidth does a multimem.st broadcast from GPU0 reach into all N GPUs' memory?
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("ERR %s line %d: %s\n", #x, __LINE__, s); return 1; } } while (0)
#define CR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("ERR %s:%d %s\n", #x, __LINE__, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void mc_store(const uint4* __restrict__ src, uint4* mc, size_t n) {
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        uint4 v = src[i];
        asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    }
}

int main(int argc, char** argv) {
    // argv[1] == "unbound-root": GPU 0 joins the multicast object but binds no memory
    const bool unbound_root = argc > 1 && std::string(argv[1]) == "unbound-root";
    // "self-src": the root reads the very memory it has bound (the executor's layout identity)
    const bool self_src = argc > 1 && std::string(argv[1]) == "self-src";
    CK(cuInit(0));
    int n = 0;
    CR(cudaGetDeviceCount(&n));
    for (int d = 0; d < n; ++d) {
        int mc = 0;
        CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
        printf("device %d multicast supported: %d\n", d, mc);
    }
    const size_t bytes = 1ull << 30;
    CUmulticastObjectProp mp = {};
    mp.numDevices = n;
    mp.size = bytes;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("multicast granularity %zu\n", gran);
    CUmemGenericAllocationHandle mch;
    CK(cuMulticastCreate(&mch, &mp));
    std::vector<CUmemGenericAllocationHandle> phys(n);
    for (int d = 0; d < n; ++d) {
        CUdevice dev;
        CK(cuDeviceGet(&dev, d));
        CK(cuMulticastAddDevice(mch, dev));
    }
    std::vector<CUdeviceptr> uc(n);
    for (int d = 0; d < n; ++d) {
        CR(cudaSetDevice(d));
        if (d == 0 && unbound_root) continue;
        CUmemAllocationProp p = {};
        p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        p.location.id = d;
        p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CK(cuMemCreate(&phys[d], bytes, &p, 0));
        CK(cuMulticastBindMem(mch, 0, phys[d], 0, bytes, 0));
        CK(cuMemAddressReserve(&uc[d], bytes, gran, 0, 0));
        CK(cuMemMap(uc[d], bytes, 0, phys[d], 0));
        CUmemAccessDesc a = {};
        a.location = p.location;
        a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CK(cuMemSetAccess(uc[d], bytes, &a, 1));
        CR(cudaMemset((void*)uc[d], 0, bytes));
    }
    CR(cudaSetDevice(0));
    CUdeviceptr mcva;
    CK(cuMemAddressReserve(&mcva, bytes, gran, 0, 0));
    CK(cuMemMap(mcva, bytes, 0, mch, 0));
    CUmemAccessDesc a = {};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = 0;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(mcva, bytes, &a, 1));
    void* src;
    if (self_src) {
        src = (void*)uc[0];
    } else {
        CR(cudaMalloc(&src, bytes));
    }
    CR(cudaMemset(src, 0x5A, bytes));
    CR(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int ctas : {148, 296, 592}) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            mc_store<<<ctas, 512>>>((const uint4*)src, (uint4*)mcva, bytes / 16);
            cudaEventRecord(e1);
            CR(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep && ms < best) best = ms;
        }
        CR(cudaGetLastError());
        printf("multimem.st broadcast to %d GPUs, ctas %d: %.3f ms, %.0f GB/s source rate (%.0f GB/s delivered)\n", n, ctas,
               best, bytes / best / 1e6, (double)n * bytes / best / 1e6);
    }
    int ok = 1;
    for (int d = unbound_root ? 1 : 0; d < n; ++d) {
        CR(cudaSetDevice(d));
        unsigned char h[16];
        CR(cudaMemcpy(h, (void*)(uc[d] + bytes - 16), 16, cudaMemcpyDeviceToHost));
        ok &= h[7] == 0x5A;
    }
    printf("check %d\n", ok);
    return 0;
}
