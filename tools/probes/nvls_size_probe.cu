// How large a multicast object (bound on every GPU, chunk by chunk in 32 MiB pieces of
// separate allocations) can the NVSwitch fabric take? Also the minimum granularity.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("  ERR %s: %s\n", #x, s); return false; } } while (0)

static bool try_size(int n, size_t bytes, size_t piece) {
    CUmulticastObjectProp mp = {};
    mp.numDevices = n;
    mp.size = bytes;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle mch;
    CK(cuMulticastCreate(&mch, &mp));
    for (int d = 0; d < n; ++d) {
        CUdevice dev;
        CK(cuDeviceGet(&dev, d));
        CK(cuMulticastAddDevice(mch, dev));
    }
    std::vector<CUmemGenericAllocationHandle> hs;
    bool ok = true;
    for (int d = 0; d < n && ok; ++d) {
        CUmemAllocationProp p = {};
        p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        p.location.id = d;
        p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        for (size_t off = 0; off < bytes; off += piece) {
            CUmemGenericAllocationHandle h;
            if (cuMemCreate(&h, piece, &p, 0) != CUDA_SUCCESS) { printf("  cuMemCreate failed\n"); ok = false; break; }
            hs.push_back(h);
            CUresult r = cuMulticastBindMem(mch, off, h, 0, piece, 0);
            if (r != CUDA_SUCCESS) {
                const char* s;
                cuGetErrorString(r, &s);
                printf("  bind failed at device %d offset %zu MiB: %s\n", d, off >> 20, s);
                ok = false;
                break;
            }
        }
    }
    for (int d = 0; d < n; ++d) {
        CUdevice dev;
        cuDeviceGet(&dev, d);
        cuMulticastUnbind(mch, dev, 0, bytes);
    }
    for (auto h : hs) cuMemRelease(h);
    cuMemRelease(mch);
    return ok;
}

int main() {
    cuInit(0);
    int n = 0;
    cudaGetDeviceCount(&n);
    for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaFree(0); }
    CUmulticastObjectProp mp = {};
    mp.numDevices = n;
    mp.size = 1 << 30;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gmin = 0, grec = 0;
    cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
    cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("%d GPUs, multicast granularity min %zu rec %zu\n", n, gmin, grec);
    for (size_t gb : {1, 4, 16, 32, 64}) {
        bool ok = try_size(n, gb << 30, 32ull << 20);
        printf("multicast object %zu GiB bound in 32 MiB pieces: %s\n", gb, ok ? "ok" : "FAILED");
        if (!ok) break;
    }
    return 0;
}
