// Probe: VMM map/unmap cost, local copy bandwidth (16-B vector kernel vs cudaMemcpy).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <chrono>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("ERR %s line %d: %s\n", #x, __LINE__, s); return 1; } } while (0)
#define CR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(r)); return 1; } } while (0)
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

__global__ void copy16(const int4* __restrict__ s, int4* __restrict__ d, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 a = s[i], b = s[i + stride], c = s[i + 2 * stride], e = s[i + 3 * stride];
    d[i] = a; d[i + stride] = b; d[i + 2 * stride] = c; d[i + 3 * stride] = e;
  }
  for (; i < n; i += stride) d[i] = s[i];
}

int main() {
  CR(cudaSetDevice(0));
  CR(cudaFree(0));
  size_t fr, tot; CR(cudaMemGetInfo(&fr, &tot));
  printf("mem free %.2f GB total %.2f GB\n", fr / 1e9, tot / 1e9);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); printf("SMs %d\n", sms);
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran; CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  size_t rgran; CK(cuMemGetAllocationGranularity(&rgran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("granularity min %zu rec %zu\n", gran, rgran);
  for (size_t chunk : {(size_t)64 << 20, (size_t)512 << 20, (size_t)2 << 30}) {
    int n = (int)((16ull << 30) / chunk);
    std::vector<CUmemGenericAllocationHandle> h(n);
    double t0 = now();
    for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], chunk, &prop, 0));
    double t1 = now();
    CUdeviceptr va; CK(cuMemAddressReserve(&va, chunk * n, 0, 0, 0));
    double t2 = now();
    for (int i = 0; i < n; ++i) CK(cuMemMap(va + i * chunk, chunk, 0, h[i], 0));
    double t3 = now();
    CUmemAccessDesc ad = {}; ad.location = prop.location; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(va, chunk * n, &ad, 1));
    double t4 = now();
    CR(cudaMemset((void*)va, 1, chunk * n)); CR(cudaDeviceSynchronize());
    double t5 = now();
    CK(cuMemUnmap(va, chunk * n));
    double t6 = now();
    for (int i = 0; i < n; ++i) CK(cuMemRelease(h[i]));
    double t7 = now();
    CK(cuMemAddressFree(va, chunk * n));
    printf("VMM 16GB in %d chunks of %zu MB: create %.3f ms, reserve %.3f, map %.3f, setaccess %.3f, memset %.3f, unmap %.3f, release %.3f ms\n",
           n, chunk >> 20, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3, (t6 - t5) * 1e3, (t7 - t6) * 1e3);
  }
  // remap cost: keep physical handles, map/setaccess/unmap repeatedly
  {
    size_t chunk = 1ull << 30; int n = 16;
    std::vector<CUmemGenericAllocationHandle> h(n);
    for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], chunk, &prop, 0));
    CUdeviceptr va; CK(cuMemAddressReserve(&va, chunk * n, 0, 0, 0));
    CUmemAccessDesc ad = {}; ad.location = prop.location; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int rep = 0; rep < 3; ++rep) {
      double t0 = now();
      for (int i = 0; i < n; ++i) { CK(cuMemMap(va + i * chunk, chunk, 0, h[(i + rep) % n], 0)); CK(cuMemSetAccess(va + i * chunk, chunk, &ad, 1)); }
      double t1 = now();
      CK(cuMemUnmap(va, chunk * n));
      double t2 = now();
      printf("remap 16x1GB: map+access %.3f ms, unmap %.3f ms\n", (t1 - t0) * 1e3, (t2 - t1) * 1e3);
    }
    for (int i = 0; i < n; ++i) CK(cuMemRelease(h[i]));
    CK(cuMemAddressFree(va, chunk * n));
  }
  // copy bandwidth
  size_t bytes = 8ull << 30;
  void *a, *b; CR(cudaMalloc(&a, bytes)); CR(cudaMalloc(&b, bytes));
  CR(cudaMemset(a, 3, bytes)); CR(cudaMemset(b, 0, bytes));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy16<<<blocks, 256>>>((const int4*)a, (int4*)b, bytes / 16);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) printf("copy16 blocks=%d: %.3f ms, %.1f GB/s (r+w)\n", blocks, ms, 2.0 * bytes / ms / 1e6);
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 2) printf("cudaMemcpy D2D: %.3f ms, %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
  }
  CR(cudaGetLastError());
  printf("done\n");
  return 0;
}
