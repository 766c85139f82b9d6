// Copy-engine peer bandwidth for the executor's op shapes (2 GPUs, one process, peer
// access, both directions at once): contiguous, 2-D strided rows of 6 KiB / 21 KiB /
// 2 KiB (the ZeRO fragment shapes of the north star), and many 512 KiB calls.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("ERR %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(r)); return 1; } } while (0)

int main() {
    int n = 0;
    CR(cudaGetDeviceCount(&n));
    if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
    const size_t bytes = 2ull << 30;
    void *src[2], *dst[2];
    cudaStream_t st[2][2];
    for (int d = 0; d < 2; ++d) {
        CR(cudaSetDevice(d));
        CR(cudaDeviceEnablePeerAccess(1 - d, 0));
        CR(cudaMalloc(&src[d], 2 * bytes));
        CR(cudaMalloc(&dst[d], 2 * bytes));
        CR(cudaMemset(src[d], 1 + d, 2 * bytes));
        for (int s = 0; s < 2; ++s) CR(cudaStreamCreateWithFlags(&st[d][s], cudaStreamNonBlocking));
    }
    struct Case { const char* name; size_t width, spitch, dpitch, call_bytes; };
    const Case cases[] = {
        {"contiguous, 1 call per 256 MiB", 0, 0, 0, 256ull << 20},
        {"contiguous, 1 call per 512 KiB", 0, 0, 0, 512ull << 10},
        {"2D rows 6144 B, src pitch 12288", 6144, 12288, 6144, 64ull << 20},
        {"2D rows 21504 B, src pitch 43008", 21504, 43008, 21504, 64ull << 20},
        {"2D rows 2048 B, src pitch 8192, dst pitch 4096", 2048, 8192, 4096, 64ull << 20},
        {"2D rows 8192 B, src pitch 16384, dst pitch 8192", 8192, 16384, 8192, 64ull << 20},
    };
    for (const Case& c : cases) {
        for (int dir_mode = 0; dir_mode < 2; ++dir_mode) {  // 0: one direction, 1: both
            double best = 1e30, issue_best = 1e30;
            for (int rep = 0; rep < 3; ++rep) {
                for (int d = 0; d < 2; ++d) { CR(cudaSetDevice(d)); CR(cudaDeviceSynchronize()); }
                auto t0 = std::chrono::steady_clock::now();
                for (int d = 0; d < (dir_mode ? 2 : 1); ++d) {
                    CR(cudaSetDevice(d));
                    size_t done = 0;
                    int k = 0;
                    while (done < bytes) {
                        cudaStream_t s = st[d][k++ & 1];
                        const size_t chunk = std::min(c.call_bytes, bytes - done);
                        if (c.width == 0) {
                            CR(cudaMemcpyAsync((char*)dst[1 - d] + done, (char*)src[d] + done, chunk, cudaMemcpyDeviceToDevice, s));
                        } else {
                            const size_t rows = chunk / c.width;
                            const size_t row0 = done / c.width;
                            CR(cudaMemcpy2DAsync((char*)dst[1 - d] + row0 * c.dpitch, c.dpitch, (char*)src[d] + row0 * c.spitch, c.spitch,
                                                 c.width, rows, cudaMemcpyDeviceToDevice, s));
                        }
                        done += chunk;
                    }
                }
                auto t1 = std::chrono::steady_clock::now();
                for (int d = 0; d < 2; ++d) { CR(cudaSetDevice(d)); CR(cudaDeviceSynchronize()); }
                auto t2 = std::chrono::steady_clock::now();
                const double s = std::chrono::duration<double>(t2 - t0).count();
                if (rep && s < best) best = s, issue_best = std::chrono::duration<double>(t1 - t0).count();
            }
            printf("%-50s %s: %7.1f GB/s per direction (host issue %.2f ms)\n", c.name, dir_mode ? "both" : "one ",
                   bytes / best / 1e9, issue_best * 1e3);
        }
    }
    return 0;
}
