// GPU planner: expands the ZeRO optimizer moves of a PlanCore (stair::Triple
// records, one per (src k, dst j, tensor)) into the reference's flat SliceTransfer
// runs, bit-exact with plan_optimizer + resolve_peers (routing.hpp:287-337,
// :360-396) — which takes hours on the reference's O(n*m) interval lists at
// Llama-3-8B scale.
//
// One thread per tensor row of every triple. A row yields 0..2 runs
// ((J ∩ K) \ I, stair.hpp); it continues the previous run when its first piece
// starts exactly where the previous row's last piece ended (same src/dst), which is
// precisely normalize_intervals' abutting-merge rule. Pass 1 counts new runs per
// row, a device-wide exclusive scan (CUB) assigns run indices, pass 2 writes lo at
// run starts and folds hi with atomicMax along continuation chains (hi only grows
// along a chain, so the result is deterministic).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <stdexcept>
#include <vector>

#include "reshard/executor_rt.hpp"
#include "reshard/plan_core.hpp"

namespace reshard {
namespace gpuplan {

namespace {

#define RS_CUDA_P(x)                                                                                      \
    do {                                                                                                  \
        cudaError_t e_ = (x);                                                                             \
        if (e_ != cudaSuccess)                                                                            \
            throw exec::CudaError(strfmt("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__)); \
    } while (0)

__device__ __forceinline__ int find_triple(const long long* __restrict__ row_off, int n, long long g) {
    int lo = 0, hi = n - 1;  // largest t with row_off[t] <= g
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (row_off[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

/// runs of row g and whether its first run continues the previous row's last run
__device__ __forceinline__ int row_eval(const stair::Triple* __restrict__ T, const long long* __restrict__ row_off,
                                        int ntrip, long long g, stair::Iv out[2], int* ti_out, bool* cont) {
    const int ti = find_triple(row_off, ntrip, g);
    const stair::Triple& X = T[ti];
    const long long q = g - row_off[ti];
    const int n = stair::triple_row_runs(X, q, out);
    *ti_out = ti;
    *cont = false;
    if (n == 0) return 0;
    stair::Iv prev[2];
    int pn = 0;
    if (q > 0) {
        pn = stair::triple_row_runs(X, q - 1, prev);
    } else if (ti > 0 && T[ti - 1].src == X.src && T[ti - 1].dst == X.dst) {
        pn = stair::triple_row_runs(T[ti - 1], T[ti - 1].nrows - 1, prev);
    }
    *cont = pn > 0 && prev[pn - 1].hi == out[0].lo;
    return n;
}

__global__ void count_kernel(const stair::Triple* __restrict__ T, const long long* __restrict__ row_off, int ntrip,
                             long long nrows, int* __restrict__ starts) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nrows; g += (long long)gridDim.x * blockDim.x) {
        stair::Iv r[2];
        int ti;
        bool cont;
        const int n = row_eval(T, row_off, ntrip, g, r, &ti, &cont);
        starts[g] = n - (cont ? 1 : 0);
    }
}

__global__ void write_kernel(const stair::Triple* __restrict__ T, const long long* __restrict__ row_off, int ntrip,
                             long long nrows, const int* __restrict__ idx, core::FlatXfer* __restrict__ out) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nrows; g += (long long)gridDim.x * blockDim.x) {
        stair::Iv r[2];
        int ti;
        bool cont;
        const int n = row_eval(T, row_off, ntrip, g, r, &ti, &cont);
        int run = idx[g] - (cont ? 1 : 0);
        for (int i = 0; i < n; ++i, ++run) {
            core::FlatXfer* f = out + run;
            if (!(i == 0 && cont)) {
                f->lo = r[i].lo;
                f->src = T[ti].src;
                f->dst = T[ti].dst;
            }
            atomicMax(reinterpret_cast<unsigned long long*>(&f->hi), static_cast<unsigned long long>(r[i].hi));
        }
    }
}

}  // namespace

/// Expand on `device`. Runs of D2-overridden destinations come from the host plan.
std::vector<core::FlatXfer> expand_flat_gpu(const core::PlanCore& P, int device, double* kernel_ms) {
    RS_CUDA_P(cudaSetDevice(device));
    std::vector<stair::Triple> trip;
    std::vector<char> d2(static_cast<size_t>(P.dst_cfg.world_size()), 0);
    for (const core::FlatXfer& f : P.d2_runs) d2[static_cast<size_t>(f.dst)] = 1;
    for (const stair::Triple& T : P.triples)
        if (!d2[static_cast<size_t>(T.dst)]) trip.push_back(T);
    std::vector<core::FlatXfer> out;
    if (!trip.empty()) {
        std::vector<long long> off(trip.size());
        long long nrows = 0;
        for (size_t i = 0; i < trip.size(); ++i) off[i] = nrows, nrows += trip[i].nrows;
        stair::Triple* dT = nullptr;
        long long* dOff = nullptr;
        int *dStarts = nullptr, *dIdx = nullptr;
        core::FlatXfer* dOut = nullptr;
        void* dTmp = nullptr;
        size_t tmp_bytes = 0;
        cudaStream_t s = nullptr;
        cudaEvent_t e0, e1, ea, eb;  // kernel time = [e0, ea] (count + scan) + [eb, e1] (write)
        RS_CUDA_P(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        RS_CUDA_P(cudaEventCreate(&e0));
        RS_CUDA_P(cudaEventCreate(&e1));
        RS_CUDA_P(cudaEventCreate(&ea));
        RS_CUDA_P(cudaEventCreate(&eb));
        try {
            RS_CUDA_P(cudaMalloc(&dT, trip.size() * sizeof(stair::Triple)));
            RS_CUDA_P(cudaMalloc(&dOff, off.size() * sizeof(long long)));
            RS_CUDA_P(cudaMalloc(&dStarts, static_cast<size_t>(nrows + 1) * sizeof(int)));
            RS_CUDA_P(cudaMalloc(&dIdx, static_cast<size_t>(nrows + 1) * sizeof(int)));
            RS_CUDA_P(cudaMemcpyAsync(dT, trip.data(), trip.size() * sizeof(stair::Triple), cudaMemcpyHostToDevice, s));
            RS_CUDA_P(cudaMemcpyAsync(dOff, off.data(), off.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
            RS_CUDA_P(cudaMemsetAsync(dStarts + nrows, 0, sizeof(int), s));
            cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, dStarts, dIdx, nrows + 1, s);
            RS_CUDA_P(cudaMalloc(&dTmp, tmp_bytes));
            const int threads = 256;
            const long long want = (nrows + threads - 1) / threads;
            const int blocks = static_cast<int>(want < 148 * 64 ? want : 148 * 64);
            RS_CUDA_P(cudaEventRecord(e0, s));
            count_kernel<<<blocks, threads, 0, s>>>(dT, dOff, static_cast<int>(trip.size()), nrows, dStarts);
            cub::DeviceScan::ExclusiveSum(dTmp, tmp_bytes, dStarts, dIdx, nrows + 1, s);
            RS_CUDA_P(cudaEventRecord(ea, s));
            int total = 0;
            RS_CUDA_P(cudaMemcpyAsync(&total, dIdx + nrows, sizeof(int), cudaMemcpyDeviceToHost, s));
            RS_CUDA_P(cudaStreamSynchronize(s));
            RS_CUDA_P(cudaMalloc(&dOut, static_cast<size_t>(total > 0 ? total : 1) * sizeof(core::FlatXfer)));
            RS_CUDA_P(cudaMemsetAsync(dOut, 0, static_cast<size_t>(total > 0 ? total : 1) * sizeof(core::FlatXfer), s));
            RS_CUDA_P(cudaEventRecord(eb, s));
            write_kernel<<<blocks, threads, 0, s>>>(dT, dOff, static_cast<int>(trip.size()), nrows, dIdx, dOut);
            RS_CUDA_P(cudaEventRecord(e1, s));
            RS_CUDA_P(cudaGetLastError());
            out.resize(static_cast<size_t>(total));
            RS_CUDA_P(cudaMemcpyAsync(out.data(), dOut, static_cast<size_t>(total) * sizeof(core::FlatXfer),
                                      cudaMemcpyDeviceToHost, s));
            RS_CUDA_P(cudaStreamSynchronize(s));
            float m1 = 0, m2 = 0;
            cudaEventElapsedTime(&m1, e0, ea);
            cudaEventElapsedTime(&m2, eb, e1);
            if (kernel_ms) *kernel_ms = m1 + m2;
        } catch (...) {
            cudaFree(dT), cudaFree(dOff), cudaFree(dStarts), cudaFree(dIdx), cudaFree(dOut), cudaFree(dTmp);
            cudaStreamDestroy(s);
            throw;
        }
        cudaFree(dT), cudaFree(dOff), cudaFree(dStarts), cudaFree(dIdx), cudaFree(dOut), cudaFree(dTmp);
        cudaEventDestroy(e0), cudaEventDestroy(e1), cudaEventDestroy(ea), cudaEventDestroy(eb);
        cudaStreamDestroy(s);
    }
    if (P.d2_runs.empty()) return out;
    std::vector<core::FlatXfer> merged;
    merged.reserve(out.size() + P.d2_runs.size());
    auto less = [](const core::FlatXfer& a, const core::FlatXfer& b) {
        if (a.src != b.src) return a.src < b.src;
        if (a.dst != b.dst) return a.dst < b.dst;
        return a.lo < b.lo;
    };
    std::merge(out.begin(), out.end(), P.d2_runs.begin(), P.d2_runs.end(), std::back_inserter(merged), less);
    return merged;
}

}  // namespace gpuplan
}  // namespace reshard
