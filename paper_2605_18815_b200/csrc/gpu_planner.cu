// GPU planner: expands the ZeRO optimizer moves of a PlanCore (stair::Triple
// records, one per (src k, dst j, tensor)) into the reference's flat SliceTransfer
// runs, bit-exact with plan_optimizer + resolve_peers (routing.hpp:287-337,
// :360-396) — which takes hours on the reference's O(n*m) interval lists at
// Llama-3-8B scale.
//
// Boxes (params, grads, replicated optimizer): one thread per (dst rank j, tensor t,
// src rank k) intersects the two ranks' boxes of t — the batched hyper-rectangle
// intersection over all (old shard, new shard) pairs. The reference splits
// D_j \ S_own(j) at the source projection grid and collects the candidates holding each
// cell (routing.hpp:197-279); since the source positions partition every tensor, its
// cells are exactly the non-empty D_j ∩ S_p over source positions p other than own(j)'s,
// with the ranks sharing position p as candidates. The lowest rank of a
// position emits the cell; resolve_peers' proximity rule picks the source on the host.
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

struct DevBox {
    long long lo[4], hi[4];
    int valid;
};

struct DevCell {
    long long lo[4], hi[4];
    unsigned long long cands;  // source ranks holding the cell (bit k)
    int j, t;
};

__device__ __forceinline__ bool same_box(const DevBox& a, const DevBox& b, int nd) {
    for (int d = 0; d < nd; ++d)
        if (a.lo[d] != b.lo[d] || a.hi[d] != b.hi[d]) return false;
    return true;
}

__global__ void box_cells_kernel(const DevBox* __restrict__ S, const DevBox* __restrict__ D, const int* __restrict__ nd_of,
                                 const int* __restrict__ own, int ns, int ndst, int nt, DevCell* __restrict__ out,
                                 unsigned long long* __restrict__ count) {
    const long long total = static_cast<long long>(ndst) * nt * ns;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x) {
        const int k = static_cast<int>(g % ns);
        const int t = static_cast<int>((g / ns) % nt);
        const int j = static_cast<int>(g / (static_cast<long long>(ns) * nt));
        const DevBox& db = D[static_cast<long long>(j) * nt + t];
        const DevBox& sb = S[static_cast<long long>(k) * nt + t];
        if (!db.valid || !sb.valid) continue;
        const int nd = nd_of[t];
        bool lowest = true;  // k is the lowest rank of its source position
        unsigned long long cands = 0;
        for (int q = 0; q < ns; ++q) {
            const DevBox& x = S[static_cast<long long>(q) * nt + t];
            if (x.valid && same_box(x, sb, nd)) {
                if (q < k) lowest = false;
                cands |= 1ull << q;
            }
        }
        if (!lowest) continue;
        const int o = own[j];
        if (o >= 0 && S[static_cast<long long>(o) * nt + t].valid && same_box(S[static_cast<long long>(o) * nt + t], sb, nd))
            continue;  // retained on the device, not moved
        DevCell c;
        bool empty = false;
        for (int d = 0; d < nd; ++d) {
            c.lo[d] = db.lo[d] > sb.lo[d] ? db.lo[d] : sb.lo[d];
            c.hi[d] = db.hi[d] < sb.hi[d] ? db.hi[d] : sb.hi[d];
            empty = empty || c.lo[d] >= c.hi[d];
        }
        if (empty) continue;
        for (int d = nd; d < 4; ++d) c.lo[d] = c.hi[d] = 0;
        c.cands = cands;
        c.j = j;
        c.t = t;
        out[atomicAdd(count, 1ull)] = c;
    }
}

}  // namespace

std::vector<core::BoxXfer> box_routes_gpu(const core::PlanCore& P, int device, double* kernel_ms) {
    const int ns = P.src_cfg.world_size(), ndst = P.dst_cfg.world_size();
    const int nt = P.ntensors();
    if (ns > 64) throw ConfigError("GPU box planner: more than 64 source ranks");
    if (P.opts.balance_fanout) {  // the round-robin cursor follows the reference's pending order
        if (kernel_ms) *kernel_ms = 0;
        return P.box;
    }
    std::vector<DevBox> S(static_cast<size_t>(ns) * nt), D(static_cast<size_t>(ndst) * nt);
    auto fill = [&](const core::Side& side, std::vector<DevBox>& v) {
        for (size_t r = 0; r < side.ranks.size(); ++r)
            for (int t = 0; t < nt; ++t) {
                DevBox& b = v[r * static_cast<size_t>(nt) + static_cast<size_t>(t)];
                const int si = side.ranks[r].seg_of[static_cast<size_t>(t)];
                b.valid = si >= 0;
                for (int d = 0; d < 4; ++d) b.lo[d] = b.hi[d] = 0;
                if (si >= 0)
                    for (int d = 0; d < 4; ++d) {
                        b.lo[d] = side.ranks[r].segs[static_cast<size_t>(si)].blo[d];
                        b.hi[d] = side.ranks[r].segs[static_cast<size_t>(si)].bhi[d];
                    }
            }
    };
    fill(P.src, S);
    fill(P.dst, D);
    std::vector<int> nd_of(static_cast<size_t>(nt)), own(static_cast<size_t>(ndst), -1);
    for (int t = 0; t < nt; ++t) nd_of[static_cast<size_t>(t)] = static_cast<int>(P.space->entries()[static_cast<size_t>(t)].spec.shape.size());
    for (int j = 0; j < ndst; ++j) own[static_cast<size_t>(j)] = P.wm.src_rank_of(P.wm.dst_phys[static_cast<size_t>(j)]);
    const long long total = static_cast<long long>(ndst) * nt * ns;
    std::vector<DevCell> cells;
    {
        RS_CUDA_P(cudaSetDevice(device));
        DevBox *dS = nullptr, *dD = nullptr;
        int *dNd = nullptr, *dOwn = nullptr;
        DevCell* dOut = nullptr;
        unsigned long long* dCount = nullptr;
        cudaStream_t st = nullptr;
        cudaEvent_t e0, e1;
        RS_CUDA_P(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        RS_CUDA_P(cudaEventCreate(&e0));
        RS_CUDA_P(cudaEventCreate(&e1));
        auto release = [&] {
            cudaFree(dS), cudaFree(dD), cudaFree(dNd), cudaFree(dOwn), cudaFree(dOut), cudaFree(dCount);
            cudaEventDestroy(e0), cudaEventDestroy(e1);
            cudaStreamDestroy(st);
        };
        try {
            RS_CUDA_P(cudaMalloc(&dS, S.size() * sizeof(DevBox)));
            RS_CUDA_P(cudaMalloc(&dD, D.size() * sizeof(DevBox)));
            RS_CUDA_P(cudaMalloc(&dNd, nd_of.size() * sizeof(int)));
            RS_CUDA_P(cudaMalloc(&dOwn, own.size() * sizeof(int)));
            RS_CUDA_P(cudaMalloc(&dOut, static_cast<size_t>(total > 0 ? total : 1) * sizeof(DevCell)));
            RS_CUDA_P(cudaMalloc(&dCount, sizeof(unsigned long long)));
            RS_CUDA_P(cudaMemcpyAsync(dS, S.data(), S.size() * sizeof(DevBox), cudaMemcpyHostToDevice, st));
            RS_CUDA_P(cudaMemcpyAsync(dD, D.data(), D.size() * sizeof(DevBox), cudaMemcpyHostToDevice, st));
            RS_CUDA_P(cudaMemcpyAsync(dNd, nd_of.data(), nd_of.size() * sizeof(int), cudaMemcpyHostToDevice, st));
            RS_CUDA_P(cudaMemcpyAsync(dOwn, own.data(), own.size() * sizeof(int), cudaMemcpyHostToDevice, st));
            RS_CUDA_P(cudaMemsetAsync(dCount, 0, sizeof(unsigned long long), st));
            const int threads = 256;
            const long long want = (total + threads - 1) / threads;
            const int blocks = static_cast<int>(want < 148 * 16 ? (want > 0 ? want : 1) : 148 * 16);
            RS_CUDA_P(cudaEventRecord(e0, st));
            box_cells_kernel<<<blocks, threads, 0, st>>>(dS, dD, dNd, dOwn, ns, ndst, nt, dOut, dCount);
            RS_CUDA_P(cudaEventRecord(e1, st));
            RS_CUDA_P(cudaGetLastError());
            unsigned long long n = 0;
            RS_CUDA_P(cudaMemcpyAsync(&n, dCount, sizeof n, cudaMemcpyDeviceToHost, st));
            RS_CUDA_P(cudaStreamSynchronize(st));
            cells.resize(static_cast<size_t>(n));
            RS_CUDA_P(cudaMemcpyAsync(cells.data(), dOut, static_cast<size_t>(n) * sizeof(DevCell), cudaMemcpyDeviceToHost, st));
            RS_CUDA_P(cudaStreamSynchronize(st));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (kernel_ms) *kernel_ms = ms;
        } catch (...) {
            release();
            throw;
        }
        release();
    }
    // resolve_peers' proximity rule (routing.hpp:360-396): the first candidate on the
    // destination's node, else the lowest rank; then every kind the plan moves as boxes
    std::vector<core::BoxXfer> out;
    const bool grads = P.opts.gradients == GradientPolicy::Migrate;
    const bool optim_boxes = !P.src_cfg.zero_enabled;
    out.reserve(cells.size() * (1 + grads + optim_boxes));
    for (const DevCell& c : cells) {
        const int dphys = P.wm.dst_phys[static_cast<size_t>(c.j)];
        int chosen = -1;
        for (int k = 0; k < ns && chosen < 0; ++k)
            if ((c.cands >> k) & 1ull)
                if (P.topo.same_node(P.wm.src_phys[static_cast<size_t>(k)], dphys)) chosen = k;
        for (int k = 0; k < ns && chosen < 0; ++k)
            if ((c.cands >> k) & 1ull) chosen = k;
        core::BoxXfer x;
        x.tensor = c.t;
        x.count = 1;
        for (int d = 0; d < 4; ++d) {
            x.lo[d] = c.lo[d];
            x.hi[d] = c.hi[d];
        }
        for (int d = 0; d < nd_of[static_cast<size_t>(c.t)]; ++d) x.count *= c.hi[d] - c.lo[d];
        x.src = chosen;
        x.dst = c.j;
        for (int kind : {0, 2, 1}) {
            if ((kind == 2 && !grads) || (kind == 1 && !optim_boxes)) continue;
            x.kind = kind;
            x.bytes = x.count * core::payload_width(*P.space, kind, c.t);
            out.push_back(x);
        }
    }
    std::sort(out.begin(), out.end(), [&](const core::BoxXfer& a, const core::BoxXfer& b) { return core::box_xfer_less(P, a, b); });
    return out;
}

/// Expand on `device`. Runs of D2-overridden destinations come from the host plan.
std::vector<core::FlatXfer> expand_flat_gpu(const core::PlanCore& P, int device, double* kernel_ms) {
    RS_CUDA_P(cudaSetDevice(device));
    const std::vector<stair::Triple>& trip = P.triples;
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
    // D2 extension: the runs inside over-sourced intervals are replaced (host, a few
    // hundred intervals)
    return core::apply_d2(P, std::move(out));
}

}  // namespace gpuplan
}  // namespace reshard
