// Copy-kernel variants on one B200: which shape reaches the HBM copy roofline.
// V1 current (512 thr, unroll 4, grid 4x148), V2 grid = residency, V3 256 thr unroll 8,
// V4 TMA bulk (cp.async.bulk g->s->g, mbarrier pipeline), V5 streaming store hints.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("ERR %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(r)); return 1; } } while (0)

struct Tile { uint64_t src, dst, src_pitch, dst_pitch; uint32_t rows, row_bytes; };

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void stcs(uint4* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

template <int T, int U, bool CS>
__global__ void __launch_bounds__(T) copy_v(const Tile* __restrict__ tiles, int ntiles) {
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const Tile tl = tiles[ti];
        const unsigned vpr = tl.row_bytes / 16;
        if (tl.rows == 1) {
            const uint4* s = reinterpret_cast<const uint4*>(tl.src);
            uint4* d = reinterpret_cast<uint4*>(tl.dst);
            unsigned i = threadIdx.x;
            for (; i + (U - 1) * T < vpr; i += U * T) {
                uint4 r[U];
#pragma unroll
                for (int u = 0; u < U; ++u) r[u] = ldnc(s + i + u * T);
#pragma unroll
                for (int u = 0; u < U; ++u) { if (CS) stcs(d + i + u * T, r[u]); else d[i + u * T] = r[u]; }
            }
            for (; i < vpr; i += T) d[i] = ldnc(s + i);
        } else {
            const unsigned n = tl.rows * vpr;
            for (unsigned i = threadIdx.x; i < n; i += U * T) {
                uint4 r[U];
                unsigned row[U], col[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const unsigned e = i + u * T;
                    row[u] = e / vpr; col[u] = e - row[u] * vpr;
                    if (e < n) r[u] = ldnc(reinterpret_cast<const uint4*>(tl.src + row[u] * tl.src_pitch) + col[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const unsigned e = i + u * T;
                    if (e < n) { uint4* p = reinterpret_cast<uint4*>(tl.dst + row[u] * tl.dst_pitch) + col[u]; if (CS) stcs(p, r[u]); else *p = r[u]; }
                }
            }
        }
    }
}

// ---- TMA bulk pipeline: one thread per CTA drives S stages of B bytes
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" :: "r"(smem_u32(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(s)), "l"(g), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(g), "r"(smem_u32(s)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct Seg { uint64_t src, dst; uint32_t bytes, pad; };

template <int S, int B>
__global__ void __launch_bounds__(32) copy_tma(const Seg* __restrict__ segs, int nseg) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar[S];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // segments for this CTA: blockIdx.x, +grid, ...
    int mine = 0;
    for (int j = blockIdx.x; j < nseg; j += gridDim.x) ++mine;
    uint32_t phase[S];
    for (int i = 0; i < S; ++i) phase[i] = 0;
    auto seg_of = [&](int k) { return segs[blockIdx.x + k * gridDim.x]; };
    // prologue: S-1 loads in flight
    int issued = 0;
    for (; issued < S - 1 && issued < mine; ++issued) {
        Seg g = seg_of(issued);
        int s = issued % S;
        mbar_expect(&bar[s], g.bytes);
        bulk_g2s(smem + s * B, reinterpret_cast<const void*>(g.src), g.bytes, &bar[s]);
    }
    for (int k = 0; k < mine; ++k) {
        if (issued < mine) {
            int s = issued % S;
            // stage s last held chunk issued-S, stored at iteration issued-S: make sure its read is done
            bulk_wait_read<S - 2>();
            Seg g = seg_of(issued);
            mbar_expect(&bar[s], g.bytes);
            bulk_g2s(smem + s * B, reinterpret_cast<const void*>(g.src), g.bytes, &bar[s]);
            ++issued;
        }
        int s = k % S;
        mbar_wait(&bar[s], phase[s]);
        phase[s] ^= 1;
        Seg g = seg_of(k);
        bulk_s2g(reinterpret_cast<void*>(g.dst), smem + s * B, g.bytes);
    }
    bulk_wait_all();
}

int main() {
    CR(cudaSetDevice(0));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = 8ull << 30;
    char *a, *b;
    CR(cudaMalloc(&a, bytes));
    CR(cudaMalloc(&b, bytes));
    CR(cudaMemset(a, 7, bytes));
    CR(cudaMemset(b, 0, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto mk_contig = [&](size_t tile) {
        std::vector<Tile> t;
        for (size_t o = 0; o < bytes; o += tile) t.push_back({(uint64_t)(a + o), (uint64_t)(b + o), 0, 0, 1, (uint32_t)tile});
        return t;
    };
    // 2-D: rows of 2 KB out of 4 KB-pitched src, dense dst (half the buffer moved)
    auto mk_2d = [&](size_t row, size_t pitch, size_t tile) {
        std::vector<Tile> t;
        size_t nrows = bytes / pitch, per = tile / row;
        for (size_t r = 0; r < nrows; r += per) {
            size_t n = std::min(per, nrows - r);
            t.push_back({(uint64_t)(a + r * pitch), (uint64_t)(b + r * row), pitch, row, (uint32_t)n, (uint32_t)row});
        }
        return t;
    };
    Tile* dt;
    CR(cudaMalloc(&dt, (bytes / 4096 + 16) * sizeof(Tile)));
    auto run = [&](const char* name, auto kern, int grid, int threads, const std::vector<Tile>& tiles, double moved) {
        CR(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice));
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            kern<<<grid, threads>>>(dt, (int)tiles.size());
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep >= 1 && ms < best) best = ms;
        }
        CR(cudaGetLastError());
        printf("%-44s grid %5d thr %3d tiles %7zu: %.3f ms  %.0f GB/s (r+w)\n", name, grid, threads, tiles.size(), best, 2 * moved / best / 1e6);
        return 0;
    };
    for (size_t tile : {256u << 10, 512u << 10, 1u << 20}) {
        auto t = mk_contig(tile);
        char nm[64];
        snprintf(nm, 64, "V1 512x4 grid4x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<512, 4, false>, sms * 4, 512, t, bytes);
        snprintf(nm, 64, "V2 512x4 grid2x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<512, 4, false>, sms * 2, 512, t, bytes);
        snprintf(nm, 64, "V3 256x8 grid4x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<256, 8, false>, sms * 4, 256, t, bytes);
        snprintf(nm, 64, "V3b 256x8 grid8x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<256, 8, false>, sms * 8, 256, t, bytes);
        snprintf(nm, 64, "V5 512x4 cs grid2x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<512, 4, true>, sms * 2, 512, t, bytes);
        snprintf(nm, 64, "V6 1024x2 grid2x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<1024, 2, false>, sms * 2, 1024, t, bytes);
        snprintf(nm, 64, "V7 128x8 grid16x (contig tile %zuK)", tile >> 10);
        run(nm, copy_v<128, 8, false>, sms * 16, 128, t, bytes);
    }
    {
        auto t = mk_2d(2048, 4096, 512 << 10);
        run("V1 2D row2K pitch4K", copy_v<512, 4, false>, sms * 4, 512, t, bytes / 2);
        run("V2 2D row2K pitch4K grid2x", copy_v<512, 4, false>, sms * 2, 512, t, bytes / 2);
        run("V3 2D 256x8 grid4x", copy_v<256, 8, false>, sms * 4, 256, t, bytes / 2);
        auto t2 = mk_2d(1024, 2048, 512 << 10);
        run("V2 2D row1K pitch2K grid2x", copy_v<512, 4, false>, sms * 2, 512, t2, bytes / 2);
        run("V3 2D row1K 256x8 grid4x", copy_v<256, 8, false>, sms * 4, 256, t2, bytes / 2);
    }
    // TMA bulk
    {
        Seg* ds;
        CR(cudaMalloc(&ds, (bytes / 8192 + 16) * sizeof(Seg)));
        auto tma = [&](const char* name, auto kern, int S, int B, int ctas_per_sm) {
            std::vector<Seg> sg;
            for (size_t o = 0; o < bytes; o += B) sg.push_back({(uint64_t)(a + o), (uint64_t)(b + o), (uint32_t)B, 0});
            CR(cudaMemcpy(ds, sg.data(), sg.size() * sizeof(Seg), cudaMemcpyHostToDevice));
            int smem = S * B;
            CR(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                kern<<<sms * ctas_per_sm, 32, smem>>>(ds, (int)sg.size());
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep >= 1 && ms < best) best = ms;
            }
            CR(cudaGetLastError());
            printf("%-44s S=%d B=%dK ctas/sm %d: %.3f ms  %.0f GB/s (r+w)\n", name, S, B >> 10, ctas_per_sm, best, 2.0 * bytes / best / 1e6);
            return 0;
        };
        tma("V4 TMA bulk", copy_tma<4, 32768>, 4, 32768, 1);
        tma("V4 TMA bulk", copy_tma<6, 32768>, 6, 32768, 1);
        tma("V4 TMA bulk", copy_tma<4, 16384>, 4, 16384, 2);
        tma("V4 TMA bulk", copy_tma<8, 16384>, 8, 16384, 1);
        tma("V4 TMA bulk", copy_tma<3, 32768>, 3, 32768, 2);
        tma("V4 TMA bulk", copy_tma<6, 16384>, 6, 16384, 2);
        tma("V4 TMA bulk", copy_tma<4, 8192>, 4, 8192, 4);
    }
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("cudaMemcpy D2D: %.3f ms, %.0f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
    }
    // check
    std::vector<char> h(1 << 20);
    CR(cudaMemcpy(h.data(), b + bytes - (1 << 20), 1 << 20, cudaMemcpyDeviceToHost));
    printf("check %d\n", h[12345] == 7);
    return 0;
}
