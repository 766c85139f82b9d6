// Executor: turns a PlanCore into copy descriptors for one GPU and runs them.
//
// Push model: every GPU executes the moves whose SOURCE virtual rank
// lives on it, reading local HBM and storing straight into the destination
// buffer at its final offset — local HBM for co-located destinations, a peer GPU's
// HBM (cudaIpc-mapped) over NVLink otherwise. No staging buffers, no unpack.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "reshard/plan_core.hpp"

namespace reshard {
namespace exec {

enum Buf : int { kParam = 0, kMaster = 1, kM = 2, kV = 3, kGrad = 4, kScalars = 5, kNumBufs = 6 };

/// 2-D strided byte copy: `rows` rows of `row_bytes`, pitches in bytes.
struct CopyOp {
    int src_side_rank, src_buf;  // src virtual rank, buffer
    int dst_rank, dst_buf;       // dst virtual rank, buffer
    std::int64_t src_off, dst_off, rows, row_bytes, src_pitch, dst_pitch;
    int tensor = -1;             // model tensor the bytes belong to (-1: scalar blob)
    int box = -1;                // index of the plan box transfer it moves (PlanCore::box), else -1
};

/// Device tile: <= kTileBytes of one CopyOp, absolute pointers.
struct Tile {
    std::uint64_t src, dst;
    std::uint64_t src_pitch, dst_pitch;
    std::uint32_t rows, row_bytes;
};
static_assert(sizeof(Tile) == 40, "tile layout");

/// Fill/verify task: a contiguous element range of one segment's row-major
/// enumeration stored at `ptr` (element width `width`).
struct FillTask {
    std::uint64_t ptr;
    stair::TensorView t;
    std::int64_t plo[2], pext_box[2], rlo, rows_box, clo, cols_box;  // box (lifted)
    std::int64_t e_lo, e_hi;  // element range within the box enumeration
    int kind;                 // 0 param, 1 master, 2 m, 3 v, 4 grad
    int width;                // bytes per element
};

/// Build every CopyOp of the transition (all GPUs), grouped by nothing.
std::vector<CopyOp> build_ops(const core::PlanCore& P);

/// Byte accounting of one GPU under contiguous-block placement (host only): what it
/// copies locally, pushes to peers (out) and receives from peers (in).
struct PlacementStats {
    std::int64_t local_bytes = 0, out_bytes = 0, in_bytes = 0, ops = 0;
};
PlacementStats placement_stats(const core::PlanCore& P, int n_gpus, int gpu);

/// The transition's copy bytes between physical devices (host only): m[s * n + d] for
/// n = highest participating phys + 1; off-diagonal entries sum to bytes_moved, the
/// diagonal holds the on-device copies (retained regions). Input of a co-location search
/// when several devices share a GPU.
std::vector<std::int64_t> traffic_matrix(const core::PlanCore& P, int* n);

/// Buffer sizes of a rank (bytes) for one side.
void buffer_sizes(const core::PlanCore& P, int side, int rank, bool with_grads, std::int64_t out[kNumBufs]);

}  // namespace exec
}  // namespace reshard
