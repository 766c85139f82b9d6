// Closed-form geometry of ZeRO optimizer shards, shared by the host planner, the
// GPU planner kernels and the executor's descriptor builder.
//
// A ZeRO shard restricted to one tensor is a contiguous range [a,b) of the
// row-major enumeration of the rank's box of that tensor (project.hpp:146-159:
// local_layout flattens visible boxes row-major; shard_range cuts a contiguous
// slice; invert_segments maps it back). We call that set a "stair": full rows in
// the middle, partial rows at both ends. The reference materializes it as one flat
// interval per row and intersects interval lists in O(n*m) (routing.hpp:317-327);
// here the transfer set of one (src k, dst j, tensor t) triple is
//        (Stair_j ∩ Stair_k) \ Stair_own(j)
// evaluated per tensor row in O(1), which is what lets the expansion run as one
// GPU thread per row.
//
// Boxes are lifted to >= 2 dims (a 1-D box [c0,c1) becomes [0,1) x [c0,c1)), then
// viewed as planes (dims 0..nd-3) x rows (dim nd-2) x cols (dim nd-1).
#pragma once

#include <cstdint>

#include "reshard/common.hpp"

namespace reshard {
namespace stair {

struct Iv {
    std::int64_t lo, hi;
};

/// A tensor in lifted coordinates.
struct TensorView {
    int np;                 // plane dims (0..2)
    std::int64_t pext[2];   // plane extents
    std::int64_t rows;      // extent of the row dim
    std::int64_t cols;      // extent of the column dim (= row width W)
    std::int64_t off;       // global flat offset of element 0
};

/// Row-major sub-range [a,b) of a lifted box.
struct Stair {
    std::int64_t plo[2], phi[2];
    std::int64_t rlo, rhi, clo, chi;
    std::int64_t a, b;
};

RS_HD bool iv_empty(Iv x) { return x.hi <= x.lo; }

/// Columns of stair X in row (p, r), or an empty interval.
RS_HD Iv stair_cols(const Stair& X, int np, const std::int64_t* p, std::int64_t r) {
    Iv none{0, 0};
    std::int64_t prank = 0;
    for (int i = 0; i < np; ++i) {
        if (p[i] < X.plo[i] || p[i] >= X.phi[i]) return none;
        prank = prank * (X.phi[i] - X.plo[i]) + (p[i] - X.plo[i]);
    }
    if (r < X.rlo || r >= X.rhi) return none;
    const std::int64_t w = X.chi - X.clo;
    const std::int64_t s = (prank * (X.rhi - X.rlo) + (r - X.rlo)) * w;
    const std::int64_t lo = X.a - s > 0 ? X.a - s : 0;
    const std::int64_t hi = X.b - s < w ? X.b - s : w;
    if (lo >= hi) return none;
    return Iv{X.clo + lo, X.clo + hi};
}

/// (J ∩ K) \ I on one row: up to two column intervals, ascending. Returns count.
RS_HD int row_pieces(const Stair& K, const Stair& J, const Stair* I, int np, const std::int64_t* p, std::int64_t r,
                     Iv out[2]) {
    const Iv k = stair_cols(K, np, p, r), j = stair_cols(J, np, p, r);
    Iv x{k.lo > j.lo ? k.lo : j.lo, k.hi < j.hi ? k.hi : j.hi};
    if (iv_empty(x)) return 0;
    if (I == nullptr) {
        out[0] = x;
        return 1;
    }
    const Iv i = stair_cols(*I, np, p, r);
    if (iv_empty(i) || i.hi <= x.lo || i.lo >= x.hi) {
        out[0] = x;
        return 1;
    }
    int n = 0;
    if (x.lo < i.lo) out[n++] = Iv{x.lo, i.lo};
    if (i.hi < x.hi) out[n++] = Iv{i.hi, x.hi};
    return n;
}

/// One (src k, dst j, tensor t) optimizer move in closed form.
struct Triple {
    TensorView t;
    Stair K, J, I;
    int has_i;
    int src, dst;  // world ranks
    int tensor;
    // iteration space: planes ∩ and rows ∩ of K and J
    std::int64_t plo[2], phi[2], rlo, rhi;
    std::int64_t nrows;  // (#planes) x (rhi - rlo)
};

/// Row q of the triple's iteration space -> plane coords and row index.
RS_HD void triple_row(const Triple& T, std::int64_t q, std::int64_t* p, std::int64_t* r) {
    const std::int64_t nr = T.rhi - T.rlo;
    std::int64_t plane = q / nr;
    *r = T.rlo + (q - plane * nr);
    for (int i = T.t.np - 1; i >= 0; --i) {
        const std::int64_t e = T.phi[i] - T.plo[i];
        p[i] = T.plo[i] + plane % e;
        plane /= e;
    }
}

/// Global flat index of (p, r, c).
RS_HD std::int64_t flat_of(const TensorView& t, const std::int64_t* p, std::int64_t r, std::int64_t c) {
    std::int64_t g = 0;
    for (int i = 0; i < t.np; ++i) g = g * t.pext[i] + p[i];
    return t.off + (g * t.rows + r) * t.cols + c;
}

/// Pieces of row q as global flat runs. Returns count (0..2).
RS_HD int triple_row_runs(const Triple& T, std::int64_t q, Iv out[2]) {
    std::int64_t p[2] = {0, 0}, r;
    triple_row(T, q, p, &r);
    Iv cols[2];
    const int n = row_pieces(T.K, T.J, T.has_i ? &T.I : nullptr, T.t.np, p, r, cols);
    for (int i = 0; i < n; ++i) out[i] = Iv{flat_of(T.t, p, r, cols[i].lo), flat_of(T.t, p, r, cols[i].hi)};
    return n;
}

}  // namespace stair
}  // namespace reshard
