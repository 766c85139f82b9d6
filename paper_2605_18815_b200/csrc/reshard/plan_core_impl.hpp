// Template helpers of plan_core.hpp.
#pragma once

#include <algorithm>
#include <vector>

namespace reshard {
namespace core {

template <class F>
void for_each_band(const stair::Triple& T, F&& emit) {
    const int np = T.t.np;
    std::int64_t p[2] = {0, 0};
    const std::int64_t e0 = np > 0 ? T.phi[0] - T.plo[0] : 1;
    const std::int64_t e1 = np > 1 ? T.phi[1] - T.plo[1] : 1;
    // at most 2 + 3 stairs x 6 row cuts per plane: a fixed array, no heap per call
    std::int64_t cuts[24];
    int nc = 0;
    const stair::Stair* stairs[3] = {&T.K, &T.J, T.has_i ? &T.I : nullptr};
    for (std::int64_t i0 = 0; i0 < e0; ++i0) {
        for (std::int64_t i1 = 0; i1 < e1; ++i1) {
            if (np > 0) p[0] = T.plo[0] + i0;
            if (np > 1) p[1] = T.plo[1] + i1;
            nc = 0;
            cuts[nc++] = T.rlo;
            cuts[nc++] = T.rhi;
            for (const stair::Stair* X : stairs) {
                if (!X) continue;
                std::int64_t prank = 0;
                bool inside = true;
                for (int d = 0; d < np; ++d) {
                    if (p[d] < X->plo[d] || p[d] >= X->phi[d]) inside = false;
                    prank = prank * (X->phi[d] - X->plo[d]) + (p[d] - X->plo[d]);
                }
                if (!inside) continue;
                const std::int64_t w = X->chi - X->clo;
                const std::int64_t q0 = prank * (X->rhi - X->rlo);
                const std::int64_t qs[4] = {X->a / w, X->a / w + 1, X->b / w, X->b / w + 1};
                for (std::int64_t q : qs) cuts[nc++] = X->rlo + (q - q0);
                cuts[nc++] = X->rlo;
                cuts[nc++] = X->rhi;
            }
            std::sort(cuts, cuts + nc);
            nc = static_cast<int>(std::unique(cuts, cuts + nc) - cuts);
            for (int c = 0; c + 1 < nc; ++c) {
                const std::int64_t u = cuts[c], v = cuts[c + 1];
                if (u < T.rlo || v > T.rhi || u >= v) continue;
                stair::Iv cols[2];
                const int n = stair::row_pieces(T.K, T.J, T.has_i ? &T.I : nullptr, np, p, u, cols);
                if (n) emit(p, u, v, cols, n);
            }
        }
    }
}

}  // namespace core
}  // namespace reshard
