// Cutting a recorded 2-D copy into copy-kernel tiles — one definition for the host
// (counting, and the tile-level interleave path) and the GPU (the descriptor cut kernel).
//
// A record is one strided copy (rows x row bytes, pitches) of a launch group `key`. Tiles
// hold <= kTile bytes: whole rows grouped when rows are short, row slices when they are
// long; a head that shares the source and destination misalignment is peeled so the body
// runs 16-byte vectors. A tile's bucket is key * 5 + its alignment class (16/8/4/2/1 B).
#pragma once

#include <cstdint>

#include "reshard/common.hpp"
#include "reshard/executor.hpp"

namespace reshard {
namespace exec {

/// a recorded copy (TileSet::add), POD so the GPU can cut it
struct CopyRec {
    std::uint64_t src, dst;
    std::int64_t rows, rb, sp, dp, kTile;
    int key, lane;
};

RS_HD int align_class(std::uint64_t x) {
    if (x % 16 == 0) return 16;
    if (x % 8 == 0) return 8;
    if (x % 4 == 0) return 4;
    if (x % 2 == 0) return 2;
    return 1;
}

RS_HD int class_index(int v) { return v == 16 ? 0 : v == 8 ? 1 : v == 4 ? 2 : v == 2 ? 3 : 4; }

/// emit(bucket, tile) for every tile of the record, in order
template <class Emit>
RS_HD void cut_tiles(const CopyRec& q, Emit& emit_to) {
    std::int64_t rows = q.rows, rb = q.rb;
    const std::int64_t sp = q.sp, dp = q.dp, kTile = q.kTile;
    if (rows > 1 && sp == rb && dp == rb) {  // contiguous block
        rb *= rows;
        rows = 1;
    }
    auto emit = [&](std::uint64_t s, std::uint64_t d, std::int64_t nr, std::int64_t nb) {
        const Tile t{s, d, static_cast<std::uint64_t>(sp), static_cast<std::uint64_t>(dp), static_cast<std::uint32_t>(nr),
                     static_cast<std::uint32_t>(nb)};
        std::uint64_t a = s | d | static_cast<std::uint64_t>(nb);
        if (nr > 1) a |= static_cast<std::uint64_t>(sp) | static_cast<std::uint64_t>(dp);
        emit_to(static_cast<int>(q.key) * 5 + class_index(align_class(a)), t);
    };
    if (rows == 1 || rb >= kTile) {
        for (std::int64_t r = 0; r < rows; ++r) {
            std::uint64_t s = q.src + static_cast<std::uint64_t>(r * sp), d = q.dst + static_cast<std::uint64_t>(r * dp);
            std::int64_t left = rb;
            // peel an unaligned head so the body runs 16-byte vectors when both sides
            // share the same misalignment (relative offsets keep it: bases are 256-B aligned)
            if ((s % 16) == (d % 16) && (s % 16) != 0) {
                const std::int64_t head = left < 16 - static_cast<std::int64_t>(s % 16) ? left : 16 - static_cast<std::int64_t>(s % 16);
                emit(s, d, 1, head);
                s += static_cast<std::uint64_t>(head);
                d += static_cast<std::uint64_t>(head);
                left -= head;
            }
            while (left > 0) {
                const std::int64_t n = left < kTile ? left : kTile;
                const bool aligned = (s % 16) == 0 && (d % 16) == 0;
                const std::int64_t body = (aligned && n > 16) ? n - n % 16 : n;
                emit(s, d, 1, body);
                s += static_cast<std::uint64_t>(body);
                d += static_cast<std::uint64_t>(body);
                left -= body;
            }
        }
    } else {
        const std::int64_t per = kTile / rb > 1 ? kTile / rb : 1;
        for (std::int64_t r = 0; r < rows; r += per) {
            const std::int64_t nr = per < rows - r ? per : rows - r;
            emit(q.src + static_cast<std::uint64_t>(r * sp), q.dst + static_cast<std::uint64_t>(r * dp), nr, rb);
        }
    }
}

}  // namespace exec
}  // namespace reshard
