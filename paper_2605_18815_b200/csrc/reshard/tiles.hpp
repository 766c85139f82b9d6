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

/// Tiles per alignment class (16/8/4/2/1 B) that cut_tiles emits for the record, added to
/// n[5], in closed form: O(1) per row of a long-row copy and O(1) for a short-row copy
/// (per-row only when every tile holds one row). Same result as counting cut_tiles'
/// emissions (tests/cpp/tiles_check.cpp); a kTile that is not a multiple of 16 is counted
/// by cutting.
template <class Int>
RS_HD void count_tiles(const CopyRec& q, Int n[5]) {
    std::int64_t rows = q.rows, rb = q.rb;
    const std::int64_t sp = q.sp, dp = q.dp, kTile = q.kTile;
    if (kTile % 16) {  // a caller-chosen tile size: count the emissions
        auto c = [&](int b, const Tile&) { ++n[b % 5]; };
        cut_tiles(q, c);
        return;
    }
    if (rows > 1 && sp == rb && dp == rb) {
        rb *= rows;
        rows = 1;
    }
    auto cls = [](std::uint64_t a) { return class_index(align_class(a)); };
    if (rows == 1 || rb >= kTile) {
        for (std::int64_t r = 0; r < rows; ++r) {
            const std::uint64_t s = q.src + static_cast<std::uint64_t>(r * sp), d = q.dst + static_cast<std::uint64_t>(r * dp);
            std::int64_t left = rb;
            if ((s % 16) == (d % 16) && (s % 16) != 0) {  // head peel, then the body is aligned
                const std::int64_t head = left < 16 - static_cast<std::int64_t>(s % 16) ? left : 16 - static_cast<std::int64_t>(s % 16);
                ++n[cls(s | d | static_cast<std::uint64_t>(head))];
                left -= head;
            }
            if (left <= 0) continue;
            if ((s % 16) == (d % 16)) {  // aligned body: full tiles, a 16-B multiple, a tail
                n[0] += static_cast<Int>(left / kTile);
                const std::int64_t rem = left % kTile;
                if (rem > 16) {
                    ++n[0];
                    if (rem % 16) ++n[cls(static_cast<std::uint64_t>(rem % 16))];
                } else if (rem > 0) {
                    ++n[cls(static_cast<std::uint64_t>(rem))];
                }
            } else {  // different misalignment: kTile pieces keep s, d mod 16
                const std::uint64_t low = (s | d) & 15;
                n[cls(low)] += static_cast<Int>(left / kTile);
                const std::int64_t rem = left % kTile;
                if (rem > 0) ++n[cls(low | static_cast<std::uint64_t>(rem))];
            }
        }
    } else {
        const std::int64_t per = kTile / rb > 1 ? kTile / rb : 1;
        if (per == 1) {  // one row per tile: each row's own alignment
            for (std::int64_t r = 0; r < rows; ++r)
                ++n[cls((q.src + static_cast<std::uint64_t>(r * sp)) | (q.dst + static_cast<std::uint64_t>(r * dp)) |
                        static_cast<std::uint64_t>(rb))];
            return;
        }
        // multi-row tiles: the pitches in the alignment make the class row-independent
        const std::int64_t full = rows / per, last = rows % per;
        const std::uint64_t a = q.src | q.dst | static_cast<std::uint64_t>(rb) | static_cast<std::uint64_t>(sp) |
                                static_cast<std::uint64_t>(dp);
        n[cls(a)] += static_cast<Int>(full);
        if (last > 1) {
            ++n[cls(a)];
        } else if (last == 1) {
            const std::int64_t r = rows - 1;
            ++n[cls((q.src + static_cast<std::uint64_t>(r * sp)) | (q.dst + static_cast<std::uint64_t>(r * dp)) |
                    static_cast<std::uint64_t>(rb))];
        }
    }
}

/// Split a copy at tile boundaries into pieces of about `piece_tiles` tiles, appended to
/// `out` (host). Cutting the pieces yields exactly the tiles of the whole copy, in order
/// (pitch fields of single-row tiles aside, which the kernels ignore).
template <class Vec>
inline void split_rec(const CopyRec& q0, std::int64_t piece_tiles, Vec& out) {
    CopyRec q = q0;
    if (q.rows > 1 && q.sp == q.rb && q.dp == q.rb) q.rb *= q.rows, q.rows = 1, q.sp = q.dp = q.rb;
    const std::int64_t piece = piece_tiles * q.kTile;
    if (q.rows * q.rb <= piece) {
        out.push_back(q0);
        return;
    }
    if (q.rows == 1) {
        // contiguous: the head peel (shared misalignment) rides with the first piece, then
        // whole multiples of kTile
        std::int64_t head = 0;
        if ((q.src % 16) == (q.dst % 16) && (q.src % 16) != 0) {
            head = 16 - static_cast<std::int64_t>(q.src % 16);
            if (head > q.rb) head = q.rb;
        }
        for (std::int64_t off = 0; off < q.rb;) {
            std::int64_t len = (off == 0 ? head : 0) + piece;
            if (len > q.rb - off) len = q.rb - off;
            CopyRec p = q;
            p.src = q.src + static_cast<std::uint64_t>(off);
            p.dst = q.dst + static_cast<std::uint64_t>(off);
            p.rb = len;
            p.sp = p.dp = len;
            out.push_back(p);
            off += len;
        }
        return;
    }
    // strided: whole tiles' worth of rows per piece
    std::int64_t step;
    if (q.rb < q.kTile) {
        const std::int64_t rows_per_tile = q.kTile / q.rb > 1 ? q.kTile / q.rb : 1;
        step = rows_per_tile * piece_tiles;
    } else {
        const std::int64_t tiles_per_row = (q.rb + q.kTile - 1) / q.kTile + 1;
        step = piece_tiles / tiles_per_row > 1 ? piece_tiles / tiles_per_row : 1;
    }
    for (std::int64_t r = 0; r < q.rows;) {
        CopyRec p = q;
        p.src = q.src + static_cast<std::uint64_t>(r * q.sp);
        p.dst = q.dst + static_cast<std::uint64_t>(r * q.dp);
        p.rows = step < q.rows - r ? step : q.rows - r;
        // a lone last row would be cut as a single-row copy (head peel); keep it with the
        // piece before, where it is the last row group exactly as in the whole copy
        if (q.rows - r - p.rows == 1) ++p.rows;
        out.push_back(p);
        r += p.rows;
    }
}

}  // namespace exec
}  // namespace reshard
