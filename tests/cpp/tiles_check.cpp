// Host check of the tile cutter shared by the host and the GPU (reshard/tiles.hpp):
// random strided / contiguous copies with every alignment, cut whole and cut after
// split_rec (the record-level interleave's pieces). The tiles must cover the copy's bytes
// exactly once, respect kTile and their alignment class, and the pieces must cut into the
// same tiles in the same order. Prints "TILES_OK <cases>" or the first failure.
#include <cstdio>
#include <random>
#include <vector>

#include "reshard/tiles.hpp"

using namespace reshard::exec;

struct T {
    int bucket;
    Tile t;
};

static std::vector<T> cut(const CopyRec& q) {
    std::vector<T> v;
    auto emit = [&](int b, const Tile& t) { v.push_back({b, t}); };
    cut_tiles(q, emit);
    return v;
}

int main() {
    std::mt19937_64 rng(2605);
    auto pick = [&](std::int64_t lo, std::int64_t hi) { return lo + static_cast<std::int64_t>(rng() % (hi - lo + 1)); };
    int cases = 0;
    for (int it = 0; it < 20000; ++it) {
        CopyRec q{};
        const std::int64_t kTiles[] = {32 << 10, 64 << 10, 512 << 10};
        q.kTile = kTiles[rng() % 3];
        q.key = static_cast<int>(rng() % 4);
        q.lane = static_cast<int>(rng() % 3);
        const int shape = static_cast<int>(rng() % 4);
        if (shape == 0) {  // contiguous, big
            q.rows = 1;
            q.rb = pick(1, 24 * q.kTile);
        } else if (shape == 1) {  // strided short rows
            q.rows = pick(2, 4000);
            q.rb = pick(1, q.kTile / 2);
        } else if (shape == 2) {  // strided long rows
            q.rows = pick(2, 40);
            q.rb = pick(q.kTile, 3 * q.kTile);
        } else {  // rows that collapse to one block
            q.rows = pick(2, 400);
            q.rb = pick(1, 2 * q.kTile);
        }
        const std::int64_t misalign_s = pick(0, 31), misalign_d = rng() % 2 ? misalign_s : pick(0, 31);
        q.sp = shape == 3 ? q.rb : q.rb + pick(0, 64);
        q.dp = shape == 3 ? q.rb : q.rb + pick(0, 64);
        q.src = (1ull << 40) + static_cast<std::uint64_t>(misalign_s);
        q.dst = (3ull << 40) + static_cast<std::uint64_t>(misalign_d);
        const std::vector<T> whole = cut(q);
        // coverage, size and class
        std::int64_t bytes = 0;
        for (const T& x : whole) {
            const std::int64_t tb = static_cast<std::int64_t>(x.t.rows) * x.t.row_bytes;
            bytes += tb;
            if (tb > q.kTile && x.t.rows > 1) return std::printf("FAIL tile over kTile (case %d)\n", it), 1;
            if (x.t.rows == 1 && x.t.row_bytes > q.kTile) return std::printf("FAIL row tile over kTile (case %d)\n", it), 1;
            const int V = 16 >> (x.bucket % 5);
            std::uint64_t a = x.t.src | x.t.dst | x.t.row_bytes;
            if (x.t.rows > 1) a |= x.t.src_pitch | x.t.dst_pitch;
            if (a % static_cast<std::uint64_t>(V)) return std::printf("FAIL alignment class (case %d)\n", it), 1;
            if (x.bucket / 5 != q.key) return std::printf("FAIL key (case %d)\n", it), 1;
        }
        // the closed-form count equals the cutter's emissions per class
        std::int64_t counted[5] = {0, 0, 0, 0, 0}, emitted[5] = {0, 0, 0, 0, 0};
        count_tiles(q, counted);
        for (const T& x : whole) ++emitted[x.bucket % 5];
        for (int c = 0; c < 5; ++c)
            if (counted[c] != emitted[c])
                return std::printf("FAIL count_tiles class %d: %lld != %lld (case %d: rows %lld rb %lld sp %lld dp %lld kTile %lld src%%16 %d dst%%16 %d)\n",
                                   c, (long long)counted[c], (long long)emitted[c], it, (long long)q.rows, (long long)q.rb,
                                   (long long)q.sp, (long long)q.dp, (long long)q.kTile, (int)(q.src % 16), (int)(q.dst % 16)), 1;
        if (bytes != q.rows * q.rb) return std::printf("FAIL coverage %lld != %lld (case %d)\n", (long long)bytes, (long long)(q.rows * q.rb), it), 1;
        // split pieces cut into the same tiles
        std::vector<CopyRec> pieces;
        split_rec(q, 1 + static_cast<std::int64_t>(rng() % 16), pieces);
        std::vector<T> again;
        for (const CopyRec& p : pieces)
            for (const T& x : cut(p)) again.push_back(x);
        if (again.size() != whole.size()) return std::printf("FAIL split tile count %zu != %zu (case %d: rows %lld rb %lld sp %lld dp %lld kTile %lld src%%16 %d dst%%16 %d pieces %zu)\n", again.size(), whole.size(), it, (long long)q.rows, (long long)q.rb, (long long)q.sp, (long long)q.dp, (long long)q.kTile, (int)(q.src%16), (int)(q.dst%16), pieces.size()), 1;
        for (size_t i = 0; i < whole.size(); ++i) {
            const Tile &a = whole[i].t, &b = again[i].t;
            const bool pitch_ok = a.rows == 1 || (a.src_pitch == b.src_pitch && a.dst_pitch == b.dst_pitch);
            if (whole[i].bucket != again[i].bucket || a.src != b.src || a.dst != b.dst || a.rows != b.rows ||
                a.row_bytes != b.row_bytes || !pitch_ok)
                return std::printf("FAIL split tile %zu differs (case %d)\n", i, it), 1;
        }
        ++cases;
    }
    std::printf("TILES_OK %d\n", cases);
    return 0;
}
