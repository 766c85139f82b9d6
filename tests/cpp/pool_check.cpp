// Stress check of the host worker pool (csrc/pool.cpp): thousands of short parallel loops
// back to back, each index must run exactly once and run() must return only after all of
// them; exceptions propagate; nested loops run inline.
#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "reshard/pool.hpp"

using namespace reshard;

int main() {
    std::vector<std::atomic<int>> hits(4096);
    for (int it = 0; it < 20000; ++it) {
        const std::size_t n = 1 + static_cast<std::size_t>((it * 2654435761u) % 97);
        for (std::size_t i = 0; i < n; ++i) hits[i].store(0);
        pool::run(n, [&](std::size_t t) { hits[t].fetch_add(1); });
        for (std::size_t i = 0; i < n; ++i)
            if (hits[i].load() != 1) {
                std::printf("FAIL loop %d: index %zu ran %d times (n=%zu)\n", it, i, hits[i].load(), n);
                return 1;
            }
        std::vector<long> out(n * 7, 0);
        pool::parallel_for(out.size(), [&](std::size_t i) { out[i] = static_cast<long>(i) * 3; });
        for (std::size_t i = 0; i < out.size(); ++i)
            if (out[i] != static_cast<long>(i) * 3) {
                std::printf("FAIL parallel_for loop %d index %zu\n", it, i);
                return 1;
            }
    }
    {  // the same under a Warm guard (workers spin between loops)
        const pool::Warm warm;
        for (int it = 0; it < 5000; ++it) {
            const std::size_t n = 1 + static_cast<std::size_t>((it * 40503u) % 61);
            for (std::size_t i = 0; i < n; ++i) hits[i].store(0);
            pool::run(n, [&](std::size_t t) { hits[t].fetch_add(1); });
            for (std::size_t i = 0; i < n; ++i)
                if (hits[i].load() != 1) return std::printf("FAIL warm loop %d index %zu\n", it, i), 1;
        }
    }
    bool threw = false;
    try {
        pool::run(64, [](std::size_t t) {
            if (t == 17) throw std::runtime_error("x");
        });
    } catch (const std::runtime_error&) {
        threw = true;
    }
    if (!threw) return std::printf("FAIL exception not propagated\n"), 1;
    std::atomic<int> nested{0};
    pool::run(8, [&](std::size_t) { pool::run(8, [&](std::size_t) { nested.fetch_add(1); }); });
    if (nested.load() != 64) return std::printf("FAIL nested %d\n", nested.load()), 1;
    std::printf("POOL_OK threads=%zu\n", pool::size());
    return 0;
}
