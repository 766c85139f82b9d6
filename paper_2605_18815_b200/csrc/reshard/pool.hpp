// A persistent host worker pool for the planner and the descriptor build: their parallel
// loops are short (sub-millisecond), so spawning threads per loop would cost as much as
// the work. Workers sleep on a condition variable between loops.
#pragma once

#include <cstddef>
#include <functional>

namespace reshard {
namespace pool {

/// number of threads parallel_for uses (workers + the caller), >= 1: the host's cores
/// divided by the rank processes sharing it (LOCAL_WORLD_SIZE), at most 16;
/// RS_HOST_THREADS overrides
std::size_t size();

/// fn(t) for t in [0, n) on the pool (the caller runs one share); returns when all are
/// done; the first exception thrown by any fn is rethrown here. Nested calls run inline.
void run(std::size_t n, const std::function<void(std::size_t)>& fn);

/// While a Warm guard lives (any thread), idle workers spin (yielding) between loops
/// instead of going to sleep: a plan or a descriptor build runs several short parallel
/// loops separated by serial work, and a condition-variable wake-up of every worker per
/// loop costs about as much as the loops. Workers sleep again ~100 us after the last
/// guard ends.
class Warm {
public:
    Warm();
    ~Warm();
    Warm(const Warm&) = delete;
    Warm& operator=(const Warm&) = delete;
};

/// fn(i) for every i in [0, n), split into contiguous slices over the pool
template <class F>
void parallel_for(std::size_t n, F&& fn) {
    if (n == 0) return;
    const std::size_t parts = n < size() ? n : size();
    run(parts, [&](std::size_t t) {
        for (std::size_t i = n * t / parts; i < n * (t + 1) / parts; ++i) fn(i);
    });
}

}  // namespace pool
}  // namespace reshard
