// A persistent host worker pool for the planner and the descriptor build: their parallel
// loops are short (sub-millisecond), so spawning threads per loop would cost as much as
// the work. Workers sleep on a condition variable between loops.
#pragma once

#include <cstddef>
#include <functional>

namespace reshard {
namespace pool {

/// number of threads parallel_for uses (workers + the caller), >= 1
std::size_t size();

/// fn(t) for t in [0, n) on the pool (the caller runs one share); returns when all are
/// done; the first exception thrown by any fn is rethrown here. Nested calls run inline.
void run(std::size_t n, const std::function<void(std::size_t)>& fn);

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
