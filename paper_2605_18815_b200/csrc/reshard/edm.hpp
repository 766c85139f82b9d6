// Elastic Device Manager, native core. See edm.cpp.
#pragma once

#include <cstdint>
#include <vector>

#include "reshard/parallel.hpp"

namespace reshard {
namespace edm {

enum class Mode { Blocking = 0, Overlapped = 1, InPlace = 2 };

struct Accounting {
    double init_s = 0, overlapped_s = 0, switch_s = 0, exposed_s = 0;
    double ratio = -1;  // overlapped / (overlapped + exposed); -1 when both are 0
};

/// simulate_scale_event's accounting. window_s >= 0: measured overlap
/// window; else train_step_s > 0: whole training steps fit into init.
Accounting account(double init_s, double switch_s, double window_s, double train_step_s, Mode mode);

class Manager {
public:
    Manager();
    ~Manager();
    Manager(const Manager&) = delete;
    Manager& operator=(const Manager&) = delete;

    /// get_or_create_groups for one dimension: cached per configuration; *hit tells
    /// whether the cache already held it (zero creation cost)
    const std::vector<std::vector<int>>& groups(const ParallelConfig& cfg, GroupDim dim, bool* hit);
    void cache_stats(std::int64_t* hits, std::int64_t* misses, double* creation_s) const;

    /// run build(arg) on a side thread (the new world's plan, executor, buffers, peer
    /// mappings) while the caller keeps training; timed as init_s
    void prepare_async(int (*build)(void*), void* arg);
    bool ready() const;
    /// join the side thread; returns build's return code
    int wait(double* init_s);

private:
    struct Impl;
    Impl* impl_;
};

}  // namespace edm
}  // namespace reshard
