// Elastic Device Manager core, native: the cache of
// communicator groups per parallel configuration (get_or_create_groups), the side thread
// that prepares the next world while the old layout keeps training (prepare_async /
// ready / wait), and the SPEC accounting of exposed vs overlapped time
// (simulate_scale_event). Communicator objects themselves belong to the
// caller's runtime (torch.distributed here); the manager caches their rank lists.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "reshard/edm.hpp"

namespace reshard {
namespace edm {

namespace {
using Key = std::tuple<int, int, int, int, int, std::string, int>;  // dp, tp, pp, ep, zero, order, dim
Key key_of(const ParallelConfig& c, GroupDim dim) {
    return Key{c.dp, c.tp, c.pp, c.ep, c.zero_enabled ? 1 : 0, c.rank_order, static_cast<int>(dim)};
}
}  // namespace

struct Manager::Impl {
    std::mutex mu;
    std::map<Key, std::vector<std::vector<int>>> cache;
    std::int64_t hits = 0, misses = 0;
    double creation_s = 0.0;
    std::thread worker;
    std::atomic<bool> running{false};
    double init_s = 0.0;
    int build_rc = 0;
};

Manager::Manager() : impl_(new Impl) {}

Manager::~Manager() {
    if (impl_->worker.joinable()) impl_->worker.join();
    delete impl_;
}

const std::vector<std::vector<int>>& Manager::groups(const ParallelConfig& cfg, GroupDim dim, bool* hit) {
    std::lock_guard<std::mutex> lock(impl_->mu);
    const Key k = key_of(cfg, dim);
    auto it = impl_->cache.find(k);
    if (it != impl_->cache.end()) {
        ++impl_->hits;
        if (hit) *hit = true;
        return it->second;
    }
    const auto t0 = std::chrono::steady_clock::now();
    auto g = parallel_groups(cfg, dim);
    impl_->creation_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ++impl_->misses;
    if (hit) *hit = false;
    return impl_->cache.emplace(k, std::move(g)).first->second;
}

void Manager::cache_stats(std::int64_t* hits, std::int64_t* misses, double* creation_s) const {
    std::lock_guard<std::mutex> lock(impl_->mu);
    *hits = impl_->hits;
    *misses = impl_->misses;
    *creation_s = impl_->creation_s;
}

void Manager::prepare_async(int (*build)(void*), void* arg) {
    if (impl_->running.load()) throw ConfigError("edm: a preparation is already running");
    if (impl_->worker.joinable()) impl_->worker.join();
    impl_->running = true;
    impl_->worker = std::thread([this, build, arg] {
        const auto t0 = std::chrono::steady_clock::now();
        const int rc = build(arg);
        impl_->init_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        impl_->build_rc = rc;
        impl_->running = false;
    });
}

bool Manager::ready() const { return impl_->worker.joinable() && !impl_->running.load(); }

int Manager::wait(double* init_s) {
    if (impl_->worker.joinable()) impl_->worker.join();
    if (init_s) *init_s = impl_->init_s;
    return impl_->build_rc;
}

Accounting account(double init_s, double switch_s, double window_s, double train_step_s, Mode mode) {
    // exposed = switch + max(0, init - overlapped);
    // ratio = overlapped / (overlapped + exposed). With a measured window the overlapped
    // part is min(init, window); with a step cost, whole training steps only.
    Accounting a;
    if (mode == Mode::InPlace) init_s = 0.0;
    double overlapped = 0.0;
    if (mode == Mode::Overlapped && init_s > 0.0) {
        if (window_s >= 0.0) overlapped = std::min(init_s, window_s);
        else if (train_step_s > 0.0) overlapped = static_cast<double>(static_cast<long long>(init_s / train_step_s)) * train_step_s;
    }
    a.init_s = init_s;
    a.overlapped_s = overlapped;
    a.switch_s = switch_s;
    a.exposed_s = switch_s + std::max(0.0, init_s - overlapped);
    a.ratio = overlapped + a.exposed_s > 0 ? overlapped / (overlapped + a.exposed_s) : -1.0;
    return a;
}

}  // namespace edm
}  // namespace reshard
