// Persistent host worker pool (reshard/pool.hpp).
#include "reshard/pool.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace reshard {
namespace pool {

namespace {

thread_local bool t_in_pool = false;
std::atomic<int> g_warm{0};  // live Warm guards

/// one parallel loop: workers claim indices of THIS loop only, so a worker still leaving
/// the previous loop can never take (or count) an index of the next one
struct Job {
    const std::function<void(std::size_t)>* fn = nullptr;
    std::size_t n = 0;
    std::atomic<std::size_t> next{0};
    std::size_t pending = 0;  // guarded by Pool::mu_
    std::exception_ptr error;  // guarded by Pool::mu_
};

class Pool {
public:
    Pool() {
        // the host's cores are shared by the rank processes on it (torchrun exports
        // LOCAL_WORLD_SIZE); RS_HOST_THREADS overrides
        const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
        std::size_t local = 1;
        if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) local = static_cast<std::size_t>(std::max(1, std::atoi(lw)));
        nthreads_ = std::max<std::size_t>(1, std::min<std::size_t>(hw / local, 16));
        if (const char* ht = std::getenv("RS_HOST_THREADS")) nthreads_ = static_cast<std::size_t>(std::max(1, std::atoi(ht)));
        for (std::size_t i = 1; i < nthreads_; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
            gen_atomic_.store(gen_, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    std::size_t size() const { return nthreads_; }

    void run(std::size_t n, const std::function<void(std::size_t)>& fn) {
        if (n == 0) return;
        if (n == 1 || t_in_pool || nthreads_ == 1) {  // inline: tiny loops and nested calls
            for (std::size_t t = 0; t < n; ++t) fn(t);
            return;
        }
        std::lock_guard<std::mutex> serial(run_mu_);  // one parallel loop at a time
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->n = n;
        job->pending = n;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = job;
            ++gen_;
            gen_atomic_.store(gen_, std::memory_order_release);
        }
        cv_.notify_all();
        work(*job);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return job->pending == 0; });
        job_.reset();
        if (job->error) std::rethrow_exception(job->error);
    }

private:
    void work(Job& j) {
        const bool was = t_in_pool;
        t_in_pool = true;
        for (;;) {
            const std::size_t t = j.next.fetch_add(1);
            if (t >= j.n) break;
            std::exception_ptr e;
            try {
                (*j.fn)(t);
            } catch (...) {
                e = std::current_exception();
            }
            std::lock_guard<std::mutex> lk(mu_);
            if (e && !j.error) j.error = e;
            if (--j.pending == 0) done_cv_.notify_all();
        }
        t_in_pool = was;
    }

    void loop() {
        std::uint64_t seen = 0;
        for (;;) {
            // a planner / descriptor build issues several short loops back to back: spin
            // briefly on the generation counter before sleeping, so the next loop does not
            // pay a condition-variable wake-up per worker
            const auto t0 = std::chrono::steady_clock::now();
            while (gen_atomic_.load(std::memory_order_acquire) == seen &&
                   (g_warm.load(std::memory_order_relaxed) > 0 ||
                    std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(100)))
                std::this_thread::yield();
            std::shared_ptr<Job> j;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                j = job_;
            }
            if (j) work(*j);
        }
    }

    std::size_t nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_, done_cv_;
    std::shared_ptr<Job> job_;  // the loop in progress (guarded by mu_)
    std::uint64_t gen_ = 0;
    std::atomic<std::uint64_t> gen_atomic_{0};  // gen_, readable without the lock (spin)
    bool stop_ = false;
};

Pool& instance() {
    static Pool p;
    return p;
}

}  // namespace

std::size_t size() { return instance().size(); }

Warm::Warm() {
    instance();  // the workers exist before the first loop
    g_warm.fetch_add(1, std::memory_order_relaxed);
}

Warm::~Warm() { g_warm.fetch_sub(1, std::memory_order_relaxed); }

void run(std::size_t n, const std::function<void(std::size_t)>& fn) { instance().run(n, fn); }

}  // namespace pool
}  // namespace reshard
