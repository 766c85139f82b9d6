// New-world NCCL communicators for the Elastic Device Manager (
// SPEC.md:443-451): built natively, non-blocking, on the EDM side thread while the old
// layout keeps training.
//
// A configuration's communicators are its world communicator — ncclCommInitRankConfig
// with blocking = 0 from a fresh unique id — and one sub-communicator per parallel
// dimension (DP, TP, PP, EP, expert-DP) split from it with ncclCommSplit (also
// non-blocking); both are polled with ncclCommGetAsyncError until ready. They are cached
// per configuration (get_or_create_groups), so a configuration seen before costs nothing.
//
// libnccl is loaded at run time (dlopen "libnccl.so.2"): inside a PyTorch process that is
// the NCCL torch already loaded, so one NCCL lives in the process.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace reshard {
namespace edm {

constexpr int kNcclIdBytes = 128;
constexpr int kCommDims = 5;  // GroupDim: dp, tp, pp, ep, expert-dp

/// ncclGetUniqueId (rank 0 of the new world draws it; the caller broadcasts it)
void nccl_unique_id(std::uint8_t out[kNcclIdBytes]);
/// "major.minor.patch" of the loaded libnccl
std::string nccl_version();

struct CommSet {
    void* world = nullptr;                 // ncclComm_t
    void* dims[kCommDims] = {};            // ncclComm_t per dimension (nullptr: not split)
    int nranks = 0, rank = 0, device = 0;
    double init_s = 0, split_s = 0;        // wall time of the world init / of the splits
};

class CommCache {
public:
    CommCache() = default;
    ~CommCache();
    CommCache(const CommCache&) = delete;
    CommCache& operator=(const CommCache&) = delete;

    /// create (or return the cached) communicators of configuration `key`: the world
    /// communicator from `uid`, then one split per dimension with colors[d] (< 0: skip the
    /// dimension). Non-blocking NCCL calls polled to completion on the calling thread
    /// (the EDM side thread); every rank of the new world must call with the same key.
    /// *hit: the cache held it already.
    const CommSet& get_or_create(const std::string& key, const std::uint8_t uid[kNcclIdBytes], int nranks, int rank,
                                 int device, const int colors[kCommDims], bool* hit);
    const CommSet* find(const std::string& key) const;
    /// an all-reduce (sum) of one float 1.0 over the world (dim < 0) or a dimension's
    /// communicator on `stream`: returns the sum (= that communicator's size)
    float check_allreduce(const std::string& key, int dim, cudaStream_t stream);
    void destroy(const std::string& key);

private:
    mutable std::mutex mu_;
    std::map<std::string, std::unique_ptr<CommSet>> cache_;
};

}  // namespace edm
}  // namespace reshard
