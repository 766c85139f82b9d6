// SynchronizeAll on the device (ExecuteSwitch): a cross-GPU flag barrier
// enqueued on a stream, so memory-aware stages and consecutive transitions follow each
// other without a host round trip.
//
// Every rank owns a small flag array in its HBM, mapped into every peer (cudaIpc). A
// barrier with epoch e: one thread per peer does a system-scope release store of e into
// slot[rank] of that peer's array (after a system fence, so every earlier write of this
// stream — the stage's peer pushes — is visible first), then spins with acquire loads
// until its own array holds >= e in every peer's slot. Epochs grow monotonically, so the
// flags never need resetting. A spin that exceeds the timeout gives up and raises a
// status word the host checks (rs_sync_status), so a missing peer cannot hang the GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace reshard {
namespace sync {

constexpr int kMaxRanks = 64;

class DeviceBarrier {
public:
    DeviceBarrier(int rank, int world, int device);
    ~DeviceBarrier();
    DeviceBarrier(const DeviceBarrier&) = delete;
    DeviceBarrier& operator=(const DeviceBarrier&) = delete;

    /// cudaIpc handle of this rank's flag array (64 bytes)
    std::vector<std::uint8_t> export_handle() const;
    /// map rank `peer`'s flag array (its export_handle); the own rank maps itself
    void import_handle(int peer, const std::uint8_t* blob, size_t len);
    /// enqueue one barrier on `stream`; every rank must enqueue the same sequence
    void arrive_and_wait(cudaStream_t stream);
    /// 1 if a barrier spin timed out since the last call (and clears it)
    int status();
    std::uint64_t epoch() const { return epoch_; }
    void set_timeout_ns(std::uint64_t ns) { timeout_ns_ = ns; }

private:
    int rank_, world_, device_;
    std::uint64_t* flags_ = nullptr;    // [kMaxRanks] own array (peers write slot[peer])
    std::uint32_t* status_ = nullptr;   // device status word
    std::uint64_t** d_peers_ = nullptr; // device copy of the peers' mapped arrays
    std::vector<std::uint64_t*> peers_;
    std::vector<void*> opened_;
    std::uint64_t epoch_ = 0;
    std::uint64_t timeout_ns_ = 20'000'000'000ull;
    bool dirty_ = true;
};

}  // namespace sync
}  // namespace reshard
