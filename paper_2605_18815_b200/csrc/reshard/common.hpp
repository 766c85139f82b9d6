// reshard-b200 — common types. Mirrors the reference's common.hpp surface
// (FlatIndex/ByteCount :25-26, ConfigError :30-33, StateKind :37, canon_value
// :77-80) so callers of the reference compile unchanged; canon_value is also
// callable from device code (fill/verify kernels).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#if defined(__CUDACC__)
#define RS_HD __host__ __device__ __forceinline__
#else
#define RS_HD inline
#endif

namespace reshard {

using FlatIndex = std::int64_t;
using ByteCount = std::int64_t;

/// Bad input (config, scenario, divisibility). C ABI status RS_ERR_CONFIG (exit 2).
class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};

/// Payload categories; the numeric order is the canonical dump order.
enum class StateKind : int { Param = 0, Optim = 1, Grad = 2, Scalar = 3 };

inline const char* to_string(StateKind k) {
    static const char* const names[] = {"param", "optim", "grad", "scalar"};
    int i = static_cast<int>(k);
    return (i >= 0 && i < 4) ? names[i] : "?";
}

inline std::string strfmt(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    va_list ap2;
    va_copy(ap2, ap);
    int n = std::vsnprintf(nullptr, 0, fmt, ap);
    va_end(ap);
    std::string s(n > 0 ? static_cast<size_t>(n) : 0, '\0');
    if (n > 0) std::vsnprintf(s.data(), s.size() + 1, fmt, ap2);
    va_end(ap2);
    return s;
}

/// splitmix64 finalizer and the per-element canonical payload: resharding is a
/// pure copy, so bit equality with canon_value is the correctness oracle.
RS_HD std::uint64_t mix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

RS_HD std::uint64_t canon_value(std::uint64_t seed, FlatIndex element, StateKind kind) {
    const std::uint64_t k = static_cast<std::uint64_t>(static_cast<int>(kind)) + 1;
    return mix64(mix64(seed ^ static_cast<std::uint64_t>(element) * 0xD6E8FEB86659FD93ull) ^
                 k * 0xA5A5A5A5A5A5A5A5ull);
}

}  // namespace reshard
