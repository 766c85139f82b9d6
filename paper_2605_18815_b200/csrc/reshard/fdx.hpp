// Descriptor exchange between local processes (fdx.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace reshard {
namespace fdx {

/// listening socket bound to the abstract name
int listen_on(const std::string& name);
/// connect to `peer` and pass descriptors (+ an opaque payload); blocks until received
void send_fds(const std::string& peer, const std::vector<int>& fds, const std::vector<std::uint8_t>& payload);
/// accept one sender and receive its descriptors (and payload)
std::vector<int> recv_fds(int listener, std::vector<std::uint8_t>* payload);
void close_fd(int fd);

}  // namespace fdx
}  // namespace reshard
