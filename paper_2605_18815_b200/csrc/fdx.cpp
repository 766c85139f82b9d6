// File-descriptor exchange between processes of one node (Unix domain sockets in the
// abstract namespace, SCM_RIGHTS). CUDA VMM allocations are shared across processes as
// POSIX file descriptors (cuMemExportToShareableHandle); cudaIpc does not cover them.
#include "reshard/fdx.hpp"

#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <stdexcept>

#include "reshard/common.hpp"

namespace reshard {
namespace fdx {

namespace {

sockaddr_un address(const std::string& name, socklen_t* len) {
    sockaddr_un a;
    std::memset(&a, 0, sizeof a);
    a.sun_family = AF_UNIX;
    if (name.size() + 1 > sizeof(a.sun_path)) throw std::runtime_error("fdx: socket name too long");
    a.sun_path[0] = '\0';  // abstract namespace: no filesystem entry to clean up
    std::memcpy(a.sun_path + 1, name.data(), name.size());
    *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + name.size());
    return a;
}

void check(bool ok, const char* what) {
    if (!ok) throw std::runtime_error(strfmt("fdx: %s failed: %s", what, std::strerror(errno)));
}

void write_all(int s, const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    while (n) {
        const ssize_t k = ::send(s, c, n, 0);
        if (k < 0 && errno == EINTR) continue;
        check(k > 0, "send");
        c += k;
        n -= static_cast<size_t>(k);
    }
}

void read_all(int s, void* p, size_t n) {
    char* c = static_cast<char*>(p);
    while (n) {
        const ssize_t k = ::recv(s, c, n, 0);
        if (k < 0 && errno == EINTR) continue;
        check(k > 0, "recv");
        c += k;
        n -= static_cast<size_t>(k);
    }
}

constexpr int kBatch = 128;  // descriptors per message (SCM_MAX_FD is 253)

}  // namespace

int listen_on(const std::string& name) {
    const int s = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    check(s >= 0, "socket");
    socklen_t len;
    sockaddr_un a = address(name, &len);
    if (::bind(s, reinterpret_cast<sockaddr*>(&a), len) != 0) {
        ::close(s);
        check(false, "bind");
    }
    check(::listen(s, 64) == 0, "listen");
    return s;
}

void send_fds(const std::string& peer, const std::vector<int>& fds, const std::vector<std::uint8_t>& payload) {
    const int s = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    check(s >= 0, "socket");
    socklen_t len;
    sockaddr_un a = address(peer, &len);
    int rc = -1;
    for (int attempt = 0; attempt < 2000 && rc != 0; ++attempt) {  // the peer may not listen yet
        rc = ::connect(s, reinterpret_cast<sockaddr*>(&a), len);
        if (rc != 0) ::usleep(5000);
    }
    if (rc != 0) {
        ::close(s);
        check(false, "connect");
    }
    const std::uint64_t hdr[2] = {fds.size(), payload.size()};
    write_all(s, hdr, sizeof hdr);
    write_all(s, payload.data(), payload.size());
    for (size_t i = 0; i < fds.size(); i += kBatch) {
        const int n = static_cast<int>(std::min<size_t>(kBatch, fds.size() - i));
        char byte = 'F';
        iovec io{&byte, 1};
        std::vector<char> ctrl(CMSG_SPACE(sizeof(int) * static_cast<size_t>(n)), 0);
        msghdr m;
        std::memset(&m, 0, sizeof m);
        m.msg_iov = &io;
        m.msg_iovlen = 1;
        m.msg_control = ctrl.data();
        m.msg_controllen = ctrl.size();
        cmsghdr* c = CMSG_FIRSTHDR(&m);
        c->cmsg_level = SOL_SOCKET;
        c->cmsg_type = SCM_RIGHTS;
        c->cmsg_len = CMSG_LEN(sizeof(int) * static_cast<size_t>(n));
        std::memcpy(CMSG_DATA(c), fds.data() + i, sizeof(int) * static_cast<size_t>(n));
        ssize_t k;
        do {
            k = ::sendmsg(s, &m, 0);
        } while (k < 0 && errno == EINTR);
        check(k == 1, "sendmsg");
    }
    char ack;
    read_all(s, &ack, 1);  // the receiver holds the descriptors before we may close ours
    ::close(s);
}

std::vector<int> recv_fds(int listener, std::vector<std::uint8_t>* payload) {
    int s;
    do {
        s = ::accept4(listener, nullptr, nullptr, SOCK_CLOEXEC);
    } while (s < 0 && errno == EINTR);
    check(s >= 0, "accept");
    // only processes of this user may hand us descriptors (abstract sockets have no
    // filesystem permissions)
    ucred cred{};
    socklen_t cl = sizeof cred;
    if (::getsockopt(s, SOL_SOCKET, SO_PEERCRED, &cred, &cl) != 0 || cred.uid != ::getuid()) {
        ::close(s);
        throw ConfigError("fdx: connection from another user refused");
    }
    std::uint64_t hdr[2];
    read_all(s, hdr, sizeof hdr);
    if (hdr[0] > (1u << 20) || hdr[1] > (1ull << 30)) {
        ::close(s);
        throw ConfigError("fdx: malformed header");
    }
    if (payload) {
        payload->resize(static_cast<size_t>(hdr[1]));
        read_all(s, payload->data(), payload->size());
    } else {
        std::vector<std::uint8_t> skip(static_cast<size_t>(hdr[1]));
        read_all(s, skip.data(), skip.size());
    }
    std::vector<int> fds;
    while (fds.size() < hdr[0]) {
        const int n = static_cast<int>(std::min<std::uint64_t>(kBatch, hdr[0] - fds.size()));
        char byte;
        iovec io{&byte, 1};
        std::vector<char> ctrl(CMSG_SPACE(sizeof(int) * static_cast<size_t>(n)), 0);
        msghdr m;
        std::memset(&m, 0, sizeof m);
        m.msg_iov = &io;
        m.msg_iovlen = 1;
        m.msg_control = ctrl.data();
        m.msg_controllen = ctrl.size();
        ssize_t k;
        do {
            k = ::recvmsg(s, &m, MSG_CMSG_CLOEXEC);
        } while (k < 0 && errno == EINTR);
        check(k == 1, "recvmsg");
        cmsghdr* c = CMSG_FIRSTHDR(&m);
        check(c && c->cmsg_type == SCM_RIGHTS, "SCM_RIGHTS");
        const size_t got = (c->cmsg_len - CMSG_LEN(0)) / sizeof(int);
        check(got > 0 && got <= static_cast<size_t>(n), "SCM_RIGHTS count");
        const int* p = reinterpret_cast<const int*>(CMSG_DATA(c));
        fds.insert(fds.end(), p, p + got);
    }
    const char ack = 'A';
    write_all(s, &ack, 1);
    ::close(s);
    return fds;
}

void close_fd(int fd) {
    if (fd >= 0) ::close(fd);
}

}  // namespace fdx
}  // namespace reshard
