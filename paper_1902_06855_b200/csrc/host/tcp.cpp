// SPDX-License-Identifier: Apache-2.0
// TcpTransport (see gflow/tcp.hpp): full-mesh GFL1 over TCP with one poll() progress thread.
// Reference behaviour kept: connection topology and handshake (src/tcp.cpp:157-253), recv
// timeout -> TransportError, a broken connection poisons the transport while frames that
// already arrived stay receivable, send never blocks the caller.
#include "gflow/tcp.hpp"

#include <arpa/inet.h>
#include <fcntl.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/eventfd.h>
#include <sys/socket.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <unordered_map>

namespace gflow {

namespace {

std::pair<std::string, std::uint16_t> split_address(const std::string& a) {
    const auto c = a.rfind(':');
    if (c == std::string::npos || c == 0) throw ConfigError("address '" + a + "' is not host:port");
    int port = 0;
    try {
        port = std::stoi(a.substr(c + 1));
    } catch (const std::exception&) {
        throw ConfigError("address '" + a + "' has no numeric port");
    }
    if (port < 1 || port > 65535) throw ConfigError("address '" + a + "' has an invalid port");
    return {a.substr(0, c), static_cast<std::uint16_t>(port)};
}

sockaddr_in ipv4(const std::string& host, std::uint16_t port) {
    sockaddr_in sa{};
    sa.sin_family = AF_INET;
    sa.sin_port = htons(port);
    const std::string h = host == "localhost" ? "127.0.0.1" : host;
    if (::inet_pton(AF_INET, h.c_str(), &sa.sin_addr) != 1) throw ConfigError("host '" + host + "' is not IPv4");
    return sa;
}

// blocking helpers, used only while the mesh is being built
void send_exact(int fd, const std::byte* p, std::size_t n) {
    while (n > 0) {
        const ssize_t k = ::send(fd, p, n, MSG_NOSIGNAL);
        if (k < 0 && errno == EINTR) continue;
        if (k <= 0) throw TransportError(std::string("handshake send failed: ") + std::strerror(errno));
        p += k;
        n -= static_cast<std::size_t>(k);
    }
}

void recv_exact(int fd, std::byte* p, std::size_t n) {
    while (n > 0) {
        const ssize_t k = ::recv(fd, p, n, 0);
        if (k < 0 && errno == EINTR) continue;
        if (k <= 0) throw TransportError("handshake: connection closed");
        p += k;
        n -= static_cast<std::size_t>(k);
    }
}

std::uint64_t box_key(int src, std::uint8_t type, std::uint32_t tag) {
    return (std::uint64_t(std::uint32_t(src)) << 40) | (std::uint64_t(type) << 32) | tag;
}

}  // namespace

struct TcpTransport::Impl {
    struct Peer {
        int fd = -1;
        bool open = false;
        // outgoing: encoded frames, the front one partly written
        std::deque<std::vector<std::byte>> out;
        std::size_t out_off = 0;
        // incoming: header, then payload
        std::byte hdr[Frame::kHeaderSize];
        std::size_t hdr_got = 0;
        Frame cur;
        std::uint64_t need = 0;
        std::size_t pay_got = 0;
        bool in_payload = false;
    };

    std::vector<Peer> peers;
    int listen_fd = -1;
    int wake_fd = -1;
    std::thread progress;
    std::atomic<bool> stopping{false};

    std::mutex send_mu;  // peers[*].out / out_off

    std::mutex box_mu;   // box, poisoned, reason
    std::condition_variable box_cv;
    std::unordered_map<std::uint64_t, std::deque<std::vector<std::byte>>> box;
    bool poisoned = false;
    std::string reason;
    std::vector<char> closed;  // per peer: orderly EOF seen (frames already received stay readable)

    void wake() const {
        const std::uint64_t one = 1;
        [[maybe_unused]] const ssize_t k = ::write(wake_fd, &one, sizeof(one));
    }

    void poison(const std::string& why) {
        {
            std::lock_guard lk(box_mu);
            if (!poisoned) {
                poisoned = true;
                reason = why;
            }
        }
        box_cv.notify_all();
    }

    void drop(int r, const std::string& why, bool orderly = false) {
        Peer& p = peers[static_cast<std::size_t>(r)];
        if (!p.open) return;
        p.open = false;
        if (stopping.load()) return;
        if (orderly) {  // the peer finished and closed: only waits on ITS frames can fail now
            {
                std::lock_guard lk(box_mu);
                if (closed.size() < peers.size()) closed.resize(peers.size(), 0);
                closed[static_cast<std::size_t>(r)] = 1;
            }
            box_cv.notify_all();
            return;
        }
        poison(why);
    }

    // reads everything available on peer r; complete frames go to the mailbox
    void on_readable(int r) {
        Peer& p = peers[static_cast<std::size_t>(r)];
        for (;;) {
            std::byte* dst;
            std::size_t want;
            if (!p.in_payload) {
                dst = p.hdr + p.hdr_got;
                want = Frame::kHeaderSize - p.hdr_got;
            } else {
                dst = p.cur.payload.data() + p.pay_got;
                want = static_cast<std::size_t>(p.need) - p.pay_got;
            }
            ssize_t k = 0;
            if (want > 0) {
                k = ::recv(p.fd, dst, want, 0);
                if (k < 0 && errno == EINTR) continue;
                if (k < 0 && (errno == EAGAIN || errno == EWOULDBLOCK)) return;
                if (k <= 0) {
                    drop(r, "connection to rank " + std::to_string(r) + (k == 0 ? " closed" : " reset"), k == 0);
                    return;
                }
            }
            if (!p.in_payload) {
                p.hdr_got += static_cast<std::size_t>(k);
                if (p.hdr_got < Frame::kHeaderSize) continue;
                try {
                    p.need = Frame::decode_header(std::span<const std::byte>(p.hdr, Frame::kHeaderSize), p.cur);
                } catch (const ProtocolError& e) {
                    drop(r, "protocol error from rank " + std::to_string(r) + ": " + e.what());
                    return;
                }
                if (p.cur.src_rank != std::uint32_t(r)) {
                    drop(r, "frame from rank " + std::to_string(r) + " claims source " +
                                std::to_string(p.cur.src_rank));
                    return;
                }
                p.cur.payload.assign(static_cast<std::size_t>(p.need), std::byte{0});
                p.pay_got = 0;
                p.in_payload = true;
            } else {
                p.pay_got += static_cast<std::size_t>(k);
            }
            if (p.in_payload && p.pay_got == p.need) {
                {
                    std::lock_guard lk(box_mu);
                    box[box_key(r, p.cur.msg_type, p.cur.tag)].push_back(std::move(p.cur.payload));
                }
                box_cv.notify_all();
                p.cur = Frame{};
                p.hdr_got = 0;
                p.in_payload = false;
            }
        }
    }

    void on_writable(int r) {
        Peer& p = peers[static_cast<std::size_t>(r)];
        std::lock_guard lk(send_mu);
        while (!p.out.empty()) {
            const auto& f = p.out.front();
            const ssize_t k = ::send(p.fd, f.data() + p.out_off, f.size() - p.out_off, MSG_NOSIGNAL);
            if (k < 0 && errno == EINTR) continue;
            if (k < 0 && (errno == EAGAIN || errno == EWOULDBLOCK)) return;
            if (k <= 0) {
                p.out.clear();
                p.out_off = 0;
                drop(r, "send to rank " + std::to_string(r) + " failed: " + std::strerror(errno));
                return;
            }
            p.out_off += static_cast<std::size_t>(k);
            if (p.out_off == f.size()) {
                p.out.pop_front();
                p.out_off = 0;
            }
        }
    }

    bool sends_pending() {
        std::lock_guard lk(send_mu);
        for (const auto& p : peers)
            if (p.open && !p.out.empty()) return true;
        return false;
    }

    void loop(std::chrono::milliseconds drain_limit) {
        std::vector<pollfd> fds;
        std::vector<int> who;
        std::chrono::steady_clock::time_point drain_deadline{};
        for (;;) {
            if (stopping.load()) {
                if (drain_deadline == std::chrono::steady_clock::time_point{})
                    drain_deadline = std::chrono::steady_clock::now() + drain_limit;
                if (!sends_pending() || std::chrono::steady_clock::now() > drain_deadline) return;
            }
            fds.clear();
            who.clear();
            fds.push_back({wake_fd, POLLIN, 0});
            who.push_back(-1);
            {
                std::lock_guard lk(send_mu);
                for (std::size_t r = 0; r < peers.size(); ++r) {
                    if (!peers[r].open) continue;
                    short ev = POLLIN;
                    if (!peers[r].out.empty()) ev |= POLLOUT;
                    fds.push_back({peers[r].fd, ev, 0});
                    who.push_back(static_cast<int>(r));
                }
            }
            const int n = ::poll(fds.data(), fds.size(), 100);
            if (n < 0 && errno != EINTR) {
                poison(std::string("poll failed: ") + std::strerror(errno));
                return;
            }
            if (n <= 0) continue;
            for (std::size_t i = 0; i < fds.size(); ++i) {
                if (fds[i].revents == 0) continue;
                if (who[i] < 0) {
                    std::uint64_t v;
                    [[maybe_unused]] const ssize_t k = ::read(wake_fd, &v, sizeof(v));
                    continue;
                }
                const int r = who[i];
                if (fds[i].revents & (POLLIN | POLLHUP | POLLERR)) on_readable(r);
                if (peers[static_cast<std::size_t>(r)].open && (fds[i].revents & POLLOUT)) on_writable(r);
            }
        }
    }
};

std::vector<std::string> TcpTransport::loopback_addresses(int world_size, std::uint16_t port_base) {
    std::vector<std::string> v;
    v.reserve(static_cast<std::size_t>(std::max(world_size, 0)));
    for (int r = 0; r < world_size; ++r) v.push_back("127.0.0.1:" + std::to_string(port_base + r));
    return v;
}

TcpTransport::TcpTransport(int rank, int world_size, const std::vector<std::string>& peers)
    : rank_(rank), world_size_(world_size), impl_(std::make_unique<Impl>()) {
    if (world_size < 1) throw ConfigError("world_size must be >= 1");
    if (rank < 0 || rank >= world_size) throw ConfigError("rank " + std::to_string(rank) + " outside the world");
    if (peers.size() != static_cast<std::size_t>(world_size))
        throw ConfigError("need one address per rank (" + std::to_string(world_size) + "), got " +
                          std::to_string(peers.size()));
    Impl& I = *impl_;
    I.peers.resize(static_cast<std::size_t>(world_size));
    if (world_size == 1) return;
    auto fail_cleanup = [&] {
        for (auto& p : I.peers)
            if (p.fd >= 0) ::close(p.fd);
        if (I.listen_fd >= 0) ::close(I.listen_fd);
    };
    try {
        // listen first, so lower-ranked peers' connects queue up while we dial
        const auto [my_host, my_port] = split_address(peers[static_cast<std::size_t>(rank)]);
        (void)my_host;
        I.listen_fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
        if (I.listen_fd < 0) throw TransportError("socket() failed");
        const int on = 1;
        ::setsockopt(I.listen_fd, SOL_SOCKET, SO_REUSEADDR, &on, sizeof(on));
        sockaddr_in any{};
        any.sin_family = AF_INET;
        any.sin_addr.s_addr = htonl(INADDR_ANY);
        any.sin_port = htons(my_port);
        if (::bind(I.listen_fd, reinterpret_cast<sockaddr*>(&any), sizeof(any)) != 0)
            throw TransportError("rank " + std::to_string(rank) + ": bind to port " + std::to_string(my_port) +
                                 " failed: " + std::strerror(errno));
        if (::listen(I.listen_fd, world_size) != 0) throw TransportError("listen() failed");

        Frame hello;
        hello.msg_type = kMsgHandshake;
        hello.src_rank = static_cast<std::uint32_t>(rank);
        hello.payload.resize(4);
        const std::uint32_t ws = static_cast<std::uint32_t>(world_size);
        for (int i = 0; i < 4; ++i) hello.payload[static_cast<std::size_t>(i)] = std::byte((ws >> (8 * i)) & 0xFFu);
        const auto hello_bytes = hello.encode();

        // dial every lower rank (retry while it comes up), then announce ourselves
        for (int j = 0; j < rank; ++j) {
            const auto [host, port] = split_address(peers[static_cast<std::size_t>(j)]);
            const sockaddr_in sa = ipv4(host, port);
            const auto deadline = std::chrono::steady_clock::now() + timeout_;
            int fd = -1;
            for (;;) {
                fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
                if (fd < 0) throw TransportError("socket() failed");
                if (::connect(fd, reinterpret_cast<const sockaddr*>(&sa), sizeof(sa)) == 0) break;
                ::close(fd);
                fd = -1;
                if (std::chrono::steady_clock::now() > deadline)
                    throw TransportError("rank " + std::to_string(j) + " unreachable at " +
                                         peers[static_cast<std::size_t>(j)]);
                std::this_thread::sleep_for(std::chrono::milliseconds(10));
            }
            I.peers[static_cast<std::size_t>(j)].fd = fd;
            send_exact(fd, hello_bytes.data(), hello_bytes.size());
        }
        // accept every higher rank; its handshake says who it is
        for (int a = rank + 1; a < world_size; ++a) {
            pollfd pf{I.listen_fd, POLLIN, 0};
            const int ready = ::poll(&pf, 1, static_cast<int>(timeout_.count()));
            if (ready <= 0) throw TransportError("rank " + std::to_string(rank) + ": peers never connected");
            const int fd = ::accept4(I.listen_fd, nullptr, nullptr, SOCK_CLOEXEC);
            if (fd < 0) throw TransportError("accept() failed");
            std::byte h[Frame::kHeaderSize];
            Frame f;
            std::uint64_t len = 0;
            try {
                recv_exact(fd, h, sizeof(h));
                len = Frame::decode_header(std::span<const std::byte>(h, sizeof(h)), f);
            } catch (...) {
                ::close(fd);
                throw;
            }
            if (f.msg_type != kMsgHandshake || len != 4) {
                ::close(fd);
                throw ProtocolError("expected a GFL1 handshake frame");
            }
            std::byte w[4];
            recv_exact(fd, w, 4);
            const std::uint32_t peer_world = std::to_integer<std::uint32_t>(w[0]) |
                                             (std::to_integer<std::uint32_t>(w[1]) << 8) |
                                             (std::to_integer<std::uint32_t>(w[2]) << 16) |
                                             (std::to_integer<std::uint32_t>(w[3]) << 24);
            const int src = static_cast<int>(f.src_rank);
            if (peer_world != ws) {
                ::close(fd);
                throw ProtocolError("world_size mismatch: rank " + std::to_string(src) + " says " +
                                    std::to_string(peer_world) + ", this rank " + std::to_string(ws));
            }
            if (src <= rank || src >= world_size || I.peers[static_cast<std::size_t>(src)].fd >= 0) {
                ::close(fd);
                throw ProtocolError("unexpected handshake from rank " + std::to_string(src));
            }
            I.peers[static_cast<std::size_t>(src)].fd = fd;
        }
        for (auto& p : I.peers) {
            if (p.fd < 0) continue;
            const int one = 1;
            ::setsockopt(p.fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
            ::fcntl(p.fd, F_SETFL, ::fcntl(p.fd, F_GETFL) | O_NONBLOCK);
            p.open = true;
        }
        I.wake_fd = ::eventfd(0, EFD_NONBLOCK | EFD_CLOEXEC);
        if (I.wake_fd < 0) throw TransportError("eventfd() failed");
    } catch (...) {
        fail_cleanup();
        throw;
    }
    const auto drain = timeout_;
    I.progress = std::thread([this, drain] { impl_->loop(drain); });
}

TcpTransport::~TcpTransport() {
    Impl& I = *impl_;
    if (I.progress.joinable()) {
        I.stopping.store(true);
        I.wake();
        I.progress.join();  // flushes queued frames first (bounded by the timeout)
    }
    for (auto& p : I.peers) {
        if (p.fd >= 0) {
            ::shutdown(p.fd, SHUT_RDWR);
            ::close(p.fd);
        }
    }
    if (I.listen_fd >= 0) ::close(I.listen_fd);
    if (I.wake_fd >= 0) ::close(I.wake_fd);
}

void TcpTransport::post(int dst, std::uint8_t type, std::uint32_t tag, std::span<const std::byte> payload) {
    if (dst < 0 || dst >= world_size_ || dst == rank_)
        throw ConfigError("invalid destination rank " + std::to_string(dst));
    Frame f;
    f.msg_type = type;
    f.tag = tag;
    f.src_rank = static_cast<std::uint32_t>(rank_);
    f.payload.assign(payload.begin(), payload.end());
    {
        std::lock_guard lk(impl_->box_mu);
        if (impl_->poisoned) throw TransportError(impl_->reason);
    }
    {
        std::lock_guard lk(impl_->send_mu);
        auto& p = impl_->peers[static_cast<std::size_t>(dst)];
        if (!p.open) throw TransportError("connection to rank " + std::to_string(dst) + " is down");
        p.out.push_back(f.encode());
    }
    impl_->wake();
}

std::vector<std::byte> TcpTransport::take(int src, std::uint8_t type, std::uint32_t tag) {
    if (src < 0 || src >= world_size_ || src == rank_)
        throw ConfigError("invalid source rank " + std::to_string(src));
    const std::uint64_t key = box_key(src, type, tag);
    std::unique_lock lk(impl_->box_mu);
    auto ready = [&] {
        auto it = impl_->box.find(key);
        return it != impl_->box.end() && !it->second.empty();
    };
    auto gone = [&] {
        return static_cast<std::size_t>(src) < impl_->closed.size() && impl_->closed[static_cast<std::size_t>(src)];
    };
    impl_->box_cv.wait_for(lk, timeout_, [&] { return ready() || impl_->poisoned || gone(); });
    if (!ready()) {
        if (impl_->poisoned) throw TransportError(impl_->reason);
        if (gone()) throw TransportError("connection to rank " + std::to_string(src) + " closed");
        throw TransportError("recv timeout at rank " + std::to_string(rank_) + " (src " + std::to_string(src) +
                             ", tag " + std::to_string(tag) + ")");
    }
    auto& q = impl_->box[key];
    std::vector<std::byte> v = std::move(q.front());
    q.pop_front();
    return v;
}

void TcpTransport::send(int dst, std::uint32_t tag, std::span<const std::byte> payload, const std::string& phase) {
    post(dst, kMsgData, tag, payload);
    stats_.record_send(phase, payload.size());
}

std::vector<std::byte> TcpTransport::recv(int src, std::uint32_t tag, const std::string& phase) {
    auto v = take(src, kMsgData, tag);
    stats_.record_recv(phase, v.size());
    return v;
}

void TcpTransport::control_send(int dst, std::uint32_t tag, std::span<const std::byte> payload) {
    post(dst, kMsgControl, tag, payload);
}

std::vector<std::byte> TcpTransport::control_recv(int src, std::uint32_t tag) {
    return take(src, kMsgControl, tag);
}

// Dissemination barrier: in round k every rank signals rank + 2^k and waits for rank - 2^k;
// after ceil(log2 N) rounds every rank has (transitively) heard from every other.
void TcpTransport::barrier() {
    const std::uint32_t seq = barrier_seq_++;
    if (world_size_ == 1) return;
    for (int k = 0, d = 1; d < world_size_; ++k, d <<= 1) {
        const std::uint32_t tag = (seq << 5) | static_cast<std::uint32_t>(k);
        post((rank_ + d) % world_size_, kMsgBarrier, tag, {});
        try {
            take((rank_ - d + world_size_) % world_size_, kMsgBarrier, tag);
        } catch (const TransportError& e) {
            throw TransportError(std::string("barrier ") + std::to_string(seq) + " failed at rank " +
                                 std::to_string(rank_) + ": " + e.what());
        }
    }
}

}  // namespace gflow
