// SPDX-License-Identifier: Apache-2.0
// Collectives of the gflow API on the B200 data plane (reference: src/collectives.cpp).
#include "gflow/collectives.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <string>

namespace gflow {

namespace {

// control-plane tag phase of the device layer; the rooted handshake's two messages add the
// disjoint bits kReady / kRelease, so no sub-phase tag can alias another
constexpr std::uint8_t kPhaseDevice = 0x10;
constexpr std::uint32_t kReady = 0x40u, kRelease = 0x80u;

std::uint32_t device_tag(Communicator& comm) {
    return (comm.acquire_collective_id() << 8) | kPhaseDevice;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Runs fn on a device view of buf: in place when buf is GPU memory on the rank's device,
// otherwise staged through device scratch (host views: H2D before, D2H after).
template <typename F>
void with_device_view(DeviceContext& ctx, ScalarBuffer buf, F&& fn) {
    const bool dev = is_device_ptr(buf.data);
    if (dev) {
        buf.residency = Residency::kDevice;
        fn(buf);
        return;
    }
    ctx.activate();
    auto* s = static_cast<std::byte*>(ctx.scratch(buf.byte_length()));
    if (cudaMemcpy(s, buf.data, buf.byte_length(), cudaMemcpyHostToDevice) != cudaSuccess)
        throw TransportError("collective: host-to-device staging failed");
    fn(ScalarBuffer{buf.type, s, buf.length, Residency::kDevice});
    if (cudaMemcpy(buf.data, s, buf.byte_length(), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw TransportError("collective: device-to-host staging failed");
}

// Host-orchestrated rooted collective: every rank publishes its device buffer, non-roots
// signal readiness, the root launches one kernel over all (peer-mapped) buffers and
// releases the others.
template <typename F>
void rooted(Communicator& comm, ScalarBuffer dev, int root, F&& launch) {
    DeviceContext& ctx = comm.device();
    Transport& tp = comm.transport();
    const std::uint32_t tag = device_tag(comm);
    cudaDeviceSynchronize();  // this rank's pending writes to its buffer are done
    auto ptrs = ctx.exchange(dev.data, tag, (static_cast<std::uint64_t>(dev.byte_length()) << 1) | static_cast<std::uint64_t>(dev.type));
    const std::vector<std::byte> token(1);
    if (comm.rank() == root) {
        for (int r = 0; r < comm.world_size(); ++r)
            if (r != root) tp.control_recv(r, tag | kReady);
        ctx.activate();
        launch(ptrs);
        if (cudaDeviceSynchronize() != cudaSuccess) throw TransportError("rooted collective failed");
        for (int r = 0; r < comm.world_size(); ++r)
            if (r != root) tp.control_send(r, tag | kRelease, token);
    } else {
        tp.control_send(root, tag | kReady, token);
        tp.control_recv(root, tag | kRelease);
    }
}

}  // namespace

Communicator::Communicator(Transport& tp, int group_size) : tp_(tp), group_size_(group_size) {
    ring_order_.resize(static_cast<std::size_t>(tp.world_size()));
    std::iota(ring_order_.begin(), ring_order_.end(), 0);
}

Communicator::~Communicator() = default;

void Communicator::set_ring_order(std::vector<int> order) {
    if (order.size() != static_cast<std::size_t>(world_size())) throw ConfigError("ring order must cover all ranks");
    std::vector<int> s = order;
    std::sort(s.begin(), s.end());
    for (int i = 0; i < world_size(); ++i)
        if (s[static_cast<std::size_t>(i)] != i) throw ConfigError("ring order is not a permutation of ranks");
    ring_order_ = std::move(order);
}

DeviceContext& Communicator::device() {
    std::lock_guard lk(device_mu_);
    if (!device_) device_ = std::make_unique<DeviceContext>(tp_, requested_device_);
    return *device_;
}

namespace detail {

Segment segment_of(std::size_t length, int n, int i) {
    const std::size_t nn = static_cast<std::size_t>(n), idx = static_cast<std::size_t>(i);
    const std::size_t base = length / nn, rem = length % nn;
    return {idx * base + std::min(idx, rem), base + (idx < rem ? 1u : 0u)};
}

void ring_allreduce_windows(Communicator& comm, ScalarBuffer buf,
                            const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                            const std::string& label) {
    const int n = comm.world_size();
    if (n == 1 || windows.empty()) return;
    DeviceContext& ctx = comm.device();
    const std::uint32_t tag = device_tag(comm);
    with_device_view(ctx, buf, [&](ScalarBuffer dev) { ctx.ring_allreduce(dev, comm.ring_order(), windows, tag); });
    record_ring_payload(comm, buf.type, windows, label);
}

void record_ring_payload(Communicator& comm, ElementType type,
                         const std::vector<std::pair<std::size_t, std::size_t>>& windows, const std::string& label) {
    const int n = comm.world_size();
    if (n == 1) return;
    // what this rank's peer stores/loads moved, counted as the reference ring's 2(N-1)
    // segment transfers per window (collectives.cpp:69-96)
    const auto& ring = comm.ring_order();
    const int pos = static_cast<int>(std::find(ring.begin(), ring.end(), comm.rank()) - ring.begin());
    for (auto& w : windows) {
        std::uint64_t sent = 0, recvd = 0, frames = 0;
        check(gf_ring_traffic(w.second, n, pos, static_cast<int>(type), &sent, &recvd, &frames), "traffic");
        comm.transport().stats().record_send(label, sent, frames);
        comm.transport().stats().record_recv(label, recvd);
    }
}

}  // namespace detail

void ring_allreduce(Communicator& comm, ScalarBuffer buf) {
    detail::ring_allreduce_windows(comm, buf, {{0, buf.length}});
}

void oracle_allreduce(Communicator& comm, ScalarBuffer buf) {
    const int n = comm.world_size();
    if (n == 1) return;
    DeviceContext& ctx = comm.device();
    with_device_view(ctx, buf, [&](ScalarBuffer dev) {
        rooted(comm, dev, 0, [&](std::vector<void*>& ptrs) {
            check(gf_oracle_allreduce_ptrs(static_cast<int>(dev.type), ptrs.data(), n, dev.length, nullptr),
                  "oracle_allreduce");
        });
    });
    // collectives.cpp:203-226 payload: rank 0 receives and sends (N-1) buffers; others one each
    const std::uint64_t b = buf.byte_length();
    auto& st = comm.transport().stats();
    if (comm.rank() == 0) {
        st.record_send("oracle", b * static_cast<std::uint64_t>(n - 1), static_cast<std::uint64_t>(n - 1));
        st.record_recv("oracle", b * static_cast<std::uint64_t>(n - 1));
    } else {
        st.record_send("oracle", b, 1);
        st.record_recv("oracle", b);
    }
}

void broadcast(Communicator& comm, ScalarBuffer buf, int root) {
    if (root < 0 || root >= comm.world_size()) throw ConfigError("broadcast root " + std::to_string(root) + " outside group");
    const int n = comm.world_size();
    if (n == 1) return;
    DeviceContext& ctx = comm.device();
    with_device_view(ctx, buf, [&](ScalarBuffer dev) {
        rooted(comm, dev, root, [&](std::vector<void*>& ptrs) {
            check(gf_broadcast_ptrs(ptrs.data(), n, root, dev.byte_length(), nullptr), "broadcast");
        });
    });
    // a forwarding chain from the root (collectives.cpp:146-170): every rank but the
    // last on the chain forwards the buffer once
    const auto& ring = comm.ring_order();
    const int p = static_cast<int>(std::find(ring.begin(), ring.end(), comm.rank()) - ring.begin());
    const int rp = static_cast<int>(std::find(ring.begin(), ring.end(), root) - ring.begin());
    const int hop = (p - rp + n) % n;
    if (hop < n - 1) comm.transport().stats().record_send("bcast", buf.byte_length(), 1);
    if (hop > 0) comm.transport().stats().record_recv("bcast", buf.byte_length());
}

namespace {

// Payload of ring_reduce_on (collectives.cpp:99-144) at ring position p of n, root at rp:
// the n-1 reduce-scatter sends, then every non-root position sends its owned segment.
void record_ring_reduce(TrafficStats& st, const std::string& label, std::size_t len, std::size_t es, int n,
                        int p, int rp) {
    if (n <= 1) return;
    auto seg = [&](int i) { return detail::segment_of(len, n, i).length * es; };
    std::uint64_t sent = 0, recvd = 0, frames = 0;
    for (int s = 0; s < n - 1; ++s) {
        sent += seg((p - s + n) % n);
        recvd += seg((p - s - 1 + n) % n);
        ++frames;
    }
    const int owned = (p + 1) % n;
    if (p != rp) {
        sent += seg(owned);
        ++frames;
    } else {
        for (int i = 0; i < n; ++i)
            if (i != owned && (i - 1 + n) % n != rp) recvd += seg(i);
    }
    st.record_send(label, sent, frames);
    st.record_recv(label, recvd);
}

int position_of(const std::vector<int>& ring, int rank) {
    return static_cast<int>(std::find(ring.begin(), ring.end(), rank) - ring.begin());
}

}  // namespace

void reduce(Communicator& comm, ScalarBuffer buf, int root) {
    if (root < 0 || root >= comm.world_size()) throw ConfigError("reduce root " + std::to_string(root) + " outside group");
    const int n = comm.world_size();
    if (n == 1) return;
    const auto ring = comm.ring_order();
    const int rp = position_of(ring, root);
    DeviceContext& ctx = comm.device();
    with_device_view(ctx, buf, [&](ScalarBuffer dev) {
        rooted(comm, dev, root, [&](std::vector<void*>& ptrs) {
            std::vector<void*> by_pos(static_cast<std::size_t>(n));
            for (int t = 0; t < n; ++t) by_pos[static_cast<std::size_t>(t)] = ptrs[static_cast<std::size_t>(ring[t])];
            check(gf_ring_reduce_ptrs(static_cast<int>(dev.type), by_pos.data(), n, rp, dev.length, nullptr),
                  "reduce");
        });
    });
    record_ring_reduce(comm.transport().stats(), "reduce", buf.length, element_size(buf.type), n,
                       position_of(ring, comm.rank()), rp);
}

// collectives.cpp:179-201: ring_reduce_on inside each group of m consecutive ranks to its
// master, ring_allreduce_on over the masters, broadcast_on from each master. On the device
// the root launches: the group reduces, a rooted reduce over the masters (its root holds the
// masters' ring-allreduce sums: same chains) and one broadcast of that buffer to every rank.
void hierarchical_allreduce(Communicator& comm, ScalarBuffer buf) {
    const int n = comm.world_size(), m = comm.group_size();
    if (m < 1 || n % m != 0) {
        throw ConfigError("group size " + std::to_string(m) + " must divide world " + std::to_string(n));
    }
    if (n == 1) return;
    const int k = n / m;
    DeviceContext& ctx = comm.device();
    with_device_view(ctx, buf, [&](ScalarBuffer dev) {
        rooted(comm, dev, 0, [&](std::vector<void*>& ptrs) {
            const int dt = static_cast<int>(dev.type);
            if (m > 1)
                for (int g = 0; g < k; ++g)
                    check(gf_ring_reduce_ptrs(dt, ptrs.data() + static_cast<std::size_t>(g) * m, m, 0, dev.length,
                                              nullptr),
                          "hierarchical_allreduce (groups)");
            if (k > 1) {
                std::vector<void*> masters;
                for (int g = 0; g < k; ++g) masters.push_back(ptrs[static_cast<std::size_t>(g) * m]);
                check(gf_ring_reduce_ptrs(dt, masters.data(), k, 0, dev.length, nullptr),
                      "hierarchical_allreduce (masters)");
            }
            check(gf_broadcast_ptrs(ptrs.data(), n, 0, dev.byte_length(), nullptr), "hierarchical_allreduce (bcast)");
        });
    });
    // payload of the three phases as the reference moves it (labels hier1/hier2/hier3)
    auto& st = comm.transport().stats();
    const std::size_t es = element_size(buf.type), len = buf.length;
    const int g = comm.rank() / m, q = comm.rank() % m;
    record_ring_reduce(st, "hier1", len, es, m, q, 0);
    if (q == 0 && k > 1) {
        std::uint64_t sent = 0, recvd = 0, frames = 0;
        check(gf_ring_traffic(len, k, g, static_cast<int>(buf.type), &sent, &recvd, &frames), "traffic");
        st.record_send("hier2", sent, frames);
        st.record_recv("hier2", recvd);
        auto seg = [&](int i) { return detail::segment_of(len, k, i).length * es; };
        for (int s = 0; s < k - 1; ++s) comm.log_phase2_segment(seg((g - s + k) % k));      // RS sends
        for (int s = 0; s < k - 1; ++s) comm.log_phase2_segment(seg((g + 1 - s + k) % k));  // AG sends
    }
    if (m > 1) {
        if (q < m - 1) st.record_send("hier3", buf.byte_length(), 1);
        if (q > 0) st.record_recv("hier3", buf.byte_length());
    }
}

}  // namespace gflow
