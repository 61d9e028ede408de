// SPDX-License-Identifier: Apache-2.0
// Collectives of the gflow API on the B200 data plane (reference: src/collectives.cpp).
#include "gflow/collectives.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <string>

namespace gflow {

namespace {

constexpr std::uint8_t kPhaseDevice = 9;  // control-plane tag phase of the device layer

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
    auto ptrs = ctx.exchange(dev.data, tag);
    const std::vector<std::byte> token(1);
    if (comm.rank() == root) {
        for (int r = 0; r < comm.world_size(); ++r)
            if (r != root) tp.control_recv(r, tag | 0x40u);
        ctx.activate();
        launch(ptrs);
        if (cudaDeviceSynchronize() != cudaSuccess) throw TransportError("rooted collective failed");
        for (int r = 0; r < comm.world_size(); ++r)
            if (r != root) tp.control_send(r, tag | 0x41u, token);
    } else {
        tp.control_send(root, tag | 0x40u, token);
        tp.control_recv(root, tag | 0x41u);
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
    // Payload accounting of the reference ring (collectives.cpp:69-96): what this rank's
    // peer stores/loads moved, counted as the 2(N-1) segment transfers per window.
    const auto& ring = comm.ring_order();
    const int pos = static_cast<int>(std::find(ring.begin(), ring.end(), comm.rank()) - ring.begin());
    for (auto& w : windows) {
        std::uint64_t sent = 0, recvd = 0, frames = 0;
        check(gf_ring_traffic(w.second, n, pos, static_cast<int>(buf.type), &sent, &recvd, &frames), "traffic");
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

void reduce(Communicator& comm, ScalarBuffer buf, int root) {
    if (root < 0 || root >= comm.world_size()) throw ConfigError("reduce root " + std::to_string(root) + " outside group");
    throw ConfigError("reduce: rooted ring reduce is not part of the B200 hot path (SURVEY.md §8f); "
                      "use ring_allreduce");
}

void hierarchical_allreduce(Communicator& comm, ScalarBuffer buf) {
    const int n = comm.world_size(), m = comm.group_size();
    if (m < 1 || n % m != 0) {
        throw ConfigError("group size " + std::to_string(m) + " must divide world " + std::to_string(n));
    }
    (void)buf;
    throw ConfigError("hierarchical_allreduce: not on the B200 path — one NVSwitch domain gives every "
                      "GPU full bandwidth to every peer (SURVEY.md §8f); use Algo::kRing");
}

}  // namespace gflow
