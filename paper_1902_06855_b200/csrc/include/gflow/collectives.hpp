// SPDX-License-Identifier: Apache-2.0
// Collectives (reference API: include/gflow/collectives.hpp:18-104).
//
// ring_allreduce runs the sm_100a peer-memory kernel (K4): each rank loads its owned
// segment from every rank's buffer in ring-arrival order and stores the sum back to all
// of them — bit-identical to the reference's RS+AG ring (segment j summed from ring
// position j onward, fp16 widened per add). TrafficStats records the payload the
// reference ring would have sent ("ring" label, 2(N-1) segment transfers per call).
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <numeric>
#include <vector>

#include "gflow/buffer.hpp"
#include "gflow/device.hpp"
#include "gflow/transport.hpp"

namespace gflow {

class Communicator {
public:
    explicit Communicator(Transport& tp, int group_size = 1);
    ~Communicator();

    Transport& transport() { return tp_; }
    int rank() const { return tp_.rank(); }
    int world_size() const { return tp_.world_size(); }
    int group_size() const { return group_size_; }

    const std::vector<int>& ring_order() const { return ring_order_; }
    void set_ring_order(std::vector<int> order);

    std::uint32_t acquire_collective_id() { return next_id_.fetch_add(1); }

    std::vector<std::size_t> phase2_segment_bytes() const {
        std::lock_guard lock(mu_);
        return phase2_segments_;
    }
    void log_phase2_segment(std::size_t bytes) {
        std::lock_guard lock(mu_);
        phase2_segments_.push_back(bytes);
    }

    // B200: the rank's GPU binding, created on first use (a collective call).
    DeviceContext& device();
    // Pins this rank to a GPU before the first device collective (-1 = automatic).
    void set_device(int device) { requested_device_ = device; }

private:
    Transport& tp_;
    int group_size_;
    std::vector<int> ring_order_;
    std::atomic<std::uint32_t> next_id_{0};
    mutable std::mutex mu_;
    std::vector<std::size_t> phase2_segments_;
    int requested_device_ = -1;
    std::unique_ptr<DeviceContext> device_;
    std::mutex device_mu_;
};

void ring_allreduce(Communicator& comm, ScalarBuffer buf);
void hierarchical_allreduce(Communicator& comm, ScalarBuffer buf);
void oracle_allreduce(Communicator& comm, ScalarBuffer buf);
void reduce(Communicator& comm, ScalarBuffer buf, int root);
void broadcast(Communicator& comm, ScalarBuffer buf, int root);

namespace detail {
struct Segment {
    std::size_t offset;
    std::size_t length;
};
Segment segment_of(std::size_t length, int n, int i);

// Ring allreduce of several windows of one buffer in one launch (FusionEngine batching);
// each window is split by segment_of on its own, exactly like separate calls.
void ring_allreduce_windows(Communicator& comm, ScalarBuffer buf,
                            const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                            const std::string& label = "ring");
// TrafficStats of the reference ring for these windows (collectives.cpp:69-96): 2(N-1)
// segment_of transfers per window at this rank's ring position.
void record_ring_payload(Communicator& comm, ElementType type,
                         const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                         const std::string& label = "ring");
}  // namespace detail

}  // namespace gflow
