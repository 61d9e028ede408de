// SPDX-License-Identifier: Apache-2.0
// The GPU side of a rank: which B200 it drives and how it reaches its peers' memory.
// (No reference counterpart: the reference moves bytes through Transport::send/recv;
// here the Transport only bootstraps and the data plane is NVLink peer memory.)
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "gflow/buffer.hpp"
#include "gflow/transport.hpp"
#include "gflow_b200.h"

namespace gflow {

// Throws the exception class matching a C-ABI status (errors.hpp taxonomy).
void check(int status, const char* what = nullptr);

// Ranks of one process that share a GPU: each collective runs as ONE launch over all
// their buffers (the kernels cannot wait on each other across launches on one device).
struct ColocatedGroup;

class DeviceContext {
public:
    enum class Mode { kSolo, kLocal, kIpc, kColocated };

    // Collective over `tp` (control plane): every rank constructs its context at the same
    // point. `device` < 0 picks: in-process ranks -> rank r on GPU r when there are enough
    // GPUs, else all on GPU 0 (colocated); separate processes -> the caller's current GPU.
    DeviceContext(Transport& tp, int device = -1);
    ~DeviceContext();
    DeviceContext(const DeviceContext&) = delete;
    DeviceContext& operator=(const DeviceContext&) = delete;

    int device() const { return device_; }
    Mode mode() const { return mode_; }
    const char* mode_name() const;
    gf_comm* comm() { return comm_; }
    int rank() const { return rank_; }
    int world() const { return world_; }

    // Makes this context's GPU current for the calling thread.
    void activate() const;

    // Collective: every rank passes its own device buffer (same call order on all ranks).
    // Returns rank r's buffer as addressable from this rank's GPU, for every r. `agree` must be
    // equal on every rank (a digest of what the collective covers), else ProtocolError.
    std::vector<void*> exchange(void* mine, std::uint32_t tag, std::uint64_t agree = 0);

    // Collective in-place sum of `windows` (element ranges of buf) with the reference's
    // ring order; buf is a DEVICE view on this rank's GPU. Blocks until done; a peer
    // timeout raises TransportError.
    void ring_allreduce(ScalarBuffer buf, const std::vector<int>& ring,
                        const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                        std::uint32_t tag);

    // Device scratch of at least `bytes` on this GPU (grown on demand, kept).
    void* scratch(std::size_t bytes, int slot = 0);

    // The rank's collective stream (a cudaStream_t, non-blocking): every device collective of
    // this context is enqueued on it, FIFO — the NVLink kernels' per-CTA epoch protocol needs
    // one collective at a time per communicator.
    void* stream() const { return stream_; }
    // True when collectives can be enqueued without a host rendezvous (peer-mapped ranks on
    // distinct GPUs); colocated ranks run each collective as one host-orchestrated launch.
    bool async_collectives() const { return mode_ == Mode::kLocal || mode_ == Mode::kIpc; }
    // Enqueue the ring allreduce of `windows` (element ranges) over rank_bufs (each rank's
    // buffer as mapped here, 16-byte aligned, from exchange()) on stream(); no host wait.
    // With `client` (a cudaStream_t) the collective is ordered after the client stream's queued
    // work and the client stream after the collective (CUDA events both ways).
    void ring_allreduce_async(ElementType type, const std::vector<void*>& rank_bufs, const std::vector<int>& ring,
                              const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                              void* client = nullptr);

private:
    Transport& tp_;
    int rank_, world_, device_ = 0;
    Mode mode_ = Mode::kSolo;
    gf_comm* comm_ = nullptr;
    std::shared_ptr<ColocatedGroup> group_;
    std::map<std::string, void*> ipc_cache_;  // peer handle bytes -> mapped base
    std::vector<std::pair<void*, std::size_t>> scratch_;
    void* stream_ = nullptr;
    void* ev_client_ = nullptr;  // client stream -> collective stream
    void* ev_done_ = nullptr;    // collective stream -> client stream
    std::mutex mu_;
};

}  // namespace gflow
