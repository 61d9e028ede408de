// SPDX-License-Identifier: Apache-2.0
// Communicator internals shared by the NVLink kernels (ring.cu, fused.cu).
//
// Per-rank device allocation: [ flag area | symmetric heap ]. The whole allocation is
// IPC-exported, so every peer can write this rank's flags and read/write its heap.
// Flag area layout (uint64 words unless noted):
//   [0, kFlagWords)                 ring barrier flags  flags[cta][src_rank]   (peers write)
//   [kFlagWords, +kMaxBlocks)       per-CTA epoch counters (local)
//   [+kMaxBlocks, +32)              ring work/done counters (local)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "gf_internal.cuh"

constexpr int kMaxBlocks = 1024;
constexpr int kMaxW = GF_MAX_WINDOWS_PER_LAUNCH;
constexpr int kRingThreads = 512;
constexpr uint64_t kFlagWords = uint64_t(kMaxBlocks) * GF_MAX_RANKS;
constexpr uint64_t kRingFlagBytes = (kFlagWords + kMaxBlocks + 32) * sizeof(uint64_t);
constexpr uint64_t kFlagBytes = kRingFlagBytes;
static_assert(kFlagBytes % 256 == 0, "the symmetric heap stays 256-byte aligned");

struct gf_comm {
    int world = 0, rank = 0, device = 0, pos = 0;
    int ring[GF_MAX_RANKS] = {};
    uint64_t heap_bytes = 0;
    char* alloc = nullptr;  // [flags | heap]
    char* peer_alloc[GF_MAX_RANKS] = {};
    bool ipc_opened[GF_MAX_RANKS] = {};
    int* err_host = nullptr;  // mapped pinned page: [0] error word, trace at +64 B
    int* err_dev = nullptr;
    bool trace = false;
    uint64_t timeout_ns = 30ull * 1000 * 1000 * 1000;  // transport.hpp:25 kDefaultTimeout
    bool connected = false;
    // gf_comm_connect_colocated: every rank of the world lives on this device (emulation of an
    // N-GPU world on one B200, the same kernels and barriers); grids are capped so all ranks'
    // barrier-waiting CTAs fit on the SMs at once
    bool colocated = false;
    int grid_cap = 0;
    int max_blocks = 0;     // gf_comm_set_max_blocks (0: automatic)
    int block_threads = 0;  // gf_comm_set_block_threads: CTA size of the CSC exchange (0: 512)
    uint64_t sel_inbox_off = UINT64_MAX;  // gf_comm_set_select_inbox (UINT64_MAX: pull protocol)
    // gf_comm_set_csc_inbox: the routed CSC exchange (UINT64_MAX: off). World-1 slots of
    // csc_slot_elems fp16 elements; slot t of the owner at position j holds position j + 1 + t.
    uint64_t csc_inbox_off = UINT64_MAX;
    uint64_t csc_slot_elems = 0;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline int comm_ready(gf_comm* c) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    if (!c->connected) return gfi::fail(GF_ERR_CONFIG, "communicator not connected");
    if (c->err_host && *reinterpret_cast<volatile int*>(c->err_host) != 0)
        return gfi::fail(GF_ERR_TRANSPORT, "communicator poisoned by an earlier peer timeout (rank " +
                                               std::to_string(c->rank) + ")");
    return GF_OK;
}

}  // namespace
