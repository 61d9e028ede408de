// SPDX-License-Identifier: Apache-2.0
// Device pieces of the NVLink ring shared by ring.cu (K4, the collective alone) and
// fused.cu (the dense step: pack + ring + unpack in one kernel): launch arguments, the
// per-CTA-pair cross-GPU barrier and the segment reduction.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "comm.cuh"
#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace {

struct RingArgs {
    char* bufs[GF_MAX_RANKS];            // buffer base of each RANK (peer-mapped)
    int ring[GF_MAX_RANKS];              // rank at each ring position
    int world, rank, pos;
    int nwin;                            // >= 0 explicit windows; -1: read plan
    uint64_t* flags_local;
    uint64_t* flags_peer[GF_MAX_RANKS];  // by rank
    uint64_t* epochs;                    // local, one per CTA
    uint64_t* work;                      // local dynamic item counter (re-armed by the last CTA)
    unsigned* done;                      // local CTA completion counter
    uint64_t timeout_ns;
    int* err;
    uint64_t* trace;                     // host-mapped [start, entered, exit_begin, end] or null
    const uint64_t* plan;
    // planned (CSC) mode only: after the exit barrier every CTA writes its staging vectors
    // back into the local fp16 pool and adds their exact |x| units to nacc (the work of
    // gf_csc_scatter, sparse.cpp:162-168, fused into the collective). Null: no write-back.
    char* wb_pool;
    uint64_t* wb_nacc;
    uint64_t wb_chunk, wb_nc;
    // routed CSC exchange (gf_comm_set_csc_inbox): the reduce-scatter's operands are local, my
    // staging buffer and my inbox slots (ring order from my position); null: pulled from the peers
    const char* csc_inbox;
    uint64_t csc_slot_bytes;
    int csc_push_ag;  // ... and the owners push the all-gather into every staging (read locally)
    uint64_t wstart[kMaxW];
    uint64_t wlen[kMaxW];
};

// ---- cross-GPU barrier (CTA b <-> CTA b of every peer) ------------------------
// release_writes: the CTA's earlier global stores (incl. pushes into peers) must be visible
// to a peer that observes the flag. bar.sync orders them before the signalling threads, whose
// system-scope fence + release store make them cumulative (the cooperative-groups grid-sync
// pattern, at .sys scope). At kernel entry nothing was written yet: no fence.
template <typename A>
__device__ bool cross_barrier(const A& a, uint64_t val, int* s_ok, bool release_writes = true) {
    __syncthreads();
    const int t = threadIdx.x;
    if (t < a.world && t != a.rank) {
        if (release_writes) __threadfence_system();
        gfd::st_release_sys(a.flags_peer[t] + blockIdx.x * GF_MAX_RANKS + a.rank, val);
        const uint64_t* f = a.flags_local + blockIdx.x * GF_MAX_RANKS + t;
        if (a.timeout_ns != 0 && gfd::ld_acquire_sys(f) < val) {  // 0: GF_DIAG_NOWAIT probe
            const uint64_t t0 = gfd::globaltimer_ns();
            uint32_t spins = 0;
            while (gfd::ld_acquire_sys(f) < val) {
                if ((++spins & 255u) == 0) {
                    if (*reinterpret_cast<volatile int*>(a.err) != 0) { *s_ok = 0; break; }
                    if (gfd::globaltimer_ns() - t0 > a.timeout_ns) {
                        *reinterpret_cast<volatile int*>(a.err) = 1;
                        *s_ok = 0;
                        break;
                    }
                }
            }
        }
    }
    __syncthreads();
    return *s_ok != 0;
}

// ---- reduction of one element range [e0, e1) -----------------------------------
template <int DT>
struct Vec;
template <>
struct Vec<GF_F16> {
    static constexpr int kElems = 8;
    __device__ static uint4 acc(uint4 local, uint4 a) { return gfd::acc16x8(local, a); }
    __device__ static void scalar(const RingArgs& a, const char* const* src, int n, uint64_t e) {
        uint16_t acc = reinterpret_cast<const uint16_t*>(src[0])[e];
        for (int t = 1; t < n; ++t) acc = gfd::acc16(reinterpret_cast<const uint16_t*>(src[t])[e], acc);
        for (int r = 0; r < a.world; ++r) reinterpret_cast<uint16_t*>(a.bufs[r])[e] = acc;
    }
};
template <>
struct Vec<GF_F32> {
    static constexpr int kElems = 4;
    __device__ static uint4 acc(uint4 local, uint4 a) { return gfd::acc32x4(local, a); }
    __device__ static void scalar(const RingArgs& a, const char* const* src, int n, uint64_t e) {
        float acc = reinterpret_cast<const float*>(src[0])[e];
        for (int t = 1; t < n; ++t) acc = gfd::add(reinterpret_cast<const float*>(src[t])[e], acc);
        for (int r = 0; r < a.world; ++r) reinterpret_cast<float*>(a.bufs[r])[e] = acc;
    }
};

// Reduction of one window's owned segment: the grid (or the CTA group given the window)
// sweeps its 16-byte vectors in lockstep (thread g takes vectors g, g+T, g+2T, ... with T =
// all threads sweeping it), so
// every thread gets the same number of vectors (+-1) and all CTAs of a rank finish
// together; U vectors x N sources of loads are in flight per thread.
template <int DT, int NT>
__device__ __forceinline__ void reduce_segment(const RingArgs& a, const char* const* src, int n,
                                               uint64_t e0, uint64_t e1, uint64_t gtid, uint64_t T,
                                               int edge_cta = 0) {
    constexpr int VE = Vec<DT>::kElems;
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int U = NMAX <= 4 ? 4 : (NMAX <= 8 ? 2 : 1);
    const uint64_t v0 = (e0 + VE - 1) / VE, v1 = e1 / VE;
    const bool edge = int(blockIdx.x) == edge_cta;  // this CTA takes the unaligned edges
    if (v0 >= v1) {  // no aligned vector inside: all scalar, the edge CTA
        if (edge)
            for (uint64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) Vec<DT>::scalar(a, src, n, e);
        return;
    }
    if (edge) {
        for (uint64_t e = e0 + threadIdx.x; e < v0 * VE; e += blockDim.x) Vec<DT>::scalar(a, src, n, e);
        for (uint64_t e = v1 * VE + threadIdx.x; e < e1; e += blockDim.x) Vec<DT>::scalar(a, src, n, e);
    }
    for (uint64_t v = v0 + gtid; v < v1; v += T * U) {
        uint4 x[U][NMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * T;
            if (vv < v1) {
#pragma unroll
                for (int t = 0; t < NMAX; ++t)
                    if (t < n) x[u][t] = gfd::ld16(src[t] + vv * 16);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * T;
            if (vv < v1) {
                uint4 acc = x[u][0];
#pragma unroll
                for (int t = 1; t < NMAX; ++t)
                    if (t < n) acc = Vec<DT>::acc(x[u][t], acc);
                // push the sum to every rank, starting with the next one on the ring so the
                // ranks' first stores spread over distinct destinations
#pragma unroll
                for (int t = 0; t < NMAX; ++t)
                    if (t < n) gfd::st16(const_cast<char*>(src[(t + 1) % n]) + vv * 16, acc);
            }
        }
    }
}

inline void fill_common(gf_comm* c, RingArgs& a, uint64_t heap_off) {
    a.world = c->world;
    a.rank = c->rank;
    a.pos = c->pos;
    for (int r = 0; r < c->world; ++r) {
        a.bufs[r] = c->peer_alloc[r] + kFlagBytes + heap_off;
        a.flags_peer[r] = reinterpret_cast<uint64_t*>(c->peer_alloc[r]);
        a.ring[r] = c->ring[r];
    }
    a.flags_local = reinterpret_cast<uint64_t*>(c->alloc);
    a.epochs = a.flags_local + kFlagWords;
    a.work = a.epochs + kMaxBlocks;
    a.done = reinterpret_cast<unsigned*>(a.work + 16);
    a.timeout_ns = c->timeout_ns;
    a.err = c->err_dev;
    a.trace = c->trace ? reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(c->err_dev) + 64) : nullptr;
}

// Explicit windows (FusionEngine theta windows, <= kMaxW per launch, lengths as they fall):
// the owned segments of all windows form ONE vector space that the grid sweeps in lockstep,
// so a launch over many small windows costs one NVLink round trip, not one per window.
// FlatWins::build runs before the entry barrier (it only reads the launch arguments).
struct FlatWins {
    uint64_t pre[kMaxW + 1];  // vectors of the owned segments of windows < w
    uint64_t v0[kMaxW];       // first aligned vector of window w's owned segment
    uint64_t e0[kMaxW], e1[kMaxW];
};

template <int VE>
__device__ __forceinline__ void flat_build(const RingArgs& a, int n, int p, FlatWins& f) {
    __shared__ uint64_t warp_tot[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();  // f may still be read by a sweep over the previous segment
    for (int w0 = 0; w0 < a.nwin; w0 += blockDim.x) {  // one pass for <= blockDim windows
        const int w = w0 + threadIdx.x;
        uint64_t cnt = 0;
        if (w < a.nwin) {
            const uint64_t wl = a.wlen[w], base = wl / uint64_t(n), rem = wl % uint64_t(n), up = uint64_t(p);
            const uint64_t e0 = a.wstart[w] + up * base + min(up, rem);  // segment_of (collectives.cpp:47-53)
            const uint64_t e1 = e0 + base + (up < rem ? 1 : 0);
            const uint64_t v0 = (e0 + VE - 1) / VE, v1 = e1 / VE;
            f.e0[w] = e0;
            f.e1[w] = e1;
            f.v0[w] = v0;
            cnt = v1 > v0 ? v1 - v0 : 0;
        }
        uint64_t x = cnt;  // block-wide inclusive scan: warps, then warp totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[warp] = x;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t run = w0 == 0 ? 0 : f.pre[w0];
            for (int q = 0; q < int(blockDim.x >> 5); ++q) {
                const uint64_t t = warp_tot[q];
                warp_tot[q] = run;
                run += t;
            }
            if (w0 == 0) f.pre[0] = 0;
        }
        __syncthreads();
        if (w < a.nwin) f.pre[w + 1] = warp_tot[warp] + x;
        __syncthreads();
    }
}

// window holding flat vector x: the last w with pre[w] <= x
__device__ __forceinline__ int flat_window(const FlatWins& f, int nwin, uint64_t x) {
    int lo = 0, hi = nwin;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (f.pre[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

template <int DT, int NT>
__device__ __forceinline__ void reduce_flat(const RingArgs& a, const char* const* src, int n, const FlatWins& f,
                                            uint64_t gtid, uint64_t T) {
    constexpr int VE = Vec<DT>::kElems;
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int U = NMAX <= 4 ? 4 : (NMAX <= 8 ? 2 : 1);
    for (int w = int(blockIdx.x); w < a.nwin; w += int(gridDim.x)) {  // unaligned edges, scalar
        const uint64_t e0 = f.e0[w], e1 = f.e1[w], v0 = f.v0[w], v1 = v0 + (f.pre[w + 1] - f.pre[w]);
        if (v1 == v0) {
            for (uint64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) Vec<DT>::scalar(a, src, n, e);
        } else {
            for (uint64_t e = e0 + threadIdx.x; e < v0 * VE; e += blockDim.x) Vec<DT>::scalar(a, src, n, e);
            for (uint64_t e = v1 * VE + threadIdx.x; e < e1; e += blockDim.x) Vec<DT>::scalar(a, src, n, e);
        }
    }
    const uint64_t total = f.pre[a.nwin];
    for (uint64_t x = gtid; x < total; x += T * U) {
        uint4 v[U][NMAX];
        uint64_t vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t xu = x + uint64_t(u) * T;
            vv[u] = ~0ull;
            if (xu < total) {
                const int w = flat_window(f, a.nwin, xu);
                vv[u] = f.v0[w] + (xu - f.pre[w]);
#pragma unroll
                for (int t = 0; t < NMAX; ++t)
                    if (t < n) v[u][t] = gfd::ld16(src[t] + vv[u] * 16);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (vv[u] == ~0ull) continue;
            uint4 acc = v[u][0];
#pragma unroll
            for (int t = 1; t < NMAX; ++t)
                if (t < n) acc = Vec<DT>::acc(v[u][t], acc);
#pragma unroll
            for (int t = 0; t < NMAX; ++t)
                if (t < n) gfd::st16(const_cast<char*>(src[(t + 1) % n]) + vv[u] * 16, acc);
        }
    }
}

// Planned (CSC) windows are all of one length except the last. With several of them the grid
// is cut into `groups` CTA groups of c CTAs; group g sweeps windows g, g + groups, ... so the
// windows' NVLink round trips overlap instead of following one another. Depends only on
// (nwin, grid), so CTA b covers the same vectors on every rank (the barriers pair CTA b only).
struct WinGroups {
    int first, step, edge_cta;  // windows first, first+step, ...; edge handler of my group
    uint64_t lg, LT;            // my thread index within the group, the group's threads
    __device__ WinGroups(int nwin, bool grouped) {
        const int G = int(gridDim.x);
        if (!grouped || nwin <= 1) {
            first = 0;
            step = 1;
            edge_cta = 0;
            lg = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
            LT = uint64_t(G) * blockDim.x;
            return;
        }
        const int c = max(1, G / nwin), groups = G / c, grp = int(blockIdx.x) / c;
        first = grp < groups ? grp : nwin;  // CTAs past the last full group sit out
        step = groups;
        edge_cta = grp * c;
        lg = uint64_t(int(blockIdx.x) % c) * blockDim.x + threadIdx.x;
        LT = uint64_t(c) * blockDim.x;
    }
};

}  // namespace

namespace gfr {
// CTAs per rank of a ring launch (ring.cu): identical on every rank for the same windows.
int ring_blocks(uint64_t max_seg_bytes);
// The same capped by the communicator (colocated ranks share one device's SMs).
int comm_blocks(const gf_comm* c, uint64_t max_seg_bytes);
// pull.cu: reduce-scatter (pulled from the peers' pools, or from my pool + my inbox slots when
// inbox != null) then pull all-gather, both unpacking from registers (<= 256 tensors).
int rsag_launch(gf_comm* c, int dtype, uint64_t pool_heap_off, const char* inbox, uint64_t slot_bytes,
                float* const* dst, const uint64_t* pool_off, const uint64_t* count, int ntensors,
                const uint64_t* win_start, const uint64_t* win_len, int nwin, int flags, void* stream,
                const char* fn);
}  // namespace gfr
