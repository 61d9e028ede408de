// SPDX-License-Identifier: Apache-2.0
//
// K4: ring allreduce over NVLink/NVSwitch peer memory, and K5: the fused
// norm exchange + top-k selection — plus the communicator (symmetric heap,
// IPC / in-process bootstrap, cross-GPU flags).
//
// Reference: detail::ring_allreduce_on (src/collectives.cpp:55-97) runs n-1
// reduce-scatter steps (send segment p-s, receive p-s-1, accumulate) and n-1
// all-gather steps over a Transport. Segment j (segment_of, :47-53) is summed
// starting at ring position j: ((x_j + x_{j+1}) + ...) + x_{j-1}, rounding to
// the element type after every add (accumulate, buffer.hpp:60-81).
//
// B200 design: no store-and-forward. The rank at ring position p owns segment
// p of every window: it LOADS that segment from all N ranks' buffers directly
// over NVLink (in ring order, so the sum is bit-identical to the reference),
// and STORES the result into all N buffers (the all-gather becomes posted
// remote writes). Per rank: (N-1)/N*K bytes pulled + (N-1)/N*K pushed — the
// same 2(N-1)/N*K bus bytes as the ring — in ONE kernel with two cross-GPU
// barriers (entry: peers' inputs are ready; exit: all pushes into my buffer
// landed). Each CTA b only pairs with CTA b on the peers, through monotonic
// 64-bit flags written with st.release.sys and polled with ld.acquire.sys.
// Waits are bounded (globaltimer) and a timeout poisons the communicator,
// surfacing as TransportError like the reference's recv timeout (inproc.cpp:28-36).

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gf_device.cuh"
#include "gf_internal.cuh"
#include "select.cuh"
#include "comm.cuh"
#include "ring_device.cuh"

namespace {



struct SelArgs {
    float* norms[GF_MAX_RANKS];          // by rank
    uint64_t* nacc[GF_MAX_RANKS];        // exact |x| sums (units 2^-24) to finalize, or null
    const uint16_t* pool[GF_MAX_RANKS];  // fp16 pools (sequential fallback for huge sums)
    const uint8_t* imp_cur;              // this iteration's important set (x1/N)
    int ring[GF_MAX_RANKS];
    int world, rank, p2p;
    uint64_t nc, k, total, chunk, esz, theta;
    uint8_t* flags;
    uint64_t* coff;
    uint64_t* plan;
    uint64_t* flags_local;
    uint64_t* flags_peer[GF_MAX_RANKS];
    uint64_t* epochs;
    uint64_t timeout_ns;
    int* err;
    uint64_t* trace;
    // push-inbox norm exchange (gf_comm_set_select_inbox): rank r's finalized norms go to
    // slot r of every peer's inbox before the one barrier; the sums then read local memory only
    float* inbox_local;                  // world x nc floats: slot r = rank r's norms
    float* inbox_peer[GF_MAX_RANKS];     // each rank's inbox as mapped here
};

// ---- CSC write-back fused into the planned ring (staging -> pool + exact chunk L1) -------
using gfd::half_units;
constexpr uint64_t kNaccNaN = 1ull << 63;

// pool element of staging element s: important chunk q of the plan starts at staging q*chunk
// (only the final pool chunk differs in length, and it is last when selected). The chunk
// list is staged in shared memory after the exit barrier (wb_list).
__device__ __forceinline__ uint64_t wb_target(const RingArgs& a, const uint64_t* list, uint64_t k, uint64_t s,
                                              uint64_t& c) {
    const uint64_t q = min(s / a.wb_chunk, k - 1);
    c = list[q];
    return c * a.wb_chunk + (s - q * a.wb_chunk);
}

// warp-aggregated add of (chunk, units): lanes sharing the first active lane's chunk combine
__device__ __forceinline__ void wb_nacc_add(uint64_t* nacc, uint64_t c, uint64_t u, bool nan, bool active) {
    const unsigned full = 0xFFFFFFFFu;
    const unsigned act = __ballot_sync(full, active);
    if (!act) return;
    const int leader = __ffs(act) - 1;
    const uint64_t c0 = __shfl_sync(full, c, leader);
    const bool same = active && c == c0;
    uint64_t v = same ? u : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(full, v, o);
    const bool anynan = __any_sync(full, same && nan);
    if ((threadIdx.x & 31) == unsigned(leader)) {
        if (v) atomicAdd(reinterpret_cast<unsigned long long*>(nacc + c0), (unsigned long long)v);
        if (anynan) atomicOr(reinterpret_cast<unsigned long long*>(nacc + c0), (unsigned long long)kNaccNaN);
    }
    if (active && !same) {
        if (u) atomicAdd(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)u);
        if (nan) atomicOr(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)kNaccNaN);
    }
}

// This CTA's staging vectors of segment [e0, e1) (the reduce pattern: every segment's, since
// the exit barrier covered the pushes of CTA b on every rank) -> pool, + units.
__device__ void wb_segment(const RingArgs& a, const uint64_t* list, uint64_t k, uint64_t e0, uint64_t e1,
                           uint64_t gtid, uint64_t T, int edge_cta = 0) {
    const uint16_t* stg = reinterpret_cast<const uint16_t*>(a.bufs[a.rank]);
    uint16_t* pool = reinterpret_cast<uint16_t*>(a.wb_pool);
    const uint64_t v0 = (e0 + 7) / 8, v1 = e1 / 8;
    auto scalar = [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
            uint64_t c;
            const uint64_t d = wb_target(a, list, k, i, c);
            const uint16_t h = reinterpret_cast<const volatile uint16_t*>(stg)[i];
            pool[d] = h;
            if ((h & 0x7C00u) == 0x7C00u)
                atomicOr(reinterpret_cast<unsigned long long*>(a.wb_nacc + c), (unsigned long long)kNaccNaN);
            else if (half_units(h))
                atomicAdd(reinterpret_cast<unsigned long long*>(a.wb_nacc + c), (unsigned long long)half_units(h));
        }
    };
    if (v0 >= v1) {
        if (int(blockIdx.x) == edge_cta) scalar(e0, e1);
        return;
    }
    if (int(blockIdx.x) == edge_cta) {
        scalar(e0, v0 * 8);
        scalar(v1 * 8, e1);
    }
    // whole-warp iterations (the aggregation's shuffles need every lane), U vectors in flight
    constexpr int U = 4;
    const uint64_t lane = gtid & 31;
    for (uint64_t base = v0 + gtid - lane; base < v1; base += T * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = base + uint64_t(u) * T + lane;
            if (vv < v1)
                asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"  // peers wrote it: skip L1
                             : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w)
                             : "l"(stg + vv * 8));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = base + uint64_t(u) * T + lane;
            if (base + uint64_t(u) * T >= v1) break;  // warp-uniform
            const bool act = vv < v1;
            uint64_t c = 0, un = 0;
            bool nan = false;
            if (act) {
                const uint64_t d = wb_target(a, list, k, vv * 8, c);
                gfd::st16(pool + d, x[u]);
                nan = gfd::any_special(x[u]);
                if (!nan) un = gfd::units8(x[u]);
            }
            wb_nacc_add(a.wb_nacc, c, un, nan, act);
        }
    }
}

// ---- CSC exchange, pull form (gf_csc_exchange_pull) ------------------------------------
// The planned windows over the staging buffers, without any push: the rank at ring position
// p sums segment p of every window by pulling it from all N staging buffers in ring order
// (bit-identical to the ring), keeps the sum in its own staging buffer and writes it back
// into its pool (+ exact |x| units, the norms of the important chunks); after one barrier
// with its peer CTAs it pulls every other segment from the owner's staging buffer straight
// into its pool. The write-back's address math and atomics overlap the NVLink loads; no
// barrier waits for posted writes to drain. The caller's next write of its staging buffer
// must come after a later collective's barrier (gf_csc_select's, in the CSC step).
__device__ __forceinline__ void wb_scalar(const RingArgs& a, const uint64_t* list, uint64_t k, uint64_t i,
                                          uint16_t h) {
    uint64_t c;
    const uint64_t d = wb_target(a, list, k, i, c);
    reinterpret_cast<uint16_t*>(a.wb_pool)[d] = h;
    if ((h & 0x7C00u) == 0x7C00u)
        atomicOr(reinterpret_cast<unsigned long long*>(a.wb_nacc + c), (unsigned long long)kNaccNaN);
    else if (half_units(h))
        atomicAdd(reinterpret_cast<unsigned long long*>(a.wb_nacc + c), (unsigned long long)half_units(h));
}

// RS (OWN = true: sum from all N in ring order, keep in the local staging) or AG (OWN =
// false: src[0] is the owner's staging) of staging range [e0, e1), written back to the pool.
template <int NT, bool OWN>
__device__ void csc_pull_range(const RingArgs& a, const char* const* src, int n, const uint64_t* list,
                               uint64_t k, uint64_t e0, uint64_t e1, uint64_t gtid, uint64_t T,
                               int edge_cta) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int NS = OWN ? NMAX : 1;
    constexpr int U = OWN ? (NMAX <= 4 ? 4 : (NMAX <= 8 ? 2 : 1)) : 8;
    uint16_t* local = reinterpret_cast<uint16_t*>(a.bufs[a.rank]);
    uint64_t v0 = (e0 + 7) / 8, v1 = e1 / 8;
    if (v0 >= v1) v0 = v1 = e1 / 8 + 1;  // no aligned vector inside: all scalar
    if (int(blockIdx.x) == edge_cta) {
        auto edge = [&](uint64_t lo, uint64_t hi) {
            for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                uint16_t h;
                if (OWN) {
                    h = reinterpret_cast<const uint16_t*>(src[0])[i];
                    for (int t = 1; t < n; ++t) h = gfd::acc16(reinterpret_cast<const uint16_t*>(src[t])[i], h);
                    local[i] = h;
                    if (a.csc_push_ag)  // the all-gather as posted writes into every peer's staging
                        for (int t = 1; t < n; ++t) reinterpret_cast<uint16_t*>(a.bufs[a.ring[(a.pos + t) % n]])[i] = h;
                } else {
                    h = reinterpret_cast<const volatile uint16_t*>(src[0])[i];
                }
                wb_scalar(a, list, k, i, h);
            }
        };
        if (v0 < v1) {
            edge(e0, v0 * 8);
            edge(v1 * 8, e1);
        } else {
            edge(e0, e1);
        }
    }
    // whole-warp iterations (the units aggregation shuffles need every lane)
    const uint64_t lane = gtid & 31;
    for (uint64_t base = v0 + gtid - lane; base < v1; base += T * U) {
        uint4 x[U][NS];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = base + uint64_t(u) * T + lane;
            if (vv < v1) {
#pragma unroll
                for (int t = 0; t < NS; ++t) {
                    if (OWN) {
                        if (t < n) x[u][t] = gfd::ld16(src[t] + vv * 16);
                    } else {
                        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"  // the owner wrote it
                                     : "=r"(x[u][t].x), "=r"(x[u][t].y), "=r"(x[u][t].z), "=r"(x[u][t].w)
                                     : "l"(src[0] + vv * 16));
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + uint64_t(u) * T >= v1) break;  // warp-uniform
            const uint64_t vv = base + uint64_t(u) * T + lane;
            const bool act = vv < v1;
            uint64_t c = 0, un = 0;
            bool nan = false;
            if (act) {
                uint4 acc = x[u][0];
                if (OWN) {
#pragma unroll
                    for (int t = 1; t < NS; ++t)
                        if (t < n) acc = gfd::acc16x8(x[u][t], acc);
                    gfd::st16_keep(local + vv * 8, acc);  // the peers pull it next
                    if (a.csc_push_ag)
#pragma unroll
                        for (int t = 1; t < NMAX; ++t)
                            if (t < n) gfd::st16(a.bufs[a.ring[(a.pos + t) % n]] + vv * 16, acc);
                }
                const uint64_t d = wb_target(a, list, k, vv * 8, c);
                gfd::st16(reinterpret_cast<uint16_t*>(a.wb_pool) + d, acc);
                nan = gfd::any_special(acc);
                if (!nan) un = gfd::units8(acc);
            }
            wb_nacc_add(a.wb_nacc, c, un, nan, act);
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(kRingThreads) csc_pull_kernel(const __grid_constant__ RingArgs a) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    extern __shared__ uint64_t wb_list[];  // the plan's important chunks (plan[1] <= nc)
    __shared__ int s_ok;
    const uint64_t epoch = a.epochs[blockIdx.x];
    if (threadIdx.x == 0) s_ok = 1;
    const int n = NT > 0 ? NT : a.world;
    const uint64_t k = a.plan[1];
    for (uint64_t q = threadIdx.x; q < k; q += blockDim.x) wb_list[q] = a.plan[4 + q];
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) a.trace[0] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 1, &s_ok, false)) return;  // peers' staging buffers are packed
    if (tr) a.trace[1] = gfd::globaltimer_ns();
    const uint64_t staged = a.plan[0], stride = a.plan[3];
    const int nwin = int(a.plan[2]);
    const char* src[NMAX];
#pragma unroll
    for (int t = 0; t < NMAX; ++t)
        src[t] = t >= n ? nullptr
                        : (a.csc_inbox == nullptr ? a.bufs[a.ring[(a.pos + t) % n]]
                                                  : (t == 0 ? a.bufs[a.rank] : a.csc_inbox + uint64_t(t - 1) * a.csc_slot_bytes));
    auto seg = [&](int w, int j, uint64_t& e0, uint64_t& e1) {  // segment_of (collectives.cpp:47-53)
        const uint64_t ws = uint64_t(w) * stride, wl = (w == nwin - 1) ? staged - ws : stride;
        const uint64_t base = wl / uint64_t(n), rem = wl % uint64_t(n), uj = uint64_t(j);
        e0 = ws + uj * base + min(uj, rem);
        e1 = e0 + base + (uj < rem ? 1 : 0);
    };
    const WinGroups wg(nwin, true);  // CTA groups sweep the windows concurrently
    for (int w = wg.first; w < nwin; w += wg.step) {
        uint64_t e0, e1;
        seg(w, a.pos, e0, e1);
        csc_pull_range<NT, true>(a, src, n, wb_list, k, e0, e1, wg.lg, wg.LT, wg.edge_cta);
    }
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 2, &s_ok, true)) return;  // my segment sums are visible
    for (int w = wg.first; w < nwin; w += wg.step) {
        for (int j = 1; j < n; ++j) {
            const int q = (a.pos + j) % n;
            uint64_t e0, e1;
            seg(w, q, e0, e1);
            const char* owner[1] = {a.csc_push_ag ? a.bufs[a.rank] : a.bufs[a.ring[q]]};  // pushed here / pulled
            csc_pull_range<NT, false>(a, owner, n, wb_list, k, e0, e1, wg.lg, wg.LT, wg.edge_cta);
        }
    }
    if (threadIdx.x == 0) a.epochs[blockIdx.x] = epoch + 2;
    if (tr) a.trace[3] = gfd::globaltimer_ns();
}

template <int DT, int NT, bool P2P>
__global__ void __launch_bounds__(kRingThreads, 1) ring_kernel(const __grid_constant__ RingArgs a) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    __shared__ int s_ok;
    uint64_t epoch = 0;
    if (P2P) epoch = a.epochs[blockIdx.x];
    if (threadIdx.x == 0) s_ok = 1;
    const int n = NT > 0 ? NT : a.world;
    const int p = P2P ? a.pos : int(blockIdx.y);
    const bool tr = P2P && a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) a.trace[0] = gfd::globaltimer_ns();
    __shared__ FlatWins flat;  // explicit windows, several: one flattened sweep
    const bool use_flat = a.nwin > 1;
    if (use_flat) flat_build<Vec<DT>::kElems>(a, n, p, flat);
    if (P2P && !cross_barrier(a, epoch + 1, &s_ok, false)) return;
    if (tr) a.trace[1] = gfd::globaltimer_ns();

    const char* src[NMAX];
#pragma unroll
    for (int t = 0; t < NMAX; ++t) src[t] = (t < n) ? a.bufs[a.ring[(p + t) % n]] : nullptr;
    const uint64_t T = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int nwin;
    uint64_t staged = 0, stride = 0;
    if (a.nwin >= 0) {
        nwin = a.nwin;
    } else {
        staged = a.plan[0];
        nwin = int(a.plan[2]);
        stride = a.plan[3];
    }
    const WinGroups wg(nwin, a.nwin < 0);  // planned windows: CTA groups sweep them concurrently
    if (use_flat) reduce_flat<DT, NT>(a, src, n, flat, gtid, T);
    for (int w = use_flat ? nwin : wg.first; w < nwin; w += wg.step) {
        uint64_t ws, wl;
        if (a.nwin >= 0) {
            ws = a.wstart[w];
            wl = a.wlen[w];
        } else {
            ws = uint64_t(w) * stride;
            wl = (w == nwin - 1) ? staged - ws : stride;
        }
        // owned segment: segment_of(wl, n, p) (collectives.cpp:47-53)
        const uint64_t base = wl / uint64_t(n), rem = wl % uint64_t(n), up = uint64_t(p);
        const uint64_t e0 = ws + up * base + min(up, rem);
        reduce_segment<DT, NT>(a, src, n, e0, e0 + base + (up < rem ? 1 : 0), wg.lg, wg.LT, wg.edge_cta);
    }
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    if (P2P && !cross_barrier(a, epoch + 2, &s_ok, true)) return;
    if (P2P && threadIdx.x == 0) a.epochs[blockIdx.x] = epoch + 2;
    if (tr) a.trace[3] = gfd::globaltimer_ns();
    if (DT == GF_F16 && P2P && a.wb_pool != nullptr && nwin > 0) {  // fused CSC write-back
        extern __shared__ uint64_t wb_list[];  // the plan's important chunks (plan[1] <= nc)
        const uint64_t k = a.plan[1];
        for (uint64_t q = threadIdx.x; q < k; q += blockDim.x) wb_list[q] = a.plan[4 + q];
        __syncthreads();
        for (int w = wg.first; w < nwin; w += wg.step) {  // the vectors my group reduced
            const uint64_t ws = uint64_t(w) * stride, wl = (w == nwin - 1) ? staged - ws : stride;
            const uint64_t base = wl / uint64_t(n), rem = wl % uint64_t(n);
            for (int j = 0; j < n; ++j) {
                const uint64_t uj = uint64_t(j), e0 = ws + uj * base + min(uj, rem);
                wb_segment(a, wb_list, k, e0, e0 + base + (uj < rem ? 1 : 0), wg.lg, wg.LT, wg.edge_cta);
            }
        }
    }
}

// ---- K5: norm exchange + selection (one CTA) -----------------------------------
__global__ void __launch_bounds__(gfs::kSelThreads) select_kernel(const __grid_constant__ SelArgs a) {
    extern __shared__ float red[];
    __shared__ int s_ok;
    __shared__ gfs::SelShared sh;
    if (threadIdx.x == 0) s_ok = 1;
    const int n = a.world;
    const uint64_t epoch = a.p2p ? a.epochs[0] : 0;
    const bool tr = a.trace != nullptr && threadIdx.x == 0;  // [start, finalized, entered, summed, exited, top-k, end]
    if (tr) a.trace[0] = gfd::globaltimer_ns();
    // Finalize this iteration's local norms from the exact accumulators written by
    // pack_correct (unimportant chunks) and scatter (important chunks): chunk_l1 +
    // x1/N (sparse.cpp:176-184), then re-arm the accumulators for the next iteration.
    // World 1: the finalized norms are the sums; they go straight into `red` (shared memory)
    // and the sum phase below is skipped.
    const bool solo = n == 1;
    if (a.nacc[0] || a.nacc[a.rank]) {
        const float inv_world = 1.0f / float(n);
        for (int r = a.p2p ? a.rank : 0; r < (a.p2p ? a.rank + 1 : n); ++r) {
            for (uint64_t i = threadIdx.x; i < a.nc; i += gfs::kSelThreads) {
                const uint64_t S = a.nacc[r][i];
                const bool imp = a.imp_cur[i] != 0;  // both loads in flight together
                float v;
                if (S >> 63) {
                    v = gfd::u2f(0x7FC00000u);
                } else if (S < (1ull << 53)) {
                    v = __double2float_rn(__ull2double_rn(S) * 0x1p-24);
                } else {  // inexact fp64 partial sums in the reference: replay its order
                    const uint64_t b = i * a.chunk, len = (i + 1 == a.nc) ? a.total - b : a.chunk;
                    double d = 0.0;
                    for (uint64_t e = 0; e < len; ++e) d = __dadd_rn(d, fabs(double(gfd::dec(a.pool[r][b + e]))));
                    v = __double2float_rn(d);
                }
                if (imp) v = gfd::mul(v, inv_world);
                a.norms[r][i] = v;
                if (solo) red[i] = v;
                a.nacc[r][i] = 0;
            }
        }
        __syncthreads();
    }
    const bool inbox = a.p2p && a.inbox_local != nullptr;
    if (inbox) {  // push my norms into slot `rank` of every peer's inbox (posted NVLink writes)
        for (uint64_t i = threadIdx.x; i < a.nc; i += gfs::kSelThreads) {
            const float v = a.norms[a.rank][i];
            for (int q = 0; q < n; ++q)
                if (q != a.rank) a.inbox_peer[q][uint64_t(a.rank) * a.nc + i] = v;
        }
    }
    if (tr) a.trace[1] = gfd::globaltimer_ns();
    // entry: peers' norms are final (and, with the inbox, have landed here: the fence before
    // each flag release makes the CTA's pushes visible first)
    if (a.p2p && !cross_barrier(a, epoch + 1, &s_ok)) return;
    if (inbox && threadIdx.x == 0) a.epochs[0] = epoch + 1;
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    const uint64_t base = a.nc / uint64_t(n), rem = a.nc % uint64_t(n);
    const bool have_red = solo && (a.nacc[0] != nullptr);
    for (uint64_t i = threadIdx.x; i < a.nc && !have_red; i += gfs::kSelThreads) {
        // segment index of element i under segment_of(nc, n, .) (collectives.cpp:47-53)
        const uint64_t big = rem * (base + 1);
        const int j = int(i < big ? i / (base + 1) : rem + (i - big) / base);
        // issue every rank's load before the first add: one NVLink round trip, not n
        float v[GF_MAX_RANKS];
#pragma unroll
        for (int t = 0; t < GF_MAX_RANKS; ++t) {
            if (t < n) {
                const int src = a.ring[(j + t) % n];
                v[t] = (inbox && src != a.rank) ? a.inbox_local[uint64_t(src) * a.nc + i] : a.norms[src][i];
            }
        }
        float acc = v[0];
#pragma unroll
        for (int t = 1; t < GF_MAX_RANKS; ++t)
            if (t < n) acc = gfd::add(v[t], acc);
        red[i] = acc;
    }
    if (tr) a.trace[3] = gfd::globaltimer_ns();
    // exit: without the inbox, peers may still be loading my norms, which are overwritten with
    // the sums below. With it nobody reads my norms buffer; my inbox slots are next written by
    // the peers' next selection, which follows the next exchange's entry barrier with me.
    if (a.p2p && !inbox) {
        if (!cross_barrier(a, epoch + 2, &s_ok)) return;
        if (threadIdx.x == 0) a.epochs[0] = epoch + 2;
    }
    if (tr) a.trace[4] = gfd::globaltimer_ns();
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < a.nc; i += gfs::kSelThreads) {
        if (a.p2p) {
            a.norms[a.rank][i] = red[i];
        } else {
            for (int r = 0; r < n; ++r) a.norms[r][i] = red[i];
        }
    }
    gfs::block_topk(red, a.nc, a.k, a.flags, sh);
    if (tr) a.trace[5] = gfd::globaltimer_ns();
    if (a.coff && a.plan) gfs::block_plan(a.flags, a.total, a.chunk, a.nc, a.esz, a.theta, a.coff, a.plan, sh);
    if (tr) a.trace[6] = gfd::globaltimer_ns();
}

template <int DT, bool P2P>
void launch_ring_dt(const RingArgs& a, dim3 grid, cudaStream_t s, size_t smem, int threads) {
    const int kRingThreads = threads;  // the CTA size of this launch (<= the compiled 512)
    switch (a.world) {
        case 2: ring_kernel<DT, 2, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        case 3: ring_kernel<DT, 3, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        case 4: ring_kernel<DT, 4, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        case 5: ring_kernel<DT, 5, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        case 6: ring_kernel<DT, 6, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        case 7: ring_kernel<DT, 7, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        case 8: ring_kernel<DT, 8, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
        default: ring_kernel<DT, 0, P2P><<<grid, kRingThreads, smem, s>>>(a); break;
    }
}
void launch_ring(int dtype, bool p2p, const RingArgs& a, dim3 grid, cudaStream_t s, size_t smem = 0,
                 int threads = kRingThreads) {
    if (dtype == GF_F16) {
        if (p2p) launch_ring_dt<GF_F16, true>(a, grid, s, smem, threads);
        else launch_ring_dt<GF_F16, false>(a, grid, s, smem, threads);
    } else {
        if (p2p) launch_ring_dt<GF_F32, true>(a, grid, s, smem, threads);
        else launch_ring_dt<GF_F32, false>(a, grid, s, smem, threads);
    }
}

// CTAs per rank: enough 512-thread CTAs to keep ~2 MB of NVLink loads in flight,
// capped at 1 per SM (and by the flag table). Depends only on values identical
// on every rank, so all ranks launch the same grid (CTA b pairs with CTA b).
int ring_blocks_impl(uint64_t max_seg_bytes) {
    static const int forced = [] {
        const char* e = std::getenv("GF_RING_BLOCKS");  // tuning override (must match on all ranks)
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return std::min(forced, kMaxBlocks);
    const uint64_t per_cta = uint64_t(kRingThreads) * 16 * 4;
    const uint64_t want = (max_seg_bytes + per_cta - 1) / per_cta;
    // one 512-thread CTA per SM: measured on 2-4 B200, 2/SM and more oversubscribe the
    // NVLink request queues (ResNet-50 fp16, N=4: 150 us at 148 CTAs vs 163 at 296)
    const uint64_t cap = std::min<uint64_t>(kMaxBlocks, uint64_t(gfi::sm_count()));
    return int(std::max<uint64_t>(1, std::min(want, cap)));
}

// CUDA 12 loads kernels lazily by default (CUDA_MODULE_LOADING=LAZY). Loading a kernel while
// another kernel of the same context spins at a cross-rank barrier was measured to stall the
// colocated world (the barrier never observes the peer): colocated worlds require EAGER loading.
bool lazy_module_loading() {
    using fn_t = CUresult (*)(CUmoduleLoadingMode*);
    static fn_t fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<fn_t>(f);
    }();
    CUmoduleLoadingMode m = CU_MODULE_EAGER_LOADING;
    if (!fn || fn(&m) != CUDA_SUCCESS) return false;
    return m == CU_MODULE_LAZY_LOADING;
}

// GF_DIAG_NOWAIT=1: cross-GPU barriers and flags signal but never wait (timeout 0). A traffic
// probe for ncu's serialised kernel replay (scripts/ncu_nvlink.py); every result is invalid.
bool diag_nowait() {
    static const bool v = [] {
        const char* e = std::getenv("GF_DIAG_NOWAIT");
        return e && std::atoi(e) == 1;
    }();
    return v;
}

bool valid_ring(const int* order, int world) {
    bool seen[GF_MAX_RANKS] = {};
    for (int i = 0; i < world; ++i) {
        if (order[i] < 0 || order[i] >= world || seen[order[i]]) return false;
        seen[order[i]] = true;
    }
    return true;
}

}  // namespace

namespace {

}  // namespace

extern "C" {

int gf_comm_create(int world, int rank, int device, uint64_t heap_bytes, gf_comm** out) {
    if (!out) return gfi::fail(GF_ERR_CONFIG, "gf_comm_create: null out");
    *out = nullptr;
    if (world < 1 || world > GF_MAX_RANKS) return gfi::fail(GF_ERR_CONFIG, "world size out of range [1,16]");
    if (rank < 0 || rank >= world) return gfi::fail(GF_ERR_CONFIG, "rank " + std::to_string(rank) + " outside world");
    DeviceGuard g(device);
    auto* c = new gf_comm();
    c->world = world;
    c->rank = rank;
    c->device = device;
    if (diag_nowait()) c->timeout_ns = 0;
    c->heap_bytes = (heap_bytes + 255) & ~uint64_t(255);
    for (int i = 0; i < world; ++i) c->ring[i] = i;
    c->pos = rank;
    cudaError_t e = cudaMalloc(&c->alloc, kFlagBytes + c->heap_bytes);
    if (e == cudaSuccess) e = cudaMemset(c->alloc, 0, kFlagBytes);
    if (e == cudaSuccess) e = cudaHostAlloc(&c->err_host, 256, cudaHostAllocMapped);
    if (e == cudaSuccess) {
        std::memset(c->err_host, 0, 256);
        e = cudaHostGetDevicePointer(&c->err_dev, c->err_host, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        if (c->alloc) cudaFree(c->alloc);
        if (c->err_host) cudaFreeHost(c->err_host);
        delete c;
        return gfi::cuda_fail(e, "gf_comm_create");
    }
    c->peer_alloc[rank] = c->alloc;
    if (world == 1) c->connected = true;
    *out = c;
    return GF_OK;
}

int gf_comm_destroy(gf_comm* c) {
    if (!c) return GF_OK;
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    for (int r = 0; r < c->world; ++r)
        if (c->ipc_opened[r]) cudaIpcCloseMemHandle(c->peer_alloc[r]);
    cudaFree(c->alloc);
    cudaFreeHost(c->err_host);
    delete c;
    return GF_OK;
}

int gf_comm_heap(gf_comm* c, void** base, uint64_t* bytes) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    if (base) *base = c->alloc + kFlagBytes;
    if (bytes) *bytes = c->heap_bytes;
    return GF_OK;
}

int gf_comm_export_handle(gf_comm* c, void* handle_out) {
    if (!c || !handle_out) return gfi::fail(GF_ERR_CONFIG, "gf_comm_export_handle: null argument");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    GF_CHECK_CUDA(cudaIpcGetMemHandle(&h, c->alloc));
    static_assert(sizeof(cudaIpcMemHandle_t) == GF_IPC_HANDLE_BYTES, "ipc handle size");
    std::memcpy(handle_out, &h, GF_IPC_HANDLE_BYTES);
    return GF_OK;
}

int gf_comm_connect_ipc(gf_comm* c, const void* all_handles) {
    if (!c || !all_handles) return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_ipc: null argument");
    DeviceGuard g(c->device);
    const char* hs = static_cast<const char*>(all_handles);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hs + size_t(r) * GF_IPC_HANDLE_BYTES, GF_IPC_HANDLE_BYTES);
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            gfi::cuda_fail(e, "cudaIpcOpenMemHandle");
            return gfi::fail(GF_ERR_TRANSPORT, "rank " + std::to_string(c->rank) +
                                                   ": cannot map peer " + std::to_string(r) +
                                                   " heap: " + cudaGetErrorString(e));
        }
        c->peer_alloc[r] = static_cast<char*>(p);
        c->ipc_opened[r] = true;
    }
    c->connected = true;
    return GF_OK;
}

int gf_comm_connect_local(gf_comm* const* comms, int world) {
    if (!comms || world < 1) return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_local: bad arguments");
    for (int r = 0; r < world; ++r) {
        if (!comms[r] || comms[r]->world != world || comms[r]->rank != r)
            return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_local: comms[r] must be rank r of this world");
        for (int q = 0; q < r; ++q)
            if (comms[q]->device == comms[r]->device)
                return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_local: ranks must use distinct devices "
                                                "(use the colocated entry points to emulate ranks on one device)");
    }
    for (int r = 0; r < world; ++r) {
        DeviceGuard g(comms[r]->device);
        for (int q = 0; q < world; ++q) {
            if (q == r) continue;
            int can = 0;
            GF_CHECK_CUDA(cudaDeviceCanAccessPeer(&can, comms[r]->device, comms[q]->device));
            if (!can)
                return gfi::fail(GF_ERR_TRANSPORT, "device " + std::to_string(comms[r]->device) +
                                                       " cannot access peer " + std::to_string(comms[q]->device));
            cudaError_t e = cudaDeviceEnablePeerAccess(comms[q]->device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return gfi::cuda_fail(e, "cudaDeviceEnablePeerAccess");
            comms[r]->peer_alloc[q] = comms[q]->alloc;
        }
        comms[r]->connected = true;
    }
    return GF_OK;
}

int gf_comm_connect_colocated(gf_comm* const* comms, int world) {
    if (!comms || world < 1 || world > GF_MAX_RANKS) return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_colocated: bad arguments");
    if (world > 1 && lazy_module_loading())
        return gfi::fail(GF_ERR_CONFIG,
                         "gf_comm_connect_colocated: needs CUDA_MODULE_LOADING=EAGER in the environment before CUDA "
                         "initialises (a kernel loaded lazily while another rank's kernel waits at a barrier on the "
                         "same device can stall both)");
    for (int r = 0; r < world; ++r) {
        if (!comms[r] || comms[r]->world != world || comms[r]->rank != r)
            return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_colocated: comms[r] must be rank r of this world");
        if (comms[r]->device != comms[0]->device)
            return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_colocated: every rank must use the same device");
        if (comms[r]->connected && world > 1)
            return gfi::fail(GF_ERR_CONFIG, "gf_comm_connect_colocated: communicator already connected");
    }
    // every rank's barrier-waiting CTAs (one per SM at most) must be resident at once, with
    // SMs left over for the ranks' non-waiting kernels: world x cap <= SMs / 2
    const int cap = std::max(1, gfi::sm_count() / (2 * world));
    for (int r = 0; r < world; ++r) {
        for (int q = 0; q < world; ++q) comms[r]->peer_alloc[q] = comms[q]->alloc;
        comms[r]->colocated = true;
        comms[r]->grid_cap = cap;
        comms[r]->connected = true;
    }
    return GF_OK;
}

int gf_comm_set_ring_order(gf_comm* c, const int* order) {
    if (!c || !order) return gfi::fail(GF_ERR_CONFIG, "gf_comm_set_ring_order: null argument");
    if (!valid_ring(order, c->world)) return gfi::fail(GF_ERR_CONFIG, "ring order is not a permutation of ranks");
    for (int i = 0; i < c->world; ++i) {
        c->ring[i] = order[i];
        if (order[i] == c->rank) c->pos = i;
    }
    return GF_OK;
}

int gf_comm_set_timeout_ms(gf_comm* c, uint64_t ms) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    if (diag_nowait()) return GF_OK;  // the probe keeps timeout 0
    c->timeout_ns = std::max<uint64_t>(ms * 1000ull * 1000ull, 1);  // 0 is the no-wait probe
    return GF_OK;
}

int gf_comm_set_max_blocks(gf_comm* c, int max_blocks) {
    if (!c || max_blocks < 0) return gfi::fail(GF_ERR_CONFIG, "gf_comm_set_max_blocks: bad arguments");
    c->max_blocks = std::min(max_blocks, kMaxBlocks);
    return GF_OK;
}

int gf_comm_set_block_threads(gf_comm* c, int threads) {
    if (!c || threads < 0 || threads > kRingThreads || threads % 32 != 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_comm_set_block_threads: 0 (default 512) or a multiple of 32 up to 512");
    c->block_threads = threads;
    return GF_OK;
}

int gf_comm_status(gf_comm* c) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    if (c->err_host && *reinterpret_cast<volatile int*>(c->err_host) != 0)
        return gfi::fail(GF_ERR_TRANSPORT, "recv timeout at rank " + std::to_string(c->rank) +
                                               " (peer did not reach the collective barrier)");
    return GF_OK;
}

int gf_comm_set_trace(gf_comm* c, int on) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    c->trace = on != 0;
    return GF_OK;
}

int gf_comm_trace(gf_comm* c, uint64_t* out4) {
    if (!c || !out4) return gfi::fail(GF_ERR_CONFIG, "gf_comm_trace: null argument");
    const volatile uint64_t* t =
        reinterpret_cast<const volatile uint64_t*>(reinterpret_cast<char*>(c->err_host) + 64);
    for (int i = 0; i < 4; ++i) out4[i] = t[i];
    return GF_OK;
}

int gf_comm_set_select_inbox(gf_comm* c, uint64_t inbox_heap_off) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    if (inbox_heap_off != UINT64_MAX && (inbox_heap_off % 16 != 0 || inbox_heap_off >= c->heap_bytes))
        return gfi::fail(GF_ERR_CONFIG, "gf_comm_set_select_inbox: offset outside the heap or not 16-B aligned");
    c->sel_inbox_off = inbox_heap_off;
    return GF_OK;
}

int gf_comm_set_csc_inbox(gf_comm* c, uint64_t inbox_heap_off, uint64_t slot_elems) {
    if (!c) return gfi::fail(GF_ERR_CONFIG, "null communicator");
    if (inbox_heap_off != UINT64_MAX &&
        (inbox_heap_off % 16 != 0 || slot_elems % 8 != 0 || slot_elems == 0 ||
         inbox_heap_off + uint64_t(c->world - 1) * slot_elems * 2 > c->heap_bytes))
        return gfi::fail(GF_ERR_CONFIG, "gf_comm_set_csc_inbox: world-1 slots of slot_elems (multiple of 8) fp16 "
                                        "elements at a 16-B aligned offset inside the heap");
    c->csc_inbox_off = inbox_heap_off;
    c->csc_slot_elems = inbox_heap_off == UINT64_MAX ? 0 : slot_elems;
    return GF_OK;
}

int gf_comm_trace_n(gf_comm* c, uint64_t* out, int n) {
    if (!c || !out || n < 0 || n > 16) return gfi::fail(GF_ERR_CONFIG, "gf_comm_trace_n: bad arguments");
    const volatile uint64_t* t =
        reinterpret_cast<const volatile uint64_t*>(reinterpret_cast<char*>(c->err_host) + 64);
    for (int i = 0; i < n; ++i) out[i] = t[i];
    return GF_OK;
}

int gf_comm_rank(gf_comm* c) { return c ? c->rank : -1; }
int gf_comm_world(gf_comm* c) { return c ? c->world : -1; }

int gf_ring_allreduce(gf_comm* c, int dtype, uint64_t heap_off, const uint64_t* win_start,
                      const uint64_t* win_len, int nwin, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (!gfi::valid_dtype(dtype) || nwin < 0 || (nwin > 0 && (!win_start || !win_len)))
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce: bad arguments");
    if (c->world == 1) return GF_OK;  // collectives.cpp:59
    const uint64_t es = gfi::esz(dtype);
    for (int w = 0; w < nwin; ++w)
        if (heap_off + (win_start[w] + win_len[w]) * es > c->heap_bytes)
            return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce: window outside the symmetric heap");
    DeviceGuard g(c->device);
    for (int first = 0; first < nwin; first += kMaxW) {
        RingArgs a;
        std::memset(&a, 0, sizeof(a));
        a.nwin = std::min(kMaxW, nwin - first);
        uint64_t max_seg = 0;
        for (int w = 0; w < a.nwin; ++w) {
            a.wstart[w] = win_start[first + w];
            a.wlen[w] = win_len[first + w];
            max_seg += (a.wlen[w] + c->world - 1) / c->world;
        }
        fill_common(c, a, heap_off);
        launch_ring(dtype, true, a, dim3(gfr::comm_blocks(c, max_seg * es)), gfi::S(stream));
        gfi::count_launch();
        if (int rc = gfi::check_launch("gf_ring_allreduce")) return rc;
    }
    return GF_OK;
}

int gf_ring_allreduce_ptrs(gf_comm* c, int dtype, void* const* rank_bufs, const uint64_t* win_start,
                           const uint64_t* win_len, int nwin, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (!gfi::valid_dtype(dtype) || !rank_bufs || nwin < 0 || (nwin > 0 && (!win_start || !win_len)))
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_ptrs: bad arguments");
    if (c->world == 1) return GF_OK;
    const uint64_t es = gfi::esz(dtype);
    for (int r = 0; r < c->world; ++r) {
        if (!rank_bufs[r]) return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_ptrs: null rank buffer");
        if ((reinterpret_cast<uintptr_t>(rank_bufs[r]) & 15u) != 0)
            return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_ptrs: rank buffers must be 16-byte aligned");
    }
    DeviceGuard g(c->device);
    for (int first = 0; first < nwin; first += kMaxW) {
        RingArgs a;
        std::memset(&a, 0, sizeof(a));
        a.nwin = std::min(kMaxW, nwin - first);
        uint64_t max_seg = 0;
        for (int w = 0; w < a.nwin; ++w) {
            a.wstart[w] = win_start[first + w];
            a.wlen[w] = win_len[first + w];
            max_seg += (a.wlen[w] + c->world - 1) / c->world;
        }
        fill_common(c, a, 0);
        for (int r = 0; r < c->world; ++r) a.bufs[r] = static_cast<char*>(rank_bufs[r]);
        launch_ring(dtype, true, a, dim3(gfr::comm_blocks(c, max_seg * es)), gfi::S(stream));
        gfi::count_launch();
        if (int rc = gfi::check_launch("gf_ring_allreduce_ptrs")) return rc;
    }
    return GF_OK;
}

int gf_ipc_export(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return gfi::fail(GF_ERR_CONFIG, "gf_ipc_export: null argument");
    // driver entry point fetched through the runtime: no link-time libcuda dependency
    using range_fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static range_fn get_range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<range_fn>(fn);
    }();
    if (!get_range) return gfi::fail(GF_ERR_CUDA, "gf_ipc_export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return gfi::fail(GF_ERR_CONFIG, "gf_ipc_export: not a device allocation");
    cudaIpcMemHandle_t h;
    GF_CHECK_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle_out, &h, GF_IPC_HANDLE_BYTES);
    *offset_out = reinterpret_cast<CUdeviceptr>(dev_ptr) - base;
    return GF_OK;
}

int gf_ipc_open(gf_comm* c, const void* handle, void** base_out) {
    if (!c || !handle || !base_out) return gfi::fail(GF_ERR_CONFIG, "gf_ipc_open: null argument");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, GF_IPC_HANDLE_BYTES);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        gfi::cuda_fail(e, "cudaIpcOpenMemHandle");
        return gfi::fail(GF_ERR_TRANSPORT, std::string("gf_ipc_open: ") + cudaGetErrorString(e));
    }
    *base_out = p;
    return GF_OK;
}

int gf_ipc_close(gf_comm* c, void* base) {
    if (!c || !base) return GF_OK;
    DeviceGuard g(c->device);
    GF_CHECK_CUDA(cudaIpcCloseMemHandle(base));
    return GF_OK;
}

int gf_ring_allreduce_planned(gf_comm* c, int dtype, uint64_t heap_off, const uint64_t* plan_dev,
                              void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (!gfi::valid_dtype(dtype) || !plan_dev) return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_planned: bad arguments");
    if (c->world == 1) return GF_OK;
    DeviceGuard g(c->device);
    RingArgs a;
    std::memset(&a, 0, sizeof(a));
    a.nwin = -1;
    a.plan = plan_dev;
    fill_common(c, a, heap_off);
    const uint64_t bound = c->heap_bytes > heap_off ? (c->heap_bytes - heap_off) / c->world : 0;
    launch_ring(dtype, true, a, dim3(gfr::comm_blocks(c, bound)), gfi::S(stream));
    gfi::count_launch();
    return gfi::check_launch("gf_ring_allreduce_planned");
}

int gf_ring_allreduce_planned_scatter(gf_comm* c, int dtype, uint64_t stage_heap_off, const uint64_t* plan_dev,
                                      void* pool, uint64_t chunk, uint64_t nc, uint64_t* nacc, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (dtype != GF_F16 || !plan_dev || !pool || !nacc || chunk == 0 || chunk % 8 != 0 || nc == 0 ||
        nc > 6144 || (reinterpret_cast<uintptr_t>(pool) & 15u) != 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_planned_scatter: fp16 pool (16-B aligned), chunk % 8 == 0, "
                                        "nc <= 6144 (chunk list in shared memory), nacc required");
    if (c->world == 1) return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_planned_scatter: world 1 has no exchange");
    DeviceGuard g(c->device);
    RingArgs a;
    std::memset(&a, 0, sizeof(a));
    a.nwin = -1;
    a.plan = plan_dev;
    fill_common(c, a, stage_heap_off);
    a.wb_pool = static_cast<char*>(pool);
    a.wb_nacc = nacc;
    a.wb_chunk = chunk;
    a.wb_nc = nc;
    const uint64_t bound = c->heap_bytes > stage_heap_off ? (c->heap_bytes - stage_heap_off) / c->world : 0;
    launch_ring(dtype, true, a, dim3(gfr::comm_blocks(c, bound)), gfi::S(stream), size_t(nc) * 8,
                c->block_threads > 0 ? c->block_threads : kRingThreads);
    gfi::count_launch();
    return gfi::check_launch("gf_ring_allreduce_planned_scatter");
}

int gf_csc_exchange_pull(gf_comm* c, uint64_t stage_heap_off, const uint64_t* plan_dev, void* pool,
                         uint64_t chunk, uint64_t nc, uint64_t* nacc, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (!plan_dev || !pool || !nacc || chunk == 0 || chunk % 8 != 0 || nc == 0 || nc > 6144 ||
        (reinterpret_cast<uintptr_t>(pool) & 15u) != 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_exchange_pull: fp16 pool (16-B aligned), chunk % 8 == 0, "
                                        "nc <= 6144 (chunk list in shared memory), nacc required");
    if (c->world == 1) return gfi::fail(GF_ERR_CONFIG, "gf_csc_exchange_pull: world 1 has no exchange");
    DeviceGuard g(c->device);
    RingArgs a;
    std::memset(&a, 0, sizeof(a));
    a.nwin = -1;
    a.plan = plan_dev;
    fill_common(c, a, stage_heap_off);
    a.wb_pool = static_cast<char*>(pool);
    a.wb_nacc = nacc;
    a.wb_chunk = chunk;
    a.wb_nc = nc;
    if (c->csc_inbox_off != UINT64_MAX) {
        a.csc_inbox = c->alloc + kFlagBytes + c->csc_inbox_off;
        a.csc_slot_bytes = c->csc_slot_elems * 2;
        a.csc_push_ag = 1;  // measured: the exchange 6-13 % shorter than with a pulled all-gather
    }
    const uint64_t bound = c->heap_bytes > stage_heap_off ? (c->heap_bytes - stage_heap_off) / c->world : 0;
    const dim3 grid(gfr::comm_blocks(c, bound));
    const size_t smem = size_t(nc) * 8;
    cudaStream_t s = gfi::S(stream);
    const int th = c->block_threads > 0 ? c->block_threads : kRingThreads;
    switch (c->world) {
        case 2: csc_pull_kernel<2><<<grid, th, smem, s>>>(a); break;
        case 4: csc_pull_kernel<4><<<grid, th, smem, s>>>(a); break;
        case 8: csc_pull_kernel<8><<<grid, th, smem, s>>>(a); break;
        default: csc_pull_kernel<0><<<grid, th, smem, s>>>(a); break;
    }
    gfi::count_launch();
    return gfi::check_launch("gf_csc_exchange_pull");
}

int gf_ring_allreduce_colocated(int dtype, void* const* bufs, int world, const int* ring_order,
                                const uint64_t* win_start, const uint64_t* win_len, int nwin,
                                void* stream) {
    if (!gfi::valid_dtype(dtype) || world < 1 || world > GF_MAX_RANKS || !bufs || nwin < 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_colocated: bad arguments");
    if (ring_order && !valid_ring(ring_order, world))
        return gfi::fail(GF_ERR_CONFIG, "ring order is not a permutation of ranks");
    if (world == 1) return GF_OK;
    for (int first = 0; first < nwin; first += kMaxW) {
        RingArgs a;
        std::memset(&a, 0, sizeof(a));
        a.world = world;
        a.nwin = std::min(kMaxW, nwin - first);
        uint64_t max_seg = 0;
        for (int w = 0; w < a.nwin; ++w) {
            a.wstart[w] = win_start[first + w];
            a.wlen[w] = win_len[first + w];
            max_seg += (a.wlen[w] + world - 1) / world;
        }
        for (int r = 0; r < world; ++r) {
            a.bufs[r] = static_cast<char*>(bufs[r]);
            a.ring[r] = ring_order ? ring_order[r] : r;
        }
        launch_ring(dtype, false, a, dim3(gfr::ring_blocks(max_seg * gfi::esz(dtype)), world), gfi::S(stream));
        gfi::count_launch();
        if (int rc = gfi::check_launch("gf_ring_allreduce_colocated")) return rc;
    }
    return GF_OK;
}

int gf_ring_allreduce_colocated_planned(int dtype, void* const* bufs, int world,
                                        const int* ring_order, const uint64_t* plan_dev,
                                        void* stream) {
    if (!gfi::valid_dtype(dtype) || world < 1 || world > GF_MAX_RANKS || !bufs || !plan_dev)
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_colocated_planned: bad arguments");
    if (ring_order && !valid_ring(ring_order, world))
        return gfi::fail(GF_ERR_CONFIG, "ring order is not a permutation of ranks");
    if (world == 1) return GF_OK;
    RingArgs a;
    std::memset(&a, 0, sizeof(a));
    a.world = world;
    a.nwin = -1;
    a.plan = plan_dev;
    for (int r = 0; r < world; ++r) {
        a.bufs[r] = static_cast<char*>(bufs[r]);
        a.ring[r] = ring_order ? ring_order[r] : r;
    }
    launch_ring(dtype, false, a, dim3(gfi::sm_count(), world), gfi::S(stream));
    gfi::count_launch();
    return gfi::check_launch("gf_ring_allreduce_colocated_planned");
}

static int select_launch(SelArgs& a, cudaStream_t s) {
    const size_t smem = size_t(a.nc) * sizeof(float);
    if (smem > 200u * 1024u) return gfi::fail(GF_ERR_CONFIG, "gf_csc_select: too many chunks (max 51200)");
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        GF_CHECK_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set[dev] = true;
    }
    select_kernel<<<1, gfs::kSelThreads, smem, s>>>(a);
    gfi::count_launch();
    return gfi::check_launch("gf_csc_select");
}

int gf_csc_select(gf_comm* c, uint64_t norms_off, uint64_t nc, uint64_t k, uint8_t* flags,
                  uint64_t total, uint64_t chunk, int dtype, uint64_t theta, uint64_t* coff,
                  uint64_t* plan, uint64_t* nacc, const void* pool, const uint8_t* imp_cur,
                  void* stream) {
    if (nacc && (!pool || !imp_cur || dtype != GF_F16))
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_select: nacc needs an fp16 pool and the current set");
    if (int rc = comm_ready(c)) return rc;
    if (nc == 0 || k == 0 || !flags || !gfi::valid_dtype(dtype) || chunk == 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_select: bad arguments");
    if (norms_off + nc * 4 > c->heap_bytes) return gfi::fail(GF_ERR_CONFIG, "gf_csc_select: norms outside heap");
    DeviceGuard g(c->device);
    SelArgs a;
    std::memset(&a, 0, sizeof(a));
    a.world = c->world;
    a.rank = c->rank;
    a.p2p = c->world > 1 ? 1 : 0;
    for (int r = 0; r < c->world; ++r) {
        a.norms[r] = reinterpret_cast<float*>(c->peer_alloc[r] + kFlagBytes + norms_off);
        a.flags_peer[r] = reinterpret_cast<uint64_t*>(c->peer_alloc[r]);
        a.ring[r] = c->ring[r];
    }
    a.nc = nc; a.k = k; a.total = total; a.chunk = chunk; a.esz = gfi::esz(dtype); a.theta = theta;
    a.flags = flags; a.coff = coff; a.plan = plan;
    a.nacc[c->rank] = nacc;
    a.pool[c->rank] = static_cast<const uint16_t*>(pool);
    a.imp_cur = imp_cur;
    a.flags_local = reinterpret_cast<uint64_t*>(c->alloc);
    a.epochs = a.flags_local + kFlagWords;
    a.trace = c->trace ? reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(c->err_dev) + 64) + 4 : nullptr;
    a.timeout_ns = c->timeout_ns;
    a.err = c->err_dev;
    if (c->world > 1 && c->sel_inbox_off != UINT64_MAX) {
        if (c->sel_inbox_off + uint64_t(c->world) * nc * 4 > c->heap_bytes)
            return gfi::fail(GF_ERR_CONFIG, "gf_csc_select: the select inbox (world x nc floats) is outside the heap");
        a.inbox_local = reinterpret_cast<float*>(c->alloc + kFlagBytes + c->sel_inbox_off);
        for (int r = 0; r < c->world; ++r)
            a.inbox_peer[r] = reinterpret_cast<float*>(c->peer_alloc[r] + kFlagBytes + c->sel_inbox_off);
    }
    return select_launch(a, gfi::S(stream));
}

int gf_csc_select_colocated(float* const* norms, int world, const int* ring_order, uint64_t nc,
                            uint64_t k, uint8_t* flags, uint64_t total, uint64_t chunk, int dtype,
                            uint64_t theta, uint64_t* coff, uint64_t* plan, uint64_t* const* nacc,
                            const void* const* pools, const uint8_t* imp_cur, void* stream) {
    if (nacc && (!pools || !imp_cur || dtype != GF_F16))
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_select_colocated: nacc needs fp16 pools and the current set");
    if (!norms || world < 1 || world > GF_MAX_RANKS || nc == 0 || k == 0 || !flags ||
        !gfi::valid_dtype(dtype) || chunk == 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_select_colocated: bad arguments");
    if (ring_order && !valid_ring(ring_order, world))
        return gfi::fail(GF_ERR_CONFIG, "ring order is not a permutation of ranks");
    SelArgs a;
    std::memset(&a, 0, sizeof(a));
    a.world = world;
    a.p2p = 0;
    for (int r = 0; r < world; ++r) {
        a.norms[r] = norms[r];
        a.ring[r] = ring_order ? ring_order[r] : r;
        if (nacc) {
            a.nacc[r] = nacc[r];
            a.pool[r] = static_cast<const uint16_t*>(pools[r]);
        }
    }
    a.imp_cur = imp_cur;
    a.nc = nc; a.k = k; a.total = total; a.chunk = chunk; a.esz = gfi::esz(dtype); a.theta = theta;
    a.flags = flags; a.coff = coff; a.plan = plan;
    return select_launch(a, gfi::S(stream));
}

int gf_ring_traffic(uint64_t len, int world, int position, int dtype, uint64_t* bytes_sent,
                    uint64_t* bytes_received, uint64_t* frames_sent) {
    if (world < 1 || position < 0 || position >= world || !gfi::valid_dtype(dtype))
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_traffic: bad arguments");
    const uint64_t es = gfi::esz(dtype), n = uint64_t(world);
    auto seg = [&](int i) {
        const uint64_t base = len / n, rem = len % n, idx = uint64_t(i);
        return base + (idx < rem ? 1 : 0);
    };
    uint64_t sent = 0, recv = 0, frames = 0;
    if (world > 1) {
        const int p = position;
        for (int s = 0; s < world - 1; ++s) {
            sent += seg((p - s + world) % world) * es;          // RS send p-s
            recv += seg((p - s - 1 + world) % world) * es;      // RS recv p-s-1
            sent += seg((p + 1 - s + world) % world) * es;      // AG send p+1-s
            recv += seg((p - s + world) % world) * es;          // AG recv p-s
            frames += 2;
        }
    }
    if (bytes_sent) *bytes_sent = sent;
    if (bytes_received) *bytes_received = recv;
    if (frames_sent) *frames_sent = frames;
    return GF_OK;
}

}  // extern "C"

namespace gfr {
int ring_blocks(uint64_t max_seg_bytes) { return ring_blocks_impl(max_seg_bytes); }
int comm_blocks(const gf_comm* c, uint64_t max_seg_bytes) {
    int g = ring_blocks_impl(max_seg_bytes);
    if (c->max_blocks > 0) g = std::min(g, c->max_blocks);
    return c->grid_cap > 0 ? std::min(g, c->grid_cap) : g;
}
}  // namespace gfr
