// SPDX-License-Identifier: Apache-2.0
//
// The dense gradient-sync step in ONE kernel per rank (gf_sync_step_dense):
// pack (K1) -> NVLink ring allreduce (K4) -> unpack (K6).
//
// Reference: the dense iteration of train_worker (src/trainer.cpp:297-347): write_tensor
// per tensor (src/gradient_pool.cpp:78-105), FusionEngine windows (src/fusion.cpp:72-109)
// each reduced by ring_allreduce_on (src/collectives.cpp:55-97), then g_avg = get(i) / N.
//
// Every CTA b owns one fixed, strided set of 16-byte pool vectors: the vectors it reduces
// in the ring (reduce_segment, ring_device.cuh: vector v0 + g + k*S of a segment, g = the
// thread's grid index, S = all threads), taken over EVERY segment of every window:
//   1. pack    its vectors of all segments, fp32 tensors -> the local fp16 pool;
//   2. entry   barrier with CTA b of every peer (which packed the same vectors);
//   3. reduce  its vectors of this rank's segment over NVLink (ring order, pushed to all);
//   4. exit    barrier with CTA b of every peer (which pushed the same vectors to me);
//   5. unpack  its vectors of all segments -> the fp32 g_avg tensors (x 1/N).
// Only CTA pairs synchronise: no grid-wide barrier and no extra launches, so a CTA that is
// done packing already moves NVLink traffic while others still pack, and unpacks while
// others still reduce. CTA 0 also takes each segment's unaligned edge elements in all three
// phases (as in reduce_segment). The results are those of gf_pack + gf_ring_allreduce +
// gf_unpack, bit for bit. At world == 1 the step is the one-pass pack_kernel<DstTable>.

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ring_device.cuh"

namespace {

constexpr int kStepMaxT = 256;
#ifndef GF_SWEEP_U
#define GF_SWEEP_U 8
#endif
constexpr int kSweepU = GF_SWEEP_U;  // pack/unpack vectors in flight per thread (1 CTA of 512 per SM)

struct StepTable {  // tensors sorted by pool offset
    int n;
    int pad;
    uint64_t off[kStepMaxT];
    uint64_t cnt[kStepMaxT];
    const float* src[kStepMaxT];
    float* dst[kStepMaxT];
};

// last tensor whose pool range starts at or before element e
__device__ __forceinline__ int tensor_at(const StepTable& T, uint64_t e) {
    int lo = 0, hi = T.n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (T.off[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint4 ld16_cv(const void* p) {  // bypass L1: peers wrote it
    uint4 v;
    asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// ---- element-wise paths: segment edges and vectors that straddle a tensor boundary ------
template <int DT>
__device__ __forceinline__ void pack_elem(const StepTable& T, char* pool, uint64_t e, int& t) {
    while (t + 1 < T.n && T.off[t + 1] <= e) ++t;
    const float x = T.src[t][e - T.off[t]];
    if (DT == GF_F16) reinterpret_cast<uint16_t*>(pool)[e] = gfd::enc(x);
    else reinterpret_cast<float*>(pool)[e] = x;
}
template <int DT>
__device__ __forceinline__ void unpack_elem(const StepTable& T, const char* pool, uint64_t e, int& t,
                                            float inv) {
    while (t + 1 < T.n && T.off[t + 1] <= e) ++t;
    const float x = DT == GF_F16 ? gfd::dec(reinterpret_cast<const volatile uint16_t*>(pool)[e])
                                 : reinterpret_cast<const volatile float*>(pool)[e];
    T.dst[t][e - T.off[t]] = gfd::mul(x, inv);
}
// [e0, e1) by the threads of one CTA
template <int DT, bool PACK>
__device__ void edge_range(const StepTable& T, char* pool, uint64_t e0, uint64_t e1, float inv) {
    for (uint64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        int t = tensor_at(T, e);
        if (PACK) pack_elem<DT>(T, pool, e, t);
        else unpack_elem<DT>(T, pool, e, t, inv);
    }
}

// ---- vector sweeps: vectors v0 + g + k*S of one segment, U in flight per thread ------------
template <int DT>
__device__ __forceinline__ void pack_vectors(const StepTable& T, char* pool, uint64_t v0, uint64_t v1,
                                             uint64_t g, uint64_t S) {
    constexpr int VE = Vec<DT>::kElems;
    constexpr int U = kSweepU;
    for (uint64_t v = v0 + g; v < v1; v += S * U) {
        gfd::F8 f[U];
        int tt[U];
        bool fast[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * S;
            fast[u] = false;
            tt[u] = 0;
            if (vv < v1) {
                const uint64_t e = vv * VE;
                const int t = tensor_at(T, e);
                tt[u] = t;
                const float* s = T.src[t] + (e - T.off[t]);
                if (e + VE <= T.off[t] + T.cnt[t] && (reinterpret_cast<uintptr_t>(s) & (VE * 4 - 1)) == 0) {
                    fast[u] = true;
                    if (DT == GF_F16) {
                        f[u] = gfd::ld32f_stream(s);  // LDG.E.256
                    } else {
                        f[u].lo = gfd::ld16f_stream(s);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * S;
            if (vv >= v1) continue;
            if (fast[u]) {
                if (DT == GF_F16) {
                    gfd::st16_keep(pool + vv * 16, gfd::enc8(f[u].lo, f[u].hi));  // peers read it next
                } else {
                    gfd::st16_keep(pool + vv * 16, *reinterpret_cast<const uint4*>(&f[u].lo));
                }
            } else {
                int t = tt[u];
                for (int k = 0; k < VE; ++k) pack_elem<DT>(T, pool, vv * VE + k, t);
            }
        }
    }
}

// one 16-byte pool vector vv holding x -> fp32 g_avg = x * (1/N) in its tensor(s)
template <int DT>
__device__ __forceinline__ void unpack_vec(const StepTable& T, uint64_t vv, uint4 x, float inv) {
    constexpr int VE = Vec<DT>::kElems;
    const uint64_t e = vv * VE;
    int t = tensor_at(T, e);
    float* d = T.dst[t] + (e - T.off[t]);
    const bool whole = e + VE <= T.off[t] + T.cnt[t];
    if (DT == GF_F16 && whole && (reinterpret_cast<uintptr_t>(d) & 31u) == 0 && !gfd::any_special(x)) {
        const float2 f0 = gfd::h2f2(x.x), f1 = gfd::h2f2(x.y);
        const float2 f2 = gfd::h2f2(x.z), f3 = gfd::h2f2(x.w);
        gfd::st32f_stream(d,  // STG.E.256; finite halves: x * (1/N) cannot produce NaN
                          make_float4(__fmul_rn(f0.x, inv), __fmul_rn(f0.y, inv), __fmul_rn(f1.x, inv),
                                      __fmul_rn(f1.y, inv)),
                          make_float4(__fmul_rn(f2.x, inv), __fmul_rn(f2.y, inv), __fmul_rn(f3.x, inv),
                                      __fmul_rn(f3.y, inv)));
    } else if (DT == GF_F32 && whole && (reinterpret_cast<uintptr_t>(d) & 15u) == 0) {
        const float4 f = *reinterpret_cast<const float4*>(&x);
        __stcs(reinterpret_cast<float4*>(d), make_float4(gfd::mul(f.x, inv), gfd::mul(f.y, inv),
                                                        gfd::mul(f.z, inv), gfd::mul(f.w, inv)));
    } else {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
        for (int k = 0; k < VE; ++k) {
            const uint64_t ek = e + k;
            while (t + 1 < T.n && T.off[t + 1] <= ek) ++t;
            const float xv = DT == GF_F16 ? gfd::dec(uint16_t((w[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu))
                                          : gfd::u2f(w[k]);
            T.dst[t][ek - T.off[t]] = gfd::mul(xv, inv);
        }
    }
}

template <int DT>
__device__ __forceinline__ void unpack_vectors(const StepTable& T, const char* pool, uint64_t v0, uint64_t v1,
                                               uint64_t g, uint64_t S, float inv) {
    constexpr int U = kSweepU;
    for (uint64_t v = v0 + g; v < v1; v += S * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * S;
            if (vv < v1) x[u] = ld16_cv(pool + vv * 16);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * S;
            if (vv < v1) unpack_vec<DT>(T, vv, x[u], inv);
        }
    }
}

// segment j of window w (segment_of, collectives.cpp:47-53)
__device__ __forceinline__ void segment(const RingArgs& a, int n, int w, int j, uint64_t& e0, uint64_t& e1) {
    const uint64_t ws = a.wstart[w], wl = a.wlen[w];
    const uint64_t base = wl / uint64_t(n), rem = wl % uint64_t(n), uj = uint64_t(j);
    e0 = ws + uj * base + min(uj, rem);
    e1 = e0 + base + (uj < rem ? 1 : 0);
}

// phases 1 and 5 over every window's every segment, in the ring's vector pattern
template <int DT, bool PACK>
__device__ void sweep_all(const RingArgs& a, const StepTable& T, int n, uint64_t g, uint64_t S, float inv) {
    constexpr int VE = Vec<DT>::kElems;
    char* pool = a.bufs[a.rank];
    for (int w = 0; w < a.nwin; ++w) {
        for (int j = 0; j < n; ++j) {
            uint64_t e0, e1;
            segment(a, n, w, j, e0, e1);
            const uint64_t v0 = (e0 + VE - 1) / VE, v1 = e1 / VE;
            if (v0 >= v1) {  // no aligned vector inside: all scalar, CTA 0 (as reduce_segment)
                if (blockIdx.x == 0) edge_range<DT, PACK>(T, pool, e0, e1, inv);
                continue;
            }
            if (blockIdx.x == 0) {
                edge_range<DT, PACK>(T, pool, e0, v0 * VE, inv);
                edge_range<DT, PACK>(T, pool, v1 * VE, e1, inv);
            }
            if (PACK) pack_vectors<DT>(T, pool, v0, v1, g, S);
            else unpack_vectors<DT>(T, pool, v0, v1, g, S, inv);
        }
    }
}

template <int DT, int NT>
__global__ void __launch_bounds__(kRingThreads)
step_kernel(const __grid_constant__ RingArgs a, const __grid_constant__ StepTable T, float inv) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    __shared__ int s_ok;
    const uint64_t epoch = a.epochs[blockIdx.x];
    if (threadIdx.x == 0) s_ok = 1;
    const int n = NT > 0 ? NT : a.world;
    const uint64_t S = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) a.trace[0] = gfd::globaltimer_ns();

    sweep_all<DT, true>(a, T, n, g, S, inv);  // 1. pack
    if (!cross_barrier(a, epoch + 1, &s_ok, true)) return;  // 2. my packed vectors are visible
    if (tr) a.trace[1] = gfd::globaltimer_ns();

    const char* src[NMAX];  // 3. reduce my segment of every window (ring order from my position)
#pragma unroll
    for (int t = 0; t < NMAX; ++t) src[t] = (t < n) ? a.bufs[a.ring[(a.pos + t) % n]] : nullptr;
    for (int w = 0; w < a.nwin; ++w) {
        uint64_t e0, e1;
        segment(a, n, w, a.pos, e0, e1);
        reduce_segment<DT, NT>(a, src, n, e0, e1, g, S);
    }
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 2, &s_ok, true)) return;  // 4. peers' pushes to me landed
    if (threadIdx.x == 0) a.epochs[blockIdx.x] = epoch + 2;
    if (tr) a.trace[3] = gfd::globaltimer_ns();

    sweep_all<DT, false>(a, T, n, g, S, inv);  // 5. unpack
}

template <int DT>
void launch_step(const RingArgs& a, const StepTable& T, float inv, int grid, cudaStream_t s) {
    switch (a.world) {
        case 2: step_kernel<DT, 2><<<grid, kRingThreads, 0, s>>>(a, T, inv); break;
        case 4: step_kernel<DT, 4><<<grid, kRingThreads, 0, s>>>(a, T, inv); break;
        case 8: step_kernel<DT, 8><<<grid, kRingThreads, 0, s>>>(a, T, inv); break;
        default: step_kernel<DT, 0><<<grid, kRingThreads, 0, s>>>(a, T, inv); break;
    }
}

// ---- gf_ring_allreduce_unpack: pull reduce-scatter, then pull all-gather fused with unpack ----
// The rank at ring position p sums segment p of every window from all N pools in ring order
// (the reference's arrival order, as reduce_segment), keeps the sum in its OWN pool only and
// unpacks it from registers. After one barrier with its peer CTAs it PULLS every other
// segment from the rank that owns it, writes it into its pool (every pool ends holding the
// sums, as after ring_allreduce) and unpacks it. Nothing is pushed, so no barrier waits for
// posted NVLink writes to drain; and the separate unpack pass (re-reading the pool) is gone.
template <int DT>
__device__ __forceinline__ uint4 ld16_cg(const void* p) {  // L2 only: a peer wrote it this launch
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Scalar reduce (or copy) + unpack of pool element e by the edge CTA.
template <int DT, bool OWN>
__device__ __forceinline__ void pull_elem(const StepTable& T, const char* const* src, int n, char* local,
                                          uint64_t e, float inv) {
    float xv;
    if (DT == GF_F16) {
        uint16_t h;
        if (OWN) {
            h = reinterpret_cast<const uint16_t*>(src[0])[e];
            for (int t = 1; t < n; ++t) h = gfd::acc16(reinterpret_cast<const uint16_t*>(src[t])[e], h);
        } else {
            h = reinterpret_cast<const volatile uint16_t*>(src[0])[e];
        }
        reinterpret_cast<uint16_t*>(local)[e] = h;
        xv = gfd::dec(h);
    } else {
        float acc;
        if (OWN) {
            acc = reinterpret_cast<const float*>(src[0])[e];
            for (int t = 1; t < n; ++t) acc = gfd::add(reinterpret_cast<const float*>(src[t])[e], acc);
        } else {
            acc = reinterpret_cast<const volatile float*>(src[0])[e];
        }
        reinterpret_cast<float*>(local)[e] = acc;
        xv = acc;
    }
    const int t = tensor_at(T, e);
    T.dst[t][e - T.off[t]] = gfd::mul(xv, inv);
}

// OWN: reduce-scatter of my segment of every window (sum of all N pools in ring order, kept
// in my pool); else all-gather of segment q from its owner (src[0]) into my pool. Both unpack
// every value from registers. f is the flattened vector space of that segment over the
// windows (FlatWins): the owner's RS and every rank's AG of segment q map flat vector x to the
// same CTA, so the middle barrier (CTA b <-> CTA b) orders exactly the vectors it needs.
template <int DT, int NT, bool OWN>
__device__ void pull_flat(const RingArgs& a, const StepTable& T, const char* const* src, int n, char* local,
                          const FlatWins& f, uint64_t g, uint64_t S, float inv) {
    constexpr int VE = Vec<DT>::kElems;
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int NS = OWN ? NMAX : 1;
    constexpr int U = OWN ? (NMAX <= 4 ? 4 : (NMAX <= 8 ? 2 : 1)) : 8;
    // unaligned edges, scalar: window w's by CTA w mod grid (the same CTA in RS and AG)
    for (int w = int(blockIdx.x); w < a.nwin; w += int(gridDim.x)) {
        const uint64_t e0 = f.e0[w], e1 = f.e1[w], v0 = f.v0[w], v1 = v0 + (f.pre[w + 1] - f.pre[w]);
        const uint64_t h0 = v1 > v0 ? min(e1, v0 * VE) : e1;
        for (uint64_t e = e0 + threadIdx.x; e < h0; e += blockDim.x) pull_elem<DT, OWN>(T, src, n, local, e, inv);
        if (v1 > v0)
            for (uint64_t e = v1 * VE + threadIdx.x; e < e1; e += blockDim.x)
                pull_elem<DT, OWN>(T, src, n, local, e, inv);
    }
    const uint64_t total = f.pre[a.nwin];
    for (uint64_t x = g; x < total; x += S * U) {
        uint4 v[U][NS];
        uint64_t vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t xu = x + uint64_t(u) * S;
            vv[u] = ~0ull;
            if (xu < total) {
                const int w = flat_window(f, a.nwin, xu);
                vv[u] = f.v0[w] + (xu - f.pre[w]);
#pragma unroll
                for (int t = 0; t < NS; ++t) {
                    if (OWN) {
                        if (t < n) v[u][t] = gfd::ld16(src[t] + vv[u] * 16);
                    } else {
                        v[u][t] = ld16_cg<DT>(src[0] + vv[u] * 16);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (vv[u] == ~0ull) continue;
            uint4 acc = v[u][0];
            if (OWN) {
#pragma unroll
                for (int t = 1; t < NS; ++t)
                    if (t < n) acc = Vec<DT>::acc(v[u][t], acc);
                gfd::st16_keep(local + vv[u] * 16, acc);  // the peers pull it next
            } else {
                gfd::st16(local + vv[u] * 16, acc);
            }
            unpack_vec<DT>(T, vv[u], acc, inv);
        }
    }
}

template <int DT, int NT>
__global__ void __launch_bounds__(kRingThreads)
rsag_kernel(const __grid_constant__ RingArgs a, const __grid_constant__ StepTable T, float inv, int exit_barrier) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    __shared__ int s_ok;
    const uint64_t epoch = a.epochs[blockIdx.x];
    if (threadIdx.x == 0) s_ok = 1;
    const int n = NT > 0 ? NT : a.world;
    const uint64_t S = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) a.trace[0] = gfd::globaltimer_ns();
    constexpr int VE = Vec<DT>::kElems;
    __shared__ FlatWins flat;
    flat_build<VE>(a, n, a.pos, flat, true);  // my segment of every window (this piece)
    if (!cross_barrier(a, epoch + 1, &s_ok, false)) return;  // peers' pools are packed
    if (tr) a.trace[1] = gfd::globaltimer_ns();
    const char* src[NMAX];
#pragma unroll
    for (int t = 0; t < NMAX; ++t) src[t] = (t < n) ? a.bufs[a.ring[(a.pos + t) % n]] : nullptr;
    char* local = a.bufs[a.rank];
    pull_flat<DT, NT, true>(a, T, src, n, local, flat, g, S, inv);
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 2, &s_ok, true)) return;  // my segment sums are visible
    for (int j = 1; j < n; ++j) {  // next ring position first: owners differ across ranks
        const int q = (a.pos + j) % n;
        flat_build<VE>(a, n, q, flat, true);
        const char* owner[1] = {a.bufs[a.ring[q]]};
        pull_flat<DT, NT, false>(a, T, owner, n, local, flat, g, S, inv);
    }
    uint64_t fin = epoch + 2;
    if (exit_barrier) {  // the peers are done reading my pool (no write drain involved)
        if (!cross_barrier(a, epoch + 3, &s_ok, false)) return;
        fin = epoch + 3;
    }
    if (threadIdx.x == 0) a.epochs[blockIdx.x] = fin;
    if (tr) a.trace[3] = gfd::globaltimer_ns();
}

template <int DT>
void launch_rsag(const RingArgs& a, const StepTable& T, float inv, int exit_barrier, int grid, cudaStream_t s) {
    switch (a.world) {
        case 2: rsag_kernel<DT, 2><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier); break;
        case 4: rsag_kernel<DT, 4><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier); break;
        case 8: rsag_kernel<DT, 8><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier); break;
        default: rsag_kernel<DT, 0><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier); break;
    }
}

// tensor table in pool order; checks the tensors tile [off[0], hi) without overlap
int build_table(const char* fn, const float* const* src, float* const* dst, const uint64_t* pool_off,
                const uint64_t* count, int ntensors, StepTable& T, uint64_t& hi) {
    std::vector<int> order(static_cast<size_t>(ntensors));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return pool_off[x] < pool_off[y]; });
    std::memset(&T, 0, sizeof(T));
    T.n = ntensors;
    hi = 0;
    for (int i = 0; i < ntensors; ++i) {
        const int k = order[static_cast<size_t>(i)];
        T.off[i] = pool_off[k];
        T.cnt[i] = count[k];
        T.src[i] = src ? src[k] : nullptr;
        T.dst[i] = dst[k];
        if ((src && !src[k]) || !dst[k]) return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": null tensor");
        if (i > 0 && T.off[i] < T.off[i - 1] + T.cnt[i - 1])
            return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": tensors overlap in the pool");
        hi = std::max(hi, T.off[i] + T.cnt[i]);
    }
    return GF_OK;
}

// the tensors and the windows must tile the same pool range: every element is reduced and
// unpacked exactly once
int check_tiling(const char* fn, const StepTable& T, uint64_t hi, const uint64_t* win_start,
                 const uint64_t* win_len, int nwin) {
    for (int i = 0; i + 1 < T.n; ++i)
        if (T.off[i] + T.cnt[i] != T.off[i + 1])
            return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": tensors must tile the pool");
    uint64_t cover = T.off[0];
    for (int w = 0; w < nwin; ++w) {
        if (win_start[w] != cover) return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": windows must tile the pool");
        cover += win_len[w];
    }
    if (cover != hi) return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": windows must tile the pool");
    return GF_OK;
}

}  // namespace

extern "C" {

int gf_sync_step_dense(gf_comm* c, int dtype, uint64_t pool_heap_off, const float* const* src,
                       float* const* dst, const uint64_t* pool_off, const uint64_t* count,
                       int ntensors, const uint64_t* win_start, const uint64_t* win_len, int nwin,
                       void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (!gfi::valid_dtype(dtype) || ntensors < 1 || ntensors > kStepMaxT || !src || !dst || !pool_off ||
        !count || nwin < 1 || !win_start || !win_len)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: bad arguments (1..256 tensors, >= 1 window)");
    const uint64_t es = gfi::esz(dtype);
    StepTable T;
    uint64_t hi = 0;
    if (int rc = build_table("gf_sync_step_dense", src, dst, pool_off, count, ntensors, T, hi)) return rc;
    if (pool_heap_off + hi * es > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: pool outside the symmetric heap");
    DeviceGuard guard(c->device);
    if (c->world == 1)  // no collective: pack and unpack in one streaming pass
        return gfi::pack_unpack_solo(dtype, c->alloc + kFlagBytes + pool_heap_off, src, dst, pool_off, count,
                                     ntensors, gfi::S(stream));
    if (int rc = check_tiling("gf_sync_step_dense", T, hi, win_start, win_len, nwin)) return rc;
    const float inv = 1.0f / static_cast<float>(c->world);
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
        fill_common(c, a, pool_heap_off);
        const int grid = gfr::ring_blocks(max_seg * es);
        if (dtype == GF_F16) launch_step<GF_F16>(a, T, inv, grid, gfi::S(stream));
        else launch_step<GF_F32>(a, T, inv, grid, gfi::S(stream));
        gfi::count_launch();
        if (int rc = gfi::check_launch("gf_sync_step_dense")) return rc;
    }
    return GF_OK;
}

int gf_ring_allreduce_unpack_part(gf_comm* c, int dtype, uint64_t pool_heap_off, float* const* dst,
                                  const uint64_t* pool_off, const uint64_t* count, int ntensors,
                                  const uint64_t* win_start, const uint64_t* win_len, int nwin,
                                  uint32_t part_lo, uint32_t part_hi, int flags, void* stream) {
    static const char* fn = "gf_ring_allreduce_unpack";
    if (part_lo >= part_hi || part_hi > GF_PART_ONE)
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_unpack_part: need 0 <= part_lo < part_hi <= GF_PART_ONE");
    if (int rc = comm_ready(c)) return rc;
    if (!gfi::valid_dtype(dtype) || ntensors < 1 || ntensors > kStepMaxT || !dst || !pool_off || !count ||
        nwin < 1 || !win_start || !win_len || (flags & ~GF_RSAG_NO_EXIT_BARRIER))
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_unpack: bad arguments (1..256 tensors, >= 1 window)");
    StepTable T;
    uint64_t hi = 0;
    if (int rc = build_table(fn, nullptr, dst, pool_off, count, ntensors, T, hi)) return rc;
    const uint64_t es = gfi::esz(dtype);
    if (pool_heap_off + hi * es > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_unpack: pool outside the symmetric heap");
    if (int rc = check_tiling(fn, T, hi, win_start, win_len, nwin)) return rc;
    DeviceGuard guard(c->device);
    if (c->world == 1) {  // the collective is the identity (collectives.cpp:59)
        if (part_lo != 0 || part_hi != GF_PART_ONE)
            return gfi::fail(GF_ERR_CONFIG, "gf_ring_allreduce_unpack_part: pieces need world > 1");
        return gf_unpack(dtype, c->alloc + kFlagBytes + pool_heap_off, dst, pool_off, count, ntensors, 1, stream);
    }
    const float inv = 1.0f / static_cast<float>(c->world);
    const int exit_barrier = (flags & GF_RSAG_NO_EXIT_BARRIER) ? 0 : 1;
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
        fill_common(c, a, pool_heap_off);
        a.part_lo = part_lo;
        a.part_hi = part_hi;
        const uint64_t part_seg = std::max<uint64_t>(1, max_seg * (part_hi - part_lo) / GF_PART_ONE);
        const int grid = gfr::ring_blocks(part_seg * es);
        if (dtype == GF_F16) launch_rsag<GF_F16>(a, T, inv, exit_barrier, grid, gfi::S(stream));
        else launch_rsag<GF_F32>(a, T, inv, exit_barrier, grid, gfi::S(stream));
        gfi::count_launch();
        if (int rc = gfi::check_launch(fn)) return rc;
    }
    return GF_OK;
}

int gf_ring_allreduce_unpack(gf_comm* c, int dtype, uint64_t pool_heap_off, float* const* dst,
                             const uint64_t* pool_off, const uint64_t* count, int ntensors,
                             const uint64_t* win_start, const uint64_t* win_len, int nwin, int flags,
                             void* stream) {
    return gf_ring_allreduce_unpack_part(c, dtype, pool_heap_off, dst, pool_off, count, ntensors, win_start,
                                         win_len, nwin, 0, GF_PART_ONE, flags, stream);
}

int gf_part_ranges(const uint64_t* win_start, const uint64_t* win_len, int nwin, int world,
                   uint32_t part_lo, uint32_t part_hi, uint64_t* lo, uint64_t* hi, int cap) {
    if (!win_start || !win_len || nwin < 0 || world < 1 || world > GF_MAX_RANKS || part_lo > part_hi ||
        part_hi > GF_PART_ONE || (cap > 0 && (!lo || !hi)))
        return gfi::fail(GF_ERR_CONFIG, "gf_part_ranges: bad arguments"), -1;
    int k = 0;
    const uint64_t n = uint64_t(world);
    for (int w = 0; w < nwin; ++w) {
        const uint64_t base = win_len[w] / n, rem = win_len[w] % n;
        for (uint64_t j = 0; j < n; ++j) {  // segment_of (collectives.cpp:47-53)
            const uint64_t e0 = win_start[w] + j * base + std::min(j, rem);
            const uint64_t e1 = e0 + base + (j < rem ? 1 : 0);
            const uint64_t a = part_cut(e0, e1, part_lo), b = part_cut(e0, e1, part_hi);
            if (a >= b) continue;
            if (k > 0 && hi[k - 1] == a) {  // adjacent: merge
                hi[k - 1] = b;
                continue;
            }
            if (k >= cap) return -1;
            lo[k] = a;
            hi[k] = b;
            ++k;
        }
    }
    return k;
}

}  // extern "C"
