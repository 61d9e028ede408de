// SPDX-License-Identifier: Apache-2.0
//
// Coarse-grained sparse communication (CSC) kernels.
//
//  K2 gf_csc_pack_correct  write_tensor + correction_pre_allreduce + staging pack,
//                          fused: src/gradient_pool.cpp:78-105, src/sparse.cpp:57-79
//                          (csc_correct sparse.hpp:34-40), src/sparse.cpp:129-140.
//                          14 B/element of HBM traffic (4 g + 4 hg in, 2 pool + 4 hg out)
//                          + 2 B per selected element (staging).
//  K3 gf_chunk_norms       GradientPool::chunk_l1 (src/gradient_pool.cpp:107-116) for all
//                          chunks, x1/N for important ones (src/sparse.cpp:176-184).
//                          The reference sums |x| sequentially in fp64. For an fp16 pool
//                          every |x| is an integer multiple of 2^-24, so we sum EXACTLY in
//                          int64 units of 2^-24 (order-free, warp-shuffle + smem tree);
//                          whenever the exact sum is < 2^53 units every fp64 partial sum
//                          of the reference was exact too, so the float result is
//                          bit-identical. Larger sums (|x| averaging > 12k) fall back to a
//                          sequential fp64 pass. 2 B/element.
//  gf_csc_compact/scatter  staging pack / write-back (src/sparse.cpp:129-140, :162-168).
//  gf_select_topk/gf_csc_plan  see select.cuh.

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "comm.cuh"
#include "gf_device.cuh"
#include "gf_internal.cuh"
#include "select.cuh"
#include "tensor_table.cuh"


namespace {

constexpr int kNormThreads = 256;

using gfd::half_units;
using gfd::units8;

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    return v;
}

// One CTA per chunk (grid-stride over chunks).
__global__ void __launch_bounds__(kNormThreads)
norms_f16_kernel(const uint16_t* __restrict__ pool, uint64_t total, uint64_t chunk, uint64_t nc,
                 const uint8_t* __restrict__ imp, float inv_world, float* __restrict__ norms) {
    __shared__ uint64_t s_sum[kNormThreads / 32];
    __shared__ int s_nan[kNormThreads / 32];
    for (uint64_t c = blockIdx.x; c < nc; c += gridDim.x) {
        const uint64_t b = c * chunk;
        const uint64_t len = (c + 1 == nc) ? total - b : chunk;
        const uint16_t* p = pool + b;
        uint64_t acc = 0;
        bool nan = false;
        uint64_t done = 0;
        if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
            const uint64_t nvec = len / 8;
            constexpr int U = 4;
            for (uint64_t v0 = threadIdx.x; v0 < nvec; v0 += uint64_t(kNormThreads) * U) {
                uint4 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t v = v0 + uint64_t(u) * kNormThreads;
                    x[u] = v < nvec ? gfd::ld16_stream(p + 8 * v) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    nan |= gfd::any_special(x[u]);
                    acc += units8(x[u]);
                }
            }
            done = nvec * 8;
        }
        for (uint64_t i = done + threadIdx.x; i < len; i += kNormThreads) {
            const uint16_t h = p[i];
            nan |= (h & 0x7C00u) == 0x7C00u;
            acc += half_units(h);
        }
        acc = warp_sum_u64(acc);
        const int any_nan = __any_sync(0xFFFFFFFFu, nan);
        if ((threadIdx.x & 31) == 0) {
            s_sum[threadIdx.x >> 5] = acc;
            s_nan[threadIdx.x >> 5] = any_nan;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t s = 0;
            int n = 0;
            for (int w = 0; w < kNormThreads / 32; ++w) { s += s_sum[w]; n |= s_nan[w]; }
            float out;
            if (n) {
                // fp16 pools only ever hold the codec's NaN (sign|0x7E00; inf is clamped):
                // fabs(double) + cast gives the positive quiet NaN.
                out = gfd::u2f(0x7FC00000u);
            } else if (s < (1ull << 53)) {
                out = __double2float_rn(__ull2double_rn(s) * 0x1p-24);
            } else {
                double d = 0.0;  // sequential fallback, exactly as the reference
                for (uint64_t i = 0; i < len; ++i) d = __dadd_rn(d, fabs(double(gfd::dec(p[i]))));
                out = __double2float_rn(d);
            }
            if (imp && imp[c]) out = gfd::mul(out, inv_world);
            norms[c] = out;
        }
        __syncthreads();
    }
}

// fp32 pools: fp64 partial sums of fp32 values are not exact in general, so the
// reference's sequential order is reproduced: CTA stages |x| in smem, one thread adds.
__global__ void __launch_bounds__(kNormThreads)
norms_f32_kernel(const float* __restrict__ pool, uint64_t total, uint64_t chunk, uint64_t nc,
                 const uint8_t* __restrict__ imp, float inv_world, float* __restrict__ norms) {
    constexpr int kStage = 2048;
    __shared__ double st[kStage];
    for (uint64_t c = blockIdx.x; c < nc; c += gridDim.x) {
        const uint64_t b = c * chunk;
        const uint64_t len = (c + 1 == nc) ? total - b : chunk;
        double d = 0.0;
        for (uint64_t base = 0; base < len; base += kStage) {
            const uint64_t n = min(uint64_t(kStage), len - base);
            for (uint64_t i = threadIdx.x; i < n; i += kNormThreads) st[i] = fabs(double(pool[b + base + i]));
            __syncthreads();
            if (threadIdx.x == 0) {
                for (uint64_t i = 0; i < n; ++i) d = __dadd_rn(d, st[i]);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            float out = __double2float_rn(d);
            if (imp && imp[c]) out = gfd::mul(out, inv_world);
            norms[c] = out;
        }
    }
}

// csc_correct element (sparse.hpp:35-40 via sparse.cpp:71-77); returns the new pool value.
__device__ __forceinline__ float correct_elem(float g, float* hg, bool imp, float mom) {
    const float gg = gfd::add(g, *hg);
    *hg = imp ? 0.0f : gfd::mul(mom, gg);
    return gg;
}

template <int DT>
__global__ void correct_kernel(void* __restrict__ pool, float* __restrict__ hg,
                               const uint8_t* __restrict__ imp, uint64_t total, uint64_t chunk,
                               uint64_t nc, uint64_t begin, uint64_t end, float mom) {
    for (uint64_t i = begin + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < end;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = min(i / chunk, nc - 1);
        const bool im = imp[c] != 0;
        if (DT == GF_F16) {
            uint16_t* p = static_cast<uint16_t*>(pool);
            p[i] = gfd::enc(correct_elem(gfd::dec(p[i]), hg + i, im, mom));
        } else {
            float* p = static_cast<float*>(pool);
            p[i] = correct_elem(p[i], hg + i, im, mom);
        }
    }
}

constexpr uint64_t kNaccNaN = 1ull << 63;  // NaN marker in an exact-norm accumulator

// Adds a per-thread (chunk, units) contribution with warp aggregation: lanes whose chunk
// equals the first active lane's chunk are summed with shuffles, the others add directly.
// Must be called by all 32 lanes.
__device__ __forceinline__ void nacc_add(uint64_t* nacc, uint64_t c, uint64_t u, bool nan, bool active) {
    const unsigned full = 0xFFFFFFFFu;
    const unsigned act = __ballot_sync(full, active);
    if (!act) return;
    const int leader = __ffs(act) - 1;
    const uint64_t c0 = __shfl_sync(full, c, leader);
    const bool same = active && c == c0;
    uint64_t v = same ? u : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(full, v, o);
    const bool anynan_same = __any_sync(full, same && nan);
    if ((threadIdx.x & 31) == unsigned(leader)) {
        if (v) atomicAdd(reinterpret_cast<unsigned long long*>(nacc + c0), (unsigned long long)v);
        if (anynan_same) atomicOr(reinterpret_cast<unsigned long long*>(nacc + c0), (unsigned long long)kNaccNaN);
    }
    if (active && !same) {
        if (u) atomicAdd(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)u);
        if (nan) atomicOr(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)kNaccNaN);
    }
}

// One 16-byte pool vector of K2: g (8 fp32) packed, corrected with hg (8 fp32) into the new
// pool halves ov and the new residual hn (write_tensor + csc_correct, sparse.hpp:35-40). The
// packed fast path runs when no half is special; otherwise the exact per-element path. nan:
// the vector holds a NaN (the pool holds no inf, so special == NaN).
__device__ __forceinline__ void correct8(const gfd::F8& gv, const float* hp, bool im, float mom, float hn[8],
                                         uint4& ov, bool& nan) {
    const uint4 h1 = gfd::enc8(gv.lo, gv.hi);  // pack (write_tensor)
    bool slow = gfd::any_special(h1);
    if (!slow) {
        const uint32_t hw[4] = {h1.x, h1.y, h1.z, h1.w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 g1 = gfd::h2f2(hw[k]);
            const float a0 = __fadd_rn(g1.x, hp[2 * k]);
            const float a1 = __fadd_rn(g1.y, hp[2 * k + 1]);
            hn[2 * k] = im ? 0.0f : __fmul_rn(mom, a0);
            hn[2 * k + 1] = im ? 0.0f : __fmul_rn(mom, a1);
            o[k] = gfd::f22h2(a0, a1);
        }
        ov = make_uint4(o[0], o[1], o[2], o[3]);
        slow = gfd::any_special(ov);  // non-finite or clamped sum: exact slow path
    }
    nan = false;
    if (slow) {
        const float g[8] = {gv.lo.x, gv.lo.y, gv.lo.z, gv.lo.w, gv.hi.x, gv.hi.y, gv.hi.z, gv.hi.w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 8; ++k) hn[k] = hp[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint16_t lo = gfd::enc(correct_elem(gfd::dec(gfd::enc(g[2 * k])), &hn[2 * k], im, mom));
            const uint16_t hi = gfd::enc(correct_elem(gfd::dec(gfd::enc(g[2 * k + 1])), &hn[2 * k + 1], im, mom));
            o[k] = uint32_t(lo) | (uint32_t(hi) << 16);
        }
        ov = make_uint4(o[0], o[1], o[2], o[3]);
        nan = gfd::any_special(ov);
    }
}

// K2 over one 8192-element tile of tensor table entry (tile index `tile`), by NTH threads.
// part: 0 every chunk, 1 the important chunks only, 2 the unimportant ones only (the CSC step
// runs part 1 first, so the exchange of the staged chunks overlaps part 2).
template <int DT, int NTH, int U>  // U: vectors per thread in flight before the math
__device__ __forceinline__ void pack_correct_tile(const TensorTable& T, uint64_t tile, void* __restrict__ pool,
                                                  float* __restrict__ hg, void* __restrict__ staging,
                                                  const uint8_t* __restrict__ imp, const uint64_t* __restrict__ coff,
                                                  uint64_t chunk, uint64_t nc, float mom, uint64_t* __restrict__ nacc,
                                                  int part) {
    const int t = find_tensor(T, tile);
    const uint64_t base = (tile - T.tiles[t]) * kTile;
    const uint64_t len = min(kTile, T.cnt[t] - base);
    const float* __restrict__ s = static_cast<const float*>(T.ptr[t]) + base;
    const uint64_t po = T.off[t] + base;
    if (part != 0) {  // a tile with no chunk of this part is skipped whole (block-uniform)
        const uint64_t c0 = min(po / chunk, nc - 1), c1 = min((po + len - 1) / chunk, nc - 1);
        bool any = c1 - c0 > 8;  // many small chunks: no shortcut
        for (uint64_t c = c0; !any && c <= c1; ++c) any = (imp[c] != 0) == (part == 1);
        if (!any) return;
    }
    uint64_t done = 0;
    if (DT == GF_F16 && (reinterpret_cast<uintptr_t>(T.ptr[t]) & 31u) == 0 && po % 8 == 0 &&
        chunk % 8 == 0 && (reinterpret_cast<uintptr_t>(hg) & 31u) == 0 &&
        (reinterpret_cast<uintptr_t>(pool) & 15u) == 0 &&
        (reinterpret_cast<uintptr_t>(staging) & 15u) == 0) {
        // 8 consecutive pool elements never straddle a chunk boundary here.
        uint16_t* __restrict__ d = static_cast<uint16_t*>(pool) + po;
        uint16_t* __restrict__ stg = static_cast<uint16_t*>(staging);
        const int nvec = int(len / 8);
        // The tile's chunks: with chunk >= kTile a tile meets at most two (c0 and c0 + 1, split at
        // element cb), so a vector's chunk and importance come from two compares, not a 64-bit
        // division and a dependent flag load per vector
        const uint64_t c0 = min(po / chunk, nc - 1), cb = (c0 + 1) * chunk;
        const bool two = chunk >= kTile && c0 + 1 < nc;
        const bool im0 = imp[c0] != 0, im1 = two ? imp[c0 + 1] != 0 : im0;
        auto chunk_of = [&](uint64_t pi) {
            return chunk >= kTile ? ((two && pi >= cb) ? c0 + 1 : c0) : min(pi / chunk, nc - 1);
        };
        for (int v0 = 0; v0 < nvec; v0 += U * NTH) {
            gfd::F8 gv[U], hv[U];
            uint64_t c[U];
            bool im[U], mine[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * NTH + threadIdx.x;
                const bool act = v < nvec;
                c[u] = 0;
                im[u] = true;
                if (act) {
                    const uint64_t pi = po + 8 * uint64_t(v);
                    c[u] = chunk_of(pi);
                    im[u] = chunk >= kTile ? (c[u] == c0 ? im0 : im1) : imp[c[u]] != 0;
                }
                mine[u] = act && (part == 0 || (part == 1) == im[u]);
                if (mine[u]) {
                    gv[u] = gfd::ld32f_stream(s + 8 * v);  // LDG.E.256
                    hv[u] = gfd::ld32f(hg + po + 8 * uint64_t(v));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * NTH + threadIdx.x;
                uint64_t units = 0;
                bool nan = false;
                if (mine[u]) {
                    const uint64_t pi = po + 8 * uint64_t(v);
                    float hn[8];
                    uint4 ov;
                    correct8(gv[u], reinterpret_cast<const float*>(&hv[u]), im[u], mom, hn, ov, nan);
                    gfd::st32f(hg + pi, make_float4(hn[0], hn[1], hn[2], hn[3]),
                               make_float4(hn[4], hn[5], hn[6], hn[7]));
                    gfd::st16(d + 8 * v, ov);
                    if (im[u] && stg) gfd::st16(stg + coff[c[u]] + (pi - c[u] * chunk), ov);
                    if ((!im[u] || !stg) && nacc) units = units8(nan ? make_uint4(0, 0, 0, 0) : ov);
                }
                if (nacc) nacc_add(nacc, c[u], units, nan, mine[u] && (!im[u] || !stg));
            }
        }
        done = uint64_t(nvec) * 8;
    }
    for (uint64_t i = done + threadIdx.x; i < len; i += NTH) {
        const uint64_t pi = po + i;
        const uint64_t c = min(pi / chunk, nc - 1);
        const bool im = imp[c] != 0;
        if (part != 0 && (part == 1) != im) continue;
        if (DT == GF_F16) {
            const uint16_t w = gfd::enc(correct_elem(gfd::dec(gfd::enc(s[i])), hg + pi, im, mom));
            static_cast<uint16_t*>(pool)[pi] = w;
            if (im && staging) static_cast<uint16_t*>(staging)[coff[c] + (pi - c * chunk)] = w;
            if ((!im || !staging) && nacc) {
                if ((w & 0x7C00u) == 0x7C00u)
                    atomicOr(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)kNaccNaN);
                else if (half_units(w))
                    atomicAdd(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)half_units(w));
            }
        } else {
            const float w = correct_elem(s[i], hg + pi, im, mom);
            static_cast<float*>(pool)[pi] = w;
            if (im && staging) static_cast<float*>(staging)[coff[c] + (pi - c * chunk)] = w;
        }
    }
}

// K2: fused pack + correction + compaction (+ exact norms of the unimportant chunks; of
// every chunk when staging is null: world 1, where the pool already holds the exchanged sums).
// U = 1 vector per thread per pass: 2 in flight spills at the 64-register cap (measured, AlexNet
// CSC N=1: 172 vs 152 us).
// 4 CTAs per SM (64 registers): measured best (AlexNet CSC: 154 us; 168 us at 78 registers
// and 3 CTAs per SM; 160 us at 5 CTAs per SM, which spills)
template <int DT, int U>
__global__ void __launch_bounds__(kThreads, 4)
pack_correct_kernel(const __grid_constant__ TensorTable T, void* __restrict__ pool,
                    float* __restrict__ hg, void* __restrict__ staging,
                    const uint8_t* __restrict__ imp, const uint64_t* __restrict__ coff,
                    uint64_t chunk, uint64_t nc, float mom, uint64_t total_tiles,
                    uint64_t* __restrict__ nacc, int part) {
    for (uint64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x)
        pack_correct_tile<DT, kThreads, U>(T, tile, pool, hg, staging, imp, coff, chunk, nc, mom, nacc, part);
}

// K2 part 1 driven by the plan: only the important chunks (plan[4 .. 4+plan[1])), each cut into
// kTile-element pieces walked by a persistent grid — its work is proportional to the staged data,
// where the tile-driven kernel visits (and skips) every tile of the gradient set. The tensor
// holding a pool element is found by binary search over the table's pool offsets, which the
// host checked to be descending (tensors in ascending id: tensor m at offset 0).
__device__ __forceinline__ int tensor_of(const TensorTable& T, uint64_t e) {
    int lo = 0, hi = T.n;  // first entry with off <= e (offsets descending)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (T.off[mid] <= e) hi = mid; else lo = mid + 1;
    }
    return (lo < T.n && e < T.off[lo] + T.cnt[lo]) ? lo : -1;
}

// Staging element s <-> pool element: s lies in important chunk q = min(s / chunk, k - 1) of the
// plan (the staging buffer holds the chunks packed ascending, all `chunk` long except the final
// pool chunk, which is last when selected).
__device__ __forceinline__ uint64_t staged_to_pool(const uint64_t* plan, uint64_t k, uint64_t chunk, uint64_t s) {
    const uint64_t q = min(s / chunk, k - 1);
    return plan[4 + q] * chunk + (s - q * chunk);
}

// Routing of staged elements to the owner of their exchange segment (gf_csc_pack_correct_routed):
// the planned windows over the staging index space (plan[2] windows of plan[3] elements, the
// last shorter) are split by segment_of (src/collectives.cpp:47-53); element s of segment j goes
// to my staging when j is my ring position, else into my slot of owner j's inbox (slot t of the
// owner at position j holds position j + 1 + t, the rspush layout). world == 0: no routing.
struct StageRoute {
    int world;
    uint16_t* dst_by_pos[GF_MAX_RANKS];  // where an element of segment j is stored (staging indices)
};

// owner position of staging element s, and the end of its segment
__device__ __forceinline__ int stage_owner(const StageRoute& R, const uint64_t* plan, uint64_t s, uint64_t& seg_end) {
    const uint64_t staged = plan[0], nwin = plan[2], stride = plan[3];
    const uint64_t w = min(s / stride, nwin - 1), ws = w * stride, wl = (w + 1 == nwin) ? staged - ws : stride;
    const uint64_t n = uint64_t(R.world), base = wl / n, rem = wl % n, off = s - ws, big = rem * (base + 1);
    const uint64_t j = off < big ? off / (base + 1) : rem + (off - big) / base;  // off >= big implies base > 0
    seg_end = ws + j * base + min(j, rem) + base + (j < rem ? 1 : 0);
    return int(j);
}

// The grid sweeps the staging index space [0, plan[0]) in 8-element vectors (kPlannedU per
// thread, every load in flight before the math); each vector maps to its pool element through
// the plan. Work is proportional to the staged data only.
constexpr int kPlannedU = 2;
template <int DT>
__global__ void __launch_bounds__(kThreads, 4)
pack_correct_planned_kernel(const __grid_constant__ TensorTable T, void* __restrict__ pool, float* __restrict__ hg,
                            void* __restrict__ staging, const uint64_t* __restrict__ plan, uint64_t chunk, float mom,
                            const __grid_constant__ StageRoute R) {
    const uint64_t staged = plan[0], k = plan[1];
    if (k == 0) return;
    const uint64_t nv = (staged + 7) / 8, G = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t v0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v0 < nv; v0 += G * kPlannedU) {
        gfd::F8 gv[kPlannedU], hv[kPlannedU];
        uint64_t pe[kPlannedU];
        bool fast[kPlannedU];
#pragma unroll
        for (int u = 0; u < kPlannedU; ++u) {
            const uint64_t v = v0 + uint64_t(u) * G, s = v * 8;
            fast[u] = false;
            pe[u] = 0;
            if (v >= nv) continue;
            const uint64_t e = staged_to_pool(plan, k, chunk, s);
            pe[u] = e;
            const int t = tensor_of(T, e);
            if (DT != GF_F16 || t < 0 || chunk % 8 != 0 || s + 8 > staged || e % 8 != 0 ||
                e + 8 > T.off[t] + T.cnt[t])
                continue;
            const float* src = static_cast<const float*>(T.ptr[t]) + (e - T.off[t]);
            if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(hg + e)) & 31u) != 0) continue;
            fast[u] = true;
            gv[u] = gfd::ld32f_stream(src);
            hv[u] = gfd::ld32f(hg + e);
        }
#pragma unroll
        for (int u = 0; u < kPlannedU; ++u) {
            const uint64_t v = v0 + uint64_t(u) * G;
            if (v >= nv) continue;
            if (fast[u]) {
                const uint64_t e = pe[u];
                float hn[8];
                uint4 ov;
                bool nan;
                correct8(gv[u], reinterpret_cast<const float*>(&hv[u]), true, mom, hn, ov, nan);
                gfd::st32f(hg + e, make_float4(hn[0], hn[1], hn[2], hn[3]), make_float4(hn[4], hn[5], hn[6], hn[7]));
                gfd::st16(static_cast<uint16_t*>(pool) + e, ov);
                if (R.world == 0) {
                    gfd::st16(static_cast<uint16_t*>(staging) + v * 8, ov);
                } else {
                    uint64_t seg_end;
                    const int j = stage_owner(R, plan, v * 8, seg_end);
                    if (v * 8 + 8 <= seg_end) {
                        gfd::st16(R.dst_by_pos[j] + v * 8, ov);
                    } else {  // a segment boundary inside the vector
                        const uint32_t w[4] = {ov.x, ov.y, ov.z, ov.w};
                        for (int q = 0; q < 8; ++q) {
                            uint64_t se;
                            const int jq = stage_owner(R, plan, v * 8 + q, se);
                            R.dst_by_pos[jq][v * 8 + q] = uint16_t((w[q >> 1] >> ((q & 1) * 16)) & 0xFFFFu);
                        }
                    }
                }
                continue;
            }
            for (uint64_t s = v * 8; s < min(v * 8 + 8, staged); ++s) {  // element by element
                const uint64_t q = staged_to_pool(plan, k, chunk, s);
                const int tq = tensor_of(T, q);
                if (tq < 0) continue;  // another table's tensor (more than 256 tensors)
                const float x = static_cast<const float*>(T.ptr[tq])[q - T.off[tq]];
                if (DT == GF_F16) {
                    const uint16_t w = gfd::enc(correct_elem(gfd::dec(gfd::enc(x)), hg + q, true, mom));
                    static_cast<uint16_t*>(pool)[q] = w;
                    if (R.world == 0) {
                        static_cast<uint16_t*>(staging)[s] = w;
                    } else {
                        uint64_t se;
                        R.dst_by_pos[stage_owner(R, plan, s, se)][s] = w;
                    }
                } else {
                    const float w = correct_elem(x, hg + q, true, mom);
                    static_cast<float*>(pool)[q] = w;
                    static_cast<float*>(staging)[s] = w;
                }
            }
        }
    }
}

// Staging pack (dir=0) / write-back (dir=1) over the important chunks listed in the plan
// (plan[4+j], j < plan[1]): grid.y walks the list, grid.x tiles a chunk; 16-B copies.
// On write-back of an fp16 pool, the exact |x| sums of the (now global) chunk values are
// accumulated into nacc — the norms of the important chunks, without re-reading the pool.
__global__ void compact_kernel(char* __restrict__ pool, char* __restrict__ staging,
                               const uint64_t* __restrict__ plan, const uint64_t* __restrict__ coff,
                               uint64_t total, uint64_t chunk, uint64_t nc, uint64_t esz, int dir,
                               uint64_t* __restrict__ nacc) {
    const uint64_t kc = plan[1];
    for (uint64_t j = blockIdx.y; j < kc; j += gridDim.y) {
        const uint64_t c = plan[4 + j];
        const uint64_t len = ((c + 1 == nc) ? total - c * chunk : chunk) * esz;
        char* p = pool + c * chunk * esz;
        char* s = staging + coff[c] * esz;
        const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(s)) & 15u) == 0;
        uint64_t done = 0, units = 0;
        bool nan = false;
        if (vec) {
            const uint64_t nv = len / 16;
            for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < nv;
                 v += uint64_t(gridDim.x) * blockDim.x) {
                if (dir == 0) {
                    gfd::st16(s + 16 * v, gfd::ld16_stream(p + 16 * v));
                } else {
                    const uint4 x = gfd::ld16_stream(s + 16 * v);
                    gfd::st16(p + 16 * v, x);
                    if (nacc) {
                        if (gfd::any_special(x)) nan = true; else units += units8(x);
                    }
                }
            }
            done = nv * 16;
        }
        for (uint64_t i = done + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < len;
             i += uint64_t(gridDim.x) * blockDim.x) {
            if (dir == 0) {
                s[i] = p[i];
            } else {
                p[i] = s[i];
                if (nacc && (i & 1)) {  // fp16: the element completes at its high byte
                    const uint16_t h = uint16_t(uint8_t(s[i - 1])) | (uint16_t(uint8_t(s[i])) << 8);
                    if ((h & 0x7C00u) == 0x7C00u) nan = true; else units += half_units(h);
                }
            }
        }
        if (nacc) {
            uint64_t v = units;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
            const bool an = __any_sync(0xFFFFFFFFu, nan);
            if ((threadIdx.x & 31) == 0) {
                if (v) atomicAdd(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)v);
                if (an) atomicOr(reinterpret_cast<unsigned long long*>(nacc + c), (unsigned long long)kNaccNaN);
            }
        }
    }
}

// CSC unpack + momentum update (sparse.cpp:206-224, csc_update sparse.hpp:42-51) over the
// important chunks of the plan: g = dec(pool)*(1/N); u = mom*hu + lr*g; hu = u; w -= u.
// kSgdU 8-element vectors per thread are loaded before any is updated (80 B each in flight):
// measured best at 1 with many short CTAs (AlexNet: 24.8 us; 28.4 us at 2 per thread).
constexpr int kSgdU = 1;
template <int DT>
__global__ void __launch_bounds__(256)
csc_sgd_kernel(const void* __restrict__ pool, const uint64_t* __restrict__ plan, uint64_t total,
               uint64_t chunk, uint64_t nc, float inv_world, float mom, float lr,
               float* __restrict__ hu, float* __restrict__ w) {
    const uint64_t kc = plan[1];
    for (uint64_t j = blockIdx.y; j < kc; j += gridDim.y) {
        const uint64_t c = plan[4 + j];
        const uint64_t b = c * chunk;
        const uint64_t len = (c + 1 == nc) ? total - b : chunk;
        uint64_t done = 0;
        if (DT == GF_F16 && b % 8 == 0 && (reinterpret_cast<uintptr_t>(pool) & 15u) == 0 &&
            (reinterpret_cast<uintptr_t>(hu) & 31u) == 0 &&
            (reinterpret_cast<uintptr_t>(w) & 31u) == 0) {
            const uint64_t nv = len / 8;
            const uint16_t* p = static_cast<const uint16_t*>(pool) + b;
            const uint64_t S = uint64_t(gridDim.x) * blockDim.x;
            for (uint64_t v0 = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v0 < nv; v0 += S * kSgdU) {
                uint4 x[kSgdU];  // every load of the kSgdU vectors in flight before any math
                gfd::F8 h[kSgdU], ww[kSgdU];
#pragma unroll
                for (int u = 0; u < kSgdU; ++u) {
                    const uint64_t v = v0 + uint64_t(u) * S;
                    if (v < nv) {
                        x[u] = gfd::ld16_stream(p + 8 * v);
                        h[u] = gfd::ld32f(hu + b + 8 * v);
                        ww[u] = gfd::ld32f(w + b + 8 * v);
                    }
                }
#pragma unroll
                for (int u = 0; u < kSgdU; ++u) {
                    const uint64_t v = v0 + uint64_t(u) * S;
                    if (v >= nv) continue;
                    float* hp = reinterpret_cast<float*>(&h[u]);
                    float* wp = reinterpret_cast<float*>(&ww[u]);
                    const uint32_t xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint16_t hv = uint16_t((xs[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu);
                        const float g = gfd::mul(gfd::dec(hv), inv_world);
                        const float uu = gfd::add(gfd::mul(mom, hp[k]), gfd::mul(lr, g));
                        hp[k] = uu;
                        wp[k] = gfd::sub(wp[k], uu);
                    }
                    gfd::st32f(hu + b + 8 * v, h[u].lo, h[u].hi);
                    gfd::st32f(w + b + 8 * v, ww[u].lo, ww[u].hi);
                }
            }
            done = nv * 8;
        }
        for (uint64_t i = b + done + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < b + len;
             i += uint64_t(gridDim.x) * blockDim.x) {
            const float x = DT == GF_F16 ? gfd::dec(static_cast<const uint16_t*>(pool)[i])
                                         : static_cast<const float*>(pool)[i];
            const float g = gfd::mul(x, inv_world);
            const float u = gfd::add(gfd::mul(mom, hu[i]), gfd::mul(lr, g));
            hu[i] = u;
            w[i] = gfd::sub(w[i], u);
        }
    }
}

__global__ void __launch_bounds__(gfs::kSelThreads)
select_plan_kernel(const float* __restrict__ norms, uint64_t nc, uint64_t k, uint8_t* flags,
                   int do_select, uint64_t total, uint64_t chunk, uint64_t esz, uint64_t theta,
                   uint64_t* coff, uint64_t* plan) {
    __shared__ gfs::SelShared sh;
    if (do_select) gfs::block_topk(norms, nc, k, flags, sh);
    __syncthreads();
    if (coff && plan) gfs::block_plan(flags, total, chunk, nc, esz, theta, coff, plan, sh);
}

int grid_y(uint64_t max_chunks, uint64_t nc) {
    return int(std::max<uint64_t>(1, std::min<uint64_t>(std::min(max_chunks, nc), 65535)));
}

int compact_launch(int dtype, void* pool, const void* staging, const uint64_t* plan,
                   const uint64_t* coff, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t max_chunks, int dir, uint64_t* nacc, void* stream) {
    if (nacc && dtype != GF_F16) return gfi::fail(GF_ERR_CONFIG, "exact norm accumulation needs an fp16 pool");
    if (!gfi::valid_dtype(dtype) || chunk == 0 || nc == 0 || !plan || !coff)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_compact/scatter: bad arguments");
    const uint64_t bytes = std::max<uint64_t>(chunk, total - (nc - 1) * chunk) * gfi::esz(dtype);
    // one 1024-thread CTA per 64 KB of chunk: 4 x 16 B per thread, one wave for k ~ 2 x #SMs
    const int gx = int(std::max<uint64_t>(1, std::min<uint64_t>((bytes + 65535) / 65536, 64)));
    compact_kernel<<<dim3(gx, grid_y(max_chunks, nc)), 1024, 0, gfi::S(stream)>>>(
        static_cast<char*>(pool), static_cast<char*>(const_cast<void*>(staging)), plan, coff,
        total, chunk, nc, gfi::esz(dtype), dir, nacc);
    gfi::count_launch();
    return gfi::check_launch("gf_csc_compact");
}

}  // namespace

extern "C" {

int gf_chunk_norms(int dtype, const void* pool, uint64_t total, uint64_t chunk, uint64_t nc,
                   const uint8_t* important, int world, float* norms, void* stream) {
    if (!gfi::valid_dtype(dtype) || chunk == 0 || nc == 0 || world < 1 || (nc - 1) * chunk >= total)
        return gfi::fail(GF_ERR_CONFIG, "gf_chunk_norms: bad arguments");
    const float inv = 1.0f / static_cast<float>(world);
    const int grid = int(std::min<uint64_t>(nc, uint64_t(gfi::sm_count()) * 16));
    if (dtype == GF_F16)
        norms_f16_kernel<<<grid, kNormThreads, 0, gfi::S(stream)>>>(
            static_cast<const uint16_t*>(pool), total, chunk, nc, important, inv, norms);
    else
        norms_f32_kernel<<<grid, kNormThreads, 0, gfi::S(stream)>>>(
            static_cast<const float*>(pool), total, chunk, nc, important, inv, norms);
    gfi::count_launch();
    return gfi::check_launch("gf_chunk_norms");
}

int gf_csc_correct(int dtype, void* pool, float* hg, const uint8_t* important, uint64_t total,
                   uint64_t chunk, uint64_t nc, uint64_t first_chunk, uint64_t num_chunks,
                   float momentum, void* stream) {
    if (!gfi::valid_dtype(dtype) || chunk == 0 || nc == 0 || first_chunk + num_chunks > nc)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_correct: chunk range out of bounds");
    if (num_chunks == 0) return GF_OK;
    const uint64_t begin = first_chunk * chunk;
    const uint64_t end = (first_chunk + num_chunks == nc) ? total : (first_chunk + num_chunks) * chunk;
    const uint64_t n = end - begin;
    const int grid = grid_for(n, 256);
    if (dtype == GF_F16)
        correct_kernel<GF_F16><<<grid, 256, 0, gfi::S(stream)>>>(pool, hg, important, total, chunk, nc, begin, end, momentum);
    else
        correct_kernel<GF_F32><<<grid, 256, 0, gfi::S(stream)>>>(pool, hg, important, total, chunk, nc, begin, end, momentum);
    gfi::count_launch();
    return gfi::check_launch("gf_csc_correct");
}

int gf_csc_pack_correct(int dtype, void* pool, float* hg, void* staging,
                        const uint8_t* important, const uint64_t* coff, uint64_t total,
                        uint64_t chunk, uint64_t nc, const float* const* src,
                        const uint64_t* pool_off, const uint64_t* count, int ntensors,
                        float momentum, uint64_t* nacc, void* stream) {
    return gf_csc_pack_correct_part(dtype, pool, hg, staging, important, coff, nullptr, total, chunk, nc, src,
                                    pool_off, count, ntensors, momentum, nacc, 0, stream);
}

int gf_csc_pack_correct_part(int dtype, void* pool, float* hg, void* staging,
                             const uint8_t* important, const uint64_t* coff, const uint64_t* plan,
                             uint64_t total, uint64_t chunk, uint64_t nc, const float* const* src,
                             const uint64_t* pool_off, const uint64_t* count, int ntensors,
                             float momentum, uint64_t* nacc, int part, void* stream) {
    if (part < 0 || part > 2) return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct_part: part is 0, 1 or 2");
    if (!gfi::valid_dtype(dtype) || chunk == 0 || nc == 0 || !pool || !hg || !important)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct: bad arguments");
    if (nacc && dtype != GF_F16) return gfi::fail(GF_ERR_CONFIG, "exact norm accumulation needs an fp16 pool");
    if (staging && !coff) return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct: staging needs coff");
    bool descending = true;
    for (int i = 1; i < ntensors; ++i) descending &= pool_off[i] < pool_off[i - 1];
    if (part == 1 && plan && staging && descending) {  // the plan-driven form
        return for_each_table(reinterpret_cast<const void* const*>(src), pool_off, count, ntensors,
                              [&](const TensorTable& T, uint64_t, int) {
                                  const int g = gfi::sm_count() * 4;
                                  if (dtype == GF_F16)
                                      pack_correct_planned_kernel<GF_F16><<<g, kThreads, 0, gfi::S(stream)>>>(
                                          T, pool, hg, staging, plan, chunk, momentum, StageRoute{});
                                  else
                                      pack_correct_planned_kernel<GF_F32><<<g, kThreads, 0, gfi::S(stream)>>>(
                                          T, pool, hg, staging, plan, chunk, momentum, StageRoute{});
                              });
    }
    return for_each_table(reinterpret_cast<const void* const*>(src), pool_off, count, ntensors,
                          [&](const TensorTable& T, uint64_t tiles, int grid) {
                              // part 1 skips most tiles: a persistent grid (4 CTAs per SM) walks
                              // them; part 2 keeps one tile per CTA, so the exchange running
                              // beside it gets SMs as CTAs retire
                              if (part == 1) grid = std::min(grid, gfi::sm_count() * 4);
                              if (dtype == GF_F16)
                                  pack_correct_kernel<GF_F16, 1><<<grid, kThreads, 0, gfi::S(stream)>>>(
                                      T, pool, hg, staging, important, coff, chunk, nc, momentum, tiles, nacc, part);
                              else
                                  pack_correct_kernel<GF_F32, 1><<<grid, kThreads, 0, gfi::S(stream)>>>(
                                      T, pool, hg, staging, important, coff, chunk, nc, momentum, tiles, nacc, part);
                          });
}

int gf_csc_pack_correct_routed(gf_comm* c, void* pool, float* hg, uint64_t stage_heap_off, const uint64_t* plan,
                               uint64_t chunk, const float* const* src, const uint64_t* pool_off, const uint64_t* count,
                               int ntensors, float momentum, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (c->csc_inbox_off == UINT64_MAX)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct_routed: no CSC inbox (gf_comm_set_csc_inbox)");
    if (!pool || !hg || !plan || !src || !pool_off || !count || ntensors < 1 || chunk == 0 || chunk % 8 != 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct_routed: fp16, chunk % 8 == 0, >= 1 tensor");
    uint64_t span = 0;
    for (int i = 0; i < ntensors; ++i) {
        if (i > 0 && pool_off[i] >= pool_off[i - 1])
            return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct_routed: tensors in ascending id (descending offsets)");
        span = std::max(span, pool_off[i] + count[i]);
    }
    if (span > c->csc_slot_elems)  // every staged element must fit an inbox slot
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct_routed: the pool is larger than the CSC inbox slots");
    if (stage_heap_off % 16 != 0 || stage_heap_off + c->csc_slot_elems * 2 > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_pack_correct_routed: staging outside the heap or not 16-B aligned");
    StageRoute R;
    std::memset(&R, 0, sizeof(R));
    R.world = c->world;
    for (int j = 0; j < c->world; ++j) {
        char* base = c->peer_alloc[c->ring[j]] + kFlagBytes;
        R.dst_by_pos[j] = j == c->pos ? reinterpret_cast<uint16_t*>(c->alloc + kFlagBytes + stage_heap_off)
                                      : reinterpret_cast<uint16_t*>(base + c->csc_inbox_off) +
                                            uint64_t((c->pos - j - 1 + c->world) % c->world) * c->csc_slot_elems;
    }
    DeviceGuard g(c->device);
    void* staging = c->alloc + kFlagBytes + stage_heap_off;
    return for_each_table(reinterpret_cast<const void* const*>(src), pool_off, count, ntensors,
                          [&](const TensorTable& T, uint64_t, int) {
                              pack_correct_planned_kernel<GF_F16><<<gfi::sm_count() * 4, kThreads, 0, gfi::S(stream)>>>(
                                  T, pool, hg, staging, plan, chunk, momentum, R);
                          });
}

int gf_csc_compact(int dtype, const void* pool, void* staging, const uint64_t* plan,
                   const uint64_t* coff, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t max_chunks, void* stream) {
    return compact_launch(dtype, const_cast<void*>(pool), staging, plan, coff, total, chunk, nc,
                          max_chunks, 0, nullptr, stream);
}

int gf_csc_scatter(int dtype, void* pool, const void* staging, const uint64_t* plan,
                   const uint64_t* coff, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t max_chunks, uint64_t* nacc, void* stream) {
    return compact_launch(dtype, pool, staging, plan, coff, total, chunk, nc, max_chunks, 1, nacc,
                          stream);
}

int gf_csc_sgd_update(int dtype, const void* pool, const uint64_t* plan, uint64_t total,
                      uint64_t chunk, uint64_t nc, uint64_t max_chunks, int world, float momentum,
                      float lr, float* hu, float* w, void* stream) {
    if (!gfi::valid_dtype(dtype) || world < 1 || chunk == 0 || nc == 0 || !plan)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_sgd_update: bad arguments");
    if (total == 0) return GF_OK;
    const float inv = 1.0f / static_cast<float>(world);
    const uint64_t longest = std::max<uint64_t>(chunk, total - (nc - 1) * chunk);
    const int gx = int(std::max<uint64_t>(1, std::min<uint64_t>((longest / 8 + 256 * kSgdU - 1) / (256 * kSgdU), 64)));
    const dim3 grid(gx, grid_y(max_chunks, nc));
    if (dtype == GF_F16)
        csc_sgd_kernel<GF_F16><<<grid, 256, 0, gfi::S(stream)>>>(pool, plan, total, chunk, nc, inv, momentum, lr, hu, w);
    else
        csc_sgd_kernel<GF_F32><<<grid, 256, 0, gfi::S(stream)>>>(pool, plan, total, chunk, nc, inv, momentum, lr, hu, w);
    gfi::count_launch();
    return gfi::check_launch("gf_csc_sgd_update");
}

int gf_csc_plan(const uint8_t* important, uint64_t total, uint64_t chunk, uint64_t nc,
                int dtype, uint64_t theta, uint64_t* coff, uint64_t* plan, void* stream) {
    if (!gfi::valid_dtype(dtype) || chunk == 0 || nc == 0 || !coff || !plan)
        return gfi::fail(GF_ERR_CONFIG, "gf_csc_plan: bad arguments");
    select_plan_kernel<<<1, gfs::kSelThreads, 0, gfi::S(stream)>>>(
        nullptr, nc, 0, const_cast<uint8_t*>(important), 0, total, chunk, gfi::esz(dtype), theta,
        coff, plan);
    gfi::count_launch();
    return gfi::check_launch("gf_csc_plan");
}

int gf_select_topk(const float* norms, uint64_t nc, uint64_t k, uint8_t* flags, void* stream) {
    if (nc == 0 || k == 0) return gfi::fail(GF_ERR_CONFIG, "gf_select_topk: empty selection");
    select_plan_kernel<<<1, gfs::kSelThreads, 0, gfi::S(stream)>>>(
        norms, nc, k, flags, 1, 0, 1, 2, 0, nullptr, nullptr);
    gfi::count_launch();
    return gfi::check_launch("gf_select_topk");
}

}  // extern "C"
