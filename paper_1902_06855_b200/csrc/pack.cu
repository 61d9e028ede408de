// SPDX-License-Identifier: Apache-2.0
//
// K1 pack (fp32 per-layer gradients -> fp16/fp32 fusion pool) and K6 unpack
// (pool -> fp32 per-layer g_avg = dec(pool) * 1/N), plus the elementwise codec,
// accumulate and momentum-SGD kernels.
//
// Reference: GradientPool::write_tensor (src/gradient_pool.cpp:78-105) does one
// ScalarBuffer::set per element (a software float_to_half_bits, half.hpp:20-59);
// the dense update loop (src/trainer.cpp:332-347) reads get(i) * inv_world.
// Here all tensors of a call go out in ONE launch: a tensor table in kernel
// parameter space, 8192-element tiles per CTA iteration, 128-bit loads/stores
// (two float4 -> one 16-B fp16 vector), streaming cache hints on data read once.
// HBM roofline: 6 B/element (4 read + 2 write) for pack and unpack.

#include <algorithm>
#include <type_traits>
#include <vector>

#include "gf_device.cuh"
#include "gf_internal.cuh"
#include "tensor_table.cuh"

namespace {

__device__ __forceinline__ float scaled(float g, float scale, bool do_scale) {
    return do_scale ? gfd::mul(g, scale) : g;
}

// ---- K1: pack (and, at world == 1, K1+K6 in one pass) ------------------------------
// Dst = NoDst: pack only. Dst = DstTable: world == 1, where the collective is the identity
// (src/collectives.cpp:59), so g_avg = dec(enc(g)) * 1/1 is written from the registers that
// hold the packed value: one HBM pass of 10 B/element instead of pack + unpack's 12.
struct NoDst {};
struct DstTable {
    float* ptr[kMaxT];
};

__device__ __forceinline__ void store_avg8(float* o, const uint4 h, float inv) {
    if (!gfd::any_special(h)) {
        const float2 g0 = gfd::h2f2(h.x), g1 = gfd::h2f2(h.y), g2 = gfd::h2f2(h.z), g3 = gfd::h2f2(h.w);
        gfd::st32f_stream(o, make_float4(__fmul_rn(g0.x, inv), __fmul_rn(g0.y, inv), __fmul_rn(g1.x, inv),
                                         __fmul_rn(g1.y, inv)),
                          make_float4(__fmul_rn(g2.x, inv), __fmul_rn(g2.y, inv), __fmul_rn(g3.x, inv),
                                      __fmul_rn(g3.y, inv)));
    } else {
        const uint32_t w[4] = {h.x, h.y, h.z, h.w};
        float r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = gfd::mul(gfd::dec(uint16_t((w[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu)), inv);
        gfd::st32f_stream(o, make_float4(r[0], r[1], r[2], r[3]), make_float4(r[4], r[5], r[6], r[7]));
    }
}

template <int DT, class Dst>
__global__ void __launch_bounds__(kThreads) pack_kernel(const __grid_constant__ TensorTable T,
                                                        const __grid_constant__ Dst D,
                                                        void* __restrict__ pool, float scale,
                                                        float inv_world, uint64_t total_tiles) {
    constexpr bool SOLO = std::is_same<Dst, DstTable>::value;
    const bool do_scale = scale != 1.0f;
    for (uint64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int t = find_tensor(T, tile);
        const uint64_t base = (tile - T.tiles[t]) * kTile;
        const uint64_t len = min(kTile, T.cnt[t] - base);
        const float* __restrict__ s = static_cast<const float*>(T.ptr[t]) + base;
        float* __restrict__ o = nullptr;
        if constexpr (SOLO) o = D.ptr[t] + base;
        const uint64_t po = T.off[t] + base;
        const bool fast = ((reinterpret_cast<uintptr_t>(T.ptr[t]) & 31u) == 0) && (po % 8 == 0) &&
                          ((reinterpret_cast<uintptr_t>(pool) & 15u) == 0) &&
                          (!SOLO || (reinterpret_cast<uintptr_t>(o) & 31u) == 0);
        if (DT == GF_F16) {
            uint16_t* __restrict__ d = static_cast<uint16_t*>(pool) + po;
            uint64_t done = 0;
            if (fast) {
                const int nvec = int(len / 8);
                float4 a[kVecPerThread], b[kVecPerThread];
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) {
                    const int v = threadIdx.x + k * kThreads;
                    if (v < nvec) {
                        const gfd::F8 f = gfd::ld32f_stream(s + 8 * v);  // LDG.E.256
                        a[k] = f.lo;
                        b[k] = f.hi;
                    }
                }
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) {
                    const int v = threadIdx.x + k * kThreads;
                    if (v < nvec) {
                        if (do_scale) {
                            a[k] = make_float4(gfd::mul(a[k].x, scale), gfd::mul(a[k].y, scale),
                                               gfd::mul(a[k].z, scale), gfd::mul(a[k].w, scale));
                            b[k] = make_float4(gfd::mul(b[k].x, scale), gfd::mul(b[k].y, scale),
                                               gfd::mul(b[k].z, scale), gfd::mul(b[k].w, scale));
                        }
                        const uint4 h = gfd::enc8(a[k], b[k]);
                        if constexpr (SOLO) {
                            gfd::st16(d + 8 * v, h);
                            store_avg8(o + 8 * v, h, inv_world);
                        } else {
                            gfd::st16_keep(d + 8 * v, h);  // the collective / unpack reads it next
                        }
                    }
                }
                done = uint64_t(nvec) * 8;
            }
            for (uint64_t i = done + threadIdx.x; i < len; i += kThreads) {
                const uint16_t h = gfd::enc(scaled(s[i], scale, do_scale));
                d[i] = h;
                if constexpr (SOLO) o[i] = gfd::mul(gfd::dec(h), inv_world);
            }
        } else {
            float* __restrict__ d = static_cast<float*>(pool) + po;
            uint64_t done = 0;
            if (fast) {
                const int nvec = int(len / 4);
                for (int v = threadIdx.x; v < nvec; v += kThreads) {
                    float4 x = gfd::ld16f_stream(s + 4 * v);
                    if (do_scale) {
                        x.x = gfd::mul(x.x, scale); x.y = gfd::mul(x.y, scale);
                        x.z = gfd::mul(x.z, scale); x.w = gfd::mul(x.w, scale);
                    }
                    *reinterpret_cast<float4*>(d + 4 * v) = x;
                    if constexpr (SOLO) {
                        __stcs(reinterpret_cast<float4*>(o + 4 * v),
                               make_float4(gfd::mul(x.x, inv_world), gfd::mul(x.y, inv_world),
                                           gfd::mul(x.z, inv_world), gfd::mul(x.w, inv_world)));
                    }
                }
                done = uint64_t(nvec) * 4;
            }
            for (uint64_t i = done + threadIdx.x; i < len; i += kThreads) {
                const float x = scaled(s[i], scale, do_scale);
                d[i] = x;
                if constexpr (SOLO) o[i] = gfd::mul(x, inv_world);
            }
        }
    }
}

// ---- K6: unpack ----------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(kThreads) unpack_kernel(const __grid_constant__ TensorTable T,
                                                          const void* __restrict__ pool,
                                                          float inv_world, uint64_t total_tiles) {
    for (uint64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int t = find_tensor(T, tile);
        const uint64_t base = (tile - T.tiles[t]) * kTile;
        const uint64_t len = min(kTile, T.cnt[t] - base);
        float* __restrict__ d = static_cast<float*>(const_cast<void*>(T.ptr[t])) + base;
        const uint64_t po = T.off[t] + base;
        const bool fast = ((reinterpret_cast<uintptr_t>(T.ptr[t]) & 31u) == 0) && (po % 8 == 0) &&
                          ((reinterpret_cast<uintptr_t>(pool) & 15u) == 0);
        uint64_t done = 0;
        if (DT == GF_F16) {
            const uint16_t* __restrict__ s = static_cast<const uint16_t*>(pool) + po;
            if (fast) {
                const int nvec = int(len / 8);
                uint4 x[kVecPerThread];
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) {
                    const int v = threadIdx.x + k * kThreads;
                    if (v < nvec) x[k] = gfd::ld16_stream(s + 8 * v);
                }
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) {
                    const int v = threadIdx.x + k * kThreads;
                    if (v < nvec && !gfd::any_special(x[k])) {
                        // fast path: finite halves, x * (1/N) cannot produce NaN
                        const float2 f0 = gfd::h2f2(x[k].x), f1 = gfd::h2f2(x[k].y);
                        const float2 f2 = gfd::h2f2(x[k].z), f3 = gfd::h2f2(x[k].w);
                        gfd::st32f_stream(d + 8 * v,  // STG.E.256
                               make_float4(__fmul_rn(f0.x, inv_world), __fmul_rn(f0.y, inv_world),
                                           __fmul_rn(f1.x, inv_world), __fmul_rn(f1.y, inv_world)),
                               make_float4(__fmul_rn(f2.x, inv_world), __fmul_rn(f2.y, inv_world),
                                           __fmul_rn(f3.x, inv_world), __fmul_rn(f3.y, inv_world)));
                    } else if (v < nvec) {
                        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x[k]);
                        float4 lo, hi;
                        lo.x = gfd::mul(gfd::dec(uint16_t(w[0] & 0xFFFF)), inv_world);
                        lo.y = gfd::mul(gfd::dec(uint16_t(w[0] >> 16)), inv_world);
                        lo.z = gfd::mul(gfd::dec(uint16_t(w[1] & 0xFFFF)), inv_world);
                        lo.w = gfd::mul(gfd::dec(uint16_t(w[1] >> 16)), inv_world);
                        hi.x = gfd::mul(gfd::dec(uint16_t(w[2] & 0xFFFF)), inv_world);
                        hi.y = gfd::mul(gfd::dec(uint16_t(w[2] >> 16)), inv_world);
                        hi.z = gfd::mul(gfd::dec(uint16_t(w[3] & 0xFFFF)), inv_world);
                        hi.w = gfd::mul(gfd::dec(uint16_t(w[3] >> 16)), inv_world);
                        gfd::st32f_stream(d + 8 * v, lo, hi);
                    }
                }
                done = uint64_t(nvec) * 8;
            }
            for (uint64_t i = done + threadIdx.x; i < len; i += kThreads) {
                d[i] = gfd::mul(gfd::dec(s[i]), inv_world);
            }
        } else {
            const float* __restrict__ s = static_cast<const float*>(pool) + po;
            if (fast) {
                const int nvec = int(len / 4);
                for (int v = threadIdx.x; v < nvec; v += kThreads) {
                    float4 x = *reinterpret_cast<const float4*>(s + 4 * v);
                    x.x = gfd::mul(x.x, inv_world); x.y = gfd::mul(x.y, inv_world);
                    x.z = gfd::mul(x.z, inv_world); x.w = gfd::mul(x.w, inv_world);
                    __stcs(reinterpret_cast<float4*>(d + 4 * v), x);
                }
                done = uint64_t(nvec) * 4;
            }
            for (uint64_t i = done + threadIdx.x; i < len; i += kThreads) {
                d[i] = gfd::mul(s[i], inv_world);
            }
        }
    }
}

// ---- elementwise ----------------------------------------------------------------
__global__ void encode_kernel(const float* __restrict__ s, uint16_t* __restrict__ d, uint64_t n,
                              float scale) {
    const bool do_scale = scale != 1.0f;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        d[i] = gfd::enc(scaled(s[i], scale, do_scale));
    }
}
__global__ void decode_kernel(const uint16_t* __restrict__ s, float* __restrict__ d, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        d[i] = gfd::dec(s[i]);
    }
}
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__global__ void digest_kernel(uint64_t first, uint64_t count, unsigned long long* out) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t b = uint32_t(first + i);
        acc += splitmix64((uint64_t(b) << 16) | gfd::enc(gfd::u2f(b)));
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}
template <int DT>
__global__ void accumulate_kernel(void* __restrict__ dst, const void* __restrict__ src, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (DT == GF_F16) {
            uint16_t* d = static_cast<uint16_t*>(dst);
            d[i] = gfd::acc16(d[i], static_cast<const uint16_t*>(src)[i]);
        } else {
            float* d = static_cast<float*>(dst);
            d[i] = gfd::add(d[i], static_cast<const float*>(src)[i]);
        }
    }
}

// trainer.cpp:337-346 / csc_update (sparse.hpp:42-51):
//   g = get(i)*inv ; u = mom*hu + lr*g ; hu = u ; w -= u
template <int DT>
__device__ __forceinline__ void sgd_elem(const void* pool, uint64_t i, float inv_world, float mom,
                                         float lr, float* hu, float* w) {
    const float x = DT == GF_F16 ? gfd::dec(static_cast<const uint16_t*>(pool)[i])
                                 : static_cast<const float*>(pool)[i];
    const float g = gfd::mul(x, inv_world);
    const float u = gfd::add(gfd::mul(mom, hu[i]), gfd::mul(lr, g));
    hu[i] = u;
    w[i] = gfd::sub(w[i], u);
}
// vec (fp16, pool 16-B and hu/w 32-B aligned): 8 elements per thread step — one 16-byte pool load
// and 32-byte hu/w loads/stores — with the per-element recurrence of sgd_elem; the tail scalar.
template <int DT>
__global__ void dense_sgd_kernel(const void* __restrict__ pool, uint64_t total, float inv_world,
                                 float mom, float lr, float* __restrict__ hu, float* __restrict__ w, int vec) {
    const uint64_t T = uint64_t(gridDim.x) * blockDim.x, g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nvec = (DT == GF_F16 && vec) ? total / 8 : 0;
    if constexpr (DT == GF_F16) for (uint64_t v = g; v < nvec; v += T) {
        const uint4 x = gfd::ld16_stream(static_cast<const uint16_t*>(pool) + 8 * v);
        gfd::F8 h = gfd::ld32f(hu + 8 * v), ww = gfd::ld32f(w + 8 * v);
        float* hp = reinterpret_cast<float*>(&h);
        float* wp = reinterpret_cast<float*>(&ww);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float gk = gfd::mul(gfd::dec(uint16_t((xs[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu)), inv_world);
            const float u = gfd::add(gfd::mul(mom, hp[k]), gfd::mul(lr, gk));
            hp[k] = u;
            wp[k] = gfd::sub(wp[k], u);
        }
        gfd::st32f(hu + 8 * v, h.lo, h.hi);
        gfd::st32f(w + 8 * v, ww.lo, ww.hi);
    }
    for (uint64_t i = nvec * 8 + g; i < total; i += T) sgd_elem<DT>(pool, i, inv_world, mom, lr, hu, w);
}
}  // namespace

extern "C" {

int gf_pack(int dtype, void* pool, const float* const* src, const uint64_t* pool_off,
            const uint64_t* count, int ntensors, float scale, void* stream) {
    if (!gfi::valid_dtype(dtype)) return gfi::fail(GF_ERR_CONFIG, "gf_pack: bad dtype");
    if (!pool && ntensors > 0) return gfi::fail(GF_ERR_CONFIG, "gf_pack: null pool");
    return for_each_table(reinterpret_cast<const void* const*>(src), pool_off, count, ntensors,
                          [&](const TensorTable& T, uint64_t tiles, int grid) {
                              if (dtype == GF_F16)
                                  pack_kernel<GF_F16, NoDst><<<grid, kThreads, 0, gfi::S(stream)>>>(T, NoDst{}, pool, scale, 1.0f, tiles);
                              else
                                  pack_kernel<GF_F32, NoDst><<<grid, kThreads, 0, gfi::S(stream)>>>(T, NoDst{}, pool, scale, 1.0f, tiles);
                          });
}

}  // extern "C"

namespace gfi {
int pack_unpack_solo(int dtype, void* pool, const float* const* src, float* const* dst,
                     const uint64_t* pool_off, const uint64_t* count, int ntensors, cudaStream_t stream) {
    if (!valid_dtype(dtype)) return fail(GF_ERR_CONFIG, "pack_unpack: bad dtype");
    if (!pool && ntensors > 0) return fail(GF_ERR_CONFIG, "pack_unpack: null pool");
    for (int t = 0; t < ntensors; ++t)
        if (count[t] && !dst[t]) return fail(GF_ERR_CONFIG, "pack_unpack: null output tensor");
    return for_each_table(reinterpret_cast<const void* const*>(src), pool_off, count, ntensors,
                          [&](const TensorTable& T, uint64_t tiles, int grid, int first) {
                              DstTable D{};
                              for (int t = first, j = 0; j < T.n; ++t)
                                  if (count[t]) D.ptr[j++] = dst[t];
                              if (dtype == GF_F16)
                                  pack_kernel<GF_F16, DstTable><<<grid, kThreads, 0, stream>>>(T, D, pool, 1.0f, 1.0f, tiles);
                              else
                                  pack_kernel<GF_F32, DstTable><<<grid, kThreads, 0, stream>>>(T, D, pool, 1.0f, 1.0f, tiles);
                          });
}
}  // namespace gfi

extern "C" {

int gf_unpack(int dtype, const void* pool, float* const* dst, const uint64_t* pool_off,
              const uint64_t* count, int ntensors, int world, void* stream) {
    if (!gfi::valid_dtype(dtype)) return gfi::fail(GF_ERR_CONFIG, "gf_unpack: bad dtype");
    if (world < 1) return gfi::fail(GF_ERR_CONFIG, "gf_unpack: world must be >= 1");
    const float inv_world = 1.0f / static_cast<float>(world);
    return for_each_table(reinterpret_cast<const void* const*>(dst), pool_off, count, ntensors,
                          [&](const TensorTable& T, uint64_t tiles, int grid) {
                              if (dtype == GF_F16)
                                  unpack_kernel<GF_F16><<<grid, kThreads, 0, gfi::S(stream)>>>(T, pool, inv_world, tiles);
                              else
                                  unpack_kernel<GF_F32><<<grid, kThreads, 0, gfi::S(stream)>>>(T, pool, inv_world, tiles);
                          });
}

int gf_encode_f16(const float* src, uint16_t* dst, uint64_t n, float scale, void* stream) {
    if (n == 0) return GF_OK;
    encode_kernel<<<grid_for(n, 256), 256, 0, gfi::S(stream)>>>(src, dst, n, scale);
    gfi::count_launch();
    return gfi::check_launch("gf_encode_f16");
}

int gf_decode_f16(const uint16_t* src, float* dst, uint64_t n, void* stream) {
    if (n == 0) return GF_OK;
    decode_kernel<<<grid_for(n, 256), 256, 0, gfi::S(stream)>>>(src, dst, n);
    gfi::count_launch();
    return gfi::check_launch("gf_decode_f16");
}

int gf_codec_digest(uint64_t first, uint64_t count, uint64_t* digest_dev, void* stream) {
    if (count == 0) return GF_OK;
    digest_kernel<<<gfi::sm_count() * 8, 256, 0, gfi::S(stream)>>>(
        first, count, reinterpret_cast<unsigned long long*>(digest_dev));
    gfi::count_launch();
    return gfi::check_launch("gf_codec_digest");
}

int gf_accumulate(int dtype, void* dst, const void* src, uint64_t n, void* stream) {
    if (!gfi::valid_dtype(dtype)) return gfi::fail(GF_ERR_CONFIG, "gf_accumulate: bad dtype");
    if (n == 0) return GF_OK;
    if (dtype == GF_F16)
        accumulate_kernel<GF_F16><<<grid_for(n, 256), 256, 0, gfi::S(stream)>>>(dst, src, n);
    else
        accumulate_kernel<GF_F32><<<grid_for(n, 256), 256, 0, gfi::S(stream)>>>(dst, src, n);
    gfi::count_launch();
    return gfi::check_launch("gf_accumulate");
}

int gf_dense_sgd_update(int dtype, const void* pool, uint64_t total, int world, float momentum,
                        float lr, float* hu, float* w, void* stream) {
    if (!gfi::valid_dtype(dtype) || world < 1)
        return gfi::fail(GF_ERR_CONFIG, "gf_dense_sgd_update: bad arguments");
    if (total == 0) return GF_OK;
    const float inv = 1.0f / static_cast<float>(world);
    if (dtype == GF_F16)
        dense_sgd_kernel<GF_F16><<<grid_for((total + 7) / 8, 256), 256, 0, gfi::S(stream)>>>(
            pool, total, inv, momentum, lr, hu, w,
            ((reinterpret_cast<uintptr_t>(pool) & 15u) | ((reinterpret_cast<uintptr_t>(hu) | reinterpret_cast<uintptr_t>(w)) & 31u)) == 0);
    else
        dense_sgd_kernel<GF_F32><<<grid_for(total, 256), 256, 0, gfi::S(stream)>>>(pool, total, inv, momentum, lr, hu, w, 0);
    gfi::count_launch();
    return gfi::check_launch("gf_dense_sgd_update");
}

}  // extern "C"

// ---- rooted helpers for the host-orchestrated oracle/broadcast collectives ---------------
// The peer-mapped buffers travel in kernel parameter space (no device pointer array, no
// allocation per call). fp16/fp32 sums go 16 bytes at a time when every buffer is 16-byte
// aligned, with the same per-element operation and operand order as the scalar form.
namespace {
struct RankPtrs {
    char* p[GF_MAX_RANKS];
};
bool all_aligned16(void* const* bufs, int n) {
    for (int r = 0; r < n; ++r)
        if ((reinterpret_cast<uintptr_t>(bufs[r]) & 15u) != 0) return false;
    return true;
}

// oracle_allreduce (collectives.cpp:203-226): rank 0 accumulates ranks 1..N-1 in order, then
// every rank gets the sum. vec: elements [0, nvec*VE) as 16-byte vectors, the rest scalar.
template <int DT>
__global__ void oracle_sum_kernel(const __grid_constant__ RankPtrs B, int world, uint64_t len, int vec) {
    constexpr int VE = DT == GF_F16 ? 8 : 4;
    const uint64_t T = uint64_t(gridDim.x) * blockDim.x, g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nvec = vec ? len / VE : 0;
    for (uint64_t v = g; v < nvec; v += T) {
        uint4 acc = gfd::ld16(B.p[0] + v * 16);
        for (int r = 1; r < world; ++r) {
            const uint4 x = gfd::ld16(B.p[r] + v * 16);
            acc = DT == GF_F16 ? gfd::acc16x8(acc, x) : gfd::acc32x4(acc, x);  // acc16(acc, x) per element
        }
        for (int r = 0; r < world; ++r) gfd::st16(B.p[r] + v * 16, acc);
    }
    for (uint64_t i = nvec * VE + g; i < len; i += T) {
        if (DT == GF_F16) {
            uint16_t acc = reinterpret_cast<const uint16_t*>(B.p[0])[i];
            for (int r = 1; r < world; ++r) acc = gfd::acc16(acc, reinterpret_cast<const uint16_t*>(B.p[r])[i]);
            for (int r = 0; r < world; ++r) reinterpret_cast<uint16_t*>(B.p[r])[i] = acc;
        } else {
            float acc = reinterpret_cast<const float*>(B.p[0])[i];
            for (int r = 1; r < world; ++r) acc = gfd::add(acc, reinterpret_cast<const float*>(B.p[r])[i]);
            for (int r = 0; r < world; ++r) reinterpret_cast<float*>(B.p[r])[i] = acc;
        }
    }
}

// ring_reduce_on (collectives.cpp:99-144) end state, one pass over every position's buffer
// (B in ring-position order): segment j's chain starts raw at position j; position j+k keeps
// the partial sum of positions j..j+k (what its RS step left), the root every full sum.
template <int DT>
__device__ __forceinline__ void ring_reduce_elem(const RankPtrs& B, int n, int root, int j, uint64_t e) {
    if (DT == GF_F16) {
        uint16_t acc = reinterpret_cast<const uint16_t*>(B.p[j])[e];
        for (int k = 1; k < n; ++k) {
            uint16_t* b = reinterpret_cast<uint16_t*>(B.p[(j + k) % n]);
            acc = gfd::acc16(b[e], acc);
            b[e] = acc;
        }
        reinterpret_cast<uint16_t*>(B.p[root])[e] = acc;
    } else {
        float acc = reinterpret_cast<const float*>(B.p[j])[e];
        for (int k = 1; k < n; ++k) {
            float* b = reinterpret_cast<float*>(B.p[(j + k) % n]);
            acc = gfd::add(b[e], acc);
            b[e] = acc;
        }
        reinterpret_cast<float*>(B.p[root])[e] = acc;
    }
}
template <int DT>
__global__ void ring_reduce_kernel(const __grid_constant__ RankPtrs B, int n, int root, uint64_t len, int vec) {
    constexpr int VE = DT == GF_F16 ? 8 : 4;
    const uint64_t base = len / uint64_t(n), rem = len % uint64_t(n), big = rem * (base + 1);
    auto seg = [&](uint64_t e) { return int(e < big ? e / (base + 1) : rem + (e - big) / base); };
    const uint64_t T = uint64_t(gridDim.x) * blockDim.x, g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nvec = vec ? len / VE : 0;
    for (uint64_t v = g; v < nvec; v += T) {
        const uint64_t e = v * VE;
        const int j = seg(e);
        if (seg(e + VE - 1) != j) {  // a segment boundary inside the vector: element by element
            for (int q = 0; q < VE; ++q) ring_reduce_elem<DT>(B, n, root, seg(e + q), e + q);
            continue;
        }
        uint4 acc = gfd::ld16(B.p[j] + v * 16);
        for (int k = 1; k < n; ++k) {
            char* b = B.p[(j + k) % n] + v * 16;
            acc = DT == GF_F16 ? gfd::acc16x8(gfd::ld16(b), acc) : gfd::acc32x4(gfd::ld16(b), acc);
            gfd::st16(b, acc);
        }
        gfd::st16(B.p[root] + v * 16, acc);
    }
    for (uint64_t e = nvec * VE + g; e < len; e += T) ring_reduce_elem<DT>(B, n, root, seg(e), e);
}

__global__ void bcast_kernel(const __grid_constant__ RankPtrs B, int world, int root, uint64_t bytes, int vec) {
    const uint64_t T = uint64_t(gridDim.x) * blockDim.x, g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nvec = vec ? bytes / 16 : 0;
    for (uint64_t v = g; v < nvec; v += T) {
        const uint4 x = gfd::ld16(B.p[root] + v * 16);
        for (int r = 0; r < world; ++r)
            if (r != root) gfd::st16(B.p[r] + v * 16, x);
    }
    for (uint64_t i = nvec * 16 + g; i < bytes; i += T) {
        const char v = B.p[root][i];
        for (int r = 0; r < world; ++r)
            if (r != root) B.p[r][i] = v;
    }
}

RankPtrs rank_ptrs(void* const* bufs, int n) {
    RankPtrs B{};
    for (int r = 0; r < n; ++r) B.p[r] = static_cast<char*>(bufs[r]);
    return B;
}
}  // namespace

extern "C" {

int gf_oracle_allreduce_ptrs(int dtype, void* const* bufs, int world, uint64_t len, void* stream) {
    if (!gfi::valid_dtype(dtype) || !bufs || world < 1 || world > GF_MAX_RANKS)
        return gfi::fail(GF_ERR_CONFIG, "gf_oracle_allreduce_ptrs: bad arguments");
    if (world == 1 || len == 0) return GF_OK;
    const RankPtrs B = rank_ptrs(bufs, world);
    const int vec = all_aligned16(bufs, world);
    const int grid = grid_for((len + 7) / 8, 256);
    if (dtype == GF_F16)
        oracle_sum_kernel<GF_F16><<<grid, 256, 0, gfi::S(stream)>>>(B, world, len, vec);
    else
        oracle_sum_kernel<GF_F32><<<grid, 256, 0, gfi::S(stream)>>>(B, world, len, vec);
    gfi::count_launch();
    return gfi::check_launch("gf_oracle_allreduce_ptrs");
}

int gf_ring_reduce_ptrs(int dtype, void* const* bufs, int n, int root_pos, uint64_t len, void* stream) {
    if (!gfi::valid_dtype(dtype) || !bufs || n < 1 || n > GF_MAX_RANKS || root_pos < 0 || root_pos >= n)
        return gfi::fail(GF_ERR_CONFIG, "gf_ring_reduce_ptrs: bad arguments");
    if (n == 1 || len == 0) return GF_OK;
    const RankPtrs B = rank_ptrs(bufs, n);
    const int vec = all_aligned16(bufs, n);
    const int grid = grid_for((len + 7) / 8, 256);
    if (dtype == GF_F16)
        ring_reduce_kernel<GF_F16><<<grid, 256, 0, gfi::S(stream)>>>(B, n, root_pos, len, vec);
    else
        ring_reduce_kernel<GF_F32><<<grid, 256, 0, gfi::S(stream)>>>(B, n, root_pos, len, vec);
    gfi::count_launch();
    return gfi::check_launch("gf_ring_reduce_ptrs");
}

int gf_broadcast_ptrs(void* const* bufs, int world, int root, uint64_t bytes, void* stream) {
    if (!bufs || world < 1 || world > GF_MAX_RANKS || root < 0 || root >= world)
        return gfi::fail(GF_ERR_CONFIG, "gf_broadcast_ptrs: bad arguments");
    if (world == 1 || bytes == 0) return GF_OK;
    bcast_kernel<<<grid_for((bytes + 15) / 16, 256), 256, 0, gfi::S(stream)>>>(rank_ptrs(bufs, world), world, root,
                                                                              bytes, all_aligned16(bufs, world));
    gfi::count_launch();
    return gfi::check_launch("gf_broadcast_ptrs");
}

}  // extern "C"
