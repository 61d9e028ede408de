// SPDX-License-Identifier: Apache-2.0
//
// Device-side numerics of the gradient-sync path, bit-compatible with the
// reference's host arithmetic (GradientFlow reference, /root/reference/proj):
//
//  * enc()/dec(): the reference binary16 codec (include/gflow/half.hpp:20-87):
//    round-to-nearest-even, but +-inf and overflow CLAMP to +-65504 (0x7BFF)
//    and NaN encodes as sign|0x7E00. Hardware cvt.rn.f16.f32 does RNE
//    (incl. subnormals) and returns inf on overflow, so we fix up inf and NaN.
//  * add/mul/sub(): IEEE single ops with x86 SSE NaN semantics (the reference
//    is compiled for baseline x86-64 with no FMA): a NaN operand propagates
//    quieted (first operand first); an invalid op (inf-inf, 0*inf) yields the
//    x86 "default NaN" 0xFFC00000. __fadd_rn/__fmul_rn are never contracted
//    into FMA (P2 in SURVEY.md).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

namespace gfd {

__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }
__device__ __forceinline__ bool isnan_(float f) { return (f2u(f) & 0x7FFFFFFFu) > 0x7F800000u; }
__device__ __forceinline__ float quiet(float f) { return u2f(f2u(f) | 0x00400000u); }

// half.hpp:20-59
__device__ __forceinline__ uint16_t enc(float v) {
    const uint32_t b = f2u(v);
    uint16_t h = __half_as_ushort(__float2half_rn(v));
    if ((h & 0x7FFFu) >= 0x7C00u) {
        // inf after rounding (overflow or inf input) clamps; NaN keeps only its sign.
        const uint16_t sign = static_cast<uint16_t>((b >> 16) & 0x8000u);
        h = ((b & 0x7FFFFFFFu) > 0x7F800000u) ? static_cast<uint16_t>(sign | 0x7E00u)
                                               : static_cast<uint16_t>(sign | 0x7BFFu);
    }
    return h;
}

// half.hpp:61-87 (exact; NaN payload and sign preserved)
__device__ __forceinline__ float dec(uint16_t h) {
    if ((h & 0x7C00u) == 0x7C00u) {
        return u2f((static_cast<uint32_t>(h & 0x8000u) << 16) | 0x7F800000u |
                   (static_cast<uint32_t>(h & 0x3FFu) << 13));
    }
    return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ float nan_result(float a, float b) {
    if (isnan_(a)) return quiet(a);
    if (isnan_(b)) return quiet(b);
    return u2f(0xFFC00000u);  // x86 default NaN for invalid operations
}
__device__ __forceinline__ float add(float a, float b) {
    const float s = __fadd_rn(a, b);
    return isnan_(s) ? nan_result(a, b) : s;
}
__device__ __forceinline__ float sub(float a, float b) {
    const float s = __fsub_rn(a, b);
    return isnan_(s) ? nan_result(a, b) : s;
}
__device__ __forceinline__ float mul(float a, float b) {
    const float s = __fmul_rn(a, b);
    return isnan_(s) ? nan_result(a, b) : s;
}

// accumulate (buffer.hpp:71-79): local + incoming, widened and rounded back.
// The reference binary (g++ -O2, x86-64) emits addss with the INCOMING value as the
// destination operand here, so when both are NaN the incoming NaN wins (measured
// against oracle/_ref). The fp32 branch (buffer.hpp:63-69, `a += b`) keeps the local one.
__device__ __forceinline__ uint16_t acc16(uint16_t local, uint16_t incoming) {
    return enc(add(dec(incoming), dec(local)));
}

// 8 x fp16 in a 16-byte vector.
struct alignas(16) H8 {
    uint32_t w[4];
    __device__ __forceinline__ uint16_t get(int i) const {
        return static_cast<uint16_t>((w[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu);
    }
    __device__ __forceinline__ void set(int i, uint16_t v) {
        const int s = (i & 1) * 16;
        w[i >> 1] = (w[i >> 1] & ~(0xFFFFu << s)) | (static_cast<uint32_t>(v) << s);
    }
};

__device__ __forceinline__ uint4 ld16(const void* p) {
    return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void st16(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }
// streaming (evict-first) variants for data touched once
__device__ __forceinline__ uint4 ld16_stream(const void* p) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld16f_stream(const float* p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// ---- packed fast paths --------------------------------------------------------------
// A half2 word holds a NaN/inf iff one of its halves has exponent 31. All fast paths
// below are taken only when no input/output half is special; then plain IEEE ops give
// exactly the reference's results and the per-element NaN/clamp fix-ups are skipped.
__device__ __forceinline__ uint32_t special2(uint32_t w) {
    return __vcmpeq2(w & 0x7C007C00u, 0x7C007C00u);  // 0xFFFF in each special half
}
__device__ __forceinline__ bool any_special(uint4 v) {
    return (special2(v.x) | special2(v.y) | special2(v.z) | special2(v.w)) != 0u;
}
__device__ __forceinline__ float2 h2f2(uint32_t w) {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
}
__device__ __forceinline__ uint32_t f22h2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);  // cvt.rn.f16x2.f32
    return *reinterpret_cast<const uint32_t*>(&h);
}
// 8 floats -> 8 halves with the reference codec; fast unless a result is inf/NaN.
__device__ __forceinline__ uint4 enc8(float4 a, float4 b) {
    uint4 o;
    o.x = f22h2(a.x, a.y);
    o.y = f22h2(a.z, a.w);
    o.z = f22h2(b.x, b.y);
    o.w = f22h2(b.z, b.w);
    if (any_special(o)) {
        o.x = uint32_t(enc(a.x)) | (uint32_t(enc(a.y)) << 16);
        o.y = uint32_t(enc(a.z)) | (uint32_t(enc(a.w)) << 16);
        o.z = uint32_t(enc(b.x)) | (uint32_t(enc(b.y)) << 16);
        o.w = uint32_t(enc(b.z)) | (uint32_t(enc(b.w)) << 16);
    }
    return o;
}

// ---- exact |x| of fp16 values in units of 2^-24 (the chunk L1 of gf_chunk_norms) ----------
// |h| * 2^24 is an integer < 2^40 for every finite half, and fp32 holds it exactly (a power
// of two times an 11-bit significand): half -> float, scale, truncate. Non-finite halves give
// meaningless units; callers track NaN separately.
__device__ __forceinline__ uint64_t half_units(uint16_t h) {
    return __float2ull_rz(fabsf(__half2float(__ushort_as_half(h))) * 16777216.0f);
}
__device__ __forceinline__ uint64_t units8(uint4 v) {
    const uint32_t w[4] = {v.x & 0x7FFF7FFFu, v.y & 0x7FFF7FFFu, v.z & 0x7FFF7FFFu, v.w & 0x7FFF7FFFu};
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 f = h2f2(w[k]);
        acc += __float2ull_rz(f.x * 16777216.0f) + __float2ull_rz(f.y * 16777216.0f);
    }
    return acc;
}

// 256-bit (32 B per thread) global access, sm_100: one LDG.E.256 / STG.E.256 per 8 floats.
// Requires 32-B alignment.
struct F8 {
    float4 lo, hi;
};
// L2 residency policies (126 MB L2): streams touched once (fp32 gradients in, fp32 g_avg
// out) are marked evict-first so that the fp16 pool written by pack stays resident for
// the ring (local + peer reads) and unpack.
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ F8 ld32f_stream(const float* p) {
    F8 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(v.lo.x), "=f"(v.lo.y), "=f"(v.lo.z), "=f"(v.lo.w), "=f"(v.hi.x), "=f"(v.hi.y),
                   "=f"(v.hi.z), "=f"(v.hi.w)
                 : "l"(p), "l"(pol_evict_first()));
    return v;
}
// fp16 pool store that asks L2 to keep the line (evict-last)
__device__ __forceinline__ void st16_keep(void* p, uint4 v) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(pol_evict_last())
                 : "memory");
}
__device__ __forceinline__ F8 ld32f(const float* p) {
    F8 v;
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.lo.x), "=f"(v.lo.y), "=f"(v.lo.z), "=f"(v.lo.w), "=f"(v.hi.x), "=f"(v.hi.y),
                   "=f"(v.hi.z), "=f"(v.hi.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st32f_stream(float* p, float4 lo, float4 hi) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p),
                 "f"(lo.x), "f"(lo.y), "f"(lo.z), "f"(lo.w), "f"(hi.x), "f"(hi.y), "f"(hi.z), "f"(hi.w),
                 "l"(pol_evict_first())
                 : "memory");
}
__device__ __forceinline__ void st32f(float* p, float4 lo, float4 hi) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(lo.x), "f"(lo.y),
                 "f"(lo.z), "f"(lo.w), "f"(hi.x), "f"(hi.y), "f"(hi.z), "f"(hi.w)
                 : "memory");
}

// fp16 vector accumulate: acc[i] = enc(add(dec(local[i]), dec(acc[i])))
__device__ __forceinline__ uint4 acc16x8(uint4 local, uint4 acc) {
    if (!any_special(local) && !any_special(acc)) {
        const uint32_t* l = reinterpret_cast<const uint32_t*>(&local);
        const uint32_t* c = reinterpret_cast<const uint32_t*>(&acc);
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 x = h2f2(l[k]), y = h2f2(c[k]);
            ow[k] = f22h2(__fadd_rn(y.x, x.x), __fadd_rn(y.y, x.y));
        }
        if (!any_special(o)) return o;  // else an add overflowed: clamp via the slow path
    }
    const uint32_t* l = reinterpret_cast<const uint32_t*>(&local);
    uint32_t* a = reinterpret_cast<uint32_t*>(&acc);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint16_t lo = acc16(static_cast<uint16_t>(l[k] & 0xFFFFu), static_cast<uint16_t>(a[k] & 0xFFFFu));
        const uint16_t hi = acc16(static_cast<uint16_t>(l[k] >> 16), static_cast<uint16_t>(a[k] >> 16));
        a[k] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
    return acc;
}
// fp32 vector accumulate: acc[i] = add(local[i], acc[i])
__device__ __forceinline__ uint4 acc32x4(uint4 local, uint4 acc) {
    uint4 r;
    r.x = f2u(add(u2f(local.x), u2f(acc.x)));
    r.y = f2u(add(u2f(local.y), u2f(acc.y)));
    r.z = f2u(add(u2f(local.z), u2f(acc.z)));
    r.w = f2u(add(u2f(local.w), u2f(acc.w)));
    return r;
}

// ---- system-scope flags for cross-GPU barriers --------------------------------
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace gfd
