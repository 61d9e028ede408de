// SPDX-License-Identifier: Apache-2.0
// Per-tensor output table of the kernels that unpack straight from registers (the pull
// all-gather of pull.cu, the push all-gather of push.cu): tensors sorted by pool offset, the
// unpack of one 16-byte pool vector into its tensor(s) as g_avg = x * (1/N)
// (src/trainer.cpp:336-342), and the host-side table builder.
#pragma once

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ring_device.cuh"

namespace {

constexpr int kStepMaxT = 256;
struct StepTable {  // tensors sorted by pool offset
    int n;
    int pad;
    uint64_t off[kStepMaxT];
    uint64_t cnt[kStepMaxT];
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
__device__ __forceinline__ uint4 ld16_cg(const void* p) {  // L2 only: a peer wrote it this launch
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

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
