// SPDX-License-Identifier: Apache-2.0
//
// Single-CTA selection + compaction plan (K5 body), shared by gf_select_topk /
// gf_csc_plan (csc.cu) and the fused NVLink norm-exchange kernel (ring.cu).
//
// Reference select_next_important (src/sparse.cpp:189-201) partial_sorts chunk
// indices by (norm desc, index asc) and flags the first k. The flagged SET is all
// that is kept, so we find it without sorting: a 4-pass 8-bit radix select finds
// the k-th largest key T and how many keys equal to T are needed; a block scan in
// index order then takes exactly that many of the ties, lowest index first.
// The compaction plan is the staging layout of sparse_exchange (sparse.cpp:129-158):
// coff[c] = sum of lengths of important chunks < c, and the theta windows.
#pragma once

#include <cstdint>

#include "gf_device.cuh"

namespace gfs {

constexpr int kSelThreads = 1024;

// Order-preserving map of a float to uint32 (-0 folded onto +0, as the
// comparator treats them equal).
__device__ __forceinline__ uint32_t norm_key(float f) {
    uint32_t b = gfd::f2u(f);
    if (b == 0x80000000u) b = 0;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Exclusive block scan of v (all kSelThreads threads participate); returns the
// exclusive prefix, *total = block sum.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total, T* warp_sums /*[32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T s = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;  // inclusive
    }
    __syncthreads();
    const T warp_off = warp == 0 ? T(0) : warp_sums[warp - 1];
    *total = warp_sums[31];
    __syncthreads();
    return warp_off + x - v;
}

constexpr int kSelBins = 2048;  // radix digits of 11, 11 and 10 bits: three passes over 32-bit keys
static_assert(kSelBins == 2 * kSelThreads, "two histogram bins per thread in the digit search");

struct SelShared {
    unsigned hist[kSelBins];
    uint64_t u64s[32];
    unsigned digit;
    unsigned long long rem;
};

// flags[c] = 1 iff chunk c is among the top k by (norm desc, index asc).
// Keys of up to kSelThreads * kKeysPerThread chunks stay in registers across the passes.
constexpr int kKeysPerThread = 4;

inline __device__ void block_topk(const float* norms, uint64_t nc, uint64_t k, uint8_t* flags,
                           SelShared& sh) {
    const int tid = threadIdx.x;
    if (k >= nc) {
        for (uint64_t i = tid; i < nc; i += kSelThreads) flags[i] = 1;
        __syncthreads();
        return;
    }
    const bool cached = nc <= uint64_t(kSelThreads) * kKeysPerThread;
    uint32_t kr[kKeysPerThread];
#pragma unroll
    for (int q = 0; q < kKeysPerThread; ++q) {
        const uint64_t i = tid + uint64_t(q) * kSelThreads;
        kr[q] = (cached && i < nc) ? norm_key(norms[i]) : 0u;
    }
    uint32_t prefix = 0;
    unsigned long long remaining = k;
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);  // digits [31:21], [20:10], [9:0]
        const uint32_t dmask = pass == 2 ? 1023u : 2047u;
        sh.hist[tid] = 0;
        sh.hist[tid + kSelThreads] = 0;
        __syncthreads();
        // Warp-aggregated: chunk norms share a few exponents, so most keys of a pass fall into one
        // or two digits and per-key shared atomics would serialise on one address.
        auto count = [&](bool valid, uint32_t key) {
            valid = valid && (pass == 0 || (key >> (pass == 1 ? 21 : 10)) == prefix);
            const uint32_t d = (key >> shift) & dmask;
            const unsigned same = __match_any_sync(0xFFFFFFFFu, valid ? d : 0xFFFFFFFFu);
            if (valid && __ffs(same) - 1 == (tid & 31)) atomicAdd(&sh.hist[d], unsigned(__popc(same)));
        };
        if (cached) {
#pragma unroll
            for (int q = 0; q < kKeysPerThread; ++q) count(tid + uint64_t(q) * kSelThreads < nc, kr[q]);
        } else {
            for (uint64_t base = 0; base < nc; base += kSelThreads) {
                const uint64_t i = base + tid;
                count(i < nc, i < nc ? norm_key(norms[i]) : 0u);
            }
        }
        __syncthreads();
        // thread t owns digits hi = top - 2t and hi - 1 (descending); one block scan finds the
        // digit where the descending cumulative count first reaches `remaining`
        const int top = int(dmask);
        const int dhi = top - 2 * tid, dlo = dhi - 1;
        const uint64_t chi = dhi >= 0 ? sh.hist[dhi] : 0, clo = dlo >= 0 ? sh.hist[dlo] : 0;
        uint64_t total;
        const uint64_t excl = block_excl_scan<uint64_t>(chi + clo, &total, sh.u64s);
        if (excl < remaining && remaining <= excl + chi + clo) {  // exactly one thread
            if (excl + chi >= remaining) {
                sh.digit = unsigned(dhi);
                sh.rem = remaining - excl;
            } else {
                sh.digit = unsigned(dlo);
                sh.rem = remaining - excl - chi;
            }
        }
        __syncthreads();
        prefix = (prefix << (pass == 2 ? 10 : 11)) | sh.digit;
        remaining = sh.rem;
        __syncthreads();
    }
    const uint32_t T = prefix;
    const uint64_t need = remaining;  // keys equal to T to take, lowest index first
    uint64_t carry = 0;
    for (uint64_t base = 0; base < nc; base += kSelThreads) {
        const uint64_t i = base + tid;
        uint32_t key = 0;
        const uint64_t q = base / kSelThreads;
        if (i < nc) {
            if (cached) {
#pragma unroll
                for (int z = 0; z < kKeysPerThread; ++z)
                    if (uint64_t(z) == q) key = kr[z];
            } else {
                key = norm_key(norms[i]);
            }
        }
        const uint64_t eq = (i < nc && key == T) ? 1 : 0;
        uint64_t tot;
        const uint64_t ex = block_excl_scan<uint64_t>(eq, &tot, sh.u64s);
        if (i < nc) flags[i] = (key > T || (eq && carry + ex < need)) ? 1 : 0;
        carry += tot;
    }
    __syncthreads();
}

// plan[0] staged elements, plan[1] important chunks, plan[2] windows, plan[3] window
// stride (elements), plan[4 .. 4+plan[1]) the important chunk indices, ascending. Windows: sparse.cpp:142-158 cuts after the selected chunk at which
// pending bytes >= theta; since only the final pool chunk differs in length, every
// window holds m = max(1, ceil(theta / (chunk*esz))) chunks except the last.
inline __device__ void block_plan(const uint8_t* flags, uint64_t total, uint64_t chunk, uint64_t nc,
                           uint64_t esz, uint64_t theta, uint64_t* coff, uint64_t* plan,
                           SelShared& sh) {
    const int tid = threadIdx.x;
    uint64_t carry_len = 0, carry_cnt = 0;
    for (uint64_t base = 0; base < nc; base += kSelThreads) {
        const uint64_t c = base + tid;
        uint64_t len = 0, one = 0;
        if (c < nc && flags[c]) {
            len = (c + 1 == nc) ? total - c * chunk : chunk;
            one = 1;
        }
        // one scan of (len << 20 | one): a round holds <= kSelThreads chunks (< 2^20), and the
        // lengths of a round sum below 2^44 whenever its chunks fit in memory; otherwise two scans
        uint64_t ex, exc, tot_len, tot_cnt;
        if (total <= (uint64_t(1) << 43)) {
            uint64_t tot;
            const uint64_t x = block_excl_scan<uint64_t>((len << 20) | one, &tot, sh.u64s);
            ex = x >> 20;
            exc = x & 0xFFFFFu;
            tot_len = tot >> 20;
            tot_cnt = tot & 0xFFFFFu;
        } else {
            ex = block_excl_scan<uint64_t>(len, &tot_len, sh.u64s);
            exc = block_excl_scan<uint64_t>(one, &tot_cnt, sh.u64s);
        }
        if (c < nc) coff[c] = carry_len + ex;
        if (one) plan[4 + carry_cnt + exc] = c;  // ascending list of important chunks
        carry_len += tot_len;
        carry_cnt += tot_cnt;
    }
    if (tid == 0) {
        uint64_t nwin = 0, stride = carry_len;
        if (carry_len > 0) {
            if (theta == UINT64_MAX) {
                nwin = 1;
            } else {
                const uint64_t per = chunk * esz;
                uint64_t m = theta / per + (theta % per != 0 ? 1 : 0);
                if (m < 1) m = 1;
                if (m > carry_cnt) m = carry_cnt;
                nwin = (carry_cnt + m - 1) / m;
                stride = m * chunk;
            }
        }
        plan[0] = carry_len;
        plan[1] = carry_cnt;
        plan[2] = nwin;
        plan[3] = stride;
    }
    __syncthreads();
}

}  // namespace gfs
