// SPDX-License-Identifier: Apache-2.0
//
// The dense step as ONE kernel per rank (gf_sync_step_dense_pipe): pack, reduce-scatter,
// all-gather and unpack overlap unit by unit over NVLink peer memory.
//
// The owned segment of every window (segment_of, src/collectives.cpp:47-53) is cut into units
// of `ue` elements; unit u of owner j is the same pool range on every rank. The grid splits in
// two roles that run at once:
//
//   producers  pack unit u of every owner (fp32 -> fp16, write_tensor src/gradient_pool.cpp:78-105)
//              and store it where the owner reduces it: my pool for my own segment, else my slot
//              of the owner's inbox (NVLink). Then they publish rs[u][me] = gen+1 at the owner.
//              Afterwards they unpack the other owners' units as those arrive (ag flags).
//   consumers  for each unit of MY segment, wait until every rank published it, sum the N
//              contributions in ring order from my position (src/collectives.cpp:69-96, the
//              reference's arrival order: bit-identical), push the sums into every rank's pool
//              (the all-gather), unpack them from registers (g = sum * 1/N, trainer.cpp:336-342)
//              and publish ag[me][u] = gen+1 at every rank.
//
// So the all-gather of unit u rides on the links while later units are still being packed and
// reduce-scattered: per rank and direction the NVLink bytes are the ring's 2(N-1)/N * K, spread
// over the whole step instead of two serial phases. Memory ordering: every publication is
// bar.sync + fence.sc.sys + st.release.sys by the signalling threads after the unit's stores
// (cumulative over the CTA's writes); every wait is ld.acquire.sys polling + bar.sync, and data
// written by peers is read with ld.global.cg. Cross-step reuse of the inboxes and pools is
// ordered by one entry barrier (CTA b <-> CTA b of every rank): a peer that entered step g+1
// has completed step g on its stream, hence every read of this rank's memory in step g.
// Flags hold generations (never reset), so a unit that is empty in some step cannot desync them.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ring_device.cuh"

namespace {

constexpr int kPipeThreads = 256;
constexpr int kPipeMaxT = 256;

struct PipeTable {  // tensors sorted by pool offset, tiling [off[0], off[n-1]+cnt[n-1])
    int n;
    int pad;
    uint64_t off[kPipeMaxT];
    uint64_t cnt[kPipeMaxT];
    const float* src[kPipeMaxT];
    float* dst[kPipeMaxT];
};

struct PipeArgs {
    int world, rank, pos, nwin;
    int ring[GF_MAX_RANKS];
    int producers;                         // CTAs [0, producers) produce, the rest consume
    uint64_t ue;                           // unit length (elements, multiple of 8)
    uint64_t slot_elems;                   // inbox slot stride (elements)
    uint16_t* pool_by_pos[GF_MAX_RANKS];   // pool of the rank at ring position j (peer-mapped)
    uint16_t* inbox_by_pos[GF_MAX_RANKS];  // inbox of the owner at position j, as mapped here
    uint64_t* rs_by_pos[GF_MAX_RANKS];     // RS flags of the owner at position j: [unit][src rank]
    uint64_t* ag_by_pos[GF_MAX_RANKS];     // AG flags of the rank at position j: [owner pos][unit]
    uint64_t* gen;                         // per-CTA generation (local)
    // entry barrier (cross_barrier)
    uint64_t* flags_local;
    uint64_t* flags_peer[GF_MAX_RANKS];  // by rank
    uint64_t* epochs;
    uint64_t timeout_ns;
    int* err;
    uint64_t* trace;
    float inv;
    uint32_t upre[kMaxW + 1];  // units per owner in windows < w (the same for every owner)
    uint64_t wstart[kMaxW];
    uint64_t wlen[kMaxW];
};

// unit u of the owner at position j: pool range [a, b) (may be empty)
__device__ __forceinline__ void unit_range(const PipeArgs& A, int j, uint32_t u, uint64_t& a, uint64_t& b) {
    int lo = 0, hi = A.nwin;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (A.upre[mid] <= u) lo = mid; else hi = mid;
    }
    const uint64_t n = uint64_t(A.world), L = A.wlen[lo], base = L / n, rem = L % n, uj = uint64_t(j);
    const uint64_t e0 = A.wstart[lo] + uj * base + min(uj, rem), e1 = e0 + base + (uj < rem ? 1 : 0);
    a = min(e1, e0 + uint64_t(u - A.upre[lo]) * A.ue);
    b = min(e1, a + A.ue);
}

// first tensor whose range ends after e
__device__ __forceinline__ int table_at(const PipeTable& T, uint64_t e) {
    int lo = 0, hi = T.n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (T.off[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

// Poll until *f >= v, bounded by the communicator timeout. Relaxed polls with exponential
// __nanosleep backoff (hundreds of CTAs wait at once: acquire-polling at system scope in a
// tight loop was measured to starve the producers), then one acquire fence.
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ bool wait_ge(const PipeArgs& A, const uint64_t* f, uint64_t v) {
    if (A.timeout_ns == 0) return true;  // GF_DIAG_NOWAIT probe
    if (ld_relaxed_sys(f) < v) {
        const uint64_t t0 = gfd::globaltimer_ns();
        unsigned ns = 32;
        uint32_t spins = 0;
        while (ld_relaxed_sys(f) < v) {
            __nanosleep(ns);
            ns = min(ns * 2, 512u);
            if ((++spins & 63u) == 0) {
                if (*reinterpret_cast<volatile int*>(A.err) != 0) return false;
                if (gfd::globaltimer_ns() - t0 > A.timeout_ns) {
                    *reinterpret_cast<volatile int*>(A.err) = 1;
                    return false;
                }
            }
        }
    }
    fence_acq_rel_sys();  // acquire: the stores published before the flag are visible from here on
    return true;
}

// publish (one thread, after bar.sync): release fence over the CTA's stores, then the flag
__device__ __forceinline__ void publish(uint64_t* flag, uint64_t v) {
    fence_acq_rel_sys();
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

// producer: pack pool range [a, b) of my gradients into dst (pool indices)
__device__ void produce_range(const PipeTable& T, uint64_t a, uint64_t b, uint16_t* __restrict__ dst) {
    constexpr int U = 4;
    int t = table_at(T, a);
    for (uint64_t e0 = a; e0 < b; ++t) {
        const uint64_t te = T.off[t] + T.cnt[t], e1 = min(b, te);
        const float* __restrict__ s = T.src[t] + (e0 - T.off[t]);  // s[i] = element e0 + i
        const uint64_t len = e1 - e0;
        // vectors: pool index and source 8-element / 32-byte aligned
        const uint64_t head = min(len, (8 - (e0 & 7)) & 7);
        const bool vec = ((reinterpret_cast<uintptr_t>(s + head)) & 31u) == 0;
        uint64_t done = 0;
        if (vec) {
            for (uint64_t i = threadIdx.x; i < head; i += kPipeThreads) dst[e0 + i] = gfd::enc(s[i]);
            const uint64_t nv = (len - head) / 8, vb = e0 + head;
            for (uint64_t v0 = threadIdx.x; v0 < nv; v0 += uint64_t(kPipeThreads) * U) {
                gfd::F8 f[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t v = v0 + uint64_t(u) * kPipeThreads;
                    if (v < nv) f[u] = gfd::ld32f_stream(s + head + 8 * v);  // LDG.E.256
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t v = v0 + uint64_t(u) * kPipeThreads;
                    if (v < nv) gfd::st16(dst + vb + 8 * v, gfd::enc8(f[u].lo, f[u].hi));
                }
            }
            done = head + nv * 8;
        }
        for (uint64_t i = done + threadIdx.x; i < len; i += kPipeThreads) dst[e0 + i] = gfd::enc(s[i]);
        e0 = e1;
    }
}

__device__ __forceinline__ uint4 ld16_cg(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// g_avg of pool elements [e, e+8) held in x (16-byte aligned pool vector)
__device__ __forceinline__ void unpack8(const PipeTable& T, uint64_t e, uint4 x, float inv) {
    int t = table_at(T, e);
    float* d = T.dst[t] + (e - T.off[t]);
    if (e + 8 <= T.off[t] + T.cnt[t] && (reinterpret_cast<uintptr_t>(d) & 31u) == 0 && !gfd::any_special(x)) {
        const float2 f0 = gfd::h2f2(x.x), f1 = gfd::h2f2(x.y), f2 = gfd::h2f2(x.z), f3 = gfd::h2f2(x.w);
        gfd::st32f_stream(d,  // finite halves: x * (1/N) cannot produce NaN
                          make_float4(__fmul_rn(f0.x, inv), __fmul_rn(f0.y, inv), __fmul_rn(f1.x, inv),
                                      __fmul_rn(f1.y, inv)),
                          make_float4(__fmul_rn(f2.x, inv), __fmul_rn(f2.y, inv), __fmul_rn(f3.x, inv),
                                      __fmul_rn(f3.y, inv)));
        return;
    }
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint64_t ek = e + k;
        while (t + 1 < T.n && T.off[t + 1] <= ek) ++t;
        T.dst[t][ek - T.off[t]] = gfd::mul(gfd::dec(uint16_t((w[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu)), inv);
    }
}
__device__ __forceinline__ void unpack1(const PipeTable& T, uint64_t e, uint16_t h, float inv) {
    const int t = table_at(T, e);
    T.dst[t][e - T.off[t]] = gfd::mul(gfd::dec(h), inv);
}

// consumer: reduce pool range [a, b) of my segment (sources in ring order from my position: my
// pool, then inbox slots 0..N-2), push the sums to every pool, unpack them
template <int NT>
__device__ void consume_range(const PipeArgs& A, const PipeTable& T, int n, uint64_t a, uint64_t b) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int U = NMAX <= 2 ? 4 : (NMAX <= 4 ? 2 : 1);
    const uint16_t* src[NMAX];
    uint16_t* dst[NMAX];
#pragma unroll
    for (int t = 0; t < NMAX; ++t) {
        src[t] = t == 0 ? A.pool_by_pos[A.pos]
                        : (t < n ? A.inbox_by_pos[A.pos] + uint64_t(t - 1) * A.slot_elems : nullptr);
        dst[t] = t < n ? A.pool_by_pos[(A.pos + 1 + t) % n] : nullptr;  // the next rank on the ring first
    }
    auto scalar = [&](uint64_t e) {
        uint16_t acc = reinterpret_cast<const volatile uint16_t*>(src[0])[e];
        for (int t = 1; t < n; ++t) acc = gfd::acc16(reinterpret_cast<const volatile uint16_t*>(src[t])[e], acc);
        for (int t = 0; t < n; ++t) dst[t][e] = acc;
        unpack1(T, e, acc, A.inv);
    };
    const uint64_t va = (a + 7) / 8, vb = b / 8;
    if (va >= vb) {
        for (uint64_t e = a + threadIdx.x; e < b; e += kPipeThreads) scalar(e);
        return;
    }
    for (uint64_t e = a + threadIdx.x; e < va * 8; e += kPipeThreads) scalar(e);
    for (uint64_t e = vb * 8 + threadIdx.x; e < b; e += kPipeThreads) scalar(e);
    const uint64_t nv = vb - va;
    for (uint64_t v0 = threadIdx.x; v0 < nv; v0 += uint64_t(kPipeThreads) * U) {
        uint4 x[U][NMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + uint64_t(u) * kPipeThreads;
            if (v < nv) {
#pragma unroll
                for (int t = 0; t < NMAX; ++t)
                    if (t < n) x[u][t] = ld16_cg(src[t] + (va + v) * 8);  // peers wrote it: L2
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + uint64_t(u) * kPipeThreads;
            if (v >= nv) continue;
            uint4 acc = x[u][0];
#pragma unroll
            for (int t = 1; t < NMAX; ++t)
                if (t < n) acc = gfd::acc16x8(x[u][t], acc);
#pragma unroll
            for (int t = 0; t < NMAX; ++t)
                if (t < n) gfd::st16(dst[t] + (va + v) * 8, acc);
            unpack8(T, (va + v) * 8, acc, A.inv);
        }
    }
}

// unpack pool range [a, b) of my pool (an owner's all-gather landed there)
__device__ void unpack_range(const PipeTable& T, const uint16_t* pool, uint64_t a, uint64_t b, float inv) {
    const uint64_t va = (a + 7) / 8, vb = b / 8;
    auto scalar = [&](uint64_t e) { unpack1(T, e, reinterpret_cast<const volatile uint16_t*>(pool)[e], inv); };
    if (va >= vb) {
        for (uint64_t e = a + threadIdx.x; e < b; e += kPipeThreads) scalar(e);
        return;
    }
    for (uint64_t e = a + threadIdx.x; e < va * 8; e += kPipeThreads) scalar(e);
    for (uint64_t e = vb * 8 + threadIdx.x; e < b; e += kPipeThreads) scalar(e);
    constexpr int U = 4;
    const uint64_t nv = vb - va;
    for (uint64_t v0 = threadIdx.x; v0 < nv; v0 += uint64_t(kPipeThreads) * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + uint64_t(u) * kPipeThreads;
            if (v < nv) x[u] = ld16_cg(pool + (va + v) * 8);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + uint64_t(u) * kPipeThreads;
            if (v < nv) unpack8(T, (va + v) * 8, x[u], inv);
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(kPipeThreads, 4)
pipe_kernel(const __grid_constant__ PipeArgs A, const __grid_constant__ PipeTable T) {
    __shared__ int s_ok;
    const int n = NT > 0 ? NT : A.world;
    const uint64_t epoch = A.epochs[blockIdx.x];
    const uint64_t g1 = A.gen[blockIdx.x] + 1;  // this step's flag value
    if (threadIdx.x == 0) s_ok = 1;
    const bool tr = A.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) A.trace[0] = gfd::globaltimer_ns();
    // entry: every rank finished its previous step (all its reads of my pool and inbox)
    if (!cross_barrier(A, epoch + 1, &s_ok, false)) return;
    if (tr) A.trace[1] = gfd::globaltimer_ns();
    const uint32_t U = A.upre[A.nwin];
    const int P = A.producers, C = int(gridDim.x) - P;
    if (int(blockIdx.x) < P) {
        // produce: item k = unit k / N of owner (pos + 1 + k) mod N, in k order on every rank so
        // the owners' units complete in order
        const uint64_t items = uint64_t(U) * uint64_t(n);
        for (uint64_t k = blockIdx.x; k < items; k += uint64_t(P)) {
            const uint32_t u = uint32_t(k / uint64_t(n));
            const int j = int((uint64_t(A.pos) + 1 + k % uint64_t(n)) % uint64_t(n));
            uint64_t a, b;
            unit_range(A, j, u, a, b);
            uint16_t* dst = j == A.pos ? A.pool_by_pos[A.pos]
                                       : A.inbox_by_pos[j] + uint64_t((A.pos - j - 1 + n) % n) * A.slot_elems;
            produce_range(T, a, b, dst);
            __syncthreads();
            if (threadIdx.x == 0) publish(A.rs_by_pos[j] + uint64_t(u) * GF_MAX_RANKS + A.rank, g1);
        }
        if (tr) A.trace[2] = gfd::globaltimer_ns();
        // then unpack the other owners' units as their all-gather lands: item k = unit k/(N-1) of
        // owner pos + 1 + k mod (N-1)
        const uint64_t uitems = uint64_t(U) * uint64_t(n - 1);
        const uint64_t* ag = A.ag_by_pos[A.pos];
        for (uint64_t k = blockIdx.x; k < uitems; k += uint64_t(P)) {
            const uint32_t u = uint32_t(k / uint64_t(n - 1));
            const int j = int((uint64_t(A.pos) + 1 + k % uint64_t(n - 1)) % uint64_t(n));
            if (threadIdx.x == 0 && !wait_ge(A, ag + uint64_t(j) * kPipeUnits + u, g1)) s_ok = 0;
            __syncthreads();
            if (!s_ok) return;
            uint64_t a, b;
            unit_range(A, j, u, a, b);
            unpack_range(T, A.pool_by_pos[A.pos], a, b, A.inv);
        }
    } else {
        // consume the units of my segment
        const uint64_t* rs = A.rs_by_pos[A.pos];
        for (uint32_t u = uint32_t(int(blockIdx.x) - P); u < U; u += uint32_t(C)) {
            if (threadIdx.x == 0)
                for (int t = 0; t < n && s_ok; ++t)
                    if (!wait_ge(A, rs + uint64_t(u) * GF_MAX_RANKS + A.ring[t], g1)) s_ok = 0;
            __syncthreads();
            if (!s_ok) return;
            uint64_t a, b;
            unit_range(A, A.pos, u, a, b);
            consume_range<NT>(A, T, n, a, b);
            __syncthreads();
            if (threadIdx.x < n && threadIdx.x != A.pos)  // every other rank: my unit u landed
                publish(A.ag_by_pos[threadIdx.x] + uint64_t(A.pos) * kPipeUnits + u, g1);
        }
        if (tr) A.trace[2] = gfd::globaltimer_ns();
    }
    if (threadIdx.x == 0) {
        A.epochs[blockIdx.x] = epoch + 1;
        A.gen[blockIdx.x] = g1;
    }
    if (tr) A.trace[3] = gfd::globaltimer_ns();
}

int pipe_ue() {  // unit length; GF_PIPE_UE overrides (multiple of 8)
    static const int v = [] {
        const char* e = std::getenv("GF_PIPE_UE");
        const int x = e ? std::atoi(e) : 16384;
        return std::max(64, (x / 8) * 8);
    }();
    return v;
}
int pipe_consumers_per_4() {  // consumer CTAs per 4 CTAs of the grid; GF_PIPE_CONS overrides (1..3)
    static const int v = [] {
        const char* e = std::getenv("GF_PIPE_CONS");
        const int x = e ? std::atoi(e) : 2;
        return std::min(3, std::max(1, x));
    }();
    return v;
}

}  // namespace

namespace gfr {
// the pipe kernel's grid: fixed per communicator (its per-CTA generations must advance together)
int pipe_grid(const gf_comm* c) {
    const int full = gfi::sm_count() * 4;
    if (!c->colocated) return std::min(full, kMaxBlocks);
    return std::max(4, full / (2 * c->world));  // every rank's CTAs resident at once
}
}  // namespace gfr

extern "C" {

int gf_sync_step_dense_pipe(gf_comm* c, int dtype, uint64_t pool_heap_off, uint64_t inbox_heap_off,
                            const float* const* src, float* const* dst, const uint64_t* pool_off,
                            const uint64_t* count, int ntensors, const uint64_t* win_start,
                            const uint64_t* win_len, int nwin, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    const char* fn = "gf_sync_step_dense_pipe";
    if (dtype != GF_F16 || ntensors < 1 || ntensors > kPipeMaxT || !src || !dst || !pool_off || !count || nwin < 1 ||
        nwin > kMaxW || !win_start || !win_len)
        return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": fp16 pool, 1..256 tensors, 1..256 windows");
    if (c->world == 1)
        return gf_sync_step_dense(c, dtype, pool_heap_off, src, dst, pool_off, count, ntensors, win_start, win_len,
                                  nwin, stream);
    PipeTable T;
    std::memset(&T, 0, sizeof(T));
    std::vector<int> order(static_cast<size_t>(ntensors));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return pool_off[x] < pool_off[y]; });
    T.n = ntensors;
    for (int i = 0; i < ntensors; ++i) {
        const int k = order[static_cast<size_t>(i)];
        T.off[i] = pool_off[k];
        T.cnt[i] = count[k];
        T.src[i] = src[k];
        T.dst[i] = dst[k];
        if (!src[k] || !dst[k] || count[k] == 0) return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": null or empty tensor");
        if (i > 0 && T.off[i] != T.off[i - 1] + T.cnt[i - 1])
            return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": tensors must tile the pool");
    }
    const uint64_t lo = T.off[0], hi = T.off[ntensors - 1] + T.cnt[ntensors - 1];
    uint64_t cover = lo;
    for (int w = 0; w < nwin; ++w) {
        if (win_start[w] != cover) return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": windows must tile the pool");
        cover += win_len[w];
    }
    if (cover != hi) return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": tensors and windows must cover the same range");
    const uint64_t slot_elems = (hi + 7) & ~uint64_t(7);
    const uint64_t pool_end = pool_heap_off + hi * 2, inbox_end = inbox_heap_off + uint64_t(c->world - 1) * slot_elems * 2;
    if (pool_end > c->heap_bytes || inbox_end > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": pool or inbox outside the symmetric heap");
    if (pool_heap_off % 16 != 0 || inbox_heap_off % 16 != 0)
        return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": pool and inbox offsets must be 16-byte aligned");
    if (pool_heap_off < inbox_end && inbox_heap_off < pool_end)
        return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": pool and inbox ranges overlap");
    PipeArgs A;
    std::memset(&A, 0, sizeof(A));
    A.world = c->world;
    A.rank = c->rank;
    A.pos = c->pos;
    A.nwin = nwin;
    A.slot_elems = slot_elems;
    A.inv = 1.0f / static_cast<float>(c->world);
    // unit length: the default, grown so every owner has <= kPipeUnits units
    uint64_t ue = uint64_t(pipe_ue());
    for (;;) {
        uint64_t u = 0;
        for (int w = 0; w < nwin; ++w) u += (win_len[w] / uint64_t(c->world) + 1 + ue - 1) / ue;
        if (u <= kPipeUnits) break;
        ue *= 2;
    }
    A.ue = ue;
    A.upre[0] = 0;
    for (int w = 0; w < nwin; ++w) {
        A.wstart[w] = win_start[w];
        A.wlen[w] = win_len[w];
        A.upre[w + 1] = A.upre[w] + uint32_t((win_len[w] / uint64_t(c->world) + 1 + ue - 1) / ue);
    }
    for (int j = 0; j < c->world; ++j) {
        char* base = c->peer_alloc[c->ring[j]];
        A.pool_by_pos[j] = reinterpret_cast<uint16_t*>(base + kFlagBytes + pool_heap_off);
        A.inbox_by_pos[j] = reinterpret_cast<uint16_t*>(base + kFlagBytes + inbox_heap_off);
        A.rs_by_pos[j] = reinterpret_cast<uint64_t*>(base + kPipeRsOff);
        A.ag_by_pos[j] = reinterpret_cast<uint64_t*>(base + kPipeAgOff);
        A.ring[j] = c->ring[j];
    }
    for (int r = 0; r < c->world; ++r) A.flags_peer[r] = reinterpret_cast<uint64_t*>(c->peer_alloc[r]);
    A.flags_local = reinterpret_cast<uint64_t*>(c->alloc);
    A.epochs = A.flags_local + kFlagWords;
    A.gen = reinterpret_cast<uint64_t*>(c->alloc + kPipeGenOff);
    A.timeout_ns = c->timeout_ns;
    A.err = c->err_dev;
    A.trace = c->trace ? reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(c->err_dev) + 64) : nullptr;
    const int grid = gfr::pipe_grid(c);
    A.producers = std::max(1, grid - std::max(1, grid * pipe_consumers_per_4() / 4));
    DeviceGuard guard(c->device);
    cudaStream_t s = gfi::S(stream);
    switch (c->world) {
        case 2: pipe_kernel<2><<<grid, kPipeThreads, 0, s>>>(A, T); break;
        case 4: pipe_kernel<4><<<grid, kPipeThreads, 0, s>>>(A, T); break;
        case 8: pipe_kernel<8><<<grid, kPipeThreads, 0, s>>>(A, T); break;
        default: pipe_kernel<0><<<grid, kPipeThreads, 0, s>>>(A, T); break;
    }
    gfi::count_launch();
    return gfi::check_launch(fn);
}

}  // extern "C"
