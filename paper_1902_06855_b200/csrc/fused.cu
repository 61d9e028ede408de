// SPDX-License-Identifier: Apache-2.0
//
// Fused gradient-sync step: pack (K1) -> NVLink ring allreduce (K4) -> unpack (K6) in ONE
// persistent kernel per rank, overlapped slab by slab (compute fused with its collective).
//
// Reference: the dense iteration of train_worker (src/trainer.cpp:297-347): write_tensor
// per tensor (src/gradient_pool.cpp:78-105), FusionEngine windows (src/fusion.cpp:72-109)
// each reduced by ring_allreduce_on (src/collectives.cpp:55-97), then g_avg = get(i)/N.
//
// Every theta window is split by segment_of; segment j (owned by ring position j) is cut
// into slabs of ~64 KB. A rank's CTAs pull tasks from one queue, in order:
//   pack   all slabs (round-robin over segments) -> release packed[slab][me] in the OWNER
//   reduce its own slabs: wait for packed[slab][*], load the slab from every rank in ring
//          order (bit-identical sums), store the result into every rank's pool, release
//          reduced[slab] in every rank
//   unpack all slabs: wait for reduced[slab], g_avg = dec(pool) * 1/N into the tensors
// No global barriers: a slab moves as soon as all ranks packed it, so HBM (pack/unpack)
// and NVLink (reduce) overlap across slabs. Pack tasks never wait and precede all waiting
// tasks in every queue, so progress needs no co-residency of the grid. Flags carry a
// device-side step epoch (CUDA-graph replayable); waits are bounded (TransportError).

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "comm.cuh"
#include "gf_device.cuh"
#include "gf_internal.cuh"

namespace {

constexpr int kStepThreads = 512;
constexpr int kStepMaxT = 256;

struct StepTable {  // tensors sorted by pool offset (pool order)
    int n;
    int pad;
    uint64_t off[kStepMaxT];
    uint64_t cnt[kStepMaxT];
    const float* src[kStepMaxT];
    float* dst[kStepMaxT];
};

struct StepArgs {
    char* pool[GF_MAX_RANKS];              // rank r's pool, peer-mapped
    uint32_t* packed_peer[GF_MAX_RANKS];   // rank r's packed[][] (written by sources)
    uint32_t* reduced_peer[GF_MAX_RANKS];  // rank r's reduced[]  (written by owners)
    uint32_t* ctl;                         // local: [0] epoch, [1] queue, [2] done
    int ring[GF_MAX_RANKS];
    int world, rank, pos;
    const uint64_t* slab_a;
    const uint64_t* slab_b;
    const uint32_t* slab_pos;
    const uint32_t* tasks;  // per-rank queue: (type << 30) | slab, software-pipelined
    uint32_t nslab, ntasks;
    float inv_world;
    uint64_t timeout_ns;
    int* err;
};

__device__ __forceinline__ void st_release_sys32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Bounded spin until *p >= e (wrap-safe). Returns false on timeout / poisoned comm.
__device__ bool wait_ge(const StepArgs& a, const uint32_t* p, uint32_t e) {
    if (int32_t(ld_acquire_sys32(p) - e) >= 0) return true;
    const uint64_t t0 = gfd::globaltimer_ns();
    for (uint32_t spins = 1;; ++spins) {
        if (int32_t(ld_acquire_sys32(p) - e) >= 0) return true;
        if ((spins & 255u) == 0) {
            if (*reinterpret_cast<volatile int*>(a.err) != 0) return false;
            if (gfd::globaltimer_ns() - t0 > a.timeout_ns) {
                *reinterpret_cast<volatile int*>(a.err) = 1;
                return false;
            }
        }
    }
}

__device__ __forceinline__ int first_tensor(const StepTable& T, uint64_t x) {
    // last tensor with off <= x
    int lo = 0, hi = T.n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (T.off[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// ---- pack / unpack of pool range [x0, x1) ----------------------------------------------
// SOLO (world == 1): the collective is the identity, so the slab is unpacked straight from
// the registers that hold its packed value (g_avg = dec(enc(g)) * 1/N): one HBM pass.
template <int DT, bool SOLO>
__device__ void pack_range(const StepArgs& a, const StepTable& T, uint64_t x0, uint64_t x1) {
    char* pool = a.pool[a.rank];
    const float inv = a.inv_world;
    for (int t = first_tensor(T, x0); t < T.n && T.off[t] < x1; ++t) {
        const uint64_t lo = max(x0, T.off[t]), hi = min(x1, T.off[t] + T.cnt[t]);
        if (lo >= hi) continue;
        const float* s = T.src[t] - T.off[t];  // indexed by pool element
        float* o = T.dst[t] - T.off[t];
        uint64_t v0 = hi, v1 = hi;
        if (DT == GF_F16 && (T.off[t] % 8) == 0 && (reinterpret_cast<uintptr_t>(T.src[t]) & 31u) == 0 &&
            (!SOLO || (reinterpret_cast<uintptr_t>(T.dst[t]) & 31u) == 0)) {
            v0 = (lo + 7) / 8 * 8;
            v1 = max(v0, hi / 8 * 8);
            uint16_t* d = reinterpret_cast<uint16_t*>(pool);
            constexpr int U = 4;  // 4 x 32 B loads in flight per thread
            const uint64_t step = 8 * uint64_t(blockDim.x);
            for (uint64_t e0 = v0 + 8 * threadIdx.x; e0 < v1; e0 += step * U) {
                gfd::F8 f[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (e0 + u * step < v1) f[u] = gfd::ld32f_stream(s + e0 + u * step);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t e = e0 + u * step;
                    if (e >= v1) break;
                    const uint4 h = gfd::enc8(f[u].lo, f[u].hi);
                    if (SOLO) {
                        gfd::st16(d + e, h);
                        if (!gfd::any_special(h)) {
                            const float2 g0 = gfd::h2f2(h.x), g1 = gfd::h2f2(h.y), g2 = gfd::h2f2(h.z), g3 = gfd::h2f2(h.w);
                            gfd::st32f_stream(o + e,
                                              make_float4(__fmul_rn(g0.x, inv), __fmul_rn(g0.y, inv),
                                                          __fmul_rn(g1.x, inv), __fmul_rn(g1.y, inv)),
                                              make_float4(__fmul_rn(g2.x, inv), __fmul_rn(g2.y, inv),
                                                          __fmul_rn(g3.x, inv), __fmul_rn(g3.y, inv)));
                        } else {
                            const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
                            for (int k = 0; k < 8; ++k)
                                o[e + k] = gfd::mul(gfd::dec(uint16_t((hw[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu)), inv);
                        }
                    } else {
                        gfd::st16_keep(d + e, h);
                    }
                }
            }
        }
        // scalar head [lo, v0) and tail [v1, hi) (everything when the tensor is unaligned)
        const uint64_t h_end = min(v0, hi), t_beg = max(v1, h_end);
        for (int part = 0; part < 2; ++part) {
            const uint64_t b0 = part == 0 ? lo : t_beg, b1 = part == 0 ? h_end : hi;
            for (uint64_t e = b0 + threadIdx.x; e < b1; e += blockDim.x) {
                if (DT == GF_F16) {
                    const uint16_t h = gfd::enc(s[e]);
                    reinterpret_cast<uint16_t*>(pool)[e] = h;
                    if (SOLO) o[e] = gfd::mul(gfd::dec(h), inv);
                } else {
                    reinterpret_cast<float*>(pool)[e] = s[e];
                    if (SOLO) o[e] = gfd::mul(s[e], inv);
                }
            }
        }
    }
}

template <int DT>
__device__ void unpack_range(const StepArgs& a, const StepTable& T, uint64_t x0, uint64_t x1) {
    const char* pool = a.pool[a.rank];
    const float inv = a.inv_world;
    for (int t = first_tensor(T, x0); t < T.n && T.off[t] < x1; ++t) {
        const uint64_t lo = max(x0, T.off[t]), hi = min(x1, T.off[t] + T.cnt[t]);
        if (lo >= hi) continue;
        float* d = T.dst[t] - T.off[t];
        uint64_t v0 = hi, v1 = hi;
        if (DT == GF_F16 && (T.off[t] % 8) == 0 && (reinterpret_cast<uintptr_t>(T.dst[t]) & 31u) == 0) {
            v0 = (lo + 7) / 8 * 8;
            v1 = max(v0, hi / 8 * 8);
            const uint16_t* p = reinterpret_cast<const uint16_t*>(pool);
            constexpr int U = 4;
            const uint64_t step = 8 * uint64_t(blockDim.x);
            for (uint64_t e0 = v0 + 8 * threadIdx.x; e0 < v1; e0 += step * U) {
              uint4 xs[U];
#pragma unroll
              for (int u = 0; u < U; ++u)
                  if (e0 + u * step < v1) xs[u] = gfd::ld16(p + e0 + u * step);
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const uint64_t e = e0 + u * step;
                if (e >= v1) break;
                const uint4 x = xs[u];
                if (!gfd::any_special(x)) {
                    const float2 f0 = gfd::h2f2(x.x), f1 = gfd::h2f2(x.y), f2 = gfd::h2f2(x.z), f3 = gfd::h2f2(x.w);
                    gfd::st32f_stream(d + e,
                                      make_float4(__fmul_rn(f0.x, inv), __fmul_rn(f0.y, inv), __fmul_rn(f1.x, inv),
                                                  __fmul_rn(f1.y, inv)),
                                      make_float4(__fmul_rn(f2.x, inv), __fmul_rn(f2.y, inv), __fmul_rn(f3.x, inv),
                                                  __fmul_rn(f3.y, inv)));
                } else {
                    for (int k = 0; k < 8; ++k) d[e + k] = gfd::mul(gfd::dec(p[e + k]), inv);
                }
              }
            }
        }
        const uint64_t h_end = min(v0, hi), t_beg = max(v1, h_end);
        for (int part = 0; part < 2; ++part) {
            const uint64_t b0 = part == 0 ? lo : t_beg, b1 = part == 0 ? h_end : hi;
            for (uint64_t e = b0 + threadIdx.x; e < b1; e += blockDim.x) {
                const float x = DT == GF_F16 ? gfd::dec(reinterpret_cast<const uint16_t*>(pool)[e])
                                             : reinterpret_cast<const float*>(pool)[e];
                d[e] = gfd::mul(x, inv);
            }
        }
    }
}

// ---- reduce of slab [x0, x1) of a segment owned by ring position p -------------------------
template <int DT, int NT>
__device__ void reduce_range(const StepArgs& a, int n, int p, uint64_t x0, uint64_t x1) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int U = NMAX <= 4 ? 4 : (NMAX <= 8 ? 2 : 1);
    constexpr int VE = DT == GF_F16 ? 8 : 4;
    const char* src[NMAX];
#pragma unroll
    for (int t = 0; t < NMAX; ++t) src[t] = (t < n) ? a.pool[a.ring[(p + t) % n]] : nullptr;
    const uint64_t v0 = (x0 + VE - 1) / VE, v1 = max(v0, x1 / VE);
    // unaligned ends [x0, v0*VE) and [v1*VE, x1)
    const uint64_t h_end = min(v0 * VE, x1), t_beg = max(v1 * VE, h_end);
    for (uint64_t k = threadIdx.x; k < (h_end - x0) + (x1 - t_beg); k += blockDim.x) {
        const uint64_t e = k < h_end - x0 ? x0 + k : t_beg + (k - (h_end - x0));
        if (DT == GF_F16) {
            uint16_t acc = reinterpret_cast<const uint16_t*>(src[0])[e];
            for (int t = 1; t < n; ++t) acc = gfd::acc16(reinterpret_cast<const uint16_t*>(src[t])[e], acc);
            for (int r = 0; r < a.world; ++r) reinterpret_cast<uint16_t*>(a.pool[r])[e] = acc;
        } else {
            float acc = reinterpret_cast<const float*>(src[0])[e];
            for (int t = 1; t < n; ++t) acc = gfd::add(reinterpret_cast<const float*>(src[t])[e], acc);
            for (int r = 0; r < a.world; ++r) reinterpret_cast<float*>(a.pool[r])[e] = acc;
        }
    }
    const uint64_t S = blockDim.x;
    for (uint64_t v = v0 + threadIdx.x; v < v1; v += S * U) {
        uint4 x[U][NMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * S;
            if (vv < v1) {
#pragma unroll
                for (int t = 0; t < NMAX; ++t)
                    if (t < n) x[u][t] = gfd::ld16(src[t] + vv * 16);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t vv = v + uint64_t(u) * S;
            if (vv < v1) {
                uint4 acc = x[u][0];
#pragma unroll
                for (int t = 1; t < NMAX; ++t)
                    if (t < n) acc = DT == GF_F16 ? gfd::acc16x8(x[u][t], acc) : gfd::acc32x4(x[u][t], acc);
#pragma unroll
                for (int r = 0; r < NMAX; ++r)
                    if (r < a.world) gfd::st16(a.pool[r] + vv * 16, acc);
            }
        }
    }
}

template <int DT, int NT>
__global__ void __launch_bounds__(kStepThreads)
step_kernel(const __grid_constant__ StepArgs a, const __grid_constant__ StepTable T) {
    __shared__ uint32_t s_task, s_epoch;
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        s_epoch = *reinterpret_cast<volatile uint32_t*>(a.ctl) + 1;
        s_ok = 1;
    }
    __syncthreads();
    const uint32_t e = s_epoch;
    const int n = NT > 0 ? NT : a.world;
    const bool solo = a.world == 1;  // no reduce tasks: unpack waits for the slab's own pack
    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(a.ctl + 1, 1u);
        __syncthreads();
        const uint32_t q = s_task;
        if (q >= a.ntasks || !s_ok) break;
        const uint32_t code = a.tasks[q], kind = code >> 30, t = code & 0x3FFFFFFFu;
        if (solo) {  // ---- world == 1: pack and unpack the slab in one pass, no flags
            pack_range<DT, true>(a, T, a.slab_a[t], a.slab_b[t]);
        } else if (kind == 0) {  // ---- pack slab t, then tell its owner
            pack_range<DT, false>(a, T, a.slab_a[t], a.slab_b[t]);
            __syncthreads();
            if (threadIdx.x == 0) {
                const int owner = a.ring[a.slab_pos[t]];
                if (owner == a.rank) {
                    __threadfence();  // only this GPU reads it: device scope suffices
                } else {
                    __threadfence_system();
                }
                st_release_sys32(a.packed_peer[owner] + uint64_t(t) * GF_MAX_RANKS + a.rank, e);
            }
        } else if (kind == 1) {  // ---- reduce one of my slabs once every rank packed it
            const uint32_t g = t;
            if (threadIdx.x < a.world &&
                !wait_ge(a, a.packed_peer[a.rank] + uint64_t(g) * GF_MAX_RANKS + threadIdx.x, e))
                s_ok = 0;
            __syncthreads();
            if (s_ok && a.world > 1) reduce_range<DT, NT>(a, n, a.pos, a.slab_a[g], a.slab_b[g]);
            __syncthreads();
            if (threadIdx.x < a.world) {
                __threadfence_system();
                st_release_sys32(a.reduced_peer[threadIdx.x] + g, e);
            }
        } else {  // ---- unpack a slab once its owner published the sum
            const uint32_t g = t;
            const uint32_t* flag = solo ? a.packed_peer[a.rank] + uint64_t(g) * GF_MAX_RANKS : a.reduced_peer[a.rank] + g;
            if (threadIdx.x == 0 && !wait_ge(a, flag, e)) s_ok = 0;
            __syncthreads();
            if (s_ok) unpack_range<DT>(a, T, a.slab_a[g], a.slab_b[g]);
        }
        __syncthreads();
    }
    // the last CTA out re-arms the queue and publishes the epoch for the next step
    if (threadIdx.x == 0 && atomicAdd(a.ctl + 2, 1u) == gridDim.x - 1) {
        reinterpret_cast<volatile uint32_t*>(a.ctl)[1] = 0;
        reinterpret_cast<volatile uint32_t*>(a.ctl)[2] = 0;
        reinterpret_cast<volatile uint32_t*>(a.ctl)[0] = e;
    }
}

template <int DT>
void launch_step(const StepArgs& a, const StepTable& T, int grid, cudaStream_t s) {
    switch (a.world) {
        case 1: step_kernel<DT, 1><<<grid, kStepThreads, 0, s>>>(a, T); break;
        case 2: step_kernel<DT, 2><<<grid, kStepThreads, 0, s>>>(a, T); break;
        case 4: step_kernel<DT, 4><<<grid, kStepThreads, 0, s>>>(a, T); break;
        case 8: step_kernel<DT, 8><<<grid, kStepThreads, 0, s>>>(a, T); break;
        default: step_kernel<DT, 0><<<grid, kStepThreads, 0, s>>>(a, T); break;
    }
}

// Slab size: 128 KB of pool (GF_STEP_SLAB=<elements> overrides).
uint64_t slab_elems(int dtype, int world, uint64_t total, int grid) {
    static const uint64_t forced = [] {
        const char* e = std::getenv("GF_STEP_SLAB");
        return e ? uint64_t(std::atoll(e)) : 0ull;
    }();
    if (forced) return forced;
    // measured (ResNet-50/AlexNet, 1-4 B200): per-task overhead outweighs a shorter tail,
    // so 128 KB slabs win at every world size
    (void)world;
    (void)total;
    (void)grid;
    return dtype == GF_F16 ? 65536 : 32768;
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
    // tensor table in pool order
    std::vector<int> order(static_cast<size_t>(ntensors));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return pool_off[x] < pool_off[y]; });
    StepTable T;
    std::memset(&T, 0, sizeof(T));
    T.n = ntensors;
    uint64_t hi = 0;
    for (int i = 0; i < ntensors; ++i) {
        const int k = order[static_cast<size_t>(i)];
        T.off[i] = pool_off[k];
        T.cnt[i] = count[k];
        T.src[i] = src[k];
        T.dst[i] = dst[k];
        if (i > 0 && T.off[i] < T.off[i - 1] + T.cnt[i - 1])
            return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: tensors overlap in the pool");
        hi = std::max(hi, T.off[i] + T.cnt[i]);
    }
    if (pool_heap_off + hi * es > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: pool outside the symmetric heap");
    DeviceGuard guard(c->device);
    if (c->world == 1)  // no collective: pack and unpack in one streaming pass
        return gfi::pack_unpack_solo(dtype, c->alloc + kFlagBytes + pool_heap_off, src, dst, pool_off, count,
                                     ntensors, gfi::S(stream));
    // ---- slab plan (cached per geometry) ---------------------------------------------
    static int grid = 0;
    if (grid == 0) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step_kernel<GF_F16, 8>, kStepThreads, 0);
        grid = std::max(1, occ) * gfi::sm_count();
    }
    uint64_t span = 0;
    for (int w = 0; w < nwin; ++w) span += win_len[w];
    const uint64_t SE = slab_elems(dtype, c->world, span, grid);
    std::string key = std::to_string(dtype) + "/" + std::to_string(c->pos) + "/" + std::to_string(SE) + "/" +
                      std::to_string(grid);
    for (int w = 0; w < nwin; ++w) key += "/" + std::to_string(win_start[w]) + ":" + std::to_string(win_len[w]);
    auto it = c->step_plans.find(key);
    if (it == c->step_plans.end()) {
        std::vector<uint64_t> A, B;
        std::vector<uint32_t> pos;
        std::vector<std::vector<uint32_t>> rounds;  // slab ids of each round
        std::vector<int64_t> mine;                  // my slab of each round (-1: none)
        const int n = c->world;
        for (int w = 0; w < nwin; ++w) {
            std::vector<std::vector<std::pair<uint64_t, uint64_t>>> segs(static_cast<size_t>(n));
            size_t most = 0;
            for (int j = 0; j < n; ++j) {  // segment_of(len, n, j) (collectives.cpp:47-53)
                const uint64_t base = win_len[w] / n, rem = win_len[w] % n;
                const uint64_t e0 = win_start[w] + j * base + std::min<uint64_t>(j, rem);
                const uint64_t e1 = e0 + base + (uint64_t(j) < rem ? 1 : 0);
                uint64_t x = e0;
                while (x < e1) {  // slab ends on absolute multiples of 8 elements
                    const uint64_t y = std::min(e1, (x / 8 * 8) + SE);
                    segs[static_cast<size_t>(j)].push_back({x, y});
                    x = y;
                }
                most = std::max(most, segs[static_cast<size_t>(j)].size());
            }
            for (size_t s = 0; s < most; ++s) {
                rounds.emplace_back();
                mine.push_back(-1);
                for (int j = 0; j < n; ++j) {
                    if (s >= segs[static_cast<size_t>(j)].size()) continue;
                    if (j == c->pos) mine.back() = static_cast<int64_t>(A.size());
                    rounds.back().push_back(static_cast<uint32_t>(A.size()));
                    A.push_back(segs[static_cast<size_t>(j)][s].first);
                    B.push_back(segs[static_cast<size_t>(j)][s].second);
                    pos.push_back(static_cast<uint32_t>(j));
                }
            }
        }
        if (A.size() > kStepMaxSlabs)
            return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: too many slabs (raise GF_STEP_SLAB)");
        // Task order over rounds: round r packs its slabs, reduces my slab of round r-D1
        // and unpacks round r-D2.
        // Measured on B200 (2-4 GPUs): lags shorter than the whole pack phase leave CTAs
        // spinning on flags that are not ready, so the default keeps the phases in order
        // (packs, then reduces, then unpacks) and overlap happens at the phase edges only.
        // GF_STEP_LAG=<rounds> enables the interleaved pipeline for experiments.
        const int64_t R = static_cast<int64_t>(rounds.size());
        static const int64_t lag = [] {
            const char* e = std::getenv("GF_STEP_LAG");
            return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(0);
        }();
        const int64_t D1 = n == 1 ? 0 : (lag ? lag : R);
        const int64_t D2 = n == 1 ? R + 1 : (lag ? 2 * lag : R + 1);  // n == 1: packs only
        std::vector<uint32_t> tasks;
        for (int64_t r = 0; r < R + D2; ++r) {
            if (r < R)
                for (uint32_t g : rounds[static_cast<size_t>(r)]) tasks.push_back((0u << 30) | g);
            if (n > 1 && r - D1 >= 0 && r - D1 < R && mine[static_cast<size_t>(r - D1)] >= 0)
                tasks.push_back((1u << 30) | static_cast<uint32_t>(mine[static_cast<size_t>(r - D1)]));
            if (n > 1 && r - D2 >= 0 && r - D2 < R)
                for (uint32_t g : rounds[static_cast<size_t>(r - D2)]) tasks.push_back((2u << 30) | g);
        }
        StepPlan sp;
        sp.nslab = static_cast<uint32_t>(A.size());
        sp.nmine = static_cast<uint32_t>(tasks.size());
        GF_CHECK_CUDA(cudaMalloc(&sp.slab_a, std::max<size_t>(A.size(), 1) * 8));
        GF_CHECK_CUDA(cudaMalloc(&sp.slab_b, std::max<size_t>(B.size(), 1) * 8));
        GF_CHECK_CUDA(cudaMalloc(&sp.slab_pos, std::max<size_t>(pos.size(), 1) * 4));
        GF_CHECK_CUDA(cudaMalloc(&sp.mine, std::max<size_t>(tasks.size(), 1) * 4));
        GF_CHECK_CUDA(cudaMemcpy(sp.slab_a, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
        GF_CHECK_CUDA(cudaMemcpy(sp.slab_b, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
        GF_CHECK_CUDA(cudaMemcpy(sp.slab_pos, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice));
        GF_CHECK_CUDA(cudaMemcpy(sp.mine, tasks.data(), tasks.size() * 4, cudaMemcpyHostToDevice));
        it = c->step_plans.emplace(key, sp).first;
    }
    const StepPlan& sp = it->second;
    StepArgs a;
    std::memset(&a, 0, sizeof(a));
    a.world = c->world;
    a.rank = c->rank;
    a.pos = c->pos;
    for (int r = 0; r < c->world; ++r) {
        a.pool[r] = c->peer_alloc[r] + kFlagBytes + pool_heap_off;
        a.packed_peer[r] = step_packed(c->peer_alloc[r]);
        a.reduced_peer[r] = step_reduced(c->peer_alloc[r]);
        a.ring[r] = c->ring[r];
    }
    a.ctl = step_ctl(c->alloc);
    a.slab_a = sp.slab_a;
    a.slab_b = sp.slab_b;
    a.slab_pos = sp.slab_pos;
    a.tasks = sp.mine;  // the plan's task queue
    a.nslab = sp.nslab;
    a.ntasks = sp.nmine;
    a.inv_world = 1.0f / static_cast<float>(c->world);
    a.timeout_ns = c->timeout_ns;
    a.err = c->err_dev;
    const int g = std::max(1, std::min<int>(grid, int(sp.nmine)));
    if (dtype == GF_F16) launch_step<GF_F16>(a, T, g, gfi::S(stream));
    else launch_step<GF_F32>(a, T, g, gfi::S(stream));
    gfi::count_launch();
    return gfi::check_launch("gf_sync_step_dense");
}

}  // extern "C"
