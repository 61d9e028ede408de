// SPDX-License-Identifier: Apache-2.0
//
// The dense step in push form (gf_sync_step_dense_push): the reduce-scatter's traffic rides
// on the pack.
//
//   1. pack_push   fp32 tensors -> fp16, and every packed vector is STORED where the ring will
//                  reduce it: the rank at ring position j owns segment j of every window
//                  (segment_of, src/collectives.cpp:47-53), so a vector of segment j goes to my
//                  own pool when j is my position, else into my slot of rank ring[j]'s inbox
//                  over NVLink. The pack's HBM reads and the scatter's NVLink writes overlap.
//   2. rsp_kernel  after the entry barrier every operand of my segments is LOCAL (my pool + my
//                  inbox slots): the sums, in ring order from my position (the reference's
//                  arrival order, bit-identical), are pushed into every rank's pool (the
//                  all-gather as posted writes), then the exit barrier.
//   3. unpack      (K6) g_avg = dec(pool) * 1/N.
//
// Per rank and direction the NVLink bytes are the ring's 2(N-1)/N * K: (N-1)/N * K pushed by
// the pack and (N-1)/N * K by the all-gather. Inbox slot s of the owner at position j holds
// the contribution of the rank at position j + 1 + s (mod N), laid out like the pool.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "ring_device.cuh"
#include "step_table.cuh"
#include "tensor_table.cuh"

namespace {

struct SegMap {  // routing of pool elements to their owners (explicit windows)
    int nwin, world, pos, diag;  // diag: GF_PUSH_DIAG timing probe (1: every store local; results invalid)
    uint64_t slot_elems;                 // elements per inbox slot (the pool span)
    char* pool_local;                    // my pool (fp16)
    char* inbox_by_pos[GF_MAX_RANKS];    // owner at ring position j: its inbox as mapped here
    uint64_t wstart[kMaxW];
    uint64_t wlen[kMaxW];
};

// Per-tile routing table in shared memory. A tile lies inside one tensor, hence inside one
// window (windows are cut at tensor boundaries), so it meets at most world-1 segment
// boundaries: one thread computes that window's segment_of starts (src/collectives.cpp:47-53,
// one 64-bit division per tile) and each owner's destination base; every vector then finds its
// owner with a few compares instead of divisions.
struct TileRoute {
    uint64_t start[GF_MAX_RANKS + 1];  // segment j of the tile's window: [start[j], start[j+1])
    uint16_t* dst[GF_MAX_RANKS];       // owner j's destination base (pool indices)
};

__device__ __forceinline__ void tile_route(const SegMap& m, uint64_t e, TileRoute& r) {
    int lo = 0, hi = m.nwin;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (m.wstart[mid] <= e) lo = mid; else hi = mid;
    }
    const uint64_t n = uint64_t(m.world), L = m.wlen[lo], ws = m.wstart[lo];
    const uint64_t base = L / n, rem = L % n;
    for (int j = 0; j <= m.world; ++j) r.start[j] = ws + uint64_t(j) * base + min(uint64_t(j), rem);
    for (int j = 0; j < m.world; ++j) {
        if (j == m.pos || m.diag == 1) {
            r.dst[j] = reinterpret_cast<uint16_t*>(m.pool_local);
        } else {  // inbox slot s of the owner at position j holds position j + 1 + s
            const int slot = (m.pos - j - 1 + m.world) % m.world;
            r.dst[j] = reinterpret_cast<uint16_t*>(m.inbox_by_pos[j]) + uint64_t(slot) * m.slot_elems;
        }
    }
}

__device__ __forceinline__ int tile_owner(const TileRoute& r, int world, uint64_t e) {
    int j = 0;
    while (j + 1 < world && r.start[j + 1] <= e) ++j;
    return j;
}

template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
pack_push_kernel(const __grid_constant__ TensorTable T, const __grid_constant__ SegMap M, uint64_t total_tiles,
                 uint64_t spread, int fence) {
    __shared__ TileRoute R;
    // CTA i packs tile (i * spread) mod tiles (spread coprime with tiles, ~tiles/N): consecutive
    // CTAs hit different segments, so every rank keeps all its peers' links busy at once
    // instead of streaming one owner's segment after another
    for (uint64_t i = blockIdx.x; i < total_tiles; i += gridDim.x) {
        const uint64_t tile = (i * spread) % total_tiles;
        const int t = find_tensor(T, tile);
        const uint64_t base = (tile - T.tiles[t]) * kTile;
        const uint64_t len = min(kTile, T.cnt[t] - base);
        const float* __restrict__ s = static_cast<const float*>(T.ptr[t]) + base;
        const uint64_t po = T.off[t] + base;
        __syncthreads();  // the previous tile's readers of R are done
        if (threadIdx.x == 0) tile_route(M, po, R);
        __syncthreads();
        auto put = [&](uint64_t e, uint16_t h) { R.dst[tile_owner(R, M.world, e)][e] = h; };
        uint64_t done = 0;
        if ((reinterpret_cast<uintptr_t>(T.ptr[t]) & 31u) == 0 && po % 8 == 0) {
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
                    const uint4 h = gfd::enc8(a[k], b[k]);
                    const uint64_t e = po + 8 * uint64_t(v);
                    const int j = tile_owner(R, M.world, e);
                    if (e + 8 <= R.start[j + 1]) {  // the whole vector belongs to one owner
                        gfd::st16(R.dst[j] + e, h);
                    } else {                         // a segment boundary inside the vector
                        const uint32_t w[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
                        for (int q = 0; q < 8; ++q) put(e + q, uint16_t((w[q >> 1] >> ((q & 1) * 16)) & 0xFFFFu));
                    }
                }
            }
            done = uint64_t(nvec) * 8;
        }
        for (uint64_t q = done + threadIdx.x; q < len; q += kThreads) put(po + q, gfd::enc(s[q]));
    }
    // No fence by default: CTAs retire with their NVLink stores in flight. The kernel boundary
    // orders all of them before rsp_kernel, whose release of the entry flag publishes them
    // (the ordering argument and the stress test that backs it). GF_PUSH_FENCE=1
    // adds a system-scope fence per thread — the provable form, for validation runs.
    if (fence) __threadfence_system();
}

// CTAs per SM the routed pack is compiled for (register cap 65536 / (256 * MINB)); 4 measured
// best so far. GF_PUSH_MINB (4, 6 or 8) is a tuning override.
int push_minb() {
    static const int v = [] {
        const char* e = std::getenv("GF_PUSH_MINB");
        const int x = e ? std::atoi(e) : 4;
        return (x == 6 || x == 8) ? x : 4;
    }();
    return v;
}

// All-local reduce of my segments (pool + inbox slots, ring order) pushed to every pool.
// UNPACK: the step's unpack is fused in — my segments' g_avg straight from the sums in
// registers while the pushes drain, and after the exit barrier the other segments from my pool:
// CTA b unpacks exactly the vectors its peer CTAs b pushed to me (the same flat sweep on the
// owner's segment), which is what its CTA-pair exit barrier covers.
template <int NT, bool UNPACK>
__global__ void __launch_bounds__(kRingThreads, 1)
rsp_kernel(const __grid_constant__ RingArgs a, const char* __restrict__ inbox_local, uint64_t slot_bytes,
           const __grid_constant__ StepTable TT, float inv) {
    constexpr int NMAX = NT > 0 ? NT : GF_MAX_RANKS;
    constexpr int U = NMAX <= 4 ? 4 : (NMAX <= 8 ? 2 : 1);
    __shared__ int s_ok;
    __shared__ FlatWins flat;
    const uint64_t epoch = a.epochs[blockIdx.x];
    if (threadIdx.x == 0) s_ok = 1;
    const int n = NT > 0 ? NT : a.world;
    flat_build<8>(a, n, a.pos, flat);
    const bool tr = a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) a.trace[0] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 1, &s_ok, false)) return;  // every peer's pack (and its pushes) is done
    if (tr) a.trace[1] = gfd::globaltimer_ns();
    const char* src[NMAX];  // ring order from my position: me, then the slots
    char* dst[NMAX];        // every rank's pool, the next one on the ring first
#pragma unroll
    for (int t = 0; t < NMAX; ++t) {
        src[t] = t == 0 ? a.bufs[a.rank] : (t < n ? inbox_local + uint64_t(t - 1) * slot_bytes : nullptr);
        dst[t] = t < n ? a.bufs[a.ring[(a.pos + 1 + t) % n]] : nullptr;
    }
    auto unpack_elem = [&](uint64_t e, uint16_t h) {
        const int t = tensor_at(TT, e);
        TT.dst[t][e - TT.off[t]] = gfd::mul(gfd::dec(h), inv);
    };
    // unaligned edges of window w: CTA w mod grid, scalar
    for (int w = int(blockIdx.x); w < a.nwin; w += int(gridDim.x)) {
        const uint64_t e0 = flat.e0[w], e1 = flat.e1[w], v0 = flat.v0[w], v1 = v0 + (flat.pre[w + 1] - flat.pre[w]);
        auto edge = [&](uint64_t lo, uint64_t hi) {
            for (uint64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
                uint16_t acc = reinterpret_cast<const uint16_t*>(src[0])[e];
                for (int t = 1; t < n; ++t) acc = gfd::acc16(reinterpret_cast<const uint16_t*>(src[t])[e], acc);
                for (int t = 0; t < n; ++t) reinterpret_cast<uint16_t*>(dst[t])[e] = acc;
                if (UNPACK) unpack_elem(e, acc);
            }
        };
        if (v1 > v0) {
            edge(e0, v0 * 8);
            edge(v1 * 8, e1);
        } else {
            edge(e0, e1);
        }
    }
    const uint64_t total = flat.pre[a.nwin];
    const uint64_t T = uint64_t(gridDim.x) * blockDim.x, g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (uint64_t x = g; x < total; x += T * U) {
        uint4 v[U][NMAX];
        uint64_t vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t xu = x + uint64_t(u) * T;
            vv[u] = ~0ull;
            if (xu < total) {
                const int w = flat_window(flat, a.nwin, xu);
                vv[u] = flat.v0[w] + (xu - flat.pre[w]);
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
                if (t < n) acc = gfd::acc16x8(v[u][t], acc);
#pragma unroll
            for (int t = 0; t < NMAX; ++t)
                if (t < n) gfd::st16(dst[t] + vv[u] * 16, acc);
            if (UNPACK) unpack_vec<GF_F16>(TT, vv[u], acc, inv);
        }
    }
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 2, &s_ok, true)) return;  // every push into my pool landed
    if (threadIdx.x == 0) a.epochs[blockIdx.x] = epoch + 2;
    if (tr) a.trace[3] = gfd::globaltimer_ns();
    if (!UNPACK) return;
    // the other owners' segments, as their CTA b pushed them
    const uint16_t* pool = reinterpret_cast<const uint16_t*>(a.bufs[a.rank]);
    for (int j = 1; j < n; ++j) {
        const int q = (a.pos + j) % n;
        flat_build<8>(a, n, q, flat);
        for (int w = int(blockIdx.x); w < a.nwin; w += int(gridDim.x)) {
            const uint64_t e0 = flat.e0[w], e1 = flat.e1[w], v0 = flat.v0[w],
                           v1 = v0 + (flat.pre[w + 1] - flat.pre[w]);
            const uint64_t h0 = v1 > v0 ? v0 * 8 : e1;
            for (uint64_t e = e0 + threadIdx.x; e < h0; e += blockDim.x)
                unpack_elem(e, reinterpret_cast<const volatile uint16_t*>(pool)[e]);
            if (v1 > v0)
                for (uint64_t e = v1 * 8 + threadIdx.x; e < e1; e += blockDim.x)
                    unpack_elem(e, reinterpret_cast<const volatile uint16_t*>(pool)[e]);
        }
        const uint64_t tq = flat.pre[a.nwin];
        for (uint64_t x = g; x < tq; x += T * 4) {
            uint4 h[4];
            uint64_t vq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t xu = x + uint64_t(u) * T;
                vq[u] = ~0ull;
                if (xu < tq) {
                    const int w = flat_window(flat, a.nwin, xu);
                    vq[u] = flat.v0[w] + (xu - flat.pre[w]);
                    h[u] = ld16_cg<GF_F16>(a.bufs[a.rank] + vq[u] * 16);  // pushed by a peer: skip L1
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (vq[u] != ~0ull) unpack_vec<GF_F16>(TT, vq[u], h[u], inv);
        }
    }
    if (tr) a.trace[3] = gfd::globaltimer_ns();
}

// GF_PUSH_DIAG timing probes (results invalid by design): 1 every routed store local, 2 the
// routed pack alone (no reduce / all-gather / unpack).
int push_fence() {
    static const int v = [] {
        const char* e = std::getenv("GF_PUSH_FENCE");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

int push_diag() {
    static const int v = [] {
        const char* e = std::getenv("GF_PUSH_DIAG");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// The routed pack of one group of <= kMaxW windows (the tensors inside them).
int routed_pack(gf_comm* c, cudaStream_t s, uint64_t pool_heap_off, uint64_t inbox_heap_off, uint64_t slot_elems,
                const float* const* src, const uint64_t* pool_off, const uint64_t* count, int ntensors,
                const uint64_t* win_start, const uint64_t* win_len, int nwin) {
    SegMap M;
    std::memset(&M, 0, sizeof(M));
    M.nwin = nwin;
    M.world = c->world;
    M.pos = c->pos;
    M.slot_elems = slot_elems;
    M.pool_local = c->alloc + kFlagBytes + pool_heap_off;
    M.diag = push_diag();
    for (int j = 0; j < c->world; ++j) M.inbox_by_pos[j] = c->peer_alloc[c->ring[j]] + kFlagBytes + inbox_heap_off;
    for (int w = 0; w < nwin; ++w) {
        M.wstart[w] = win_start[w];
        M.wlen[w] = win_len[w];
    }
    return for_each_table(reinterpret_cast<const void* const*>(src), pool_off, count, ntensors,
                          [&](const TensorTable& T, uint64_t tiles, int grid) {
                              uint64_t spread = std::max<uint64_t>(1, tiles / uint64_t(c->world));
                              while (std::gcd(spread, tiles) != 1) ++spread;
                              switch (push_minb()) {
                                  case 6: pack_push_kernel<6><<<grid, kThreads, 0, s>>>(T, M, tiles, spread, push_fence()); break;
                                  case 8: pack_push_kernel<8><<<grid, kThreads, 0, s>>>(T, M, tiles, spread, push_fence()); break;
                                  default: pack_push_kernel<4><<<grid, kThreads, 0, s>>>(T, M, tiles, spread, push_fence()); break;
                              }
                          });
}

// The unpack fused into rsp_kernel or a separate unpack launch. Measured: fused wins
// at N=2 (the own half is unpacked while the pushes drain; AlexNet 0.274 vs 0.285 ms), but from
// N=4 the (N-1)/N of the pool unpacked after the exit barrier by the 1-CTA-per-SM grid costs more
// than a separate full-grid unpack (ResNet-50 0.187 vs 0.178 ms). GF_FUSE_UNPACK=0/1 overrides.
bool fuse_unpack(int world) {
    static const int v = [] {
        const char* e = std::getenv("GF_FUSE_UNPACK");
        return e ? std::atoi(e) : -1;
    }();
    return v < 0 ? world == 2 : v != 0;
}

}  // namespace

extern "C" {

int gf_sync_step_dense_push(gf_comm* c, int dtype, uint64_t pool_heap_off, uint64_t inbox_heap_off,
                            const float* const* src, float* const* dst, const uint64_t* pool_off,
                            const uint64_t* count, int ntensors, const uint64_t* win_start,
                            const uint64_t* win_len, int nwin, void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (dtype != GF_F16 || ntensors < 1 || !src || !dst || !pool_off || !count || nwin < 1 || !win_start || !win_len)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: fp16 pool, >= 1 tensor, >= 1 window");
    if (c->world == 1)  // no collective: the one-pass pack + unpack
        return gf_sync_step_dense(c, dtype, pool_heap_off, src, dst, pool_off, count, ntensors, win_start, win_len,
                                  nwin, stream);
    uint64_t lo = UINT64_MAX, hi = 0, cover = win_start[0];
    for (int i = 0; i < ntensors; ++i) {
        lo = std::min(lo, pool_off[i]);
        hi = std::max(hi, pool_off[i] + count[i]);
    }
    for (int w = 0; w < nwin; ++w) {
        if (win_start[w] != cover) return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: windows must be contiguous");
        cover += win_len[w];
    }
    if (lo != win_start[0] || hi != cover)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: tensors and windows must cover the same pool range");
    // an inbox slot mirrors pool indices [0, hi); its stride is rounded up to 8 elements so every
    // slot base stays 16-byte aligned for the vector stores and loads
    const uint64_t slot_elems = (hi + 7) & ~uint64_t(7);
    const uint64_t pool_end = pool_heap_off + hi * 2, inbox_end = inbox_heap_off + uint64_t(c->world - 1) * slot_elems * 2;
    if (pool_end > c->heap_bytes || inbox_end > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: pool or inbox outside the symmetric heap");
    if (pool_heap_off % 16 != 0 || inbox_heap_off % 16 != 0)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: pool and inbox offsets must be 16-byte aligned");
    if (pool_heap_off < inbox_end && inbox_heap_off < pool_end)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: pool and inbox ranges overlap");
    DeviceGuard guard(c->device);
    cudaStream_t s = gfi::S(stream);
    const char* inbox_local = c->alloc + kFlagBytes + inbox_heap_off;
    // the unpack rides in rsp_kernel when the tensors fit its table and one launch covers the
    // windows (the usual case); otherwise a separate unpack follows
    const bool fused = ntensors <= kStepMaxT && nwin <= kMaxW && fuse_unpack(c->world);
    StepTable TT;
    std::memset(&TT, 0, sizeof(TT));
    if (fused) {
        uint64_t hi2 = 0;
        if (int rc = build_table("gf_sync_step_dense_push", nullptr, dst, pool_off, count, ntensors, TT, hi2)) return rc;
    }
    const float inv = 1.0f / static_cast<float>(c->world);
    // Windows go in groups of <= kMaxW per launch pair; windows are cut at tensor boundaries,
    // so every tensor belongs to exactly one group.
    std::vector<const void*> gsrc;
    std::vector<uint64_t> goff, gcnt;
    for (int first = 0; first < nwin; first += kMaxW) {
        const int nw = std::min(kMaxW, nwin - first);
        const uint64_t g0 = win_start[first], g1 = win_start[first + nw - 1] + win_len[first + nw - 1];
        gsrc.clear();
        goff.clear();
        gcnt.clear();
        for (int i = 0; i < ntensors; ++i) {
            if (pool_off[i] < g0 || pool_off[i] >= g1) continue;
            if (pool_off[i] + count[i] > g1)
                return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense_push: a tensor straddles a window boundary");
            gsrc.push_back(src[i]);
            goff.push_back(pool_off[i]);
            gcnt.push_back(count[i]);
        }
        // 1. pack, routed to the owners
        gfi::phase("pack_push", s);
        if (int rc = routed_pack(c, s, pool_heap_off, inbox_heap_off, slot_elems,
                                 reinterpret_cast<const float* const*>(gsrc.data()), goff.data(), gcnt.data(),
                                 int(gsrc.size()), win_start + first, win_len + first, nw))
            return rc;
        if (push_diag() == 2) continue;  // timing probe: the routed pack alone (results invalid)
        // 2. local reduce + all-gather push (+ the unpack when fused)
        RingArgs a;
        std::memset(&a, 0, sizeof(a));
        a.nwin = nw;
        uint64_t max_seg = 0;
        for (int w = 0; w < nw; ++w) {
            a.wstart[w] = win_start[first + w];
            a.wlen[w] = win_len[first + w];
            max_seg += (a.wlen[w] + c->world - 1) / c->world;
        }
        fill_common(c, a, pool_heap_off);
        const int grid = gfr::comm_blocks(c, max_seg * 2);
        gfi::phase("rsp", s);
        const uint64_t sb = slot_elems * 2;
#define GF_RSP(NT_)                                                                                  \
    if (fused) rsp_kernel<NT_, true><<<grid, kRingThreads, 0, s>>>(a, inbox_local, sb, TT, inv);     \
    else rsp_kernel<NT_, false><<<grid, kRingThreads, 0, s>>>(a, inbox_local, sb, TT, inv);
        switch (c->world) {
            case 2: GF_RSP(2) break;
            case 4: GF_RSP(4) break;
            case 8: GF_RSP(8) break;
            default: GF_RSP(0) break;
        }
#undef GF_RSP
        gfi::count_launch();
        if (int rc = gfi::check_launch("gf_sync_step_dense_push")) return rc;
    }
    if (fused || push_diag() == 2) return GF_OK;
    // 3. unpack
    gfi::phase("unpack", s);
    return gf_unpack(dtype, c->alloc + kFlagBytes + pool_heap_off, dst, pool_off, count, ntensors, c->world, stream);
}

}  // extern "C"
