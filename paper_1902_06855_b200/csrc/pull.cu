// SPDX-License-Identifier: Apache-2.0
//
// Dense allreduce in pull form fused with the unpack (gf_ring_allreduce_unpack), and the
// dense-step entry point gf_sync_step_dense.
//
// Reference: ring_allreduce_on (src/collectives.cpp:55-97) over the FusionEngine windows
// (src/fusion.cpp:72-109), then the update read g_avg = get(i) * (1/N) (src/trainer.cpp:336-342).
//
// rsag_kernel: the rank at ring position p sums segment p of every window by PULLING it from
// all N pools in ring order (bit-identical to the reference's arrival order), keeps the sum in
// its own pool and unpacks it from registers; after one barrier with its peer CTAs it pulls
// every other segment from its owner into its pool and unpacks it. Nothing is pushed, so no
// barrier waits for posted NVLink writes to drain, and the separate unpack pass is gone.
//
// gf_sync_step_dense: world 1 is the one-pass pack_kernel<DstTable> (the collective is the
// identity, collectives.cpp:59); world > 1 is gf_pack -> gf_ring_allreduce -> gf_unpack.

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ring_device.cuh"
#include "step_table.cuh"

namespace {

// ---- gf_ring_allreduce_unpack: pull reduce-scatter, then pull all-gather fused with unpack ----
// The rank at ring position p sums segment p of every window from all N pools in ring order
// (the reference's arrival order, as reduce_segment), keeps the sum in its OWN pool only and
// unpacks it from registers. After one barrier with its peer CTAs it PULLS every other
// segment from the rank that owns it, writes it into its pool (every pool ends holding the
// sums, as after ring_allreduce) and unpacks it. Nothing is pushed, so no barrier waits for
// posted NVLink writes to drain; and the separate unpack pass (re-reading the pool) is gone.
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
rsag_kernel(const __grid_constant__ RingArgs a, const __grid_constant__ StepTable T, float inv, int exit_barrier,
            const char* __restrict__ inbox, uint64_t slot_bytes) {
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
    flat_build<VE>(a, n, a.pos, flat);  // my segment of every window
    if (!cross_barrier(a, epoch + 1, &s_ok, false)) return;  // peers' pools are packed
    if (tr) a.trace[1] = gfd::globaltimer_ns();
    // reduce-scatter operands in ring order from my position: pulled from the peers' pools, or
    // (inbox != null, the push form) my pool + my inbox slots, where the peers' routed packs
    // stored them: slot s holds position pos+1+s (gf_sync_step_dense_push)
    const char* src[NMAX];
#pragma unroll
    for (int t = 0; t < NMAX; ++t) {
        if (t >= n) src[t] = nullptr;
        else if (inbox) src[t] = t == 0 ? a.bufs[a.rank] : inbox + uint64_t(t - 1) * slot_bytes;
        else src[t] = a.bufs[a.ring[(a.pos + t) % n]];
    }
    char* local = a.bufs[a.rank];
    pull_flat<DT, NT, true>(a, T, src, n, local, flat, g, S, inv);
    if (tr) a.trace[2] = gfd::globaltimer_ns();
    if (!cross_barrier(a, epoch + 2, &s_ok, true)) return;  // my segment sums are visible
    for (int j = 1; j < n; ++j) {  // next ring position first: owners differ across ranks
        const int q = (a.pos + j) % n;
        flat_build<VE>(a, n, q, flat);
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
void launch_rsag(const RingArgs& a, const StepTable& T, float inv, int exit_barrier, const char* inbox,
                 uint64_t slot_bytes, int grid, cudaStream_t s) {
    switch (a.world) {
        case 2: rsag_kernel<DT, 2><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier, inbox, slot_bytes); break;
        case 3: rsag_kernel<DT, 3><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier, inbox, slot_bytes); break;
        case 4: rsag_kernel<DT, 4><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier, inbox, slot_bytes); break;
        case 8: rsag_kernel<DT, 8><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier, inbox, slot_bytes); break;
        default: rsag_kernel<DT, 0><<<grid, kRingThreads, 0, s>>>(a, T, inv, exit_barrier, inbox, slot_bytes); break;
    }
}

// tensor table in pool order; checks the tensors tile [off[0], hi) without overlap
}  // namespace

namespace gfr {

int rsag_launch(gf_comm* c, int dtype, uint64_t pool_heap_off, const char* inbox, uint64_t slot_bytes,
                float* const* dst, const uint64_t* pool_off, const uint64_t* count, int ntensors,
                const uint64_t* win_start, const uint64_t* win_len, int nwin, int flags, void* stream,
                const char* fn) {
    if (!gfi::valid_dtype(dtype) || ntensors < 1 || ntensors > kStepMaxT || !dst || !pool_off || !count ||
        nwin < 1 || !win_start || !win_len || (flags & ~GF_RSAG_NO_EXIT_BARRIER))
        return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": bad arguments (1..256 tensors, >= 1 window)");
    StepTable T;
    uint64_t hi = 0;
    if (int rc = build_table(fn, nullptr, dst, pool_off, count, ntensors, T, hi)) return rc;
    const uint64_t es = gfi::esz(dtype);
    if (pool_heap_off + hi * es > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, std::string(fn) + ": pool outside the symmetric heap");
    if (int rc = check_tiling(fn, T, hi, win_start, win_len, nwin)) return rc;
    DeviceGuard guard(c->device);
    if (c->world == 1)  // the collective is the identity (collectives.cpp:59)
        return gf_unpack(dtype, c->alloc + kFlagBytes + pool_heap_off, dst, pool_off, count, ntensors, 1, stream);
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
        const int grid = gfr::comm_blocks(c, max_seg * es);
        if (dtype == GF_F16) launch_rsag<GF_F16>(a, T, inv, exit_barrier, inbox, slot_bytes, grid, gfi::S(stream));
        else launch_rsag<GF_F32>(a, T, inv, exit_barrier, inbox, slot_bytes, grid, gfi::S(stream));
        gfi::count_launch();
        if (int rc = gfi::check_launch(fn)) return rc;
    }
    return GF_OK;
}

}  // namespace gfr

extern "C" {

int gf_sync_step_dense(gf_comm* c, int dtype, uint64_t pool_heap_off, const float* const* src,
                       float* const* dst, const uint64_t* pool_off, const uint64_t* count,
                       int ntensors, const uint64_t* win_start, const uint64_t* win_len, int nwin,
                       void* stream) {
    if (int rc = comm_ready(c)) return rc;
    if (!gfi::valid_dtype(dtype) || ntensors < 1 || !src || !dst || !pool_off || !count || nwin < 1 || !win_start ||
        !win_len)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: bad arguments (>= 1 tensor, >= 1 window)");
    const uint64_t es = gfi::esz(dtype);
    uint64_t hi = 0;
    for (int t = 0; t < ntensors; ++t) hi = std::max(hi, pool_off[t] + count[t]);
    if (pool_heap_off + hi * es > c->heap_bytes)
        return gfi::fail(GF_ERR_CONFIG, "gf_sync_step_dense: pool outside the symmetric heap");
    DeviceGuard guard(c->device);
    char* pool = c->alloc + kFlagBytes + pool_heap_off;
    if (c->world == 1)  // no collective: pack and unpack in one streaming pass
        return gfi::pack_unpack_solo(dtype, pool, src, dst, pool_off, count, ntensors, gfi::S(stream));
    if (int rc = gf_pack(dtype, pool, src, pool_off, count, ntensors, 1.0f, stream)) return rc;
    if (int rc = gf_ring_allreduce(c, dtype, pool_heap_off, win_start, win_len, nwin, stream)) return rc;
    return gf_unpack(dtype, pool, dst, pool_off, count, ntensors, c->world, stream);
}

int gf_ring_allreduce_unpack(gf_comm* c, int dtype, uint64_t pool_heap_off, float* const* dst,
                             const uint64_t* pool_off, const uint64_t* count, int ntensors,
                             const uint64_t* win_start, const uint64_t* win_len, int nwin, int flags,
                             void* stream) {
    if (int rc = comm_ready(c)) return rc;
    return gfr::rsag_launch(c, dtype, pool_heap_off, nullptr, 0, dst, pool_off, count, ntensors, win_start, win_len,
                            nwin, flags, stream, "gf_ring_allreduce_unpack");
}

}  // extern "C"
