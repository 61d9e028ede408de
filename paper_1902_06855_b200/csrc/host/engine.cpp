// SPDX-License-Identifier: Apache-2.0
//
// gf_engine: one rank's whole gradient-synchronisation iteration on the device (C-ABI in
// include/gflow_b200.h). This is the sync half of the reference's train_worker
// (src/trainer.cpp:297-347) with its FusionEngine (src/fusion.cpp:25-123) and SparseState
// (src/sparse.cpp:57-224), re-planned for one B200 per rank:
//
//   dense, world 1   gf_sync_step_dense: one streaming pass (the collective is the identity,
//                    collectives.cpp:59)
//   dense, world > 1 RSPUSH  gf_sync_step_dense_push: the pack routes every vector to the owner of
//                            its segment (NVLink stores); local reduce + all-gather push with
//                            the unpack fused in
//                    PULL    gf_pack -> gf_ring_allreduce_unpack (two pools used alternately)
//                    PUSH    gf_pack -> gf_ring_allreduce -> gf_unpack
//   CSC              the other chunks' gf_csc_pack_correct_part on a side stream, beside the
//                    selected chunks' pack (routed to the exchange owners from 4 ranks) and the
//                    exchange + write-back + exact L1 (ring or routed form) on a highest-priority
//                    stream -> gf_csc_select (next set) beside gf_csc_sgd_update
//
// Every FusionEngine theta window of an iteration goes into ONE flattened launch (they are all
// known up front); the overlap API (begin_iteration / tensor_complete / finalize) launches
// each window on a communication stream as it closes, FIFO like the reference's progress
// thread. Nothing here synchronises with the host inside a step.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "gflow/sparse.hpp"  // sparsity_at / selection_count (sparse.cpp:13-24)
#include "gflow_b200.h"

namespace gfi {
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
using PhaseHook = void (*)(void* ctx, const char* name, cudaStream_t s);
void set_phase_hook(PhaseHook hook, void* ctx);
}  // namespace gfi

namespace {

constexpr uint64_t align_up(uint64_t x, uint64_t a = 256) { return (x + a - 1) / a * a; }

#define GF_ENG_CUDA(expr)                                       \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return gfi::cuda_fail(_e, #expr); \
    } while (0)
#define GF_ENG_OK(expr)               \
    do {                              \
        int _rc = (expr);             \
        if (_rc != GF_OK) return _rc; \
    } while (0)

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

struct gf_engine {
    gf_engine_config cfg{};
    int m = 0;  // tensors
    std::vector<uint64_t> sizes, offs;  // by id-1; offs: pool offset (tensor m at 0)
    uint64_t total = 0, nc = 0, esz = 2;
    int dense_mode = GF_DENSE_PUSH;
    // symmetric heap layout (bytes)
    uint64_t pool_off = 0, pull_pools[2] = {0, 0}, push_inbox = UINT64_MAX, stage_off = 0, norms_off = 0,
             inbox_off = 0, heap = 0;
    uint64_t csc_inbox = UINT64_MAX, csc_slot = 0;  // routed CSC exchange (csc_mode PULL, fp16)
    int pull_flip = 0;
    bool pull_two_pools = false;
    gf_comm* comm = nullptr;
    char* heap_base = nullptr;
    char* last_pool = nullptr;
    std::vector<uint64_t> ws, wl;  // dense theta windows
    // CSC state (one device allocation)
    char* state = nullptr;
    float *hg = nullptr, *hu = nullptr, *w = nullptr;
    uint8_t* imp[2] = {};
    uint64_t* coff[2] = {};
    uint64_t* plan[2] = {};
    uint64_t* nacc = nullptr;
    uint64_t iteration = 0;
    int xblocks = 0;   // CTAs of the CSC exchange (the packing of the other chunks runs beside it)
    int xthreads = 0;  // their size (0: 512)
    // streams / events (created on the engine's device, non-blocking)
    cudaStream_t side = nullptr, comm_s = nullptr;
    cudaStream_t hp = nullptr;  // highest priority: the CSC critical path (selected chunks + exchange)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_ready = nullptr, ev_done = nullptr, ev_sel = nullptr,
                ev_rest = nullptr, ev_x = nullptr;
    // overlap state
    bool ov_on = false;
    std::vector<const float*> ov_grad;
    std::vector<float*> ov_out;
    cudaStream_t ov_stream = nullptr;
    uint64_t ov_ws = 0, ov_we = 0;
    std::vector<int> ov_ids;
    int ov_launched = 0;
    // per-kernel timing marks
    bool marks_on = false;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;  // in launch order, "" = step end
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
};

namespace {

void mark(gf_engine* e, const char* name, cudaStream_t s) {
    if (!e->marks_on) return;
    if (e->ev_used == e->ev_pool.size()) {
        cudaEvent_t ev;
        if (cudaEventCreate(&ev) != cudaSuccess) return;
        e->ev_pool.push_back(ev);
    }
    cudaEvent_t ev = e->ev_pool[e->ev_used++];
    cudaEventRecord(ev, s);
    e->marks.emplace_back(name ? name : "", ev);
}

void phase_hook(void* ctx, const char* name, cudaStream_t s) { mark(static_cast<gf_engine*>(ctx), name, s); }

struct PhaseScope {  // routes the C-ABI's inner phase marks to this engine while a step runs
    bool on;
    PhaseScope(gf_engine* e) : on(e->marks_on) {
        if (on) gfi::set_phase_hook(phase_hook, e);
    }
    ~PhaseScope() {
        if (on) gfi::set_phase_hook(nullptr, nullptr);
    }
};

// FusionEngine windows of one iteration (fusion.cpp:72-109): tensors complete in descending
// id, a window closes when its bytes reach theta, finalize flushes the rest.
void dense_windows(gf_engine* e) {
    uint64_t a = 0, b = 0;
    for (int id = e->m; id >= 0; --id) {
        const bool flush = id == 0;
        if (!flush) b = e->offs[id - 1] + e->sizes[id - 1];
        const bool hit = e->cfg.theta_bytes != GF_THETA_INFINITE && (b - a) * e->esz >= e->cfg.theta_bytes;
        if (b > a && (hit || flush)) {
            e->ws.push_back(a);
            e->wl.push_back(b - a);
            a = b;
        }
    }
}

int create_streams(gf_engine* e) {
    GF_ENG_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    GF_ENG_CUDA(cudaStreamCreateWithFlags(&e->comm_s, cudaStreamNonBlocking));
    int least = 0, greatest = 0;
    GF_ENG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    GF_ENG_CUDA(cudaStreamCreateWithPriority(&e->hp, cudaStreamNonBlocking, greatest));
    for (cudaEvent_t* ev : {&e->ev_a, &e->ev_b, &e->ev_ready, &e->ev_done, &e->ev_sel, &e->ev_rest, &e->ev_x})
        GF_ENG_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    return GF_OK;
}

int alloc_csc_state(gf_engine* e) {
    const uint64_t T = e->total, nc = e->nc;
    const uint64_t sz_f = align_up(T * 4), sz_imp = align_up(nc), sz_coff = align_up(nc * 8),
                   sz_plan = align_up((4 + nc) * 8), sz_nacc = align_up(nc * 8);
    const uint64_t bytes = 3 * sz_f + 2 * (sz_imp + sz_coff + sz_plan) + sz_nacc;
    GF_ENG_CUDA(cudaMalloc(&e->state, bytes));
    GF_ENG_CUDA(cudaMemsetAsync(e->state, 0, bytes, e->side));
    char* p = e->state;
    e->hg = reinterpret_cast<float*>(p); p += sz_f;
    e->hu = reinterpret_cast<float*>(p); p += sz_f;
    e->w = reinterpret_cast<float*>(p); p += sz_f;
    for (int i = 0; i < 2; ++i) {
        e->imp[i] = reinterpret_cast<uint8_t*>(p); p += sz_imp;
        e->coff[i] = reinterpret_cast<uint64_t*>(p); p += sz_coff;
        e->plan[i] = reinterpret_cast<uint64_t*>(p); p += sz_plan;
    }
    e->nacc = e->cfg.dtype == GF_F16 ? reinterpret_cast<uint64_t*>(p) : nullptr;
    // iteration 0 is dense (sparse.cpp:45-51): every chunk important, its plan built up front
    GF_ENG_CUDA(cudaMemsetAsync(e->imp[0], 1, nc, e->side));
    GF_ENG_OK(gf_csc_plan(e->imp[0], T, e->cfg.chunk, nc, e->cfg.dtype, e->cfg.theta_bytes, e->coff[0], e->plan[0],
                          e->side));
    GF_ENG_CUDA(cudaStreamSynchronize(e->side));
    return GF_OK;
}

int after_connect(gf_engine* e) {
    if (e->cfg.csc && e->cfg.world > 1) GF_ENG_OK(gf_comm_set_select_inbox(e->comm, e->inbox_off));
    if (e->csc_inbox != UINT64_MAX) GF_ENG_OK(gf_comm_set_csc_inbox(e->comm, e->csc_inbox, e->csc_slot));
    return GF_OK;
}

int launch_window(gf_engine* e) {
    const int n = static_cast<int>(e->ov_ids.size());
    std::vector<const float*> src(n);
    std::vector<float*> dst(n);
    std::vector<uint64_t> off(n), cnt(n);
    for (int i = 0; i < n; ++i) {
        const int t = e->ov_ids[i] - 1;
        src[i] = e->ov_grad[t];
        dst[i] = e->ov_out[t];
        off[i] = e->offs[t];
        cnt[i] = e->sizes[t];
    }
    GF_ENG_CUDA(cudaEventRecord(e->ev_ready, e->ov_stream));  // the window's gradients are final
    GF_ENG_CUDA(cudaStreamWaitEvent(e->comm_s, e->ev_ready, 0));
    const uint64_t w0 = e->ov_ws, wlen = e->ov_we - e->ov_ws;
    char* pool = e->heap_base + e->pool_off;
    if (e->cfg.world == 1) {
        GF_ENG_OK(gf_sync_step_dense(e->comm, e->cfg.dtype, e->pool_off, src.data(), dst.data(), off.data(), cnt.data(),
                                     n, &w0, &wlen, 1, e->comm_s));
    } else {
        GF_ENG_OK(gf_pack(e->cfg.dtype, pool, src.data(), off.data(), cnt.data(), n, 1.0f, e->comm_s));
        GF_ENG_OK(gf_ring_allreduce(e->comm, e->cfg.dtype, e->pool_off, &w0, &wlen, 1, e->comm_s));
        GF_ENG_OK(gf_unpack(e->cfg.dtype, pool, dst.data(), off.data(), cnt.data(), n, e->cfg.world, e->comm_s));
    }
    GF_ENG_CUDA(cudaEventRecord(e->ev_done, e->comm_s));
    e->last_pool = pool;
    e->ov_launched += n;
    e->ov_ids.clear();
    e->ov_ws = e->ov_we;
    return GF_OK;
}

}  // namespace

extern "C" {

void gf_engine_config_init(gf_engine_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->world = 1;
    c->dtype = GF_F16;
    c->theta_bytes = 64ull << 20;
    c->chunk = 32000;
    c->dense_mode = GF_DENSE_AUTO;
    c->csc_mode = GF_CSC_AUTO;
    c->final_sparsity = 0.9;
    c->momentum = 0.9;
    c->learning_rate = 0.01;
    c->timeout_ms = 30000;
}

int gf_engine_create(const gf_engine_config* cfg, const uint64_t* sizes, int ntensors, gf_engine** out) {
    if (!out) return gfi::fail(GF_ERR_CONFIG, "gf_engine_create: null out");
    *out = nullptr;
    if (!cfg || !sizes || ntensors < 1) return gfi::fail(GF_ERR_CONFIG, "gradient pool needs at least one tensor");
    if (cfg->chunk == 0) return gfi::fail(GF_ERR_CONFIG, "chunk_size must be positive");
    if (cfg->dtype != GF_F16 && cfg->dtype != GF_F32) return gfi::fail(GF_ERR_CONFIG, "gf_engine_create: bad dtype");
    if (cfg->world < 1 || cfg->world > GF_MAX_RANKS || cfg->rank < 0 || cfg->rank >= cfg->world)
        return gfi::fail(GF_ERR_CONFIG, "gf_engine_create: rank/world out of range");
    if (cfg->dense_mode < GF_DENSE_AUTO || cfg->dense_mode > GF_DENSE_PUSH || cfg->csc_mode < GF_CSC_PUSH ||
        cfg->csc_mode > GF_CSC_AUTO)
        return gfi::fail(GF_ERR_CONFIG, "gf_engine_create: bad dense_mode / csc_mode");
    if (cfg->csc && (cfg->final_sparsity < 0.0 || cfg->final_sparsity >= 1.0))
        return gfi::fail(GF_ERR_CONFIG, "final_sparsity must be in [0, 1)");  // sparse.cpp:28-33
    for (int i = 0; i < ntensors; ++i)
        if (sizes[i] == 0) return gfi::fail(GF_ERR_CONFIG, "tensor sizes must be positive");
    auto* e = new gf_engine();
    e->cfg = *cfg;
    e->m = ntensors;
    e->esz = cfg->dtype == GF_F16 ? 2 : 4;
    e->sizes.assign(sizes, sizes + ntensors);
    e->offs.assign(ntensors, 0);
    uint64_t o = 0;  // gradient_pool.cpp:24-31: tensor m at offset 0, id 1 last
    for (int id = ntensors; id >= 1; --id) {
        e->offs[id - 1] = o;
        o += sizes[id - 1];
    }
    e->total = o;
    const double q = static_cast<double>(o) / static_cast<double>(cfg->chunk);  // llround, at least one chunk
    const long long r = std::llround(q);
    e->nc = std::max<uint64_t>(1, static_cast<uint64_t>(std::max(0LL, r)));
    const int W = cfg->world;
    int mode = cfg->dense_mode;
    if (mode == GF_DENSE_AUTO)  // measured: rspush ahead at 2 and 4 ranks; fp16 pools only
        mode = cfg->dtype == GF_F16 ? GF_DENSE_RSPUSH : (W == 2 ? GF_DENSE_PULL : GF_DENSE_PUSH);
    if (mode == GF_DENSE_RSPUSH && cfg->dtype != GF_F16) mode = GF_DENSE_PUSH;
    if (mode == GF_DENSE_PULL && ntensors > GF_MAX_WINDOWS_PER_LAUNCH) mode = GF_DENSE_PUSH;  // 256-tensor table
    e->dense_mode = mode;
    dense_windows(e);
    // the CSC exchange beside the packing of the unselected chunks: 64 CTAs of 256 threads, so
    // that packing CTAs share the exchange's SMs (measured at N=2/4: 0.226 / 0.234 ms
    // AlexNet CSC against 0.232 / 0.242 with 64 CTAs of 512 threads)
    e->xblocks = 64;
    e->xthreads = 256;
    if (const char* xb = std::getenv("GF_CSC_XBLOCKS")) e->xblocks = std::max(0, std::atoi(xb));
    if (const char* xt = std::getenv("GF_CSC_XTHREADS")) e->xthreads = std::max(0, std::atoi(xt));
    // symmetric heap: [pool | (pull: 2nd pool) | (rspush: N-1 inbox slots) | (CSC: staging) | norms | (CSC N>1: select inbox)]
    const uint64_t pool_bytes = align_up(e->total * e->esz);
    e->pool_off = 0;
    uint64_t at = pool_bytes;
    if (!cfg->csc && W > 1 && mode == GF_DENSE_PULL) {
        e->pull_two_pools = true;
        e->pull_pools[0] = 0;
        e->pull_pools[1] = at;
        at += pool_bytes;
    }
    if (!cfg->csc && W > 1 && mode == GF_DENSE_RSPUSH) {
        e->push_inbox = at;  // slot stride: a multiple of 8 elements (16-byte aligned slots)
        at += align_up(uint64_t(W - 1) * align_up(e->total, 8) * e->esz);
    }
    e->stage_off = at;
    e->norms_off = e->stage_off + (cfg->csc ? pool_bytes : 0);
    // the routed CSC exchange (pull form, fp16 with exact norms): world-1 inbox slots of the
    // staging capacity; the selected chunks' pack stores every staged element at its owner
    const bool routable = cfg->csc && W > 1 && cfg->dtype == GF_F16 && cfg->chunk % 8 == 0 && e->nc <= 6144;
    // AUTO, measured: the routed exchange from 4 ranks (ResNet-50 CSC at N=4:
    // 0.117-0.128 ms vs 0.122-0.135 with the ring); at N=2 the ring is ahead on ResNet-50
    if (e->cfg.csc_mode == GF_CSC_AUTO) e->cfg.csc_mode = (routable && W >= 4) ? GF_CSC_PULL : GF_CSC_PUSH;
    if (routable && e->cfg.csc_mode == GF_CSC_PULL) {
        e->csc_slot = align_up(e->total, 8);
        e->csc_inbox = e->norms_off;
        e->norms_off += align_up(uint64_t(W - 1) * e->csc_slot * 2);
    }
    e->inbox_off = e->norms_off + align_up(e->nc * 4);
    e->heap = e->inbox_off + ((cfg->csc && W > 1) ? align_up(uint64_t(W) * e->nc * 4) : 0);
    DevGuard g(cfg->device);
    int rc = gf_comm_create(W, cfg->rank, cfg->device, e->heap, &e->comm);
    if (rc == GF_OK) rc = gf_comm_set_timeout_ms(e->comm, cfg->timeout_ms);
    if (rc == GF_OK) {
        void* base = nullptr;
        rc = gf_comm_heap(e->comm, &base, nullptr);
        e->heap_base = static_cast<char*>(base);
        e->last_pool = e->heap_base + e->pool_off;
    }
    if (rc == GF_OK) rc = create_streams(e);
    if (rc == GF_OK && cfg->csc) rc = alloc_csc_state(e);
    if (rc != GF_OK) {
        const std::string msg = gf_last_error();
        gf_engine_destroy(e);
        return gfi::fail(rc, msg);
    }
    *out = e;
    return GF_OK;
}

int gf_engine_destroy(gf_engine* e) {
    if (!e) return GF_OK;
    DevGuard g(e->cfg.device);
    if (e->side) cudaStreamSynchronize(e->side);
    if (e->comm_s) cudaStreamSynchronize(e->comm_s);
    if (e->hp) cudaStreamSynchronize(e->hp);
    for (cudaEvent_t ev : {e->ev_a, e->ev_b, e->ev_ready, e->ev_done, e->ev_sel, e->ev_rest, e->ev_x})
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->ev_pool) cudaEventDestroy(ev);
    if (e->side) cudaStreamDestroy(e->side);
    if (e->comm_s) cudaStreamDestroy(e->comm_s);
    if (e->hp) cudaStreamDestroy(e->hp);
    if (e->state) cudaFree(e->state);
    if (e->comm) gf_comm_destroy(e->comm);
    delete e;
    return GF_OK;
}

gf_comm* gf_engine_comm(gf_engine* e) { return e ? e->comm : nullptr; }

int gf_engine_connect_ipc(gf_engine* e, const void* all_handles) {
    if (!e) return gfi::fail(GF_ERR_CONFIG, "null engine");
    GF_ENG_OK(gf_comm_connect_ipc(e->comm, all_handles));
    return after_connect(e);
}

static int connect_many(gf_engine* const* es, int world, int (*fn)(gf_comm* const*, int)) {
    if (!es || world < 1) return gfi::fail(GF_ERR_CONFIG, "gf_engine_connect: bad arguments");
    std::vector<gf_comm*> cs(world);
    for (int r = 0; r < world; ++r) {
        if (!es[r]) return gfi::fail(GF_ERR_CONFIG, "gf_engine_connect: null engine");
        cs[r] = es[r]->comm;
    }
    GF_ENG_OK(fn(cs.data(), world));
    for (int r = 0; r < world; ++r) GF_ENG_OK(after_connect(es[r]));
    return GF_OK;
}

int gf_engine_connect_local(gf_engine* const* es, int world) { return connect_many(es, world, gf_comm_connect_local); }
int gf_engine_connect_colocated(gf_engine* const* es, int world) {
    return connect_many(es, world, gf_comm_connect_colocated);
}

int gf_engine_info_get(gf_engine* e, gf_engine_info* out) {
    if (!e || !out) return gfi::fail(GF_ERR_CONFIG, "gf_engine_info_get: null argument");
    out->total = e->total;
    out->num_chunks = e->nc;
    out->heap_bytes = e->heap;
    out->nwin = static_cast<int>(e->ws.size());
    out->dense_mode = e->dense_mode;
    out->csc_mode = e->cfg.csc_mode;
    out->iteration = e->iteration;
    return GF_OK;
}

int gf_engine_state(gf_engine* e, int which, void** ptr, uint64_t* bytes) {
    if (!e || !ptr) return gfi::fail(GF_ERR_CONFIG, "gf_engine_state: null argument");
    void* p = nullptr;
    uint64_t b = 0;
    const uint64_t T = e->total, nc = e->nc;
    const int cur = int(e->iteration & 1), nxt = int((e->iteration + 1) & 1);
    switch (which) {
        case GF_STATE_POOL: p = e->last_pool; b = T * e->esz; break;
        case GF_STATE_NORMS: p = e->heap_base + e->norms_off; b = nc * 4; break;
        case GF_STATE_HG: p = e->hg; b = T * 4; break;
        case GF_STATE_HU: p = e->hu; b = T * 4; break;
        case GF_STATE_W: p = e->w; b = T * 4; break;
        case GF_STATE_IMP_NEXT: p = e->imp[cur]; b = nc; break;   // written by the last step's selection
        case GF_STATE_IMP_CUR: p = e->imp[nxt]; b = nc; break;    // the set the last step used
        case GF_STATE_PLAN_CUR: p = e->plan[nxt]; b = (4 + nc) * 8; break;
        case GF_STATE_PLAN_NEXT: p = e->plan[cur]; b = (4 + nc) * 8; break;
        case GF_STATE_NACC: p = e->nacc; b = e->nacc ? nc * 8 : 0; break;
        default: return gfi::fail(GF_ERR_CONFIG, "gf_engine_state: unknown buffer");
    }
    if (!p) return gfi::fail(GF_ERR_CONFIG, "gf_engine_state: buffer not allocated in this mode");
    *ptr = p;
    if (bytes) *bytes = b;
    return GF_OK;
}

int gf_engine_dense_step(gf_engine* e, const float* const* grads, float* const* out, void* stream) {
    if (!e || !grads || !out) return gfi::fail(GF_ERR_CONFIG, "gf_engine_dense_step: null argument");
    if (e->cfg.csc) return gfi::fail(GF_ERR_CONFIG, "gf_engine_dense_step on a CSC engine");
    if (e->ov_on) return gfi::fail(GF_ERR_CONFIG, "gf_engine_dense_step inside an overlapped iteration");
    DevGuard g(e->cfg.device);
    PhaseScope ps(e);
    auto s = static_cast<cudaStream_t>(stream);
    const int dt = e->cfg.dtype, m = e->m, nw = static_cast<int>(e->ws.size());
    const uint64_t* offs = e->offs.data();
    const uint64_t* cnts = e->sizes.data();
    int rc = GF_OK;
    if (e->cfg.world == 1) {  // no collective (collectives.cpp:59): one pass
        mark(e, "pack_unpack", s);
        e->last_pool = e->heap_base + e->pool_off;
        rc = gf_sync_step_dense(e->comm, dt, e->pool_off, grads, out, offs, cnts, m, e->ws.data(), e->wl.data(),
                                nw, s);
    } else if (e->dense_mode == GF_DENSE_RSPUSH) {
        e->last_pool = e->heap_base + e->pool_off;
        rc = gf_sync_step_dense_push(e->comm, dt, e->pool_off, e->push_inbox, grads, out, offs, cnts, m, e->ws.data(),
                                     e->wl.data(), nw, s);
    } else if (e->dense_mode == GF_DENSE_PULL) {
        // two pools used alternately: the next step's entry barrier orders the peers' last
        // reads of a pool before its reuse, so no exit barrier (GF_RSAG_NO_EXIT_BARRIER)
        const uint64_t po = e->pull_pools[e->pull_flip];
        e->pull_flip ^= 1;
        e->last_pool = e->heap_base + po;
        mark(e, "pack", s);
        rc = gf_pack(dt, e->last_pool, grads, offs, cnts, m, 1.0f, s);
        if (rc == GF_OK) {
            mark(e, "ring_unpack", s);
            rc = gf_ring_allreduce_unpack(e->comm, dt, po, out, offs, cnts, m, e->ws.data(), e->wl.data(), nw,
                                          GF_RSAG_NO_EXIT_BARRIER, s);
        }
    } else {
        char* pool = e->heap_base + e->pool_off;
        e->last_pool = pool;
        mark(e, "pack", s);
        rc = gf_pack(dt, pool, grads, offs, cnts, m, 1.0f, s);
        if (rc == GF_OK) {
            mark(e, "ring", s);
            rc = gf_ring_allreduce(e->comm, dt, e->pool_off, e->ws.data(), e->wl.data(), nw, s);
        }
        if (rc == GF_OK) {
            mark(e, "unpack", s);
            rc = gf_unpack(dt, pool, out, offs, cnts, m, e->cfg.world, s);
        }
    }
    mark(e, nullptr, s);
    return rc;
}

int gf_engine_csc_step(gf_engine* e, const float* const* grads, void* stream) {
    if (!e || !grads) return gfi::fail(GF_ERR_CONFIG, "gf_engine_csc_step: null argument");
    if (!e->cfg.csc) return gfi::fail(GF_ERR_CONFIG, "gf_engine_csc_step on a dense engine");
    DevGuard g(e->cfg.device);
    PhaseScope ps(e);
    auto s = static_cast<cudaStream_t>(stream);
    const gf_engine_config& C = e->cfg;
    const int dt = C.dtype, W = C.world;
    const uint64_t T = e->total, nc = e->nc, chunk = C.chunk;
    const int cur = int(e->iteration & 1), nxt = int((e->iteration + 1) & 1);
    char* pool = e->heap_base + e->pool_off;
    char* stage = e->heap_base + e->stage_off;
    e->last_pool = pool;
    const bool solo = W == 1;  // the exchange is the identity: no staging, no scatter
    // chunks selected for this iteration (iteration 0 is dense, sparse.cpp:45-51)
    const uint64_t k_cur = e->iteration == 0
                               ? nc
                               : gflow::selection_count(gflow::sparsity_at(e->iteration, C.warmup_iters, C.final_sparsity),
                                                        nc);
    const bool fused_wb = !solo && e->nacc && chunk % 8 == 0 && nc <= 6144;
    auto exchange = [&](cudaStream_t xs) -> int {
        if (fused_wb && C.csc_mode == GF_CSC_PULL) {
            // routed (csc_inbox set): local RS from my staging + inbox slots, the AG pushed into
            // every staging and written back locally; otherwise pull RS + pull AG straight into the
            // pool. Either way + the exact L1; the staging buffer is next rewritten after
            // gf_csc_select's barrier, so no exit barrier is needed
            mark(e, "ring_scatter", xs);
            return gf_csc_exchange_pull(e->comm, e->stage_off, e->plan[cur], pool, chunk, nc, e->nacc, xs);
        }
        if (fused_wb) {  // exchange + write-back + exact L1 of the exchanged chunks, one launch
            mark(e, "ring_scatter", xs);
            return gf_ring_allreduce_planned_scatter(e->comm, dt, e->stage_off, e->plan[cur], pool, chunk, nc,
                                                     e->nacc, xs);
        }
        mark(e, "ring", xs);
        GF_ENG_OK(gf_ring_allreduce_planned(e->comm, dt, e->stage_off, e->plan[cur], xs));
        mark(e, "scatter", xs);
        return gf_csc_scatter(dt, pool, stage, e->plan[cur], e->coff[cur], T, chunk, nc, k_cur, e->nacc, xs);
    };
    auto pack_correct = [&](int part, cudaStream_t st) {
        if (part == 1 && e->csc_inbox != UINT64_MAX)  // routed to the exchange owners
            return gf_csc_pack_correct_routed(e->comm, pool, e->hg, e->stage_off, e->plan[cur], chunk, grads,
                                              e->offs.data(), e->sizes.data(), e->m, static_cast<float>(C.momentum), st);
        return gf_csc_pack_correct_part(dt, pool, e->hg, solo ? nullptr : stage, e->imp[cur], e->coff[cur],
                                        e->plan[cur], T, chunk, nc, grads, e->offs.data(), e->sizes.data(), e->m,
                                        static_cast<float>(C.momentum), e->nacc, part, st);
    };
    auto update = [&](cudaStream_t us) {
        return gf_csc_sgd_update(dt, pool, e->plan[cur], T, chunk, nc, k_cur, W, static_cast<float>(C.momentum),
                                 static_cast<float>(C.learning_rate), e->hu, e->w, us);
    };
    if (solo) {
        mark(e, "pack_correct", s);
        GF_ENG_OK(pack_correct(0, s));
    } else {
        // the staged (important) chunks and their exchange beside the correction of the other
        // chunks (disjoint pool / hg / nacc elements), the exchange's grid capped so that the
        // packing CTAs keep the rest of the SMs
        auto capped_exchange = [&](cudaStream_t xs) {
            GF_ENG_OK(gf_comm_set_max_blocks(e->comm, e->xblocks));
            GF_ENG_OK(gf_comm_set_block_threads(e->comm, e->xthreads));
            const int rc = exchange(xs);
            gf_comm_set_max_blocks(e->comm, 0);
            gf_comm_set_block_threads(e->comm, 0);
            return rc;
        };
        if (e->marks_on) {  // per-kernel timing: one stream, kernels in order
            mark(e, "pack_correct_sel", s);
            GF_ENG_OK(pack_correct(1, s));
            GF_ENG_OK(capped_exchange(s));
            mark(e, "pack_correct_rest", s);
            GF_ENG_OK(pack_correct(2, s));
        } else {
            // The other chunks' correction starts at once on the side stream; the selected
            // chunks' pack and their exchange — the step's critical path — run on the
            // highest-priority stream, so the block scheduler hands them SMs first and the
            // other chunks' tiles fill the rest. Disjoint chunks: no ordering between the two.
            GF_ENG_CUDA(cudaEventRecord(e->ev_sel, s));
            GF_ENG_CUDA(cudaStreamWaitEvent(e->hp, e->ev_sel, 0));
            GF_ENG_CUDA(cudaStreamWaitEvent(e->side, e->ev_sel, 0));
            GF_ENG_OK(pack_correct(1, e->hp));
            GF_ENG_OK(capped_exchange(e->hp));
            GF_ENG_CUDA(cudaEventRecord(e->ev_x, e->hp));
            GF_ENG_OK(pack_correct(2, e->side));
            GF_ENG_CUDA(cudaEventRecord(e->ev_rest, e->side));
            GF_ENG_CUDA(cudaStreamWaitEvent(s, e->ev_x, 0));
            GF_ENG_CUDA(cudaStreamWaitEvent(s, e->ev_rest, 0));
        }
    }
    if (!e->nacc) {  // fp32 pool: separate norm pass (sequential fp64, as the reference)
        mark(e, "norms", s);
        GF_ENG_OK(gf_chunk_norms(dt, pool, T, chunk, nc, e->imp[cur], W,
                                 reinterpret_cast<float*>(e->heap_base + e->norms_off), s));
    }
    const uint64_t k =
        gflow::selection_count(gflow::sparsity_at(e->iteration + 1, C.warmup_iters, C.final_sparsity), nc);
    auto select = [&]() {
        return gf_csc_select(e->comm, e->norms_off, nc, k, e->imp[nxt], T, chunk, dt, C.theta_bytes, e->coff[nxt],
                             e->plan[nxt], e->nacc, e->nacc ? pool : nullptr, e->nacc ? e->imp[cur] : nullptr, s);
    };
    if (e->marks_on) {  // per-kernel timing: one stream, kernels in order
        mark(e, "select", s);
        GF_ENG_OK(select());
        mark(e, "sgd_update", s);
        GF_ENG_OK(update(s));
    } else {
        // The update reads this iteration's pool and plan; the selection reads the pool and
        // writes the NEXT plan and norms: independent. The one-CTA, latency-bound selection
        // runs beside the bandwidth-bound update on a second stream; the step ends when both
        // did (the next pack_correct overwrites the pool).
        GF_ENG_CUDA(cudaEventRecord(e->ev_a, s));
        GF_ENG_CUDA(cudaStreamWaitEvent(e->side, e->ev_a, 0));
        GF_ENG_OK(update(e->side));
        GF_ENG_CUDA(cudaEventRecord(e->ev_b, e->side));
        GF_ENG_OK(select());
        GF_ENG_CUDA(cudaStreamWaitEvent(s, e->ev_b, 0));
    }
    mark(e, nullptr, s);
    e->iteration++;
    return GF_OK;
}

int gf_engine_begin_iteration(gf_engine* e, const float* const* grads, float* const* out, void* stream) {
    if (!e || !grads || !out) return gfi::fail(GF_ERR_CONFIG, "gf_engine_begin_iteration: null argument");
    if (e->cfg.csc) return gfi::fail(GF_ERR_CONFIG, "the overlapped iteration is the dense path");
    e->ov_on = true;
    e->ov_grad.assign(grads, grads + e->m);
    e->ov_out.assign(out, out + e->m);
    e->ov_stream = static_cast<cudaStream_t>(stream);
    e->ov_ws = e->ov_we = 0;
    e->ov_ids.clear();
    e->ov_launched = 0;
    return GF_OK;
}

int gf_engine_tensor_complete(gf_engine* e, int tid) {
    if (!e) return gfi::fail(GF_ERR_CONFIG, "null engine");
    if (!e->ov_on) return gfi::fail(GF_ERR_CONFIG, "tensor_complete before begin_iteration");
    const int expect = e->m - static_cast<int>(e->ov_ids.size()) - e->ov_launched;
    if (tid != expect)  // fusion.cpp:74-78
        return gfi::fail(GF_ERR_CONFIG, "fusion: out-of-order tensor completion: got " + std::to_string(tid) +
                                            ", expected " + std::to_string(expect));
    DevGuard g(e->cfg.device);
    e->ov_ids.push_back(tid);
    e->ov_we = e->offs[tid - 1] + e->sizes[tid - 1];
    if (e->cfg.theta_bytes != GF_THETA_INFINITE && (e->ov_we - e->ov_ws) * e->esz >= e->cfg.theta_bytes)
        return launch_window(e);
    return GF_OK;
}

int gf_engine_finalize_iteration(gf_engine* e) {
    if (!e) return gfi::fail(GF_ERR_CONFIG, "null engine");
    if (!e->ov_on) return gfi::fail(GF_ERR_CONFIG, "finalize_iteration before begin_iteration");
    DevGuard g(e->cfg.device);
    if (e->ov_we > e->ov_ws) GF_ENG_OK(launch_window(e));
    if (e->ov_launched != e->m) return gfi::fail(GF_ERR_CONFIG, "finalize_iteration before every tensor completed");
    GF_ENG_CUDA(cudaStreamWaitEvent(e->ov_stream, e->ev_done, 0));
    e->ov_on = false;
    return GF_OK;
}

int gf_engine_set_marks(gf_engine* e, int on) {
    if (!e) return gfi::fail(GF_ERR_CONFIG, "null engine");
    e->marks_on = on != 0;
    return GF_OK;
}

int gf_engine_marks(gf_engine* e, char* names, int names_cap, float* ms, int cap) {
    if (!e || (cap > 0 && !ms) || (names_cap > 0 && !names)) return gfi::fail(GF_ERR_CONFIG, "gf_engine_marks: bad arguments");
    DevGuard g(e->cfg.device);
    std::vector<std::string> order;
    std::map<std::string, std::pair<double, int>> acc;
    for (size_t i = 0; i + 1 < e->marks.size(); ++i) {
        const std::string& name = e->marks[i].first;
        if (name.empty()) continue;  // step end -> next step's first mark
        GF_ENG_CUDA(cudaEventSynchronize(e->marks[i + 1].second));
        float t = 0.0f;
        GF_ENG_CUDA(cudaEventElapsedTime(&t, e->marks[i].second, e->marks[i + 1].second));
        auto it = acc.find(name);
        if (it == acc.end()) {
            order.push_back(name);
            acc[name] = {t, 1};
        } else {
            it->second.first += t;
            it->second.second += 1;
        }
    }
    e->marks.clear();
    e->ev_used = 0;
    std::string joined;
    int k = 0;
    for (const auto& nm : order) {
        if (k < cap) ms[k] = static_cast<float>(acc[nm].first / acc[nm].second);
        joined += (k ? ";" : "") + nm;
        ++k;
    }
    if (names_cap > 0) {
        std::strncpy(names, joined.c_str(), static_cast<size_t>(names_cap - 1));
        names[names_cap - 1] = '\0';
    }
    return k;
}

}  // extern "C"
