/* SPDX-License-Identifier: Apache-2.0
 *
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see gf_oracle.h). A restatement of the
 * reference's algorithm, written from its behaviour; every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 *
 * Built with baseline x86-64 flags (no FMA, no F16C), like the reference, so
 * that float arithmetic here rounds exactly as the reference's does.
 */
#include "gf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* half.hpp:20-59 — RNE encode; overflow and +-inf clamp to +-65504 (0x7BFF);
 * NaN -> sign | 0x7E00; results below half the smallest subnormal -> signed 0. */
uint16_t go_f2h(float v) {
    const uint32_t b = f2u(v);
    const uint16_t sign = (uint16_t)((b >> 16) & 0x8000u);
    const uint32_t e = (b >> 23) & 0xFFu;
    const uint32_t mant = b & 0x7FFFFFu;
    if (e == 0xFFu) return (uint16_t)(sign | (mant ? 0x7E00u : 0x7BFFu));
    const int he = (int)e - 112; /* rebias 127 -> 15 */
    if (he >= 31) return (uint16_t)(sign | 0x7BFFu);
    if (he <= 0) {
        if (he < -10) return sign;
        const uint32_t full = mant | 0x800000u;
        const int sh = 14 - he; /* 14..24 */
        uint32_t q = full >> sh;
        const uint32_t r = full & ((1u << sh) - 1u), half = 1u << (sh - 1);
        if (r > half || (r == half && (q & 1u))) q++;
        return (uint16_t)(sign | q);
    }
    uint32_t out = ((uint32_t)he << 10) | (mant >> 13);
    const uint32_t r = mant & 0x1FFFu;
    if (r > 0x1000u || (r == 0x1000u && (out & 1u))) out++;
    if (out >= 0x7C00u) return (uint16_t)(sign | 0x7BFFu);
    return (uint16_t)(sign | out);
}

/* half.hpp:61-87 — exact widening, subnormals normalised, NaN payload kept. */
float go_h2f(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1Fu, mant = h & 0x3FFu;
    if (e == 0x1Fu) return u2f(sign | 0x7F800000u | (mant << 13));
    if (e != 0) return u2f(sign | ((e + 112u) << 23) | (mant << 13));
    if (mant == 0) return u2f(sign);
    /* subnormal: value = mant * 2^-24; normalise */
    int sh = 0;
    uint32_t mm = mant;
    while (!(mm & 0x400u)) { mm <<= 1; sh++; }
    return u2f(sign | ((uint32_t)(113 - sh) << 23) | ((mm & 0x3FFu) << 13));
}

void go_f2h_array(const float* in, uint16_t* out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) out[i] = go_f2h(in[i]);
}
void go_h2f_array(const uint16_t* in, float* out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) out[i] = go_h2f(in[i]);
}

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

typedef struct { uint64_t first, count, acc; } digest_job;
static void* digest_worker(void* p) {
    digest_job* j = (digest_job*)p;
    uint64_t acc = 0;
    for (uint64_t x = j->first; x < j->first + j->count; ++x) {
        const uint32_t b = (uint32_t)x;
        acc += splitmix64(((uint64_t)b << 16) | go_f2h(u2f(b)));
    }
    j->acc = acc;
    return NULL;
}
uint64_t go_codec_digest(uint64_t first, uint64_t count, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 64) nthreads = 64;
    pthread_t th[64];
    digest_job jobs[64];
    const uint64_t per = count / (uint64_t)nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].first = first + per * (uint64_t)t;
        jobs[t].count = (t == nthreads - 1) ? count - per * (uint64_t)t : per;
        pthread_create(&th[t], NULL, digest_worker, &jobs[t]);
    }
    uint64_t acc = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); acc += jobs[t].acc; }
    return acc;
}

/* x86 SSE addss semantics made explicit (so the oracle does not depend on which operand
 * its own compiler puts in the destination register): a NaN operand propagates quieted;
 * if both are NaN the DESTINATION operand wins; an invalid op yields the default NaN
 * 0xFFC00000 (the hardware produces that itself). The reference's fp16 accumulate has
 * the incoming value as destination, its fp32 accumulate the local one (measured). */
static int isnan_f(float x) { return (f2u(x) & 0x7FFFFFFFu) > 0x7F800000u; }
static float addss(float dst, float src) {
    if (isnan_f(dst) && isnan_f(src)) return u2f(f2u(dst) | 0x400000u);
    return dst + src;
}
/* buffer.hpp:71-79 */
static uint16_t acc16(uint16_t local, uint16_t incoming) {
    return go_f2h(addss(go_h2f(incoming), go_h2f(local)));
}
/* buffer.hpp:63-69 */
static float acc32(float local, float incoming) { return addss(local, incoming); }

/* buffer.hpp:60-81 — dst[i] = dst[i] + src[i]; fp16 widened to fp32 and re-encoded. */
void go_accumulate(int dtype, void* dst, const void* src, uint64_t n) {
    if (dtype == 0) {
        float* d = (float*)dst; const float* s = (const float*)src;
        for (uint64_t i = 0; i < n; ++i) d[i] = acc32(d[i], s[i]);
    } else {
        uint16_t* d = (uint16_t*)dst; const uint16_t* s = (const uint16_t*)src;
        for (uint64_t i = 0; i < n; ++i) d[i] = acc16(d[i], s[i]);
    }
}

/* collectives.cpp:47-53 */
void go_segment_of(uint64_t len, int n, int i, uint64_t* off, uint64_t* cnt) {
    const uint64_t base = len / (uint64_t)n, rem = len % (uint64_t)n, idx = (uint64_t)i;
    *off = idx * base + (idx < rem ? idx : rem);
    *cnt = base + (idx < rem ? 1u : 0u);
}

/* gradient_pool.cpp:11-41: tensor id m at offset 0, id 1 last; nc = max(1, llround(total/chunk)). */
uint64_t go_pool_layout(const uint64_t* sizes, int m, uint64_t chunk, uint64_t* offsets) {
    if (m < 1 || chunk == 0) return 0;
    uint64_t off = 0;
    for (int id = m; id >= 1; --id) {
        if (sizes[id - 1] == 0) return 0;
        if (offsets) offsets[id - 1] = off;
        off += sizes[id - 1];
    }
    const long long nc = llround((double)off / (double)chunk);
    return nc < 1 ? 1u : (uint64_t)nc;
}
uint64_t go_chunk_begin(uint64_t chunk, uint64_t c) { return c * chunk; }
uint64_t go_chunk_len(uint64_t total, uint64_t chunk, uint64_t nc, uint64_t c) {
    return (c + 1 == nc) ? total - c * chunk : chunk; /* gradient_pool.cpp:62-66 */
}

static uint64_t esz_of(int dtype) { return dtype == 0 ? 4u : 2u; }
static float load_el(int dtype, const void* p, uint64_t i) {
    return dtype == 0 ? ((const float*)p)[i] : go_h2f(((const uint16_t*)p)[i]);
}
static void store_el(int dtype, void* p, uint64_t i, float v) {
    if (dtype == 0) ((float*)p)[i] = v; else ((uint16_t*)p)[i] = go_f2h(v);
}

/* gradient_pool.cpp:78-105 (write_tensor for ids m..1, ScalarBuffer::set per element). */
void go_pack(int dtype, const float* flat_asc, const uint64_t* sizes, int m, void* pool, float scale) {
    uint64_t* asc = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m + 1));
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m);
    asc[0] = 0;
    for (int i = 0; i < m; ++i) asc[i + 1] = asc[i] + sizes[i];
    go_pool_layout(sizes, m, 1, off);
    for (int id = m; id >= 1; --id) {
        const float* g = flat_asc + asc[id - 1];
        for (uint64_t i = 0; i < sizes[id - 1]; ++i) {
            const float v = (scale == 1.0f) ? g[i] : g[i] * scale;
            store_el(dtype, pool, off[id - 1] + i, v);
        }
    }
    free(asc); free(off);
}

/* trainer.cpp:336-342: g_avg = v.get(i) * inv_world with inv_world = 1.0f / N. */
void go_unpack(int dtype, const void* pool, uint64_t total, int world, float* out) {
    const float inv_world = 1.0f / (float)world;
    for (uint64_t i = 0; i < total; ++i) out[i] = load_el(dtype, pool, i) * inv_world;
}

/* collectives.cpp:55-97 — the RS accumulates segment j starting at ring position j:
 * at position j+t the receiver computes local + incoming (accumulate, buffer.hpp:71-79),
 * rounding to the element type each step; AG copies the owner's result everywhere. */
static void ring_one(int dtype, void* const* bufs, int n, uint64_t base, uint64_t len, const int* ring) {
    for (int j = 0; j < n; ++j) {
        uint64_t off, cnt;
        go_segment_of(len, n, j, &off, &cnt);
        for (uint64_t e = base + off; e < base + off + cnt; ++e) {
            if (dtype == 1) {
                uint16_t acc = ((const uint16_t*)bufs[ring[j]])[e];
                for (int t = 1; t < n; ++t) acc = acc16(((const uint16_t*)bufs[ring[(j + t) % n]])[e], acc);
                for (int r = 0; r < n; ++r) ((uint16_t*)bufs[r])[e] = acc;
            } else {
                float acc = ((const float*)bufs[ring[j]])[e];
                for (int t = 1; t < n; ++t) acc = acc32(((const float*)bufs[ring[(j + t) % n]])[e], acc);
                for (int r = 0; r < n; ++r) ((float*)bufs[r])[e] = acc;
            }
        }
    }
}
void go_ring_allreduce_windows(int dtype, void* const* bufs, int n, const uint64_t* wstart,
                               const uint64_t* wlen, int nwin, const int* ring_order) {
    if (n <= 1) return; /* collectives.cpp:59 */
    int* ring = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) ring[i] = ring_order ? ring_order[i] : i;
    for (int w = 0; w < nwin; ++w) ring_one(dtype, bufs, n, wstart[w], wlen[w], ring);
    free(ring);
}
void go_ring_allreduce(int dtype, void* const* bufs, int n, uint64_t len, const int* ring_order) {
    const uint64_t s = 0;
    go_ring_allreduce_windows(dtype, bufs, n, &s, &len, 1, ring_order);
}

/* collectives.cpp:99-144 ring_reduce_on: the RS of ring_allreduce_on, then every position
 * but the root sends its owned segment to the root. End state: position j+k (k = 1..n-1)
 * holds segment j's partial chain (positions j..j+k), position j keeps its raw segment j,
 * and the root holds every full sum. bufs[t] = buffer of ring position t. */
void go_ring_reduce(int dtype, void* const* bufs, int n, int root_pos, uint64_t len) {
    if (n <= 1) return; /* collectives.cpp:104 */
    for (int j = 0; j < n; ++j) {
        uint64_t off, cnt;
        go_segment_of(len, n, j, &off, &cnt);
        for (uint64_t e = off; e < off + cnt; ++e) {
            if (dtype == 1) {
                uint16_t acc = ((const uint16_t*)bufs[j])[e];
                for (int k = 1; k < n; ++k) {
                    uint16_t* b = (uint16_t*)bufs[(j + k) % n];
                    acc = acc16(b[e], acc);
                    b[e] = acc;
                }
                ((uint16_t*)bufs[root_pos])[e] = acc;
            } else {
                float acc = ((const float*)bufs[j])[e];
                for (int k = 1; k < n; ++k) {
                    float* b = (float*)bufs[(j + k) % n];
                    acc = acc32(b[e], acc);
                    b[e] = acc;
                }
                ((float*)bufs[root_pos])[e] = acc;
            }
        }
    }
}

/* collectives.cpp:179-201 hierarchical_allreduce: ring_reduce_on inside each group of m
 * consecutive ranks to its master (rank g*m), ring_allreduce_on over the masters in
 * group order, broadcast_on from each master to its group. bufs[r] = rank r. */
void go_hier_allreduce(int dtype, void* const* bufs, int n, int m, uint64_t len) {
    const int k = n / m;
    const size_t es = dtype == 1 ? 2u : 4u;
    for (int g = 0; g < k; ++g) go_ring_reduce(dtype, bufs + (size_t)g * (size_t)m, m, 0, len);
    void** masters = (void**)malloc(sizeof(void*) * (size_t)k);
    for (int g = 0; g < k; ++g) masters[g] = bufs[(size_t)g * (size_t)m];
    go_ring_allreduce(dtype, masters, k, len, NULL);
    for (int g = 0; g < k; ++g)
        for (int r = 1; r < m; ++r) memcpy(bufs[(size_t)g * (size_t)m + (size_t)r], masters[g], len * es);
    free(masters);
}

/* fusion.cpp:72-109: on_tensor_complete extends [start,end) to the tensor's end;
 * maybe_launch fires when pending bytes >= theta (theta != kThetaInfinite);
 * finalize flushes the residual. */
int go_dense_windows(const uint64_t* sizes, int m, uint64_t esz, uint64_t theta,
                     uint64_t* wstart, uint64_t* wlen, int cap) {
    uint64_t* off = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m);
    go_pool_layout(sizes, m, 1, off);
    uint64_t ws = 0, we = 0;
    int nw = 0;
    for (int id = m; id >= 0; --id) {
        const int flush = (id == 0);
        if (!flush) we = off[id - 1] + sizes[id - 1];
        const uint64_t pending = (we - ws) * esz;
        const int hit = theta != UINT64_MAX && pending >= theta;
        if (we > ws && (hit || flush)) {
            if (nw < cap) { wstart[nw] = ws; wlen[nw] = we - ws; }
            nw++;
            ws = we;
        }
    }
    free(off);
    return nw;
}

/* sparse.cpp:142-158: windows over the staging buffer cut at selected-chunk ends. */
int go_csc_windows(const uint8_t* imp, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t esz, uint64_t theta, uint64_t* wstart, uint64_t* wlen, int cap) {
    uint64_t ws = 0, pos = 0;
    int nw = 0;
    for (uint64_t c = 0; c < nc; ++c) {
        if (!imp[c]) continue;
        pos += go_chunk_len(total, chunk, nc, c);
        if (theta != UINT64_MAX && (pos - ws) * esz >= theta) {
            if (nw < cap) { wstart[nw] = ws; wlen[nw] = pos - ws; }
            nw++;
            ws = pos;
        }
    }
    if (pos > ws) {
        if (nw < cap) { wstart[nw] = ws; wlen[nw] = pos - ws; }
        nw++;
    }
    return nw;
}

/* gradient_pool.cpp:107-116: double sum of fabs(double(x)), sequential, cast to float. */
float go_chunk_l1(int dtype, const void* pool, uint64_t begin, uint64_t len) {
    double s = 0.0;
    for (uint64_t i = 0; i < len; ++i) s += fabs((double)load_el(dtype, pool, begin + i));
    return (float)s;
}
void go_chunk_norms(int dtype, const void* pool, uint64_t total, uint64_t chunk, uint64_t nc,
                    const uint8_t* imp, int world, float* norms) {
    const float inv_world = 1.0f / (float)world;
    for (uint64_t c = 0; c < nc; ++c) {
        float v = go_chunk_l1(dtype, pool, c * chunk, go_chunk_len(total, chunk, nc, c));
        if (imp && imp[c]) v *= inv_world;
        norms[c] = v;
    }
}

/* sparse.cpp:57-79 with csc_correct<float> (sparse.hpp:34-40):
 * g = dec(pool) ; g += hg ; hg = imp ? 0 : mom*g ; pool = enc(g). */
void go_csc_correct(int dtype, void* pool, float* hg, const uint8_t* imp, uint64_t total,
                    uint64_t chunk, uint64_t nc, float momentum) {
    for (uint64_t c = 0; c < nc; ++c) {
        const uint64_t b = c * chunk, len = go_chunk_len(total, chunk, nc, c);
        for (uint64_t i = b; i < b + len; ++i) {
            float g = load_el(dtype, pool, i);
            g = addss(g, hg[i]); /* g[i] += hg[i] (sparse.hpp:37) */
            hg[i] = imp[c] ? 0.0f : momentum * g;
            store_el(dtype, pool, i, g);
        }
    }
}

/* sparse.cpp:129-140 (pack queued chunks ascending) and :162-168 (write-back). */
uint64_t go_csc_compact(int dtype, const void* pool, const uint8_t* imp, uint64_t total,
                        uint64_t chunk, uint64_t nc, void* staging) {
    const uint64_t es = esz_of(dtype);
    uint64_t cur = 0;
    for (uint64_t c = 0; c < nc; ++c) {
        if (!imp[c]) continue;
        const uint64_t len = go_chunk_len(total, chunk, nc, c);
        memcpy((char*)staging + cur * es, (const char*)pool + c * chunk * es, len * es);
        cur += len;
    }
    return cur;
}
void go_csc_scatter(int dtype, void* pool, const uint8_t* imp, uint64_t total, uint64_t chunk,
                    uint64_t nc, const void* staging) {
    const uint64_t es = esz_of(dtype);
    uint64_t cur = 0;
    for (uint64_t c = 0; c < nc; ++c) {
        if (!imp[c]) continue;
        const uint64_t len = go_chunk_len(total, chunk, nc, c);
        memcpy((char*)pool + c * chunk * es, (const char*)staging + cur * es, len * es);
        cur += len;
    }
}

/* sparse.cpp:13-17 */
double go_sparsity_at(uint64_t t, uint64_t warmup, double final_sparsity) {
    if (warmup == 0) return final_sparsity;
    double ramp = (double)t / (double)warmup;
    if (ramp > 1.0) ramp = 1.0;
    return final_sparsity * ramp;
}
/* sparse.cpp:19-24: k = max(1, min(nc, llround((1-s)*nc))) — llround, half away from zero. */
uint64_t go_selection_count(double sparsity, uint64_t nc) {
    const double fraction = 1.0 - sparsity;
    const uint64_t k = (uint64_t)llround(fraction * (double)nc);
    const uint64_t kk = k < nc ? k : nc;
    return kk < 1 ? 1 : kk;
}

/* sparse.cpp:189-201: partial_sort by (norm desc, index asc), first k flagged.
 * Restated as a rank count: chunk i is selected iff fewer than k chunks precede it. */
typedef struct { float v; uint64_t i; } norm_key;
static int key_cmp(const void* a, const void* b) {
    const norm_key* x = (const norm_key*)a; const norm_key* y = (const norm_key*)b;
    if (x->v != y->v) return x->v > y->v ? -1 : 1;
    return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}
void go_select_topk(const float* norms, uint64_t nc, uint64_t k, uint8_t* flags) {
    norm_key* keys = (norm_key*)malloc(sizeof(norm_key) * (size_t)nc);
    for (uint64_t i = 0; i < nc; ++i) { keys[i].v = norms[i]; keys[i].i = i; }
    qsort(keys, (size_t)nc, sizeof(norm_key), key_cmp);
    memset(flags, 0, (size_t)nc);
    for (uint64_t i = 0; i < k && i < nc; ++i) flags[keys[i].i] = 1;
    free(keys);
}

/* sparse.cpp:96-104 */
uint64_t go_fnv1a(const uint8_t* bytes, uint64_t n) {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t i = 0; i < n; ++i) { h ^= bytes[i]; h *= 1099511628211ull; }
    return h;
}

/* sparse.cpp:206-224 + csc_update<float> (sparse.hpp:42-51). */
void go_csc_sgd_update(int dtype, const void* pool, const uint8_t* imp, uint64_t total,
                       uint64_t chunk, uint64_t nc, int world, float momentum, float lr,
                       float* hu, float* w) {
    const float inv_world = 1.0f / (float)world;
    for (uint64_t c = 0; c < nc; ++c) {
        if (!imp[c]) continue;
        const uint64_t b = c * chunk, len = go_chunk_len(total, chunk, nc, c);
        for (uint64_t i = b; i < b + len; ++i) {
            const float g_avg = load_el(dtype, pool, i) * inv_world;
            const float u = momentum * hu[i] + lr * g_avg;
            hu[i] = u;
            w[i] -= u;
        }
    }
}

/* trainer.cpp:297-330 (CSC branch) + sparse.cpp:106-204, composed. */
int go_csc_iteration(int dtype, int n, const uint64_t* sizes, int m, uint64_t chunk,
                     uint64_t theta, float momentum, const float* const* grads,
                     void* const* pool, float* const* hg, void* const* staging,
                     float* const* norms, const uint8_t* imp, uint64_t k_next,
                     uint8_t* next_imp) {
    uint64_t total = 0;
    for (int i = 0; i < m; ++i) total += sizes[i];
    const uint64_t nc = go_pool_layout(sizes, m, chunk, NULL);
    uint64_t staged = 0;
    for (int r = 0; r < n; ++r) {
        go_pack(dtype, grads[r], sizes, m, pool[r], 1.0f);
        go_csc_correct(dtype, pool[r], hg[r], imp, total, chunk, nc, momentum);
        staged = go_csc_compact(dtype, pool[r], imp, total, chunk, nc, staging[r]);
    }
    const int cap = (int)nc + 1;
    uint64_t* ws = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)cap);
    uint64_t* wl = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)cap);
    const int nw = go_csc_windows(imp, total, chunk, nc, esz_of(dtype), theta, ws, wl, cap);
    (void)staged;
    go_ring_allreduce_windows(dtype, staging, n, ws, wl, nw, NULL);
    for (int r = 0; r < n; ++r) {
        go_csc_scatter(dtype, pool[r], imp, total, chunk, nc, staging[r]);
        go_chunk_norms(dtype, pool[r], total, chunk, nc, imp, n, norms[r]);
    }
    go_ring_allreduce(0, (void* const*)norms, n, nc, NULL);
    go_select_topk(norms[0], nc, k_next, next_imp);
    free(ws); free(wl);
    return nw;
}

void go_gen_grads(uint64_t seed, const uint64_t* sizes, int m, float* out) {
    uint64_t o = 0, st = seed * 0x2545F4914F6CDD1Dull + 1;
    for (int id = 1; id <= m; ++id) {
        const float s = ldexpf(1.0f, -(id % 7));
        for (uint64_t i = 0; i < sizes[id - 1]; ++i) {
            st = splitmix64(st);
            const float u = (float)(st >> 40) * (1.0f / 16777216.0f); /* [0,1) 24-bit */
            out[o++] = (2.0f * u - 1.0f) * s;
        }
    }
}
