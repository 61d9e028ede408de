/* SPDX-License-Identifier: Apache-2.0
 *
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's gradient-synchronisation path
 * (GradientFlow reference, /root/reference/proj), used ONLY by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, and only as the
 * checker. The product (paper_1902_06855_b200) never links or calls it.
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against
 * (a) the reference's own known-answer tests (test_half.cpp, test_pool.cpp,
 * test_sparse.cpp, test_collectives.cpp) and (b) golden vectors produced by
 * the UNMODIFIED reference library compiled into oracle/_ref/ (see Makefile,
 * ref_driver.cpp, tests/golden/gen_golden.py). Parity is therefore pinned.
 *
 * dtype: 0 = fp32 (ElementType::kF32), 1 = fp16 (ElementType::kF16) — buffer.hpp:15.
 */
#ifndef GF_ORACLE_H
#define GF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* binary16 codec: half.hpp:20-59 / :61-87 */
uint16_t go_f2h(float v);
float go_h2f(uint16_t h);
void go_f2h_array(const float* in, uint16_t* out, uint64_t n);
void go_h2f_array(const uint16_t* in, float* out, uint64_t n);
/* sum mod 2^64 of splitmix64(bits<<16 | f2h(bits)) over fp32 patterns [first, first+count) */
uint64_t go_codec_digest(uint64_t first, uint64_t count, int nthreads);

/* accumulate dst += src elementwise: buffer.hpp:60-81 */
void go_accumulate(int dtype, void* dst, const void* src, uint64_t n);

/* segment_of: collectives.cpp:47-53 */
void go_segment_of(uint64_t len, int n, int i, uint64_t* off, uint64_t* cnt);

/* pool layout: gradient_pool.cpp:11-41 (offsets) and :32-38 (llround chunk count).
 * offsets[id-1] = pool offset of tensor id. Returns num_chunks (0 on error). */
uint64_t go_pool_layout(const uint64_t* sizes, int m, uint64_t chunk, uint64_t* offsets);
/* chunk_begin/chunk_length: gradient_pool.cpp:55-66 */
uint64_t go_chunk_begin(uint64_t chunk, uint64_t c);
uint64_t go_chunk_len(uint64_t total, uint64_t chunk, uint64_t nc, uint64_t c);

/* PACK: write_tensor for ids m..1 (gradient_pool.cpp:78-105). flat_asc holds the
 * gradients in ascending tensor id order; scale multiplies first when != 1. */
void go_pack(int dtype, const float* flat_asc, const uint64_t* sizes, int m, void* pool, float scale);
/* UNPACK: g_avg = dec(pool[i]) * (1/N) in pool order (trainer.cpp:336-342). */
void go_unpack(int dtype, const void* pool, uint64_t total, int world, float* out);

/* Ring allreduce, result of ring_allreduce_on (collectives.cpp:55-97) computed by
 * direct per-segment summation in ring-arrival order (P4). bufs[r] is rank r's
 * buffer; ring_order may be NULL (identity). In place on all ranks. */
void go_ring_allreduce(int dtype, void* const* bufs, int n, uint64_t len, const int* ring_order);
/* Same over a list of windows (each window has its own segment_of split). */
void go_ring_allreduce_windows(int dtype, void* const* bufs, int n, const uint64_t* wstart,
                               const uint64_t* wlen, int nwin, const int* ring_order);

/* Rooted ring reduce (collectives.cpp:99-144), end state of every position; bufs[t] is
 * ring position t's buffer. In place. */
void go_ring_reduce(int dtype, void* const* bufs, int n, int root_pos, uint64_t len);
/* hierarchical_allreduce (collectives.cpp:179-201) with groups of m ranks; bufs[r] = rank r. */
void go_hier_allreduce(int dtype, void* const* bufs, int n, int m, uint64_t len);

/* FusionEngine windows for one iteration (fusion.cpp:72-109): tensors complete in
 * descending id; window [start,end) launched when bytes >= theta (theta = UINT64_MAX
 * means never), residual at finalize. Returns window count; fills start/len (elements). */
int go_dense_windows(const uint64_t* sizes, int m, uint64_t esz, uint64_t theta,
                     uint64_t* wstart, uint64_t* wlen, int cap);
/* sparse_exchange windows over the staging buffer (sparse.cpp:142-158). */
int go_csc_windows(const uint8_t* imp, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t esz, uint64_t theta, uint64_t* wstart, uint64_t* wlen, int cap);

/* chunk_l1: sequential fp64 sum of |x|, cast to float (gradient_pool.cpp:107-116). */
float go_chunk_l1(int dtype, const void* pool, uint64_t begin, uint64_t len);
/* norms[c] = chunk_l1(c) * (imp[c] ? 1/N : 1) (sparse.cpp:176-184). */
void go_chunk_norms(int dtype, const void* pool, uint64_t total, uint64_t chunk, uint64_t nc,
                    const uint8_t* imp, int world, float* norms);

/* correction_pre_allreduce over every chunk (sparse.cpp:57-79 + csc_correct sparse.hpp:34-40). */
void go_csc_correct(int dtype, void* pool, float* hg, const uint8_t* imp, uint64_t total,
                    uint64_t chunk, uint64_t nc, float momentum);
/* staging pack / write-back (sparse.cpp:129-140, :162-168). Return staged element count. */
uint64_t go_csc_compact(int dtype, const void* pool, const uint8_t* imp, uint64_t total,
                        uint64_t chunk, uint64_t nc, void* staging);
void go_csc_scatter(int dtype, void* pool, const uint8_t* imp, uint64_t total, uint64_t chunk,
                    uint64_t nc, const void* staging);

/* selection: sparsity_at (sparse.cpp:13-17), selection_count (:19-24),
 * top-k by (norm desc, index asc) (:189-201). */
double go_sparsity_at(uint64_t t, uint64_t warmup, double final_sparsity);
uint64_t go_selection_count(double sparsity, uint64_t nc);
void go_select_topk(const float* norms, uint64_t nc, uint64_t k, uint8_t* flags);
/* FNV-1a 64 over the importance bytes (sparse.cpp:96-104). */
uint64_t go_fnv1a(const uint8_t* bytes, uint64_t n);

/* sgd_update (sparse.cpp:206-224 + csc_update sparse.hpp:42-51): important chunks only. */
void go_csc_sgd_update(int dtype, const void* pool, const uint8_t* imp, uint64_t total,
                       uint64_t chunk, uint64_t nc, int world, float momentum, float lr,
                       float* hu, float* w);

/* One full CSC iteration for n ranks (trainer.cpp:297-330 + sparse.cpp), composed
 * from the functions above. Per rank r: grads[r] flat ascending; pool[r] (fp16/fp32,
 * pool-shaped, written), hg[r] (in/out), staging[r] (scratch, >= total), norms[r]
 * (out, allreduced nc floats). imp (nc, this step's set, same on all ranks);
 * next_imp (out). Returns the number of exchange windows. */
int go_csc_iteration(int dtype, int n, const uint64_t* sizes, int m, uint64_t chunk,
                     uint64_t theta, float momentum, const float* const* grads,
                     void* const* pool, float* const* hg, void* const* staging,
                     float* const* norms, const uint8_t* imp, uint64_t k_next,
                     uint8_t* next_imp);

/* Synthetic gradients (SURVEY.md §8d scheme, different PRNG): a deterministic
 * splitmix64-based uniform(-1,1) * 2^-(id mod 7), ascending id. */
void go_gen_grads(uint64_t seed, const uint64_t* sizes, int m, float* out);

#ifdef __cplusplus
}
#endif
#endif
