/* SPDX-License-Identifier: Apache-2.0
 *
 * gflow_b200 — C-ABI of the B200-native gradient-synchronisation path
 * (GradientFlow, arXiv 1902.06855). This is the drop-in boundary: the
 * reference's C++ API (gflow::GradientPool / FusionEngine / SparseState /
 * ring_allreduce, re-stated in paper_1902_06855_b200/csrc/include/gflow/) and
 * the gflowpy bindings sit on top of these entry points, and any other host
 * (ctypes, cgo, JNI) can bind them directly.
 *
 * Conventions
 *  - Plain pointers and sizes only. Buffer pointers are DEVICE pointers unless
 *    stated otherwise; `stream` is a cudaStream_t (NULL = legacy default).
 *  - Every entry point returns gf_status (0 = OK). Errors map onto the
 *    reference's exception taxonomy (include/gflow/errors.hpp:11-33) and the
 *    message is available from gf_last_error() on the calling thread.
 *  - dtype follows ElementType (include/gflow/buffer.hpp:15): 0 fp32, 1 fp16.
 *  - Numerics are bit-exact with the reference CPU implementation: the
 *    binary16 codec clamps instead of overflowing (half.hpp:20-59), fp16
 *    accumulation widens to fp32 per element (buffer.hpp:60-81), no FMA.
 *  - "Pool order": tensor id m at offset 0, id 1 last (gradient_pool.cpp:24-31).
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *  gf_encode_f16 / gf_decode_f16    float_to_half_bits / half_bits_to_float  include/gflow/half.hpp:20-87
 *  gf_accumulate                    accumulate(ScalarBuffer, bytes)         include/gflow/buffer.hpp:60-81
 *  gf_pack                          GradientPool::write_tensor               src/gradient_pool.cpp:78-105
 *  gf_unpack                        dense update read g = get(i)*(1/N)       src/trainer.cpp:332-347
 *  gf_chunk_norms                   GradientPool::chunk_l1 (+ x1/N)          src/gradient_pool.cpp:107-116, src/sparse.cpp:176-184
 *  gf_csc_correct                   SparseState::correction_pre_allreduce    src/sparse.cpp:57-79, include/gflow/sparse.hpp:34-40
 *  gf_csc_pack_correct              write_tensor + correction + staging pack src/gradient_pool.cpp:78-105, src/sparse.cpp:57-79,:129-140
 *  gf_csc_compact / gf_csc_scatter  sparse_exchange staging pack/write-back  src/sparse.cpp:129-140, :162-168
 *  gf_csc_plan                      sparse_exchange theta windows            src/sparse.cpp:142-158
 *  gf_select_topk                   select_next_important partial_sort       src/sparse.cpp:189-201
 *  gf_csc_sgd_update                SparseState::sgd_update / csc_update     src/sparse.cpp:206-224, include/gflow/sparse.hpp:42-51
 *  gf_dense_sgd_update              dense momentum update loop               src/trainer.cpp:332-347
 *  gf_comm_*                        Communicator + Transport (data plane)    include/gflow/collectives.hpp:25-61, include/gflow/transport.hpp:96-120
 *  gf_ring_allreduce[_planned]      ring_allreduce / ring_allreduce_on       src/collectives.cpp:55-97, :174-177
 *  gf_ring_allreduce_colocated      same, all ranks' buffers on one device   src/collectives.cpp:55-97
 *  gf_ring_allreduce_unpack         ring_allreduce of the windows + the update read g = get(i)*(1/N)
 *                                   src/collectives.cpp:55-97, src/trainer.cpp:332-347
 *  gf_sync_step_dense_push          the same with the reduce-scatter pushed by the pack (write_tensor
 *                                   src/gradient_pool.cpp:78-105 + ring_allreduce_on src/collectives.cpp:55-97)
 *  gf_sync_step_dense               one dense iteration: write_tensor x m + FusionEngine windows +
 *                                   update read (src/trainer.cpp:297-347); one pass at world 1
 *  gf_engine_*                      one rank's whole iteration: train_worker's sync half
 *                                   (src/trainer.cpp:297-347), FusionEngine (src/fusion.cpp:25-123),
 *                                   SparseState (src/sparse.cpp:57-224)
 *  gf_csc_exchange_pull             sparse_exchange ring + write-back (pull form) src/sparse.cpp:106-170
 *  gf_csc_pack_correct_routed       correction_pre_allreduce + staging pack, routed to the exchange owners
 *                                   src/sparse.cpp:57-79, :129-140
 *  gf_csc_select                    select_next_important (norm allreduce + top-k) src/sparse.cpp:172-204
 *  gf_ring_traffic                  TrafficStats record_send/recv of the ring include/gflow/transport.hpp:48-91, src/collectives.cpp:69-96
 *  gf_oracle_allreduce_ptrs         oracle_allreduce                         src/collectives.cpp:203-226
 *  gf_broadcast_ptrs                broadcast / broadcast_on                 src/collectives.cpp:146-170, :237-242
 *  gf_ring_reduce_ptrs              reduce / ring_reduce_on (+ hierarchical)  src/collectives.cpp:99-144, :179-201, :229-235
 */
#ifndef GFLOW_B200_H
#define GFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_ABI_VERSION 1
#define GF_MAX_RANKS 16
#define GF_IPC_HANDLE_BYTES 64
#define GF_MAX_WINDOWS_PER_LAUNCH 256
#define GF_THETA_INFINITE UINT64_MAX

typedef enum {
    GF_OK = 0,
    GF_ERR_CONFIG = 1,    /* gflow::ConfigError    — bad arguments or call order */
    GF_ERR_PROTOCOL = 2,  /* gflow::ProtocolError  — ranks disagree (sizes, important set) */
    GF_ERR_TRANSPORT = 3, /* gflow::TransportError — peer timeout / unreachable / comm poisoned */
    GF_ERR_TRAINING = 4,  /* gflow::TrainingError */
    GF_ERR_CUDA = 5       /* CUDA runtime failure (reported as TransportError by the C++ layer) */
} gf_status;

typedef enum { GF_F32 = 0, GF_F16 = 1 } gf_dtype;

typedef struct gf_comm gf_comm;

int gf_abi_version(void);
const char* gf_last_error(void);
/* Number of this library's kernels launched by the calling process so far. */
uint64_t gf_kernel_launches(void);

/* ---- codec ---------------------------------------------------------------- */
/* dst[i] = float_to_half_bits(scale * src[i]) (scale == 1 skips the multiply). */
int gf_encode_f16(const float* src, uint16_t* dst, uint64_t n, float scale, void* stream);
/* dst[i] = half_bits_to_float(src[i]). */
int gf_decode_f16(const uint16_t* src, float* dst, uint64_t n, void* stream);
/* Self-test digest of the DEVICE encoder over fp32 bit patterns [first, first+count):
 * *digest_dev (device u64, accumulated into) += sum of splitmix64(bits<<16 | enc(bits)). */
int gf_codec_digest(uint64_t first, uint64_t count, uint64_t* digest_dev, void* stream);
/* dst[i] = dst[i] + src[i] in the element type (fp16: widen, add in fp32, re-encode). */
int gf_accumulate(int dtype, void* dst, const void* src, uint64_t n, void* stream);

/* ---- pack / unpack (multi-tensor, one launch per call) ----------------------- */
/* pool[pool_off[t] + i] = enc(scale * src[t][i]) for i < count[t], t < ntensors.
 * src/pool_off/count are HOST arrays (copied into the launch); src[t] are device ptrs. */
int gf_pack(int dtype, void* pool, const float* const* src, const uint64_t* pool_off,
            const uint64_t* count, int ntensors, float scale, void* stream);
/* dst[t][i] = dec(pool[pool_off[t] + i]) * (1.0f / world). */
int gf_unpack(int dtype, const void* pool, float* const* dst, const uint64_t* pool_off,
              const uint64_t* count, int ntensors, int world, void* stream);

/* ---- CSC kernels ----------------------------------------------------------------- */
/* norms[c] = (float)sum_i |x_i| over chunk c (exact, as the sequential fp64 sum),
 * times (1.0f/world) when important != NULL && important[c]. */
int gf_chunk_norms(int dtype, const void* pool, uint64_t total, uint64_t chunk, uint64_t nc,
                   const uint8_t* important, int world, float* norms, void* stream);
/* In place over chunks [first_chunk, first_chunk+num_chunks):
 * g = dec(pool)+hg ; hg = imp ? 0 : momentum*g ; pool = enc(g). */
int gf_csc_correct(int dtype, void* pool, float* hg, const uint8_t* important, uint64_t total,
                   uint64_t chunk, uint64_t nc, uint64_t first_chunk, uint64_t num_chunks,
                   float momentum, void* stream);
/* Fused pack + correction + compaction over all tensors: for pool element i in chunk c
 *   g = dec(enc(src)) + hg ; hg = imp ? 0 : momentum*g ; pool = enc(g) ;
 *   if imp[c]: staging[coff[c] + (i - c*chunk)] = enc(g).
 * coff (device, nc entries) comes from gf_csc_plan.
 * nacc (device, nc uint64, fp16 pools only, nullable): the exact sum of |pool| of every
 * UNIMPORTANT chunk is added in units of 2^-24 (bit 63 = NaN seen) — K3 fused into K2.
 * staging may be NULL: no compaction. That is the world-1 step, where the exchange is the
 * identity (collectives.cpp:59): nacc then also takes the important chunks, and no
 * gf_csc_scatter follows. */
int gf_csc_pack_correct(int dtype, void* pool, float* hg, void* staging,
                        const uint8_t* important, const uint64_t* coff, uint64_t total,
                        uint64_t chunk, uint64_t nc, const float* const* src,
                        const uint64_t* pool_off, const uint64_t* count, int ntensors,
                        float momentum, uint64_t* nacc, void* stream);
/* The same restricted to a part of the chunks: part 0 all, 1 the important chunks only (every
 * staged chunk), 2 the unimportant ones only. A CSC step runs part 1, starts the exchange of the
 * staging buffer, and runs part 2 beside it (they touch disjoint pool/hg/nacc elements). With
 * `plan` (device, gf_csc_plan of the same set; nullable) and the tensors in ascending id, part 1
 * walks only the planned chunks. */
int gf_csc_pack_correct_part(int dtype, void* pool, float* hg, void* staging,
                             const uint8_t* important, const uint64_t* coff, const uint64_t* plan,
                             uint64_t total, uint64_t chunk, uint64_t nc, const float* const* src,
                             const uint64_t* pool_off, const uint64_t* count, int ntensors,
                             float momentum, uint64_t* nacc, int part, void* stream);
/* Staging pack / write-back over the important chunks listed in `plan` (see gf_csc_plan):
 * staging[coff[c] + i] <-> pool[c*chunk + i]. max_chunks bounds plan[1] (launch size; nc is safe). */
int gf_csc_compact(int dtype, const void* pool, void* staging, const uint64_t* plan,
                   const uint64_t* coff, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t max_chunks, void* stream);
/* nacc (nullable, fp16): adds the exact |x| sums of the written-back important chunks. */
int gf_csc_scatter(int dtype, void* pool, const void* staging, const uint64_t* plan,
                   const uint64_t* coff, uint64_t total, uint64_t chunk, uint64_t nc,
                   uint64_t max_chunks, uint64_t* nacc, void* stream);
/* From important flags (device): coff[c] = sum of lengths of important chunks < c;
 * plan (device, 4 + nc uint64): plan[0] = staged elements, plan[1] = important chunk
 * count, plan[2] = window count, plan[3] = elements per full window (theta policy of
 * sparse.cpp:142-158), plan[4 .. 4+plan[1]) = the important chunk indices, ascending. */
int gf_csc_plan(const uint8_t* important, uint64_t total, uint64_t chunk, uint64_t nc,
                int dtype, uint64_t theta, uint64_t* coff, uint64_t* plan, void* stream);
/* flags[c] = 1 for the k chunks with largest norm (ties: lower index), else 0. */
int gf_select_topk(const float* norms, uint64_t nc, uint64_t k, uint8_t* flags, void* stream);
/* For the important chunks of `plan`: g = dec(pool)*(1/world); u = mom*hu + lr*g; hu = u; w -= u. */
int gf_csc_sgd_update(int dtype, const void* pool, const uint64_t* plan, uint64_t total,
                      uint64_t chunk, uint64_t nc, uint64_t max_chunks, int world, float momentum,
                      float lr, float* hu, float* w, void* stream);
/* Whole pool: same recurrence as above without importance (trainer.cpp:337-346). */
int gf_dense_sgd_update(int dtype, const void* pool, uint64_t total, int world, float momentum,
                        float lr, float* hu, float* w, void* stream);

/* ---- communicator (data plane over NVLink peer memory) ---------------------------- */
/* Allocates this rank's symmetric heap (heap_bytes, 256-B aligned base) plus flags on
 * `device`. All ranks must create heaps of the same size. */
int gf_comm_create(int world, int rank, int device, uint64_t heap_bytes, gf_comm** out);
int gf_comm_destroy(gf_comm* comm);
int gf_comm_heap(gf_comm* comm, void** base, uint64_t* bytes);
/* Cross-process bootstrap: export this rank's handle, gather all ranks' handles
 * (rank order, world * GF_IPC_HANDLE_BYTES) over any control plane, then connect. */
int gf_comm_export_handle(gf_comm* comm, void* handle_out);
int gf_comm_connect_ipc(gf_comm* comm, const void* all_handles);
/* In-process bootstrap: comms[r] for every rank r, each on a distinct device. */
int gf_comm_connect_local(gf_comm* const* comms, int world);
/* Emulated world on ONE device: comms[r] for every rank r, all created on the same device.
 * Every kernel runs exactly as across GPUs (same instantiations, same cross-rank flags and
 * barriers, "peer" memory = the other ranks' allocations on this device); each rank must
 * launch on its own non-blocking stream. Grids are capped so that all ranks' barrier-waiting
 * CTAs are resident at once. Used to prove the multi-GPU kernels on a single B200. Requires
 * CUDA_MODULE_LOADING=EAGER (and, for worlds with more than 8 active streams,
 * CUDA_DEVICE_MAX_CONNECTIONS >= their count) in the environment before CUDA initialises. */
int gf_comm_connect_colocated(gf_comm* const* comms, int world);
/* Ring order (collectives.hpp:37-38): a permutation of ranks, identical on all ranks. */
int gf_comm_set_ring_order(gf_comm* comm, const int* order);
int gf_comm_set_timeout_ms(gf_comm* comm, uint64_t ms);
/* Upper bound on the CTAs per rank of this communicator's NVLink kernels (0: automatic). Must be
 * the same on every rank (CTA b pairs with CTA b). A CSC step caps its exchange so the rest of
 * the SMs keep packing beside it. */
int gf_comm_set_max_blocks(gf_comm* comm, int max_blocks);
/* CTA size (threads, multiple of 32, <= 512; 0: 512) of the CSC exchange kernels
 * (gf_ring_allreduce_planned_scatter, gf_csc_exchange_pull). Same on every rank. */
int gf_comm_set_block_threads(gf_comm* comm, int threads);
/* GF_OK, or GF_ERR_TRANSPORT once a device-side wait timed out (comm is then poisoned). */
int gf_comm_status(gf_comm* comm);
/* Tracing: when on, CTA 0 of every NVLink ring launch stamps %globaltimer (ns) into a
 * host-mapped record [kernel start, entry barrier passed, exit barrier begin, end];
 * gf_comm_trace copies the latest record (call after the launch completed). */
int gf_comm_set_trace(gf_comm* comm, int on);
int gf_comm_trace(gf_comm* comm, uint64_t* out4);
/* Words 0..n-1 (n <= 16) of the trace area: [0,4) the last collective kernel's CTA 0
 * [start, entered, exit begin, end]; [4,11) gf_csc_select's [start, norms finalized, entry
 * barrier passed, ring-order sums done, exit barrier passed, top-k done, end] (globaltimer ns). */
int gf_comm_trace_n(gf_comm* comm, uint64_t* out, int n);
int gf_comm_rank(gf_comm* comm);
int gf_comm_world(gf_comm* comm);

/* In-place allreduce (sum) of nwin windows of the symmetric buffer at heap offset
 * heap_off. Each window [win_start[w], +win_len[w]) (elements, relative to heap_off)
 * is split by segment_of and reduced in ring-arrival order (bit-exact with
 * ring_allreduce). One kernel launch per <= GF_MAX_WINDOWS_PER_LAUNCH windows. */
int gf_ring_allreduce(gf_comm* comm, int dtype, uint64_t heap_off, const uint64_t* win_start,
                      const uint64_t* win_len, int nwin, void* stream);
/* Same over explicit per-rank buffers (rank_bufs[r] = rank r's buffer as mapped on THIS
 * rank's GPU, 16-byte aligned; windows relative to each buffer start). Used for
 * registered user buffers (e.g. a GradientPool) instead of the symmetric heap. */
int gf_ring_allreduce_ptrs(gf_comm* comm, int dtype, void* const* rank_bufs,
                           const uint64_t* win_start, const uint64_t* win_len, int nwin,
                           void* stream);
/* Buffer registration across processes: export the IPC handle of the allocation holding
 * dev_ptr (+ its offset), open a peer's handle (mapped base on this rank's GPU), close. */
int gf_ipc_export(const void* dev_ptr, void* handle_out, uint64_t* offset_out);
int gf_ipc_open(gf_comm* comm, const void* handle, void** base_out);
int gf_ipc_close(gf_comm* comm, void* base);
/* Same with windows described by a device plan written by gf_csc_plan / gf_csc_select. */
int gf_ring_allreduce_planned(gf_comm* comm, int dtype, uint64_t heap_off,
                              const uint64_t* plan_dev, void* stream);
/* The planned exchange of the staging buffer at stage_heap_off WITH the write-back fused in:
 * after its exit barrier each CTA copies its staging vectors into `pool` (local, fp16) and
 * adds their exact |x| units to nacc — gf_ring_allreduce_planned + gf_csc_scatter in one
 * launch (sparse.cpp:142-168). fp16 only, chunk % 8 == 0, nc <= 6144, world > 1. */
int gf_ring_allreduce_planned_scatter(gf_comm* comm, int dtype, uint64_t stage_heap_off,
                                      const uint64_t* plan_dev, void* pool, uint64_t chunk,
                                      uint64_t nc, uint64_t* nacc, void* stream);
/* The same exchange + write-back without pushes: the owner of each segment pulls it from all
 * staging buffers (ring order), keeps the sum and writes it back; after one barrier every
 * rank pulls the other segments from their owners straight into its pool (+ exact |x|
 * units into nacc). Same results as gf_ring_allreduce_planned_scatter, bit for bit. The
 * staging buffer must not be rewritten before the next collective on the communicator
 * (gf_csc_select's barrier, in a CSC step). fp16, chunk % 8 == 0, nc <= 6144, world > 1. */
int gf_csc_exchange_pull(gf_comm* comm, uint64_t stage_heap_off, const uint64_t* plan_dev, void* pool,
                         uint64_t chunk, uint64_t nc, uint64_t* nacc, void* stream);
/* One dense sync step (pack -> ring allreduce of the theta windows -> unpack), bit-identical to
 * gf_pack + gf_ring_allreduce + gf_unpack. At world 1 the collective is the identity
 * (collectives.cpp:59) and the step is ONE streaming pass (pack_kernel<DstTable>: each value
 * is encoded, stored to the pool and decoded to g_avg from registers). The fp16/fp32 pool
 * lives at pool_heap_off in the symmetric heap; src/dst/pool_off/count are HOST arrays of
 * device pointers / sizes (any number of tensors, tiling the windows). */
int gf_sync_step_dense(gf_comm* comm, int dtype, uint64_t pool_heap_off, const float* const* src,
                       float* const* dst, const uint64_t* pool_off, const uint64_t* count,
                       int ntensors, const uint64_t* win_start, const uint64_t* win_len, int nwin,
                       void* stream);
/* The allreduce of the theta windows fused with the unpack (gf_ring_allreduce + gf_unpack):
 * the rank at ring position p sums segment p of every window by pulling it from all pools in
 * ring order, then pulls every other segment from its owner; each value is unpacked to
 * dst as x * (1/N) straight from registers and every pool ends holding the sums. Nothing is
 * pushed over NVLink. dst/pool_off/count are HOST arrays (<= 256 tensors tiling the windows).
 * flags: GF_RSAG_NO_EXIT_BARRIER skips the final "peers are done reading my pool" barrier; the
 * caller must then not rewrite this pool before its next collective on the communicator
 * (alternate two pools: the next collective's entry barrier orders the reuse). */
#define GF_RSAG_NO_EXIT_BARRIER 1
int gf_ring_allreduce_unpack(gf_comm* comm, int dtype, uint64_t pool_heap_off, float* const* dst,
                             const uint64_t* pool_off, const uint64_t* count, int ntensors,
                             const uint64_t* win_start, const uint64_t* win_len, int nwin, int flags,
                             void* stream);
/* One dense sync step with the reduce-scatter's traffic riding on the pack (push form): the
 * pack stores each packed vector straight into the owner of its segment (my pool, or my slot
 * of the owner's inbox over NVLink); then one kernel sums every owned segment from LOCAL memory
 * (pool + inbox slots, ring order from the owner: bit-identical), pushes the sums into every
 * rank's pool and unpacks them from registers, and after its exit barrier unpacks the segments
 * the peers pushed to it. Same results as gf_pack + gf_ring_allreduce + gf_unpack, bit for bit.
 * fp16; the inbox (world-1 slots of round_up(pool span, 8) elements each, at inbox_heap_off,
 * same offset on every rank) lives in the symmetric heap; pool and inbox offsets are 16-byte
 * aligned and must not overlap. src/dst/pool_off/count are HOST arrays. Beyond 256 tensors or
 * windows (or with GF_FUSE_UNPACK=0) a separate unpack launch follows. */
int gf_sync_step_dense_push(gf_comm* comm, int dtype, uint64_t pool_heap_off, uint64_t inbox_heap_off,
                            const float* const* src, float* const* dst, const uint64_t* pool_off,
                            const uint64_t* count, int ntensors, const uint64_t* win_start,
                            const uint64_t* win_len, int nwin, void* stream);
/* Emulation of `world` ranks whose buffers all live on the current device (no waits). */
int gf_ring_allreduce_colocated(int dtype, void* const* bufs, int world, const int* ring_order,
                                const uint64_t* win_start, const uint64_t* win_len, int nwin,
                                void* stream);
int gf_ring_allreduce_colocated_planned(int dtype, void* const* bufs, int world,
                                        const int* ring_order, const uint64_t* plan_dev,
                                        void* stream);
/* Norm exchange + selection for the next iteration (sparse.cpp:185-201), one kernel:
 * norms (nc fp32 at heap offset norms_off on every rank) are summed over ranks in
 * ring order (as the fp32 ring_allreduce would), written back to every rank's local
 * norms, top-k selected -> flags (device, nc bytes); then coff/plan as gf_csc_plan. */
/* With nacc != NULL the local norms are first finalized from the exact accumulators
 * (float(sum), x1/N where imp_cur[c]) and nacc is zeroed for the next iteration. */
/* Switches this communicator's gf_csc_select to the push-inbox norm exchange: every rank
 * writes its finalized norms into slot `rank` of each peer's inbox (world x nc floats at
 * inbox_heap_off in the symmetric heap, same offset on every rank), so the selection needs one
 * cross-GPU barrier instead of two and reads only local memory. Same results. All ranks must
 * switch together; UINT64_MAX switches back. The caller must not rewrite its norms or
 * inbox before its next exchange (the CSC step order guarantees it). */
int gf_comm_set_select_inbox(gf_comm* comm, uint64_t inbox_heap_off);
/* Switches this communicator's CSC exchange to the routed form: world-1 inbox slots of
 * slot_elems fp16 elements (a multiple of 8, >= the staging capacity) at inbox_heap_off (same
 * offset on every rank); gf_csc_pack_correct_routed stores every staged element at the owner of
 * its exchange segment (my staging, or my slot of the owner's inbox over NVLink), so
 * gf_csc_exchange_pull reduces from local memory and pulls only the all-gather. Same results.
 * All ranks switch together; UINT64_MAX switches back. */
int gf_comm_set_csc_inbox(gf_comm* comm, uint64_t inbox_heap_off, uint64_t slot_elems);
/* Part 1 of gf_csc_pack_correct_part (the chunks of the device-side `plan`, fp16, tensors in
 * ascending id) with every staged element routed to its exchange owner (gf_comm_set_csc_inbox);
 * the staging buffer is at stage_heap_off in the symmetric heap. */
int gf_csc_pack_correct_routed(gf_comm* comm, void* pool, float* hg, uint64_t stage_heap_off,
                               const uint64_t* plan, uint64_t chunk, const float* const* src,
                               const uint64_t* pool_off, const uint64_t* count, int ntensors,
                               float momentum, void* stream);
int gf_csc_select(gf_comm* comm, uint64_t norms_off, uint64_t nc, uint64_t k,
                  uint8_t* flags, uint64_t total, uint64_t chunk, int dtype, uint64_t theta,
                  uint64_t* coff, uint64_t* plan, uint64_t* nacc, const void* pool,
                  const uint8_t* imp_cur, void* stream);
int gf_csc_select_colocated(float* const* norms, int world, const int* ring_order,
                            uint64_t nc, uint64_t k, uint8_t* flags, uint64_t total,
                            uint64_t chunk, int dtype, uint64_t theta, uint64_t* coff,
                            uint64_t* plan, uint64_t* const* nacc, const void* const* pools,
                            const uint8_t* imp_cur, void* stream);

/* Rooted helpers over peer-addressable per-rank buffers, launched by ONE rank after the
 * others signalled readiness over the control plane (host-orchestrated collectives):
 * oracle_allreduce (collectives.cpp:203-226): every buffer = ((b0 + b1) + ...) + b[N-1];
 * broadcast: every buffer = bufs[root]. */
int gf_oracle_allreduce_ptrs(int dtype, void* const* bufs, int world, uint64_t len, void* stream);
int gf_broadcast_ptrs(void* const* bufs, int world, int root, uint64_t bytes, void* stream);
/* Rooted ring reduce (reduce(), collectives.cpp:99-144, 229-235), bufs in RING-POSITION
 * order: the root position gets every full sum; position j+k keeps segment j's partial sum
 * of positions j..j+k (the reference's reduce-scatter state), position j its raw segment j.
 * hierarchical_allreduce (collectives.cpp:179-201) = this per group + ring allreduce over
 * the masters + broadcast. */
int gf_ring_reduce_ptrs(int dtype, void* const* bufs, int n, int root_pos, uint64_t len, void* stream);

/* Payload bytes the reference ring records for one allreduce of len elements at ring
 * position `position` (collectives.cpp:69-96): 2(N-1) sends of segment_of sizes. */
int gf_ring_traffic(uint64_t len, int world, int position, int dtype, uint64_t* bytes_sent,
                    uint64_t* bytes_received, uint64_t* frames_sent);


/* ---- synthetic inputs (harness) --------------------------------------------------------------
 * The benchmark's seeded gradient sets (extends bench_allreduce's stream,
 * src/harness.cpp:280-283): std::mt19937_64(1234 + rank + 7919*step), tensors in ascending id,
 * uniform_real_distribution<float>(-1,1) * 2^-(id mod 7). out: HOST buffer of sum(sizes) floats,
 * ascending id. Host-only, no GPU. */
int gf_synth_grads(int rank, int step, const uint64_t* sizes, int ntensors, float* out);

/* ---- engine: one rank's whole gradient-sync step ---------------------------------------------
 * The launch sequence a data-parallel trainer runs per iteration (trainer.cpp:297-347 with
 * FusionEngine fusion.cpp:72-109 and SparseState sparse.cpp:57-224), device-resident and
 * asynchronous on the caller's stream: no host synchronisation inside a step, so a step can be
 * captured into a CUDA graph. Gradient/output tables are HOST arrays of per-tensor DEVICE
 * pointers in ascending tensor id (id 1 first), as the reference's write_tensor(id, span). */
typedef struct gf_engine gf_engine;
enum { GF_DENSE_AUTO = 0, GF_DENSE_RSPUSH = 1, GF_DENSE_PULL = 2, GF_DENSE_PUSH = 3 };
enum { GF_CSC_PUSH = 0, GF_CSC_PULL = 1, GF_CSC_AUTO = 2 };
typedef struct {
    int world, rank, device, dtype;
    uint64_t theta_bytes;     /* FusionConfig::threshold_bytes (fusion.hpp:27-30) */
    uint64_t chunk;           /* GradientPool chunk size (gradient_pool.hpp:16) */
    int csc;                  /* 0: dense lazy allreduce; 1: CSC (TrainOptions::csc) */
    int dense_mode;           /* GF_DENSE_*: N>1 dense exchange (AUTO = RSPUSH for fp16) */
    int csc_mode;             /* GF_CSC_*: N>1 CSC exchange form (AUTO: routed PULL from 4 ranks, else PUSH) */
    double final_sparsity;    /* SparseConfig (sparse.hpp:21-26) */
    uint64_t warmup_iters;
    double momentum, learning_rate;
    uint64_t timeout_ms;      /* device-side barrier timeout (transport.hpp:25) */
} gf_engine_config;
typedef struct {
    uint64_t total, num_chunks, heap_bytes;
    int nwin;                 /* dense theta windows per iteration */
    int dense_mode;           /* resolved GF_DENSE_* */
    uint64_t iteration;       /* CSC iterations run */
    int csc_mode;             /* resolved GF_CSC_* */
} gf_engine_info;
enum { GF_STATE_POOL = 0, GF_STATE_HG, GF_STATE_HU, GF_STATE_W, GF_STATE_IMP_NEXT, GF_STATE_NORMS,
       GF_STATE_NACC, GF_STATE_PLAN_NEXT, GF_STATE_IMP_CUR, GF_STATE_PLAN_CUR };
/* Defaults: world 1, fp16, theta 64 MiB, chunk 32000, dense, AUTO, momentum 0.9, lr 0.01,
 * final_sparsity 0.9, timeout 30 s (trainer.hpp / fusion.hpp / sparse.hpp defaults). */
void gf_engine_config_init(gf_engine_config* cfg);
int gf_engine_create(const gf_engine_config* cfg, const uint64_t* sizes, int ntensors, gf_engine** out);
int gf_engine_destroy(gf_engine* e);
/* The engine's communicator: bootstrap with gf_comm_export_handle + gf_engine_connect_ipc. */
gf_comm* gf_engine_comm(gf_engine* e);
int gf_engine_connect_ipc(gf_engine* e, const void* all_handles);
int gf_engine_connect_local(gf_engine* const* engines, int world);
int gf_engine_connect_colocated(gf_engine* const* engines, int world);
int gf_engine_info_get(gf_engine* e, gf_engine_info* out);
/* Device buffers the engine owns (GF_STATE_*): pool (the one holding the last dense step's
 * sums), CSC residual hg, momentum hu, weights w (zero-initialised), the next important set,
 * the chunk norms, the exact-L1 accumulators, the next plan, the current set. */
int gf_engine_state(gf_engine* e, int which, void** ptr, uint64_t* bytes);
/* Dense iteration: out[t] = g_avg of tensor t (sum over ranks x 1/N, via the fp16/fp32 pool). */
int gf_engine_dense_step(gf_engine* e, const float* const* grads, float* const* out, void* stream);
/* CSC iteration (Algorithm 1): pack+correct+compact, exchange + write-back + exact L1, norm
 * exchange + top-k of the next set, momentum update of the important chunks of w. */
int gf_engine_csc_step(gf_engine* e, const float* const* grads, void* stream);
/* Overlap with backward (fusion.cpp:72-123): tensors become final in descending id; each theta
 * window is launched on a communication stream when it closes; finalize makes `stream` wait. */
int gf_engine_begin_iteration(gf_engine* e, const float* const* grads, float* const* out, void* stream);
int gf_engine_tensor_complete(gf_engine* e, int tensor_id);
int gf_engine_finalize_iteration(gf_engine* e);
/* Per-kernel timing: with marks on, every step records an event before each kernel phase;
 * gf_engine_marks synchronises and returns the mean ms per phase ("name" strings separated by
 * ';' in names) over the steps since the last call, then clears. Returns the phase count. */
int gf_engine_set_marks(gf_engine* e, int on);
int gf_engine_marks(gf_engine* e, char* names, int names_cap, float* ms, int cap);

#ifdef __cplusplus
}
#endif
#endif /* GFLOW_B200_H */
