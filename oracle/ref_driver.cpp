// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY. A C-ABI shim over the UNMODIFIED reference library
// (compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// It drives the reference's own public C++ API exactly the way its callers do
// (trainer.cpp:264-382 emit/sync/update, harness.cpp:245-339 bench) so that
// tests can (1) pin the C restatement in gf_oracle.c and generate golden
// fixtures, and (2) time the reference CPU path for bench.py's cpu_baseline
// and `--impl reference` arm. Nothing here is part of the product.

#include <algorithm>
#include <array>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "gflow/collectives.hpp"
#include "gflow/fusion.hpp"
#include "gflow/gradient_pool.hpp"
#include "gflow/half.hpp"
#include "gflow/harness.hpp"
#include "gflow/inproc.hpp"
#include "gflow/sparse.hpp"
#include "gflow/trainer.hpp"

using namespace gflow;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const ProtocolError& e) {
        g_err = e.what();
        return 2;
    } catch (const TransportError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

template <typename F>
void run_world(int n, F body) {
    auto world = make_inproc_world(n);
    std::vector<std::thread> ts;
    std::vector<std::exception_ptr> errors(static_cast<std::size_t>(n));
    for (int r = 0; r < n; ++r) {
        ts.emplace_back([&, r] {
            try {
                body(r, *world[static_cast<std::size_t>(r)]);
            } catch (...) {
                errors[static_cast<std::size_t>(r)] = std::current_exception();
            }
        });
    }
    for (auto& t : ts) t.join();
    for (auto& e : errors) {
        if (e) std::rethrow_exception(e);
    }
}

std::vector<std::size_t> to_sizes(const std::uint64_t* sizes, int m) {
    return std::vector<std::size_t>(sizes, sizes + m);
}

// Ascending-id offsets into a flat per-rank gradient array (id 1 first).
std::vector<std::size_t> asc_offsets(const std::vector<std::size_t>& s) {
    std::vector<std::size_t> o(s.size() + 1, 0);
    for (std::size_t i = 0; i < s.size(); ++i) o[i + 1] = o[i] + s[i];
    return o;
}

Algo algo_of(int a) { return a == 1 ? Algo::kHierarchical : a == 2 ? Algo::kOracle : Algo::kRing; }

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace

extern "C" {

const char* refd_last_error() { return g_err.c_str(); }

// ---- binary16 codec (half.hpp:20-87) -------------------------------------------
void refd_f2h_array(const float* in, std::uint16_t* out, std::uint64_t n) {
    for (std::uint64_t i = 0; i < n; ++i) out[i] = float_to_half_bits(in[i]);
}
void refd_h2f_array(const std::uint16_t* in, float* out, std::uint64_t n) {
    for (std::uint64_t i = 0; i < n; ++i) out[i] = half_bits_to_float(in[i]);
}
// Order-independent digest of float_to_half_bits over the fp32 bit patterns
// [first, first+count): sum mod 2^64 of splitmix64(bits<<16 | half). The GPU
// codec self-test computes the same digest with the device encoder.
std::uint64_t refd_codec_digest(std::uint64_t first, std::uint64_t count) {
    std::uint64_t acc = 0;
    for (std::uint64_t x = first; x < first + count; ++x) {
        const std::uint32_t b = static_cast<std::uint32_t>(x);
        const std::uint16_t h = float_to_half_bits(std::bit_cast<float>(b));
        acc += splitmix64((static_cast<std::uint64_t>(b) << 16) | h);
    }
    return acc;
}
// accumulate (buffer.hpp:60-81) over raw element arrays.
void refd_accumulate(int dtype, void* dst, const void* src, std::uint64_t n) {
    ScalarBuffer d{dtype == 1 ? ElementType::kF16 : ElementType::kF32,
                   static_cast<std::byte*>(dst), n};
    accumulate(d, std::span<const std::byte>(static_cast<const std::byte*>(src),
                                             n * element_size(d.type)));
}

// ---- pool layout (gradient_pool.cpp:11-70) -------------------------------------
int refd_pool_layout(const std::uint64_t* sizes, int m, std::uint64_t chunk,
                     std::uint64_t* offsets_out, std::uint64_t* nc_out,
                     std::uint64_t* chunk_len_out, std::uint64_t cap) {
    return guarded([&] {
        GradientPool pool(to_sizes(sizes, m), chunk, ElementType::kF32);
        for (int id = 1; id <= m; ++id) offsets_out[id - 1] = pool.desc(id).pool_offset;
        *nc_out = pool.num_chunks();
        for (std::size_t c = 0; c < pool.num_chunks() && c < cap; ++c) {
            chunk_len_out[c] = pool.chunk_length(c);
        }
    });
}

std::uint64_t refd_selection_count(double s, std::uint64_t nc) { return selection_count(s, nc); }
double refd_sparsity_at(std::uint64_t t, std::uint64_t w, double s) { return sparsity_at(t, w, s); }

// ---- ring allreduce on raw arrays, ranks as threads (collectives.cpp:55-97) ----
// bufs[r] holds rank r's `len` elements of `dtype`; reduced in place.
// algo: 0 ring, 1 hierarchical(group), 2 oracle. sent_out[r] = payload bytes sent.
int refd_allreduce(int n, int dtype, std::uint64_t len, void* const* bufs, int algo,
                   int group_size, const int* ring_order, std::uint64_t* sent_out) {
    return guarded([&] {
        run_world(n, [&](int r, Transport& tp) {
            Communicator comm(tp, group_size);
            if (ring_order) comm.set_ring_order(std::vector<int>(ring_order, ring_order + n));
            ScalarBuffer b{dtype == 1 ? ElementType::kF16 : ElementType::kF32,
                           static_cast<std::byte*>(bufs[r]), len};
            switch (algo_of(algo)) {
                case Algo::kRing: ring_allreduce(comm, b); break;
                case Algo::kHierarchical: hierarchical_allreduce(comm, b); break;
                case Algo::kOracle: oracle_allreduce(comm, b); break;
            }
            if (sent_out) sent_out[r] = tp.stats().total().payload_bytes_sent;
        });
    });
}

// ---- rooted ring reduce on raw arrays (collectives.cpp:99-144, 229-235) ----------
int refd_reduce(int n, int dtype, std::uint64_t len, void* const* bufs, int root,
                const int* ring_order, std::uint64_t* sent_out) {
    return guarded([&] {
        run_world(n, [&](int r, Transport& tp) {
            Communicator comm(tp);
            if (ring_order) comm.set_ring_order(std::vector<int>(ring_order, ring_order + n));
            ScalarBuffer b{dtype == 1 ? ElementType::kF16 : ElementType::kF32,
                           static_cast<std::byte*>(bufs[r]), len};
            reduce(comm, b, root);
            if (sent_out) sent_out[r] = tp.stats().total().payload_bytes_sent;
        });
    });
}

// ---- dense lazy-allreduce step (trainer.cpp:297-347 without the model) ---------
// grads[r]: rank r's gradients, flat in ASCENDING tensor id. Outputs (nullable):
// pools_out[r] raw pool bytes after the fused windows, gavg_out[r] pool-ordered
// dec(pool)*(1/N) (the update loop's read, trainer.cpp:336-342),
// window_bytes_out (rank 0, cap entries), sent_out[r] payload bytes.
int refd_dense_sync(int n, const std::uint64_t* sizes, int m, std::uint64_t chunk, int dtype,
                    std::uint64_t theta, int algo, int group_size,
                    const float* const* grads, void* const* pools_out,
                    float* const* gavg_out, std::uint64_t* window_bytes_out,
                    std::uint64_t cap, std::uint64_t* nwin_out, std::uint64_t* sent_out) {
    return guarded([&] {
        const auto sz = to_sizes(sizes, m);
        const auto ao = asc_offsets(sz);
        run_world(n, [&](int r, Transport& tp) {
            GradientPool pool(sz, chunk, dtype == 1 ? ElementType::kF16 : ElementType::kF32);
            Communicator comm(tp, group_size);
            FusionEngine engine(pool, comm, FusionConfig{theta, algo_of(algo)});
            pool.begin_iteration();
            engine.begin_iteration();
            std::vector<FusedHandle> handles;
            for (int id = m; id >= 1; --id) {
                pool.write_tensor(id, std::span<const float>(grads[r] + ao[id - 1], sz[id - 1]));
                for (auto& h : engine.on_tensor_complete(id)) handles.push_back(std::move(h));
            }
            if (auto h = engine.finalize_iteration()) handles.push_back(std::move(*h));
            FusionEngine::wait_all(handles);
            ScalarBuffer v = pool.view();
            if (pools_out && pools_out[r]) std::memcpy(pools_out[r], v.data, v.byte_length());
            if (gavg_out && gavg_out[r]) {
                const float inv_world = 1.0f / static_cast<float>(n);
                for (std::size_t i = 0; i < pool.total_elements(); ++i) {
                    gavg_out[r][i] = v.get(i) * inv_world;
                }
            }
            if (r == 0) {
                const auto& wb = engine.last_log().window_bytes;
                if (nwin_out) *nwin_out = wb.size();
                for (std::size_t i = 0; i < wb.size() && i < cap; ++i) window_bytes_out[i] = wb[i];
            }
            if (sent_out) sent_out[r] = tp.stats().total().payload_bytes_sent;
        });
    });
}

// ---- CSC, T iterations (trainer.cpp:297-330 CSC branch + sparse.cpp) ----------
// grads[t*n + r]: flat ascending-id gradients of rank r at step t.
// weights0: initial pool-shaped master weights (nullable = zeros).
// Per-step outputs, each indexed [(t*n + r)] and nullable:
//   pool_corr  raw pool bytes after write_tensor+correction (before exchange)
//   hg         fp32 residual after correction
//   pool_x     raw pool bytes after sparse_exchange
//   norms_loc  chunk_l1(c) * (important ? 1/N : 1)   (sparse.cpp:176-184)
//   norms_sum  the same vector ring-allreduced in fp32 (sparse.cpp:185-187)
//   imp        the important set used this step (nc bytes)
//   next_imp   select_next_important result (nc bytes)
//   hu, w      after sgd_update (sparse.cpp:206-224)
//   csum       checksum() this step
int refd_csc_run(int n, const std::uint64_t* sizes, int m, std::uint64_t chunk, int dtype,
                 std::uint64_t theta, double final_sparsity, std::uint64_t warmup,
                 double momentum, double lr, int steps, const float* const* grads,
                 const float* weights0, void* const* pool_corr, float* const* hg_out,
                 void* const* pool_x, float* const* norms_loc, float* const* norms_sum,
                 std::uint8_t* const* imp_out, std::uint8_t* const* next_imp,
                 float* const* hu_out, float* const* w_out, std::uint64_t* csum,
                 std::uint64_t* windows_out) {
    return guarded([&] {
        const auto sz = to_sizes(sizes, m);
        const auto ao = asc_offsets(sz);
        run_world(n, [&](int r, Transport& tp) {
            const ElementType et = dtype == 1 ? ElementType::kF16 : ElementType::kF32;
            GradientPool pool(sz, chunk, et);
            Communicator comm(tp);
            FusionEngine engine(pool, comm, FusionConfig{theta, Algo::kRing});
            SparseState sparse(pool, SparseConfig{momentum, lr, final_sparsity, warmup});
            std::vector<float> w(pool.total_elements(), 0.0f);
            if (weights0) std::copy(weights0, weights0 + w.size(), w.begin());
            const std::size_t nc = pool.num_chunks();
            const std::size_t total = pool.total_elements();
            const std::size_t esz = element_size(et);
            for (int t = 0; t < steps; ++t) {
                const std::size_t k = static_cast<std::size_t>(t) * n + r;
                pool.begin_iteration();
                engine.begin_iteration();
                sparse.begin_iteration(static_cast<std::uint64_t>(t));
                if (imp_out && imp_out[k]) std::memcpy(imp_out[k], sparse.important().data(), nc);
                for (int id = m; id >= 1; --id) {
                    auto done = pool.write_tensor(
                        id, std::span<const float>(grads[k] + ao[id - 1], sz[id - 1]));
                    for (auto c : done) sparse.correction_pre_allreduce(c);
                }
                if (pool_corr && pool_corr[k]) std::memcpy(pool_corr[k], pool.view().data, total * esz);
                if (hg_out && hg_out[k]) std::memcpy(hg_out[k], sparse.hg().data(), total * 4);
                if (csum) csum[k] = sparse.checksum();
                sparse.sparse_exchange(comm, engine);
                if (windows_out) windows_out[k] = sparse.last_exchange_windows();
                if (pool_x && pool_x[k]) std::memcpy(pool_x[k], pool.view().data, total * esz);
                if ((norms_loc && norms_loc[k]) || (norms_sum && norms_sum[k])) {
                    std::vector<float> nv(nc);
                    const float inv_world = 1.0f / static_cast<float>(comm.world_size());
                    for (std::size_t c = 0; c < nc; ++c) {
                        float v = pool.chunk_l1(c);
                        if (sparse.important()[c]) v *= inv_world;
                        nv[c] = v;
                    }
                    if (norms_loc && norms_loc[k]) std::memcpy(norms_loc[k], nv.data(), nc * 4);
                    ScalarBuffer nb{ElementType::kF32, reinterpret_cast<std::byte*>(nv.data()), nc};
                    ring_allreduce(comm, nb);
                    if (norms_sum && norms_sum[k]) std::memcpy(norms_sum[k], nv.data(), nc * 4);
                }
                const auto& nx = sparse.select_next_important(comm, static_cast<std::uint64_t>(t));
                if (next_imp && next_imp[k]) std::memcpy(next_imp[k], nx.data(), nc);
                sparse.sgd_update(w, n);
                if (hu_out && hu_out[k]) std::memcpy(hu_out[k], sparse.hu().data(), total * 4);
                if (w_out && w_out[k]) std::memcpy(w_out[k], w.data(), total * 4);
            }
        });
    });
}

// ---- bench_allreduce (harness.cpp:245-339) --------------------------------------
int refd_bench_allreduce(int ranks, std::uint64_t bytes, int algo, int group_size, int dtype,
                         std::uint64_t* sent, std::uint64_t* predicted, int* matches) {
    return guarded([&] {
        auto r = bench_allreduce(ranks, bytes, algo_of(algo), group_size, "inproc",
                                 dtype == 1 ? ElementType::kF16 : ElementType::kF32);
        *sent = r.per_rank_payload_sent;
        *predicted = r.predicted_payload;
        *matches = r.matches_oracle ? 1 : 0;
    });
}

// ---- whole training runs (trainer.cpp:264-382), ranks as threads -------------------
// dims: model_dims (nd entries). Outputs (rank 0): losses[iterations], grad_bytes[iterations],
// weights[n_params] (final); returns the parameter count in *n_params.
int refd_train(int ranks, const std::uint64_t* dims, int nd, int logistic, std::uint64_t iterations,
               std::uint64_t n_examples, std::uint64_t batch, double lr, double momentum, std::uint64_t seed,
               int algo, int dtype, std::uint64_t theta, int csc, double final_sparsity, std::uint64_t warmup,
               std::uint64_t chunk, double* losses, std::uint64_t* grad_bytes, float* weights,
               std::uint64_t cap, std::uint64_t* n_params) {
    return guarded([&] {
        TrainOptions o;
        o.model_dims.assign(dims, dims + nd);
        o.task = logistic ? Task::kLogistic : Task::kLinearRegression;
        o.iterations = iterations;
        o.n_examples = n_examples;
        o.batch = batch;
        o.learning_rate = lr;
        o.momentum = momentum;
        o.seed = seed;
        o.algorithm = algo_of(algo);
        o.wire_precision = dtype == 1 ? ElementType::kF16 : ElementType::kF32;
        o.theta_bytes = theta;
        o.csc = csc != 0;
        o.final_sparsity = final_sparsity;
        o.warmup_iters = warmup;
        o.chunk_size = chunk;
        std::vector<TrainResult> res(static_cast<std::size_t>(ranks));
        run_world(ranks, [&](int r, Transport& tp) { res[static_cast<std::size_t>(r)] = train_worker(o, tp); });
        const auto& r0 = res[0];
        for (std::size_t t = 0; t < r0.metrics.size(); ++t) {
            losses[t] = r0.metrics[t].loss;
            grad_bytes[t] = r0.metrics[t].grad_payload_bytes;
        }
        *n_params = r0.final_weights.size();
        for (std::size_t i = 0; i < r0.final_weights.size() && i < cap; ++i) weights[i] = r0.final_weights[i];
    });
}

// ---- seeded synthetic gradients ---------------------------------
// mt19937_64(1234 + r + 7919 t), tensors in ascending id, uniform(-1,1) * 2^-(id mod 7).
void refd_gen_grads(int r, int t, const std::uint64_t* sizes, int m, float* out) {
    std::mt19937_64 rng(1234 + static_cast<std::uint64_t>(r) + 7919ull * static_cast<std::uint64_t>(t));
    std::uniform_real_distribution<float> uni(-1.0f, 1.0f);
    std::size_t o = 0;
    for (int id = 1; id <= m; ++id) {
        const float s = std::ldexp(1.0f, -(id % 7));
        for (std::uint64_t i = 0; i < sizes[id - 1]; ++i) out[o++] = uni(rng) * s;
    }
}

// ---- CPU baseline timing: the reference path, ranks as threads ------------------
// Per step (after `warmup` untimed steps): each rank thread times
//   pack     write_tensor loop (+ correction_pre_allreduce when csc)
//   exchange FusionEngine windows + wait_all, or sparse_exchange
//   select   select_next_important (csc only)
//   unpack   g_avg = dec(pool)*(1/N) over the pool (dense) or sgd_update (csc)
// stats_out[0..4] = median over steps of the max over ranks of
// {pack, exchange, select, unpack, total}. Gradients are generated outside the
// timed region with refd_gen_grads.
int refd_time_step(int n, const std::uint64_t* sizes, int m, std::uint64_t chunk, int dtype,
                   std::uint64_t theta, int csc, double final_sparsity, int steps, int warmup,
                   double* stats_out) {
    return guarded([&] {
        const auto sz = to_sizes(sizes, m);
        const auto ao = asc_offsets(sz);
        std::uint64_t total = 0;
        for (auto s : sz) total += s;
        // per-rank, per-step stage times
        std::vector<std::vector<std::array<double, 5>>> rec(
            static_cast<std::size_t>(n), std::vector<std::array<double, 5>>(static_cast<std::size_t>(steps)));
        run_world(n, [&](int r, Transport& tp) {
            const ElementType et = dtype == 1 ? ElementType::kF16 : ElementType::kF32;
            GradientPool pool(sz, chunk, et);
            Communicator comm(tp);
            FusionEngine engine(pool, comm, FusionConfig{theta, Algo::kRing});
            SparseState sparse(pool, SparseConfig{0.9, 0.01, csc ? final_sparsity : 0.0, 0});
            std::vector<float> g(total), gavg(total), w(total, 0.0f);
            for (int t = 0; t < warmup + steps; ++t) {
                refd_gen_grads(r, t, sizes, m, g.data());
                tp.barrier();
                const double t0 = now_ms();
                pool.begin_iteration();
                engine.begin_iteration();
                if (csc) sparse.begin_iteration(static_cast<std::uint64_t>(t));
                std::vector<FusedHandle> handles;
                for (int id = m; id >= 1; --id) {
                    auto done = pool.write_tensor(
                        id, std::span<const float>(g.data() + ao[id - 1], sz[id - 1]));
                    if (csc) {
                        for (auto c : done) sparse.correction_pre_allreduce(c);
                    }
                }
                const double t1 = now_ms();
                if (csc) {
                    sparse.sparse_exchange(comm, engine);
                } else {
                    for (int id = m; id >= 1; --id) {
                        for (auto& h : engine.on_tensor_complete(id)) handles.push_back(std::move(h));
                    }
                    if (auto h = engine.finalize_iteration()) handles.push_back(std::move(*h));
                    FusionEngine::wait_all(handles);
                }
                const double t2 = now_ms();
                if (csc) sparse.select_next_important(comm, static_cast<std::uint64_t>(t));
                const double t3 = now_ms();
                if (csc) {
                    sparse.sgd_update(w, n);
                } else {
                    const float inv_world = 1.0f / static_cast<float>(n);
                    ScalarBuffer v = pool.view();
                    for (std::size_t i = 0; i < total; ++i) gavg[i] = v.get(i) * inv_world;
                }
                const double t4 = now_ms();
                if (t >= warmup) {
                    rec[static_cast<std::size_t>(r)][static_cast<std::size_t>(t - warmup)] =
                        {t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0};
                }
            }
        });
        for (int s = 0; s < 5; ++s) {
            std::vector<double> per_step;
            for (int t = 0; t < steps; ++t) {
                double mx = 0.0;
                for (int r = 0; r < n; ++r) mx = std::max(mx, rec[r][t][s]);
                per_step.push_back(mx);
            }
            std::sort(per_step.begin(), per_step.end());
            stats_out[s] = per_step[per_step.size() / 2];
        }
    });
}

}  // extern "C"
