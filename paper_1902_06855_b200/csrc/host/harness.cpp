// SPDX-License-Identifier: Apache-2.0
// Experiment harness on B200 (behaviour of the reference's src/harness.cpp: validate :111-130,
// predict_traffic :132-159, bench_allreduce :245-339, run_experiment :161-243). Ranks are host
// threads; each drives a GPU through DeviceContext (the data plane), with the in-process or a
// loopback TCP transport as the control plane.
#include "gflow/harness.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <memory>
#include <random>
#include <thread>
#include <vector>

#include "gflow/collectives.hpp"
#include "gflow/fusion.hpp"
#include "gflow/inproc.hpp"
#include "gflow/sparse.hpp"
#include "gflow/tcp.hpp"

namespace gflow {

namespace {

// weights + biases of the MLP the trainer builds (trainer.hpp Model: layer l has
// dims[l] x dims[l-1] weights and dims[l] biases)
std::uint64_t model_parameter_count(const std::vector<std::size_t>& dims) {
    std::uint64_t n = 0;
    for (std::size_t l = 1; l < dims.size(); ++l) n += dims[l] * dims[l - 1] + dims[l];
    return n;
}

std::vector<std::unique_ptr<Transport>> make_world(int ranks, const std::string& transport) {
    std::vector<std::unique_ptr<Transport>> out;
    if (transport == "inproc") {
        for (auto& t : make_inproc_world(ranks)) out.push_back(std::move(t));
        return out;
    }
    if (transport != "tcp") throw ConfigError("transport must be inproc or tcp");
    const auto peers = TcpTransport::loopback_addresses(ranks, port_base_from_env());
    out.resize(static_cast<std::size_t>(ranks));
    std::vector<std::thread> connect;
    std::vector<std::exception_ptr> err(static_cast<std::size_t>(ranks));
    for (int r = 0; r < ranks; ++r) {
        connect.emplace_back([&, r] {
            try {
                out[static_cast<std::size_t>(r)] = std::make_unique<TcpTransport>(r, ranks, peers);
            } catch (...) {
                err[static_cast<std::size_t>(r)] = std::current_exception();
            }
        });
    }
    for (auto& t : connect) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
    return out;
}

// body(rank, transport) on one thread per rank, each bound to its GPU; first error rethrown.
template <typename F>
void on_rank_threads(std::vector<std::unique_ptr<Transport>>& world, F body) {
    const int n = static_cast<int>(world.size());
    std::vector<std::thread> ts;
    std::vector<std::exception_ptr> err(static_cast<std::size_t>(n));
    for (int r = 0; r < n; ++r) {
        ts.emplace_back([&, r] {
            try {
                cudaSetDevice(thread_rank_device(r, n));
                body(r, *world[static_cast<std::size_t>(r)]);
            } catch (...) {
                err[static_cast<std::size_t>(r)] = std::current_exception();
            }
        });
    }
    for (auto& t : ts) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

}  // namespace

int thread_rank_device(int rank, int ranks) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    return n >= ranks ? rank : 0;
}

std::uint16_t port_base_from_env() {
    if (const char* s = std::getenv("GFLOW_PORT_BASE")) {
        const int p = std::atoi(s);
        if (p > 0 && p < 65000) return static_cast<std::uint16_t>(p);
    }
    return 28500;
}

void validate(const RunConfig& c) {
    const TrainOptions& t = c.train;
    if (c.ranks < 1) throw ConfigError("ranks must be >= 1");
    if (c.transport != "inproc" && c.transport != "tcp") throw ConfigError("transport must be inproc or tcp");
    if (t.model_dims.size() < 2) throw ConfigError("model needs >= 2 dims");
    if (t.batch < 1) throw ConfigError("batch must be >= 1");
    if (t.group_size < 1 || c.ranks % t.group_size != 0)
        throw ConfigError("group size " + std::to_string(t.group_size) + " must divide ranks " +
                          std::to_string(c.ranks));
    if (t.chunk_size == 0) throw ConfigError("chunk-size must be positive");
    if (t.csc && !(t.final_sparsity >= 0.0 && t.final_sparsity < 1.0)) throw ConfigError("sparsity must be in [0, 1)");
    if (t.n_examples % static_cast<std::size_t>(c.ranks) != 0)
        throw ConfigError("n_examples must be divisible by ranks");
}

TrafficPrediction predict_traffic(std::uint64_t pool_elements, std::size_t element_bytes, int ranks,
                                  double sparsity, std::size_t chunk_size, bool csc) {
    TrafficPrediction p;
    const double n = static_cast<double>(ranks);
    const double ring = ranks > 1 ? 2.0 * (n - 1.0) / n : 0.0;  // the ring's 2(N-1)/N law
    const double pool_bytes = static_cast<double>(pool_elements) * static_cast<double>(element_bytes);
    if (!csc) {
        p.grad_bytes = ring * pool_bytes;
        return p;
    }
    // steady state: the k selected chunks travel, plus the fp32 norm vector (the chunk count
    // here is the ceiling, as the reference's analytic anchor uses)
    const std::size_t nc = static_cast<std::size_t>((pool_elements + chunk_size - 1) / chunk_size);
    const std::size_t k = selection_count(sparsity, nc);
    const double sel = static_cast<double>(k) * static_cast<double>(chunk_size) * static_cast<double>(element_bytes);
    p.grad_bytes = ring * std::min(pool_bytes, sel);
    p.norm_bytes = ring * static_cast<double>(nc) * 4.0;
    return p;
}

TrafficPrediction predict_traffic(const RunConfig& c) {
    const TrainOptions& t = c.train;
    return predict_traffic(model_parameter_count(t.model_dims), element_size(t.wire_precision), c.ranks,
                           t.csc ? t.final_sparsity : 0.0, t.chunk_size, t.csc);
}

BenchResult bench_allreduce(int ranks, std::uint64_t bytes, Algo algo, int group_size, const std::string& transport,
                            ElementType precision) {
    if (ranks < 1) throw ConfigError("ranks must be >= 1");
    const std::size_t esz = element_size(precision), n = static_cast<std::size_t>(bytes / esz);
    if (n == 0) throw ConfigError("buffer too small for element type");
    if (algo == Algo::kHierarchical && (group_size < 1 || ranks % group_size != 0))
        throw ConfigError("group size " + std::to_string(group_size) + " must divide world " + std::to_string(ranks));
    auto world = make_world(ranks, transport);
    BenchResult out;
    std::vector<std::vector<float>> got(static_cast<std::size_t>(ranks)), want(static_cast<std::size_t>(ranks));
    on_rank_threads(world, [&](int r, Transport& tp) {
        Communicator comm(tp, group_size);
        // the reference's seeded buffers (harness.cpp:280-283)
        std::mt19937_64 rng(1234 + static_cast<std::uint64_t>(r));
        std::uniform_real_distribution<float> uni(-1.0f, 1.0f);
        std::vector<float> v(n);
        for (auto& x : v) x = uni(rng);
        auto buf = OwnedBuffer::from_floats(precision, v);
        auto ref = OwnedBuffer::from_floats(precision, v);
        switch (algo) {
            case Algo::kRing: ring_allreduce(comm, buf.view()); break;
            case Algo::kHierarchical: hierarchical_allreduce(comm, buf.view()); break;
            case Algo::kOracle: oracle_allreduce(comm, buf.view()); break;
        }
        oracle_allreduce(comm, ref.view());
        got[static_cast<std::size_t>(r)] = buf.to_floats();
        want[static_cast<std::size_t>(r)] = ref.to_floats();
        if (r == 0) {
            for (const auto& [label, c] : tp.stats().snapshot())
                if (label != "oracle") out.per_rank_payload_sent += c.payload_bytes_sent;
            const auto segs = comm.phase2_segment_bytes();
            out.phase2_segment_bytes = segs.empty() ? 0 : segs.front();
        }
    });
    if (algo == Algo::kRing && ranks > 1) {  // rank 0's ring sends: RS segment -s, AG segment 1-s
        for (int s = 0; s < ranks - 1; ++s)
            out.predicted_payload += (detail::segment_of(n, ranks, (ranks - s) % ranks).length +
                                      detail::segment_of(n, ranks, (1 - s + ranks) % ranks).length) * esz;
    }
    double max_rel = 0.0;  // |got - want| / max(1, |want|): cancellation-safe relative error
    for (int r = 0; r < ranks; ++r)
        for (std::size_t i = 0; i < n; ++i) {
            const double w = want[static_cast<std::size_t>(r)][i], g = got[static_cast<std::size_t>(r)][i];
            max_rel = std::max(max_rel, std::fabs(g - w) / std::max(1.0, std::fabs(w)));
        }
    out.matches_oracle = max_rel <= (precision == ElementType::kF32 ? 1e-6 : 1e-2);
    return out;
}

RunSummary run_experiment(const RunConfig& config, std::optional<int> /*worker_rank*/) {
    validate(config);
    auto world = make_world(config.ranks, config.transport);
    std::vector<TrainResult> res(static_cast<std::size_t>(config.ranks));
    on_rank_threads(world, [&](int r, Transport& tp) { res[static_cast<std::size_t>(r)] = train_worker(config.train, tp); });
    const TrainResult& r0 = res[0];
    RunSummary s;
    s.iterations = r0.metrics.size();
    s.final_loss = r0.final_loss;
    double sum = 0.0;
    for (const auto& m : r0.metrics) {
        s.total_payload_bytes += m.grad_payload_bytes;
        sum += static_cast<double>(m.grad_payload_bytes);
    }
    s.grad_bytes_per_iteration = s.iterations ? sum / static_cast<double>(s.iterations) : 0.0;
    s.predicted_bytes_per_iteration = predict_traffic(config).total();
    s.predicted_vs_measured_delta = s.predicted_bytes_per_iteration > 0.0
                                        ? (s.grad_bytes_per_iteration - s.predicted_bytes_per_iteration) /
                                              s.predicted_bytes_per_iteration
                                        : 0.0;
    if (!config.out_path.empty()) {
        std::ofstream csv(config.out_path);
        csv << "iteration,loss,grad_payload_bytes,sparsity\n";
        for (std::size_t t = 0; t < r0.metrics.size(); ++t)
            csv << t << ',' << r0.metrics[t].loss << ',' << r0.metrics[t].grad_payload_bytes << ','
                << r0.metrics[t].sparsity << '\n';
        std::ofstream js(config.out_path + ".summary.json");
        js << "{\"final_loss\": " << s.final_loss << ", \"total_payload_bytes\": " << s.total_payload_bytes
           << ", \"grad_bytes_per_iteration\": " << s.grad_bytes_per_iteration
           << ", \"predicted_bytes_per_iteration\": " << s.predicted_bytes_per_iteration
           << ", \"predicted_vs_measured_delta\": " << s.predicted_vs_measured_delta
           << ", \"iterations\": " << s.iterations << ", \"ranks\": " << config.ranks << "}\n";
    }
    return s;
}

ApiBenchResult bench_api_sync(const std::vector<std::size_t>& sizes, int steps, int warmup, std::uint64_t theta,
                              bool csc, double final_sparsity) {
    if (sizes.empty() || steps < 1 || warmup < 0) throw ConfigError("bench_api_sync: bad arguments");
    auto world = make_inproc_world(1);
    Transport& tp = *world[0];
    GradientPool pool(sizes, kDefaultChunkSize, ElementType::kF16);
    Communicator comm(tp);
    FusionEngine engine(pool, comm, FusionConfig{theta, Algo::kRing});
    SparseState sparse(pool, SparseConfig{0.9, 0.01, csc ? final_sparsity : 0.0, 0});
    pool.set_async_host_input(true);  // the loop keeps each input set intact until it is synced
    const std::size_t total = pool.total_elements(), m = sizes.size();
    std::vector<std::size_t> asc(m + 1, 0);  // ascending-id offsets into a flat input set
    for (std::size_t i = 0; i < m; ++i) asc[i + 1] = asc[i] + sizes[i];
    // two pinned input sets (seeded gradients of steps 0 and 1) and two pinned result buffers
    float* in[2] = {nullptr, nullptr};
    float* out[2] = {nullptr, nullptr};
    auto ok = [](cudaError_t e, const char* w) {
        if (e != cudaSuccess) throw TransportError(std::string(w) + ": " + cudaGetErrorString(e));
    };
    std::vector<std::uint64_t> sz(sizes.begin(), sizes.end());
    for (int k = 0; k < 2; ++k) {
        ok(cudaMallocHost(&in[k], total * 4), "cudaMallocHost");
        ok(cudaMallocHost(&out[k], total * 4), "cudaMallocHost");
        check(gf_synth_grads(0, k, sz.data(), static_cast<int>(m), in[k]), "gf_synth_grads");
    }
    std::vector<float> weights(total, 0.0f);
    std::vector<FusedHandle> handles;
    ApiBenchResult res;
    auto one = [&](int t) {
        const float* g = in[t & 1];
        pool.begin_iteration();
        engine.begin_iteration();
        if (csc) sparse.begin_iteration(static_cast<std::uint64_t>(t));
        handles.clear();
        for (int id = static_cast<int>(m); id >= 1; --id) {
            const auto done = pool.write_tensor(id, std::span<const float>(g + asc[id - 1], sizes[id - 1]));
            if (csc) {
                for (auto c : done) sparse.correction_pre_allreduce(c);
            } else {
                for (auto& h : engine.on_tensor_complete(id)) handles.push_back(std::move(h));
            }
        }
        if (csc) {
            sparse.sparse_exchange(comm, engine);
            sparse.select_next_important(comm, static_cast<std::uint64_t>(t));
            sparse.sgd_update(weights, 1);
        } else {
            if (auto h = engine.finalize_iteration()) handles.push_back(std::move(*h));
            FusionEngine::wait_all(handles);
            pool.read_averaged(std::span<float>(out[t & 1], total), 1, /*wait=*/false);
        }
    };
    try {
        for (int t = 0; t < warmup; ++t) one(t);
        pool.synchronize();
        const auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < steps; ++t) one(warmup + t);
        pool.synchronize();
        const auto t1 = std::chrono::steady_clock::now();
        res.ms_per_step = std::chrono::duration<double, std::milli>(t1 - t0).count() / steps;
        res.steps = steps;
        res.h2d_bytes_per_step = total * 4;
        if (csc) {  // the important chunks of w move in and out, plus the selected set
            const std::size_t nc = pool.num_chunks();
            const std::size_t k = selection_count(final_sparsity, nc);
            res.h2d_bytes_per_step += k * kDefaultChunkSize * 4 + nc;
            res.d2h_bytes_per_step = k * kDefaultChunkSize * 4 + nc;
        } else {
            res.d2h_bytes_per_step = total * 4;
        }
    } catch (...) {
        for (int k = 0; k < 2; ++k) {
            cudaFreeHost(in[k]);
            cudaFreeHost(out[k]);
        }
        throw;
    }
    for (int k = 0; k < 2; ++k) {
        cudaFreeHost(in[k]);
        cudaFreeHost(out[k]);
    }
    return res;
}

}  // namespace gflow
