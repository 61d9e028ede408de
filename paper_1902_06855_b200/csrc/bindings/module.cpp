// SPDX-License-Identifier: Apache-2.0
//
// gflowpy — Python bindings of the B200 gradient-sync path. The module-level functions
// keep the reference's gflowpy names, keyword arguments and defaults
// (reference: bindings/module.cpp:158-199; ConfigError -> ValueError); the classes expose
// the C++ API (GradientPool, FusionEngine, SparseState, Communicator, collectives) so that
// parity tests can drive it the way the reference's C++ tests do, ranks as threads.
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <random>
#include <thread>

#include "gflow/collectives.hpp"
#include "gflow/fusion.hpp"
#include "gflow/gradient_pool.hpp"
#include "gflow/half.hpp"
#include "gflow/harness.hpp"
#include "gflow/inproc.hpp"
#include "gflow/sparse.hpp"
#include "gflow/tcp.hpp"
#include "gflow/trainer.hpp"

namespace py = pybind11;
using namespace gflow;

namespace {

using release = py::call_guard<py::gil_scoped_release>;

Algo algo_from_name(const std::string& name) {
    if (name == "ring") return Algo::kRing;
    if (name == "hierarchical") return Algo::kHierarchical;
    if (name == "oracle") return Algo::kOracle;
    throw ConfigError("unknown algorithm: " + name);
}

ElementType precision_from_name(const std::string& name) {
    if (name == "fp32") return ElementType::kF32;
    if (name == "fp16") return ElementType::kF16;
    throw ConfigError("unknown precision: " + name);
}

// Layout only (no device allocation): gradient_pool.cpp:11-41 semantics.
py::dict pool_info(const std::vector<std::size_t>& sizes, std::size_t chunk_size) {
    if (sizes.empty()) throw ConfigError("gradient pool needs at least one tensor");
    if (chunk_size == 0) throw ConfigError("chunk_size must be positive");
    std::size_t total = 0;
    for (auto s : sizes) {
        if (s == 0) throw ConfigError("tensor sizes must be positive");
        total += s;
    }
    const std::size_t nc = std::max<std::size_t>(
        1, static_cast<std::size_t>(std::llround(static_cast<double>(total) / static_cast<double>(chunk_size))));
    py::dict offsets;
    std::size_t off = 0;
    for (int id = static_cast<int>(sizes.size()); id >= 1; --id) {
        offsets[py::int_(id)] = off;
        off += sizes[static_cast<std::size_t>(id - 1)];
    }
    std::vector<std::size_t> lens(nc, chunk_size);
    lens.back() = total - (nc - 1) * chunk_size;
    py::dict out;
    out["total_elements"] = total;
    out["num_chunks"] = nc;
    out["tensor_offsets"] = offsets;
    out["chunk_lengths"] = lens;
    return out;
}

// harness.cpp:132-159 (gflow::predict_traffic, host/harness.cpp)
py::dict py_predict_traffic(std::uint64_t pool_elements, std::size_t element_bytes, int ranks, double sparsity,
                         std::size_t chunk_size, bool csc) {
    const TrafficPrediction p = gflow::predict_traffic(pool_elements, element_bytes, ranks, sparsity, chunk_size, csc);
    py::dict out;
    out["grad_bytes"] = p.grad_bytes;
    out["norm_bytes"] = p.norm_bytes;
    out["total_bytes"] = p.total();
    return out;
}

int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

template <typename F>
void run_ranks(int ranks, F body) {
    auto world = make_inproc_world(ranks);
    std::vector<std::thread> ts;
    std::vector<std::exception_ptr> errors(static_cast<std::size_t>(ranks));
    for (int r = 0; r < ranks; ++r) {
        ts.emplace_back([&, r] {
            try {
                cudaSetDevice(gflow::thread_rank_device(r, ranks));
                body(r, *world[static_cast<std::size_t>(r)]);
            } catch (...) {
                errors[static_cast<std::size_t>(r)] = std::current_exception();
            }
        });
    }
    for (auto& t : ts) t.join();
    for (auto& e : errors)
        if (e) std::rethrow_exception(e);
}

// harness.cpp:245-339 (gflow::bench_allreduce, host/harness.cpp): ranks as threads, the
// allreduce on the GPU.
py::dict py_bench_allreduce(int ranks, std::uint64_t bytes, const std::string& algo, int group_size,
                         const std::string& precision) {
    const Algo a = algo_from_name(algo);
    const ElementType et = precision_from_name(precision);
    BenchResult r;
    {
        py::gil_scoped_release nogil;
        r = gflow::bench_allreduce(ranks, bytes, a, group_size, "inproc", et);
    }
    py::dict out;
    out["per_rank_payload_sent"] = r.per_rank_payload_sent;
    out["predicted_payload"] = r.predicted_payload;
    out["phase2_segment_bytes"] = r.phase2_segment_bytes;
    out["matches_oracle"] = r.matches_oracle;
    return out;
}

py::dict train(int ranks, const std::vector<std::size_t>& model_dims, const std::string& task,
               std::uint64_t iterations, std::size_t n_examples, std::size_t batch, double learning_rate,
               double momentum, std::uint64_t seed, const std::string& algo, int group_size,
               const std::string& precision, std::uint64_t theta_bytes, bool csc, double final_sparsity,
               std::uint64_t warmup_iters, std::size_t chunk_size) {
    TrainOptions o;
    o.model_dims = model_dims;
    o.task = task == "logistic" ? Task::kLogistic : Task::kLinearRegression;
    o.iterations = iterations;
    o.n_examples = n_examples;
    o.batch = batch;
    o.learning_rate = learning_rate;
    o.momentum = momentum;
    o.seed = seed;
    o.algorithm = algo_from_name(algo);
    o.group_size = group_size;
    o.wire_precision = precision_from_name(precision);
    o.theta_bytes = theta_bytes;
    o.csc = csc;
    o.final_sparsity = final_sparsity;
    o.warmup_iters = warmup_iters;
    o.chunk_size = chunk_size;
    std::vector<TrainResult> res(static_cast<std::size_t>(ranks));
    {
        py::gil_scoped_release nogil;
        run_ranks(ranks, [&](int r, Transport& tp) { res[static_cast<std::size_t>(r)] = train_worker(o, tp); });
    }
    const auto& r0 = res[0];
    std::vector<double> losses, sparsity;
    std::vector<std::uint64_t> gb;
    for (const auto& m : r0.metrics) {
        losses.push_back(m.loss);
        gb.push_back(m.grad_payload_bytes);
        sparsity.push_back(m.sparsity);
    }
    py::dict out;
    out["final_loss"] = r0.final_loss;
    out["final_weights"] = r0.final_weights;
    out["loss"] = losses;
    out["grad_payload_bytes"] = gb;
    out["sparsity"] = sparsity;
    return out;
}

// ---- array helpers for the class API ------------------------------------------------------
struct Span {
    float* ptr;
    std::size_t n;
};
// numpy float32 array (host) or any object with data_ptr()/numel() (torch CUDA tensor)
Span as_float_span(py::object o) {
    if (py::hasattr(o, "data_ptr") && py::hasattr(o, "numel")) {
        return {reinterpret_cast<float*>(o.attr("data_ptr")().cast<std::uintptr_t>()),
                o.attr("numel")().cast<std::size_t>()};
    }
    auto a = o.cast<py::array_t<float, py::array::c_style>>();
    return {a.mutable_data(), static_cast<std::size_t>(a.size())};
}

ScalarBuffer as_buffer(py::array a) {
    if (!(a.flags() & py::array::c_style)) throw ConfigError("buffer must be C-contiguous");
    if (a.dtype().is(py::dtype::of<float>()))
        return {ElementType::kF32, static_cast<std::byte*>(a.mutable_data()), static_cast<std::size_t>(a.size())};
    if (a.dtype().is(py::dtype::of<std::uint16_t>()))
        return {ElementType::kF16, static_cast<std::byte*>(a.mutable_data()), static_cast<std::size_t>(a.size())};
    throw ConfigError("buffer must be float32 (fp32) or uint16 (fp16 bits)");
}

py::dict stats_dict(const TrafficStats& s) {
    py::dict out;
    for (const auto& [label, c] : s.snapshot()) {
        py::dict d;
        d["payload_bytes_sent"] = c.payload_bytes_sent;
        d["payload_bytes_received"] = c.payload_bytes_received;
        d["frames_sent"] = c.frames_sent;
        out[py::str(label)] = d;
    }
    return out;
}

// futures of the fusion engine, opaque to Python
struct Handles {
    std::vector<FusedHandle> h;
    Handles() = default;
    explicit Handles(std::vector<FusedHandle> v) : h(std::move(v)) {}
    Handles(const Handles&) = delete;
    Handles& operator=(const Handles&) = delete;
    Handles(Handles&&) = default;
    Handles& operator=(Handles&&) = default;
};

}  // namespace

PYBIND11_MODULE(gflowpy, m) {
    m.doc() = "GradientFlow gradient synchronisation on B200 (sm_100a kernels, NVLink peer memory)";

    auto config_error = py::register_exception<ConfigError>(m, "ConfigError", PyExc_ValueError);
    py::register_exception<ProtocolError>(m, "ProtocolError", PyExc_RuntimeError);
    py::register_exception<TransportError>(m, "TransportError", PyExc_RuntimeError);
    py::register_exception<TrainingError>(m, "TrainingError", PyExc_RuntimeError);
    (void)config_error;

    // ---- the reference's module functions (bindings/module.cpp:158-199) --------------
    m.def("float_to_half_bits", &float_to_half_bits, py::arg("value"));
    m.def("half_bits_to_float", &half_bits_to_float, py::arg("bits"));
    m.def("encode_half", [](const std::vector<float>& v) {
        const auto b = encode_half(v);
        return py::bytes(reinterpret_cast<const char*>(b.data()), b.size());
    }, py::arg("values"));
    m.def("decode_half", [](const py::bytes& raw) {
        std::string s = raw;
        return decode_half(std::span<const std::byte>(reinterpret_cast<const std::byte*>(s.data()), s.size()));
    }, py::arg("data"));
    m.def("pool_info", &pool_info, py::arg("tensor_sizes"), py::arg("chunk_size") = 32000);
    m.def("sparsity_at", &sparsity_at, py::arg("iteration"), py::arg("warmup_iters"), py::arg("final_sparsity"));
    m.def("selection_count", &selection_count, py::arg("sparsity"), py::arg("num_chunks"));
    m.def("predict_traffic", &py_predict_traffic, py::arg("pool_elements"), py::arg("element_bytes"),
          py::arg("ranks"), py::arg("sparsity") = 0.0, py::arg("chunk_size") = 32000, py::arg("csc") = false);
    m.def(
        "bench_api",
        [](const std::vector<std::size_t>& sizes, int steps, int warmup, std::uint64_t theta, bool csc,
           double final_sparsity) {
            ApiBenchResult r;
            {
                py::gil_scoped_release nogil;
                r = gflow::bench_api_sync(sizes, steps, warmup, theta, csc, final_sparsity);
            }
            py::dict d;
            d["ms_per_step"] = r.ms_per_step;
            d["h2d_bytes_per_step"] = r.h2d_bytes_per_step;
            d["d2h_bytes_per_step"] = r.d2h_bytes_per_step;
            d["steps"] = r.steps;
            return d;
        },
        py::arg("sizes"), py::arg("steps") = 20, py::arg("warmup") = 3, py::arg("theta") = 64ull << 20,
        py::arg("csc") = false, py::arg("final_sparsity") = 0.9);
    m.def("bench_allreduce", &py_bench_allreduce, py::arg("ranks"), py::arg("bytes"), py::arg("algo") = "ring",
          py::arg("group_size") = 1, py::arg("precision") = "fp32");
    m.def("train", &train, py::arg("ranks") = 2, py::arg("model_dims") = std::vector<std::size_t>{64, 32, 1},
          py::arg("task") = "linear", py::arg("iterations") = 50, py::arg("n_examples") = 1024,
          py::arg("batch") = 16, py::arg("learning_rate") = 0.01, py::arg("momentum") = 0.9,
          py::arg("seed") = 1, py::arg("algo") = "ring", py::arg("group_size") = 1,
          py::arg("precision") = "fp32", py::arg("theta_bytes") = 64ull << 20, py::arg("csc") = false,
          py::arg("final_sparsity") = 0.0, py::arg("warmup_iters") = 0, py::arg("chunk_size") = 1000);

    // ---- the C++ API ----------------------------------------------------------------
    py::enum_<ElementType>(m, "ElementType").value("kF32", ElementType::kF32).value("kF16", ElementType::kF16);
    py::enum_<Algo>(m, "Algo").value("kRing", Algo::kRing).value("kHierarchical", Algo::kHierarchical)
        .value("kOracle", Algo::kOracle);
    m.attr("THETA_INFINITE") = py::int_(kThetaInfinite);
    m.def("device_count", &device_count);
    m.def("set_device", [](int d) {
        if (cudaSetDevice(d) != cudaSuccess) throw ConfigError("cudaSetDevice(" + std::to_string(d) + ") failed");
    });

    py::class_<Transport, std::shared_ptr<Transport>>(m, "Transport")
        .def_property_readonly("rank", &Transport::rank)
        .def_property_readonly("world_size", &Transport::world_size)
        .def("barrier", &Transport::barrier, release())
        .def("stats", [](Transport& t) { return stats_dict(t.stats()); })
        .def("total_payload_sent", [](Transport& t) { return t.stats().total().payload_bytes_sent; })
        .def("set_timeout_ms", [](Transport& t, int ms) { t.set_timeout(std::chrono::milliseconds(ms)); })
        .def("send", [](Transport& t, int dst, std::uint32_t tag, const py::bytes& data, const std::string& phase) {
            const std::string s = data;
            const auto* p = reinterpret_cast<const std::byte*>(s.data());
            py::gil_scoped_release nogil;
            t.send(dst, tag, std::span<const std::byte>(p, s.size()), phase);
        }, py::arg("dst"), py::arg("tag"), py::arg("data"), py::arg("phase") = "data")
        .def("recv", [](Transport& t, int src, std::uint32_t tag, const std::string& phase) {
            std::vector<std::byte> v;
            {
                py::gil_scoped_release nogil;
                v = t.recv(src, tag, phase);
            }
            return py::bytes(reinterpret_cast<const char*>(v.data()), v.size());
        }, py::arg("src"), py::arg("tag"), py::arg("phase") = "data");
    // Multi-process control plane (reference: include/gflow/tcp.hpp:18-47): GFL1 over TCP.
    m.def("make_tcp_transport", [](int rank, int world_size, const std::vector<std::string>& peers) {
        std::shared_ptr<Transport> t;
        {
            py::gil_scoped_release nogil;
            t = std::make_shared<TcpTransport>(rank, world_size, peers);
        }
        return t;
    }, py::arg("rank"), py::arg("world_size"), py::arg("peers"));
    m.def("tcp_loopback_addresses", &TcpTransport::loopback_addresses, py::arg("world_size"),
          py::arg("port_base"));
    m.def("make_inproc_world", [](int n) {
        std::vector<std::shared_ptr<Transport>> out;
        for (auto& t : make_inproc_world(n)) out.emplace_back(t.release());
        return out;
    }, py::arg("world_size"));

    py::class_<Communicator>(m, "Communicator")
        .def(py::init<Transport&, int>(), py::arg("transport"), py::arg("group_size") = 1, py::keep_alive<1, 2>())
        .def_property_readonly("rank", &Communicator::rank)
        .def_property_readonly("world_size", &Communicator::world_size)
        .def_property_readonly("ring_order", &Communicator::ring_order)
        .def("set_ring_order", &Communicator::set_ring_order)
        .def("set_device", &Communicator::set_device)
        .def_property_readonly("group_size", &Communicator::group_size)
        .def("phase2_segment_bytes", &Communicator::phase2_segment_bytes)
        .def("device_mode", [](Communicator& c) { return std::string(c.device().mode_name()); }, release())
        .def("device", [](Communicator& c) { return c.device().device(); }, release());

    m.def("ring_allreduce", [](Communicator& c, py::array a) {
        ScalarBuffer b = as_buffer(a);
        py::gil_scoped_release nogil;
        ring_allreduce(c, b);
    }, py::arg("comm"), py::arg("buf"));
    m.def("oracle_allreduce", [](Communicator& c, py::array a) {
        ScalarBuffer b = as_buffer(a);
        py::gil_scoped_release nogil;
        oracle_allreduce(c, b);
    }, py::arg("comm"), py::arg("buf"));
    m.def("broadcast", [](Communicator& c, py::array a, int root) {
        ScalarBuffer b = as_buffer(a);
        py::gil_scoped_release nogil;
        broadcast(c, b, root);
    }, py::arg("comm"), py::arg("buf"), py::arg("root"));
    m.def("reduce", [](Communicator& c, py::array a, int root) {
        ScalarBuffer b = as_buffer(a);
        py::gil_scoped_release nogil;
        reduce(c, b, root);
    }, py::arg("comm"), py::arg("buf"), py::arg("root"));
    m.def("hierarchical_allreduce", [](Communicator& c, py::array a) {
        ScalarBuffer b = as_buffer(a);
        py::gil_scoped_release nogil;
        hierarchical_allreduce(c, b);
    }, py::arg("comm"), py::arg("buf"));
    m.def("segment_of", [](std::size_t len, int n, int i) {
        auto s = detail::segment_of(len, n, i);
        return py::make_tuple(s.offset, s.length);
    });

    py::class_<GradientPool>(m, "GradientPool")
        .def(py::init<const std::vector<std::size_t>&, std::size_t, ElementType>(), py::arg("tensor_sizes"),
             py::arg("chunk_size") = kDefaultChunkSize, py::arg("element_type") = ElementType::kF32)
        .def_property_readonly("total_elements", &GradientPool::total_elements)
        .def_property_readonly("chunk_size", &GradientPool::chunk_size)
        .def_property_readonly("num_chunks", &GradientPool::num_chunks)
        .def_property_readonly("num_tensors", &GradientPool::num_tensors)
        .def_property_readonly("device", &GradientPool::device)
        .def("desc", [](const GradientPool& p, int id) {
            const auto& d = p.desc(id);
            return py::make_tuple(d.tensor_id, d.element_count, d.pool_offset);
        })
        .def("chunk_begin", &GradientPool::chunk_begin)
        .def("chunk_length", &GradientPool::chunk_length)
        .def("begin_iteration", &GradientPool::begin_iteration, release())
        .def("write_tensor", [](GradientPool& p, int id, py::object values) {
            Span s = as_float_span(values);
            py::gil_scoped_release nogil;
            return p.write_tensor(id, std::span<const float>(s.ptr, s.n));
        })
        .def_property_readonly("written_elements", &GradientPool::written_elements)
        .def("iteration_complete", &GradientPool::iteration_complete)
        .def("get", &GradientPool::get, release())
        .def("set", &GradientPool::set, release())
        .def("synchronize", &GradientPool::synchronize, release())
        .def("chunk_l1", &GradientPool::chunk_l1, release())
        .def("device_ptr", [](GradientPool& p) { return reinterpret_cast<std::uintptr_t>(p.device_data()); })
        .def("to_numpy", [](GradientPool& p) {
            {
                py::gil_scoped_release nogil;
                p.synchronize();  // the pool's queued packs / collectives / corrections
            }
            const std::size_t n = p.total_elements();
            if (p.element_type() == ElementType::kF16) {
                py::array_t<std::uint16_t> a(n);
                p.invalidate_host();
                if (cudaMemcpy(a.mutable_data(), p.device_data(), n * 2, cudaMemcpyDeviceToHost) != cudaSuccess)
                    throw TransportError("pool D2H");
                return py::array(a);
            }
            py::array_t<float> a(n);
            if (cudaMemcpy(a.mutable_data(), p.device_data(), n * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
                throw TransportError("pool D2H");
            return py::array(a);
        });

    py::class_<Handles>(m, "FusedHandles")
        .def("__len__", [](const Handles& h) { return h.h.size(); })
        .def("extend", [](Handles& a, Handles& b) {
            for (auto& x : b.h) a.h.push_back(std::move(x));
            b.h.clear();
        })
        .def("wait_all", [](Handles& h) { FusionEngine::wait_all(h.h); }, release());
    py::class_<FusionEngine>(m, "FusionEngine")
        .def(py::init([](GradientPool& p, Communicator& c, std::uint64_t theta, Algo a) {
                 return new FusionEngine(p, c, FusionConfig{theta, a});
             }),
             py::arg("pool"), py::arg("comm"), py::arg("threshold_bytes") = 64ull << 20,
             py::arg("algorithm") = Algo::kRing, py::keep_alive<1, 2>(), py::keep_alive<1, 3>())
        .def("begin_iteration", &FusionEngine::begin_iteration)
        // a window launch may bootstrap the device context (a collective): no GIL while in C++
        .def("on_tensor_complete", [](FusionEngine& e, int id) { return Handles{e.on_tensor_complete(id)}; },
             release())
        .def("finalize_iteration", [](FusionEngine& e) {
            Handles h;
            if (auto f = e.finalize_iteration()) h.h.push_back(std::move(*f));
            return h;
        }, release())
        .def("enqueue_collective", [](FusionEngine& e, GradientPool& p, std::size_t first, std::size_t count) {
            if (first + count > p.total_elements()) throw ConfigError("enqueue_collective: range outside the pool");
            const std::size_t es = element_size(p.element_type());
            Handles h;
            h.h.push_back(e.enqueue_collective(
                ScalarBuffer{p.element_type(), p.device_data() + first * es, count, Residency::kDevice}));
            return h;
        }, release())
        .def("window_bytes", [](const FusionEngine& e) { return e.last_log().window_bytes; })
        .def("log_csv_line", &FusionEngine::log_csv_line);

    py::class_<SparseState>(m, "SparseState")
        .def(py::init([](GradientPool& p, double mom, double lr, double s, std::uint64_t w) {
                 return new SparseState(p, SparseConfig{mom, lr, s, w});
             }),
             py::arg("pool"), py::arg("momentum") = 0.9, py::arg("learning_rate") = 0.01,
             py::arg("final_sparsity") = 0.0, py::arg("warmup_iters") = 0, py::keep_alive<1, 2>())
        .def("begin_iteration", &SparseState::begin_iteration, release())
        .def("correction_pre_allreduce", &SparseState::correction_pre_allreduce, release())
        .def("sparse_exchange", &SparseState::sparse_exchange, release())
        .def("select_next_important", &SparseState::select_next_important, release())
        .def("sgd_update", [](SparseState& s, py::object w, int world) {
            Span sp = as_float_span(w);
            py::gil_scoped_release nogil;
            s.sgd_update(std::span<float>(sp.ptr, sp.n), world);
        })
        .def_property_readonly("important", &SparseState::important)
        .def("hg", [](const SparseState& s) { auto v = s.hg(); return std::vector<float>(v.begin(), v.end()); },
             release())
        .def("hu", [](const SparseState& s) { auto v = s.hu(); return std::vector<float>(v.begin(), v.end()); },
             release())
        .def("selected_chunks", &SparseState::selected_chunks)
        .def("selected_payload_bytes", &SparseState::selected_payload_bytes)
        .def_property_readonly("current_sparsity", &SparseState::current_sparsity)
        .def_property_readonly("last_exchange_windows", &SparseState::last_exchange_windows)
        .def("checksum", &SparseState::checksum);
}
