// SPDX-License-Identifier: Apache-2.0
// Coarse-grained sparse communication on the GPU (reference: src/sparse.cpp). Device work is
// ordered on the pool's stream; see gflow/sparse.hpp for where the host waits.
#include "gflow/sparse.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

namespace gflow {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw TransportError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
T* dalloc(std::size_t n, cudaStream_t s) {
    T* p = nullptr;
    cuda_ok(cudaMalloc(&p, std::max<std::size_t>(n * sizeof(T), 16)), "cudaMalloc");
    cuda_ok(cudaMemsetAsync(p, 0, std::max<std::size_t>(n * sizeof(T), 16), s), "cudaMemset");
    return p;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct OnDevice {
    int prev = -1;
    explicit OnDevice(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~OnDevice() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

double sparsity_at(std::uint64_t t, std::uint64_t warmup, double final_sparsity) {
    if (warmup == 0) return final_sparsity;
    return final_sparsity * std::min(1.0, static_cast<double>(t) / static_cast<double>(warmup));
}

std::size_t selection_count(double sparsity, std::size_t nc) {
    const long long k = std::llround((1.0 - sparsity) * static_cast<double>(nc));
    return std::max<std::size_t>(1, std::min<std::size_t>(static_cast<std::size_t>(std::max(0LL, k)), nc));
}

SparseState::SparseState(GradientPool& pool, SparseConfig config) : pool_(pool), config_(config) {
    if (config_.final_sparsity < 0.0 || config_.final_sparsity >= 1.0)
        throw ConfigError("final_sparsity must be in [0, 1)");
    if (config_.momentum < 0.0 || config_.momentum >= 1.0) throw ConfigError("momentum must be in [0, 1)");
    if (config_.learning_rate <= 0.0) throw ConfigError("learning_rate must be positive");
    const std::size_t nc = pool_.num_chunks(), total = pool_.total_elements();
    important_.assign(nc, 1);
    next_important_.assign(nc, 1);
    corrected_.assign(nc, 0);
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    d_hg_ = dalloc<float>(total, ps);
    d_hu_ = dalloc<float>(total, ps);
    d_imp_ = dalloc<std::uint8_t>(nc, ps);
    d_coff_ = dalloc<std::uint64_t>(nc, ps);
    d_plan_ = dalloc<std::uint64_t>(4 + nc, ps);
    d_staging_ = dalloc<std::byte>(total * element_size(pool_.element_type()), ps);
    d_norms_ = dalloc<float>(nc, ps);
    cuda_ok(cudaMallocHost(&h_imp_, nc), "cudaMallocHost");
    cuda_ok(cudaMallocHost(&h_coff_, nc * 8), "cudaMallocHost");
    cuda_ok(cudaMallocHost(&h_plan_, (4 + nc) * 8), "cudaMallocHost");
    cuda_ok(cudaStreamSynchronize(ps), "sparse state init");
    pool_.set_pending_work([this] { flush_corrections(); });
}

SparseState::~SparseState() {
    pool_.set_pending_work(nullptr);
    OnDevice g(pool_.device());
    cudaStreamSynchronize(static_cast<cudaStream_t>(pool_.stream()));
    for (void* p : {static_cast<void*>(d_hg_), static_cast<void*>(d_hu_), static_cast<void*>(d_imp_),
                    static_cast<void*>(d_coff_), static_cast<void*>(d_plan_), static_cast<void*>(d_staging_),
                    static_cast<void*>(d_norms_), static_cast<void*>(d_w_)})
        if (p) cudaFree(p);
    for (void* p : {static_cast<void*>(h_imp_), static_cast<void*>(h_coff_), static_cast<void*>(h_plan_)})
        if (p) cudaFreeHost(p);
}

// The pinned control arrays are reused every iteration: earlier copies out of them have
// completed by the time they are rewritten (the iteration's host-visible results synchronise
// the pool stream), and a stream sync guards the rare early reuse.
void SparseState::upload_important() {
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    cuda_ok(cudaStreamSynchronize(ps), "pool stream");
    std::memcpy(h_imp_, important_.data(), important_.size());
    cuda_ok(cudaMemcpyAsync(d_imp_, h_imp_, important_.size(), cudaMemcpyHostToDevice, ps), "H2D flags");
}

// plan[0] staged elements, plan[1] chunk count, plan[4..] the chunks in the given (queue)
// order; coff[c] = staging offset of chunk c (sparse.cpp:129-140)
void SparseState::upload_plan(const std::vector<std::size_t>& chunks, bool with_coff) {
    const std::size_t nc = pool_.num_chunks();
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    cuda_ok(cudaStreamSynchronize(ps), "pool stream");
    std::uint64_t staged = 0;
    for (std::size_t j = 0; j < chunks.size(); ++j) {
        if (with_coff) h_coff_[chunks[j]] = staged;
        h_plan_[4 + j] = chunks[j];
        staged += pool_.chunk_length(chunks[j]);
    }
    h_plan_[0] = staged;
    h_plan_[1] = chunks.size();
    h_plan_[2] = h_plan_[3] = 0;
    cuda_ok(cudaMemcpyAsync(d_plan_, h_plan_, (4 + chunks.size()) * 8, cudaMemcpyHostToDevice, ps), "H2D plan");
    if (with_coff) cuda_ok(cudaMemcpyAsync(d_coff_, h_coff_, nc * 8, cudaMemcpyHostToDevice, ps), "H2D coff");
}

void SparseState::begin_iteration(std::uint64_t t) {
    iteration_ = t;
    current_sparsity_ = sparsity_at(t, config_.warmup_iters, config_.final_sparsity);
    if (has_selection_) important_ = next_important_;
    else std::fill(important_.begin(), important_.end(), 1);  // iteration 0 is dense
    queued_.clear();
    std::fill(corrected_.begin(), corrected_.end(), 0);
    run_lo_ = run_hi_ = 0;
    exchanged_ = false;
    upload_important();
}

void SparseState::flush_corrections() {
    if (run_hi_ == run_lo_) return;
    pool_.flush_writes();  // the chunks' packs precede their correction on the pool stream
    OnDevice g(pool_.device());
    check(gf_csc_correct(static_cast<int>(pool_.element_type()), pool_.device_data(), d_hg_, d_imp_,
                         pool_.total_elements(), pool_.chunk_size(), pool_.num_chunks(), run_lo_, run_hi_ - run_lo_,
                         static_cast<float>(config_.momentum), pool_.stream()),
          "correction_pre_allreduce");
    run_lo_ = run_hi_ = 0;
}

void SparseState::correction_pre_allreduce(std::size_t c) {
    if (c >= pool_.num_chunks()) throw ConfigError("chunk index out of range");
    const std::size_t begin = pool_.chunk_begin(c), len = pool_.chunk_length(c);
    if (begin + len > pool_.written_elements())
        throw ConfigError("correction on incomplete chunk " + std::to_string(c));
    if (corrected_[c]) throw ConfigError("chunk " + std::to_string(c) + " corrected twice");
    corrected_[c] = 1;
    // consecutive chunks (the watermark's order) join one pending K2 launch
    if (run_hi_ > run_lo_ && c == run_hi_) {
        ++run_hi_;
    } else {
        flush_corrections();
        run_lo_ = c;
        run_hi_ = c + 1;
    }
    pool_.invalidate_host();
    if (important_[c]) queued_.push_back(c);
}

std::size_t SparseState::selected_chunks() const {
    return static_cast<std::size_t>(std::count(important_.begin(), important_.end(), std::uint8_t{1}));
}

std::uint64_t SparseState::selected_payload_bytes() const {
    std::uint64_t b = 0;
    for (std::size_t c = 0; c < important_.size(); ++c)
        if (important_[c]) b += pool_.chunk_length(c) * element_size(pool_.element_type());
    return b;
}

std::uint64_t SparseState::checksum() const {
    std::uint64_t h = 1469598103934665603ull;  // FNV-1a 64 (sparse.cpp:96-104)
    for (std::uint8_t b : important_) {
        h ^= b;
        h *= 1099511628211ull;
    }
    return h;
}

void SparseState::device_allreduce(Communicator& comm, std::vector<void*>& ranks, std::byte* buf, ElementType type,
                                   std::size_t length, const std::vector<std::pair<std::size_t, std::size_t>>& windows,
                                   std::uint32_t phase) {
    DeviceContext& ctx = comm.device();
    if (ranks.empty()) {  // first use: every rank registers this buffer at the same call
        pool_.synchronize();
        ranks = ctx.exchange(buf, (comm.acquire_collective_id() << 8) | phase, (static_cast<std::uint64_t>(length) << 1) | static_cast<std::uint64_t>(type));
    }
    ctx.ring_allreduce_async(type, ranks, comm.ring_order(), windows, pool_.stream());
    detail::record_ring_payload(comm, type, windows, "ring");
}

void SparseState::sparse_exchange(Communicator& comm, FusionEngine& engine) {
    if (exchanged_) throw ConfigError("sparse_exchange called twice in one iteration");
    // every rank must hold the same important set before gradients move (sparse.cpp:109-127)
    const std::uint64_t local = checksum();
    Transport& tp = comm.transport();
    if (comm.world_size() > 1) {
        const std::uint32_t tag = (comm.acquire_collective_id() << 8) | 7;
        std::vector<std::byte> payload(8);
        std::memcpy(payload.data(), &local, 8);
        if (comm.rank() == 0) {
            for (int r = 1; r < comm.world_size(); ++r) tp.send(r, tag, payload, "csc_check");
        } else {
            auto ref = tp.recv(0, tag, "csc_check");
            std::uint64_t expected = 0;
            std::memcpy(&expected, ref.data(), 8);
            if (expected != local)
                throw ProtocolError("important-set divergence at rank " + std::to_string(comm.rank()));
        }
    }
    flush_corrections();
    const std::size_t nc = pool_.num_chunks(), esz = element_size(pool_.element_type());
    const int dt = static_cast<int>(pool_.element_type());
    OnDevice g(pool_.device());
    // staging layout: the queued chunks in queue order (sparse.cpp:129-140)
    upload_plan(queued_, true);
    check(gf_csc_compact(dt, pool_.device_data(), d_staging_, d_plan_, d_coff_, pool_.total_elements(),
                         pool_.chunk_size(), nc, queued_.size(), pool_.stream()),
          "sparse_exchange compact");
    // theta windows over the staging buffer (sparse.cpp:142-158), all reduced in one launch
    const std::uint64_t theta = engine.config().threshold_bytes;
    std::vector<std::pair<std::size_t, std::size_t>> windows;
    std::size_t ws = 0, pos = 0;
    for (std::size_t c : queued_) {
        pos += pool_.chunk_length(c);
        if (theta != kThetaInfinite && (pos - ws) * esz >= theta) {
            windows.emplace_back(ws, pos - ws);
            ws = pos;
        }
    }
    if (pos > ws) windows.emplace_back(ws, pos - ws);
    last_exchange_windows_ = windows.size();
    if (comm.world_size() > 1 && !windows.empty()) {
        if (engine.config().algorithm == Algo::kRing && comm.device().async_collectives()) {
            device_allreduce(comm, stage_ranks_, d_staging_, pool_.element_type(), pos, windows, 0x21u);
        } else {  // colocated ranks / rooted algorithms: the engine's synchronous collectives
            pool_.synchronize();
            ScalarBuffer stage{pool_.element_type(), d_staging_, pos, Residency::kDevice};
            std::vector<FusedHandle> handles;
            for (auto& w : windows) handles.push_back(engine.enqueue_collective(stage.subspan(w.first, w.second)));
            FusionEngine::wait_all(handles);
        }
    }
    // global sums back into the pool (sparse.cpp:162-168)
    check(gf_csc_scatter(dt, pool_.device_data(), d_staging_, d_plan_, d_coff_, pool_.total_elements(),
                         pool_.chunk_size(), nc, queued_.size(), nullptr, pool_.stream()),
          "sparse_exchange write-back");
    pool_.invalidate_host();
    exchanged_ = true;
}

const std::vector<std::uint8_t>& SparseState::select_next_important(Communicator& comm, std::uint64_t t) {
    if (!exchanged_) throw ConfigError("select_next_important before sparse_exchange");
    const std::size_t nc = pool_.num_chunks();
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    // exact chunk L1 (K3), x1/N on important chunks (sparse.cpp:176-184)
    check(gf_chunk_norms(static_cast<int>(pool_.element_type()), pool_.device_data(), pool_.total_elements(),
                         pool_.chunk_size(), nc, d_imp_, comm.world_size(), d_norms_, ps),
          "chunk norms");
    // fp32 ring allreduce of the norms (sparse.cpp:185-187), on the NVLink ring
    if (comm.world_size() > 1) {
        if (comm.device().async_collectives()) {
            device_allreduce(comm, norm_ranks_, reinterpret_cast<std::byte*>(d_norms_), ElementType::kF32, nc,
                             {{0, nc}}, 0x22u);
        } else {
            pool_.synchronize();
            ring_allreduce(comm, ScalarBuffer{ElementType::kF32, reinterpret_cast<std::byte*>(d_norms_), nc,
                                              Residency::kDevice});
        }
    }
    const std::size_t k = selection_count(sparsity_at(t + 1, config_.warmup_iters, config_.final_sparsity), nc);
    check(gf_select_topk(d_norms_, nc, k, d_imp_, ps), "select");  // d_imp_ reloaded below
    cuda_ok(cudaMemcpyAsync(h_imp_, d_imp_, nc, cudaMemcpyDeviceToHost, ps), "D2H selection");
    cuda_ok(cudaStreamSynchronize(ps), "select");
    if (comm.world_size() > 1 && comm.device().comm()) check(gf_comm_status(comm.device().comm()), "select");
    next_important_.assign(h_imp_, h_imp_ + nc);
    upload_important();  // d_imp_ keeps THIS iteration's set for sgd_update
    has_selection_ = true;
    return next_important_;
}

void SparseState::sgd_update(std::span<float> weights, int world_size) {
    if (weights.size() != pool_.total_elements()) throw ConfigError("weight vector does not match pool layout");
    flush_corrections();
    const std::size_t nc = pool_.num_chunks(), total = pool_.total_elements(), chunk = pool_.chunk_size();
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    std::vector<std::size_t> imp;  // the current important set, ascending
    for (std::size_t c = 0; c < nc; ++c)
        if (important_[c]) imp.push_back(c);
    upload_plan(imp, false);
    float* w = weights.data();
    const bool host = !is_device_ptr(w);
    // runs of consecutive important chunks: the only part of w the update touches
    std::vector<std::pair<std::size_t, std::size_t>> runs;
    for (std::size_t c : imp) {
        const std::size_t b = c * chunk, e = b + pool_.chunk_length(c);
        if (!runs.empty() && runs.back().second == b) runs.back().second = e;
        else runs.emplace_back(b, e);
    }
    if (host) {
        if (!d_w_) d_w_ = dalloc<float>(total, ps);
        for (auto& r : runs)
            cuda_ok(cudaMemcpyAsync(d_w_ + r.first, w + r.first, (r.second - r.first) * 4, cudaMemcpyHostToDevice, ps),
                    "H2D weights");
        w = d_w_;
    }
    check(gf_csc_sgd_update(static_cast<int>(pool_.element_type()), pool_.device_data(), d_plan_, total, chunk, nc,
                            imp.size(), world_size, static_cast<float>(config_.momentum),
                            static_cast<float>(config_.learning_rate), d_hu_, w, ps),
          "sgd_update");
    if (host)
        for (auto& r : runs)
            cuda_ok(cudaMemcpyAsync(weights.data() + r.first, d_w_ + r.first, (r.second - r.first) * 4,
                                    cudaMemcpyDeviceToHost, ps),
                    "D2H weights");
    cuda_ok(cudaStreamSynchronize(ps), "sgd_update");
}

std::span<const float> SparseState::hg() const {
    const_cast<SparseState*>(this)->flush_corrections();
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    hg_host_.resize(pool_.total_elements());
    cuda_ok(cudaMemcpyAsync(hg_host_.data(), d_hg_, hg_host_.size() * 4, cudaMemcpyDeviceToHost, ps), "D2H hg");
    cuda_ok(cudaStreamSynchronize(ps), "D2H hg");
    return hg_host_;
}

std::span<const float> SparseState::hu() const {
    OnDevice g(pool_.device());
    const auto ps = static_cast<cudaStream_t>(pool_.stream());
    hu_host_.resize(pool_.total_elements());
    cuda_ok(cudaMemcpyAsync(hu_host_.data(), d_hu_, hu_host_.size() * 4, cudaMemcpyDeviceToHost, ps), "D2H hu");
    cuda_ok(cudaStreamSynchronize(ps), "D2H hu");
    return hu_host_;
}

}  // namespace gflow
