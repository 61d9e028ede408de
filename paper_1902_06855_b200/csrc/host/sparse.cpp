// SPDX-License-Identifier: Apache-2.0
// Coarse-grained sparse communication on the GPU (reference: src/sparse.cpp).
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
T* dalloc(std::size_t n) {
    T* p = nullptr;
    cuda_ok(cudaMalloc(&p, std::max<std::size_t>(n * sizeof(T), 16)), "cudaMalloc");
    cuda_ok(cudaMemset(p, 0, std::max<std::size_t>(n * sizeof(T), 16)), "cudaMemset");
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
    d_hg_ = dalloc<float>(total);
    d_hu_ = dalloc<float>(total);
    d_imp_ = dalloc<std::uint8_t>(nc);
    d_coff_ = dalloc<std::uint64_t>(nc);
    d_plan_ = dalloc<std::uint64_t>(4 + nc);
    d_staging_ = dalloc<std::byte>(total * element_size(pool_.element_type()));
    d_norms_ = dalloc<float>(nc);
}

SparseState::~SparseState() {
    OnDevice g(pool_.device());
    cudaDeviceSynchronize();
    for (void* p : {static_cast<void*>(d_hg_), static_cast<void*>(d_hu_), static_cast<void*>(d_imp_),
                    static_cast<void*>(d_coff_), static_cast<void*>(d_plan_), static_cast<void*>(d_staging_),
                    static_cast<void*>(d_norms_), static_cast<void*>(d_w_)})
        cudaFree(p);
}

void SparseState::upload_important() {
    OnDevice g(pool_.device());
    cuda_ok(cudaMemcpy(d_imp_, important_.data(), important_.size(), cudaMemcpyHostToDevice), "H2D flags");
}

void SparseState::begin_iteration(std::uint64_t t) {
    iteration_ = t;
    current_sparsity_ = sparsity_at(t, config_.warmup_iters, config_.final_sparsity);
    if (has_selection_) important_ = next_important_;
    else std::fill(important_.begin(), important_.end(), 1);  // iteration 0 is dense
    queued_.clear();
    std::fill(corrected_.begin(), corrected_.end(), 0);
    exchanged_ = false;
    upload_important();
}

void SparseState::correction_pre_allreduce(std::size_t c) {
    if (c >= pool_.num_chunks()) throw ConfigError("chunk index out of range");
    const std::size_t begin = pool_.chunk_begin(c), len = pool_.chunk_length(c);
    if (begin + len > pool_.written_elements())
        throw ConfigError("correction on incomplete chunk " + std::to_string(c));
    if (corrected_[c]) throw ConfigError("chunk " + std::to_string(c) + " corrected twice");
    corrected_[c] = 1;
    OnDevice g(pool_.device());
    check(gf_csc_correct(static_cast<int>(pool_.element_type()), pool_.device_data(), d_hg_, d_imp_,
                         pool_.total_elements(), pool_.chunk_size(), pool_.num_chunks(), c, 1,
                         static_cast<float>(config_.momentum), nullptr),
          "correction_pre_allreduce");
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
    // staging layout: queued chunks in queue order (sparse.cpp:129-140)
    const std::size_t nc = pool_.num_chunks(), esz = element_size(pool_.element_type());
    std::vector<std::uint64_t> coff(nc, 0), plan(4 + nc, 0);
    std::uint64_t total = 0;
    for (std::size_t j = 0; j < queued_.size(); ++j) {
        coff[queued_[j]] = total;
        plan[4 + j] = queued_[j];
        total += pool_.chunk_length(queued_[j]);
    }
    plan[0] = total;
    plan[1] = queued_.size();
    OnDevice g(pool_.device());
    cuda_ok(cudaMemcpy(d_coff_, coff.data(), nc * 8, cudaMemcpyHostToDevice), "H2D coff");
    cuda_ok(cudaMemcpy(d_plan_, plan.data(), (4 + nc) * 8, cudaMemcpyHostToDevice), "H2D plan");
    const int dt = static_cast<int>(pool_.element_type());
    check(gf_csc_compact(dt, pool_.device_data(), d_staging_, d_plan_, d_coff_, pool_.total_elements(),
                         pool_.chunk_size(), nc, queued_.size(), nullptr),
          "sparse_exchange compact");
    cuda_ok(cudaDeviceSynchronize(), "compact");
    // theta windows over the staging buffer (sparse.cpp:142-158)
    ScalarBuffer stage{pool_.element_type(), d_staging_, total, Residency::kDevice};
    const std::uint64_t theta = engine.config().threshold_bytes;
    std::vector<FusedHandle> handles;
    std::size_t ws = 0, pos = 0;
    for (std::size_t c : queued_) {
        pos += pool_.chunk_length(c);
        if (theta != kThetaInfinite && (pos - ws) * esz >= theta) {
            handles.push_back(engine.enqueue_collective(stage.subspan(ws, pos - ws)));
            ws = pos;
        }
    }
    if (pos > ws) handles.push_back(engine.enqueue_collective(stage.subspan(ws, pos - ws)));
    last_exchange_windows_ = handles.size();
    FusionEngine::wait_all(handles);
    // global sums back into the pool (sparse.cpp:162-168)
    check(gf_csc_scatter(dt, pool_.device_data(), d_staging_, d_plan_, d_coff_, pool_.total_elements(),
                         pool_.chunk_size(), nc, queued_.size(), nullptr, nullptr),
          "sparse_exchange write-back");
    cuda_ok(cudaDeviceSynchronize(), "write-back");
    pool_.invalidate_host();
    exchanged_ = true;
}

const std::vector<std::uint8_t>& SparseState::select_next_important(Communicator& comm, std::uint64_t t) {
    if (!exchanged_) throw ConfigError("select_next_important before sparse_exchange");
    const std::size_t nc = pool_.num_chunks();
    OnDevice g(pool_.device());
    // exact chunk L1 (K3), x1/N on important chunks (sparse.cpp:176-184)
    check(gf_chunk_norms(static_cast<int>(pool_.element_type()), pool_.device_data(), pool_.total_elements(),
                         pool_.chunk_size(), nc, d_imp_, comm.world_size(), d_norms_, nullptr),
          "chunk norms");
    cuda_ok(cudaDeviceSynchronize(), "chunk norms");
    // fp32 ring allreduce of the norms (sparse.cpp:185-187), on the NVLink ring
    ring_allreduce(comm, ScalarBuffer{ElementType::kF32, reinterpret_cast<std::byte*>(d_norms_), nc,
                                      Residency::kDevice});
    const std::size_t k = selection_count(sparsity_at(t + 1, config_.warmup_iters, config_.final_sparsity), nc);
    check(gf_select_topk(d_norms_, nc, k, d_imp_, nullptr), "select");  // d_imp_ reloaded next iteration
    cuda_ok(cudaMemcpy(next_important_.data(), d_imp_, nc, cudaMemcpyDeviceToHost), "D2H selection");
    upload_important();  // d_imp_ keeps THIS iteration's set for sgd_update
    has_selection_ = true;
    return next_important_;
}

void SparseState::sgd_update(std::span<float> weights, int world_size) {
    if (weights.size() != pool_.total_elements()) throw ConfigError("weight vector does not match pool layout");
    const std::size_t nc = pool_.num_chunks(), total = pool_.total_elements();
    OnDevice g(pool_.device());
    // plan of the current important set (all of its chunks, ascending)
    std::vector<std::uint64_t> plan(4 + nc, 0);
    std::uint64_t k = 0;
    for (std::size_t c = 0; c < nc; ++c)
        if (important_[c]) plan[4 + k++] = c;
    plan[1] = k;
    cuda_ok(cudaMemcpy(d_plan_, plan.data(), (4 + nc) * 8, cudaMemcpyHostToDevice), "H2D plan");
    float* w = weights.data();
    const bool host = !is_device_ptr(w);
    if (host) {
        if (!d_w_) d_w_ = dalloc<float>(total);
        cuda_ok(cudaMemcpy(d_w_, w, total * 4, cudaMemcpyHostToDevice), "H2D weights");
        w = d_w_;
    }
    check(gf_csc_sgd_update(static_cast<int>(pool_.element_type()), pool_.device_data(), d_plan_, total,
                            pool_.chunk_size(), nc, k, world_size, static_cast<float>(config_.momentum),
                            static_cast<float>(config_.learning_rate), d_hu_, w, nullptr),
          "sgd_update");
    if (host) cuda_ok(cudaMemcpy(weights.data(), d_w_, total * 4, cudaMemcpyDeviceToHost), "D2H weights");
    else cuda_ok(cudaDeviceSynchronize(), "sgd_update");
}

std::span<const float> SparseState::hg() const {
    OnDevice g(pool_.device());
    hg_host_.resize(pool_.total_elements());
    cuda_ok(cudaMemcpy(hg_host_.data(), d_hg_, hg_host_.size() * 4, cudaMemcpyDeviceToHost), "D2H hg");
    return hg_host_;
}

std::span<const float> SparseState::hu() const {
    OnDevice g(pool_.device());
    hu_host_.resize(pool_.total_elements());
    cuda_ok(cudaMemcpy(hu_host_.data(), d_hu_, hu_host_.size() * 4, cudaMemcpyDeviceToHost), "D2H hu");
    return hu_host_;
}

}  // namespace gflow
