// SPDX-License-Identifier: Apache-2.0
// GradientPool on the GPU (reference: src/gradient_pool.cpp — layout :11-41, chunking
// :55-70, write_tensor :78-105, chunk_l1 :107-116, dump_snapshot :118-128).
#include "gflow/gradient_pool.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "gflow/device.hpp"

namespace gflow {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw TransportError(std::string(what) + ": " + cudaGetErrorString(e));
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

GradientPool::GradientPool(const std::vector<std::size_t>& sizes, std::size_t chunk_size, ElementType type)
    : chunk_size_(chunk_size), element_type_(type) {
    if (sizes.empty()) throw ConfigError("gradient pool needs at least one tensor");
    if (chunk_size == 0) throw ConfigError("chunk_size must be positive");
    for (std::size_t s : sizes)
        if (s == 0) throw ConfigError("tensor sizes must be positive");
    const int m = static_cast<int>(sizes.size());
    descs_.resize(sizes.size());
    std::size_t off = 0;
    for (int id = m; id >= 1; --id) {  // tensor m first: backward emits m..1
        descs_[static_cast<std::size_t>(id - 1)] = {id, sizes[static_cast<std::size_t>(id - 1)], off};
        off += sizes[static_cast<std::size_t>(id - 1)];
    }
    total_elements_ = off;
    num_chunks_ = std::max<std::size_t>(
        1, static_cast<std::size_t>(std::llround(static_cast<double>(off) / static_cast<double>(chunk_size))));
    next_expected_id_ = m;
    cuda_ok(cudaGetDevice(&device_), "cudaGetDevice");
    const std::size_t bytes = total_elements_ * element_size(type);
    cuda_ok(cudaMalloc(&data_, std::max<std::size_t>(bytes, 16)), "cudaMalloc pool");
    cuda_ok(cudaMemset(data_, 0, bytes), "cudaMemset pool");
    cuda_ok(cudaMalloc(&norm_out_, sizeof(float)), "cudaMalloc");
    host_.assign(bytes, std::byte{0});
    host_valid_ = true;
}

GradientPool::GradientPool(GradientPool&& o) noexcept
    : descs_(std::move(o.descs_)), total_elements_(o.total_elements_), chunk_size_(o.chunk_size_),
      num_chunks_(o.num_chunks_), element_type_(o.element_type_), device_(o.device_), data_(o.data_),
      stage_(o.stage_), stage_elems_(o.stage_elems_), norm_out_(o.norm_out_), host_(std::move(o.host_)),
      host_valid_(o.host_valid_), watermark_(o.watermark_), chunks_reported_(o.chunks_reported_),
      next_expected_id_(o.next_expected_id_) {
    o.data_ = nullptr;
    o.stage_ = nullptr;
    o.norm_out_ = nullptr;
}

GradientPool::~GradientPool() {
    if (!data_ && !stage_ && !norm_out_) return;
    OnDevice g(device_);
    cudaDeviceSynchronize();
    cudaFree(data_);
    cudaFree(stage_);
    cudaFree(norm_out_);
}

const TensorDesc& GradientPool::desc(int tensor_id) const {
    if (tensor_id < 1 || tensor_id > num_tensors())
        throw ConfigError("tensor id " + std::to_string(tensor_id) + " out of range");
    return descs_[static_cast<std::size_t>(tensor_id - 1)];
}

ScalarBuffer GradientPool::view() {
    host_valid_ = false;  // the caller may write through the view
    return {element_type_, data_, total_elements_, Residency::kDevice};
}

ScalarBuffer GradientPool::tensor_view(int tensor_id) {
    const TensorDesc& d = desc(tensor_id);
    return view().subspan(d.pool_offset, d.element_count);
}

std::size_t GradientPool::chunk_begin(std::size_t c) const {
    if (c >= num_chunks_) throw ConfigError("chunk index " + std::to_string(c) + " out of range");
    return c * chunk_size_;
}

std::size_t GradientPool::chunk_length(std::size_t c) const {
    const std::size_t b = chunk_begin(c);
    return c + 1 == num_chunks_ ? total_elements_ - b : chunk_size_;
}

ScalarBuffer GradientPool::chunk_view(std::size_t c) {
    return view().subspan(chunk_begin(c), chunk_length(c));
}

void GradientPool::begin_iteration() {
    watermark_ = 0;
    chunks_reported_ = 0;
    next_expected_id_ = num_tensors();
}

std::vector<std::size_t> GradientPool::write_tensor(int tensor_id, std::span<const float> values) {
    const TensorDesc& d = desc(tensor_id);
    if (tensor_id > next_expected_id_)
        throw ConfigError("tensor " + std::to_string(tensor_id) + " written twice in one iteration");
    if (tensor_id < next_expected_id_)
        throw ConfigError("out-of-order tensor write: got " + std::to_string(tensor_id) + ", expected " +
                          std::to_string(next_expected_id_));
    if (values.size() != d.element_count)
        throw ConfigError("tensor " + std::to_string(tensor_id) + " length mismatch: " +
                          std::to_string(values.size()) + " vs " + std::to_string(d.element_count));
    OnDevice g(device_);
    const float* src = values.data();
    if (!is_device_ptr(src)) {  // host gradients: one H2D copy into the staging buffer
        if (stage_elems_ < values.size()) {
            cudaFree(stage_);
            stage_ = nullptr;
            cuda_ok(cudaMalloc(&stage_, values.size() * sizeof(float)), "cudaMalloc stage");
            stage_elems_ = values.size();
        }
        cuda_ok(cudaMemcpy(stage_, src, values.size() * sizeof(float), cudaMemcpyHostToDevice), "H2D");
        src = stage_;
    }
    const std::uint64_t off = d.pool_offset, cnt = d.element_count;
    check(gf_pack(static_cast<int>(element_type_), data_, &src, &off, &cnt, 1, 1.0f, nullptr), "write_tensor");
    host_valid_ = false;
    next_expected_id_ = tensor_id - 1;
    watermark_ = d.pool_offset + d.element_count;
    std::vector<std::size_t> done;
    while (chunks_reported_ < num_chunks_ &&
           chunk_begin(chunks_reported_) + chunk_length(chunks_reported_) <= watermark_) {
        done.push_back(chunks_reported_++);
    }
    return done;
}

void GradientPool::sync_host() {
    if (host_valid_) return;
    OnDevice g(device_);
    cuda_ok(cudaMemcpy(host_.data(), data_, host_.size(), cudaMemcpyDeviceToHost), "pool D2H");
    host_valid_ = true;
}

float GradientPool::get(std::size_t i) {
    sync_host();
    ScalarBuffer h{element_type_, host_.data(), total_elements_, Residency::kHost};
    return h.get(i);
}

void GradientPool::set(std::size_t i, float v) {
    sync_host();
    ScalarBuffer h{element_type_, host_.data(), total_elements_, Residency::kHost};
    h.set(i, v);
    const std::size_t es = element_size(element_type_);
    OnDevice g(device_);
    cuda_ok(cudaMemcpy(data_ + i * es, host_.data() + i * es, es, cudaMemcpyHostToDevice), "pool set");
}

float GradientPool::chunk_l1(std::size_t c) {
    const std::size_t b = chunk_begin(c), len = chunk_length(c);
    OnDevice g(device_);
    // one-chunk launch of K3 (exact; bit-identical to the reference's fp64 loop)
    check(gf_chunk_norms(static_cast<int>(element_type_), data_ + b * element_size(element_type_), len, len, 1,
                         nullptr, 1, norm_out_, nullptr),
          "chunk_l1");
    float out = 0.0f;
    cuda_ok(cudaMemcpy(&out, norm_out_, sizeof(float), cudaMemcpyDeviceToHost), "chunk_l1 D2H");
    return out;
}

void GradientPool::dump_snapshot(std::ostream& os) {
    sync_host();
    const std::uint64_t total = total_elements_, chunk = chunk_size_;
    const std::uint8_t type = static_cast<std::uint8_t>(element_type_);
    os.write(reinterpret_cast<const char*>(&total), 8);
    os.write(reinterpret_cast<const char*>(&chunk), 8);
    os.write(reinterpret_cast<const char*>(&type), 1);
    os.write(reinterpret_cast<const char*>(host_.data()), static_cast<std::streamsize>(host_.size()));
}

GradientPool build_pool(const std::vector<std::size_t>& sizes, std::size_t chunk_size, ElementType type) {
    return GradientPool(sizes, chunk_size, type);
}

}  // namespace gflow
