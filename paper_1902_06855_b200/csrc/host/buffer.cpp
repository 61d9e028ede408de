// SPDX-License-Identifier: Apache-2.0
// ScalarBuffer helpers (reference: include/gflow/buffer.hpp:37-122) with device residency.
#include "gflow/buffer.hpp"

#include <cuda_runtime.h>

#include "gflow/device.hpp"
#include "gflow/errors.hpp"

namespace gflow {

namespace detail {

float device_get(ElementType t, const std::byte* data, std::size_t i) {
    const std::size_t es = element_size(t);
    std::byte tmp[4];
    if (cudaMemcpy(tmp, data + es * i, es, cudaMemcpyDefault) != cudaSuccess)
        throw TransportError("ScalarBuffer::get: device read failed");
    ScalarBuffer h{t, tmp, 1, Residency::kHost};
    return h.get(0);
}

void device_set(ElementType t, std::byte* data, std::size_t i, float v) {
    const std::size_t es = element_size(t);
    std::byte tmp[4];
    ScalarBuffer h{t, tmp, 1, Residency::kHost};
    h.set(0, v);
    if (cudaMemcpy(data + es * i, tmp, es, cudaMemcpyDefault) != cudaSuccess)
        throw TransportError("ScalarBuffer::set: device write failed");
}

void device_copy(void* dst, const void* src, std::size_t bytes) {
    if (bytes == 0) return;
    if (cudaMemcpy(dst, src, bytes, cudaMemcpyDefault) != cudaSuccess)
        throw TransportError("device copy failed");
}

}  // namespace detail

void accumulate(ScalarBuffer dst, std::span<const std::byte> src) {
    const std::size_t n = src.size() / element_size(dst.type);
    if (n > dst.length) throw ProtocolError("accumulate: source longer than destination");
    if (dst.on_device()) {
        // device destination: stage the source next to it and run the sm_100a kernel
        void* tmp = nullptr;
        if (cudaMalloc(&tmp, src.size()) != cudaSuccess) throw TransportError("accumulate: cudaMalloc");
        detail::device_copy(tmp, src.data(), src.size());
        const int rc = gf_accumulate(static_cast<int>(dst.type), dst.data, tmp, n, nullptr);
        cudaDeviceSynchronize();
        cudaFree(tmp);
        check(rc, "accumulate");
        return;
    }
    if (dst.type == ElementType::kF32) {
        for (std::size_t i = 0; i < n; ++i) {
            float a, b;
            std::memcpy(&a, dst.data + 4 * i, 4);
            std::memcpy(&b, src.data() + 4 * i, 4);
            a += b;
            std::memcpy(dst.data + 4 * i, &a, 4);
        }
    } else {
        for (std::size_t i = 0; i < n; ++i) {
            std::uint16_t a, b;
            std::memcpy(&a, dst.data + 2 * i, 2);
            std::memcpy(&b, src.data() + 2 * i, 2);
            // the reference binary adds the incoming value as the destination operand
            const float incoming = half_bits_to_float(b), local = half_bits_to_float(a);
            const std::uint16_t r = float_to_half_bits(incoming + local);
            std::memcpy(dst.data + 2 * i, &r, 2);
        }
    }
}

std::vector<std::byte> to_bytes(ScalarBuffer buf) {
    std::vector<std::byte> out(buf.byte_length());
    if (buf.on_device()) detail::device_copy(out.data(), buf.data, out.size());
    else std::memcpy(out.data(), buf.data, out.size());
    return out;
}

void from_bytes(ScalarBuffer buf, std::span<const std::byte> bytes) {
    if (buf.on_device()) detail::device_copy(buf.data, bytes.data(), bytes.size());
    else std::memcpy(buf.data, bytes.data(), bytes.size());
}

OwnedBuffer OwnedBuffer::from_floats(ElementType type, std::span<const float> values) {
    OwnedBuffer b(type, values.size());
    ScalarBuffer v = b.view();
    for (std::size_t i = 0; i < values.size(); ++i) v.set(i, values[i]);
    return b;
}

std::vector<float> OwnedBuffer::to_floats() {
    ScalarBuffer v = view();
    std::vector<float> out(length_);
    for (std::size_t i = 0; i < length_; ++i) out[i] = v.get(i);
    return out;
}

}  // namespace gflow
