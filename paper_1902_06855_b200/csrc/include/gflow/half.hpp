// SPDX-License-Identifier: Apache-2.0
// binary16 codec of the gflow API (reference: include/gflow/half.hpp:17-93):
// round-to-nearest-even, overflow and +-inf clamp to +-65504, NaN -> sign|0x7E00.
// Host versions for API parity; the device path uses the same rules (csrc/gf_device.cuh).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

namespace gflow {

inline constexpr std::uint16_t kHalfMaxFiniteBits = 0x7BFF;
inline constexpr float kHalfMaxFinite = 65504.0f;

std::uint16_t float_to_half_bits(float value);
float half_bits_to_float(std::uint16_t bits);

// Little-endian byte codec (wire / snapshot format).
std::vector<std::byte> encode_half(std::span<const float> values);
std::vector<float> decode_half(std::span<const std::byte> bytes);

}  // namespace gflow
