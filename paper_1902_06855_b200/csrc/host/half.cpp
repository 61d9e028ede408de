// SPDX-License-Identifier: Apache-2.0
// Host binary16 codec (API parity with include/gflow/half.hpp:20-93 of the reference).
#include "gflow/half.hpp"

#include <bit>
#include <cstring>

#include "gflow/errors.hpp"

namespace gflow {

std::uint16_t float_to_half_bits(float value) {
    const std::uint32_t b = std::bit_cast<std::uint32_t>(value);
    const std::uint16_t sign = static_cast<std::uint16_t>((b >> 16) & 0x8000u);
    const std::uint32_t exp8 = (b >> 23) & 0xFFu, frac = b & 0x7FFFFFu;
    if (exp8 == 0xFFu) return static_cast<std::uint16_t>(sign | (frac ? 0x7E00u : kHalfMaxFiniteBits));
    const int e = static_cast<int>(exp8) - 112;
    if (e >= 31) return static_cast<std::uint16_t>(sign | kHalfMaxFiniteBits);
    if (e <= 0) {
        if (e < -10) return sign;
        const std::uint32_t m = frac | 0x800000u;
        const int shift = 14 - e;
        std::uint32_t q = m >> shift;
        const std::uint32_t rest = m & ((1u << shift) - 1u), tie = 1u << (shift - 1);
        if (rest > tie || (rest == tie && (q & 1u))) ++q;
        return static_cast<std::uint16_t>(sign | q);
    }
    std::uint32_t h = (static_cast<std::uint32_t>(e) << 10) | (frac >> 13);
    const std::uint32_t rest = frac & 0x1FFFu;
    if (rest > 0x1000u || (rest == 0x1000u && (h & 1u))) ++h;
    if (h >= 0x7C00u) return static_cast<std::uint16_t>(sign | kHalfMaxFiniteBits);
    return static_cast<std::uint16_t>(sign | h);
}

float half_bits_to_float(std::uint16_t h) {
    const std::uint32_t sign = static_cast<std::uint32_t>(h & 0x8000u) << 16;
    const std::uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
    std::uint32_t bits;
    if (e == 0x1Fu) {
        bits = sign | 0x7F800000u | (m << 13);
    } else if (e != 0) {
        bits = sign | ((e + 112u) << 23) | (m << 13);
    } else if (m == 0) {
        bits = sign;
    } else {
        // normalise: shift the leading one of the 10-bit field up to bit 10
        const int sh = std::countl_zero(m) - 21;
        const std::uint32_t mm = (m << sh) & 0x3FFu;
        bits = sign | (static_cast<std::uint32_t>(113 - sh) << 23) | (mm << 13);
    }
    return std::bit_cast<float>(bits);
}

std::vector<std::byte> encode_half(std::span<const float> values) {
    std::vector<std::byte> out(values.size() * 2);
    for (std::size_t i = 0; i < values.size(); ++i) {
        const std::uint16_t h = float_to_half_bits(values[i]);
        out[2 * i] = static_cast<std::byte>(h & 0xFFu);
        out[2 * i + 1] = static_cast<std::byte>(h >> 8);
    }
    return out;
}

std::vector<float> decode_half(std::span<const std::byte> bytes) {
    if (bytes.size() % 2 != 0) throw ConfigError("half payload has odd length");
    std::vector<float> out(bytes.size() / 2);
    for (std::size_t i = 0; i < out.size(); ++i) {
        const std::uint16_t h = static_cast<std::uint16_t>(std::to_integer<std::uint16_t>(bytes[2 * i]) |
                                                           (std::to_integer<std::uint16_t>(bytes[2 * i + 1]) << 8));
        out[i] = half_bits_to_float(h);
    }
    return out;
}

}  // namespace gflow
