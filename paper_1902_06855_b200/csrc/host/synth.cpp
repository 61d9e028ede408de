// SPDX-License-Identifier: Apache-2.0
// Synthetic gradient sets of the benchmark: the seeded stream the
// reference's bench_allreduce draws its buffers from (src/harness.cpp:280-283,
// std::mt19937_64(1234 + r) with uniform_real_distribution<float>(-1, 1)), extended per
// step and scaled per tensor so that chunk norms differ and the CSC top-k is non-trivial:
//   rank r, step t: std::mt19937_64(1234 + r + 7919 t); tensors in ascending id 1..m;
//   element = uniform(-1, 1) * 2^-(id mod 7).
// Host code, compiled with the same standard library as the reference build, so the CPU
// reference arm and the GPU arm of bench.py sync the very same gradients.
#include <cmath>
#include <cstdint>
#include <random>

#include "gflow_b200.h"

extern "C" int gf_synth_grads(int rank, int step, const uint64_t* sizes, int ntensors, float* out) {
    if (rank < 0 || step < 0 || ntensors < 0 || (ntensors > 0 && (!sizes || !out))) return GF_ERR_CONFIG;
    std::mt19937_64 rng(1234 + static_cast<uint64_t>(rank) + 7919ull * static_cast<uint64_t>(step));
    std::uniform_real_distribution<float> uni(-1.0f, 1.0f);
    uint64_t o = 0;
    for (int id = 1; id <= ntensors; ++id) {
        const float s = std::ldexp(1.0f, -(id % 7));
        for (uint64_t i = 0; i < sizes[id - 1]; ++i) out[o++] = uni(rng) * s;
    }
    return GF_OK;
}
