// SPDX-License-Identifier: Apache-2.0
// Host-side helpers shared by the kernel translation units: status/error
// plumbing of the C-ABI, launch accounting, device properties.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "gflow_b200.h"

namespace gfi {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(uint64_t n = 1);
int sm_count();              // SMs of the current device (cached per device)
int check_launch(const char* what);  // cudaGetLastError -> status

// Phase marks between the launches of a multi-kernel entry point (per calling thread): the
// engine's per-kernel timing records an event on the launching stream at each mark.
using PhaseHook = void (*)(void* ctx, const char* name, cudaStream_t s);
void set_phase_hook(PhaseHook hook, void* ctx);
void phase(const char* name, cudaStream_t s);

// world == 1 dense step (pack.cu): pack and unpack in one pass (the collective is the identity)
int pack_unpack_solo(int dtype, void* pool, const float* const* src, float* const* dst,
                     const uint64_t* pool_off, const uint64_t* count, int ntensors, cudaStream_t stream);

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline uint64_t esz(int dtype) { return dtype == GF_F32 ? 4u : 2u; }
inline bool valid_dtype(int d) { return d == GF_F32 || d == GF_F16; }

}  // namespace gfi

#define GF_CHECK_CUDA(expr)                                        \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return gfi::cuda_fail(_e, #expr);   \
    } while (0)
