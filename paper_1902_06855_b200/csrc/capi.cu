// SPDX-License-Identifier: Apache-2.0
// C-ABI plumbing: error reporting, launch accounting, device properties.

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <string>

#include "gf_internal.cuh"

namespace {
thread_local std::string g_last_error;
thread_local gfi::PhaseHook g_phase_hook = nullptr;
thread_local void* g_phase_ctx = nullptr;
std::atomic<uint64_t> g_launches{0};
std::mutex g_sm_mu;
int g_sm_count[64] = {};
}  // namespace

namespace gfi {

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return GF_ERR_CUDA;
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    std::lock_guard<std::mutex> lk(g_sm_mu);
    if (g_sm_count[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        g_sm_count[dev] = n;
    }
    return g_sm_count[dev];
}

void set_phase_hook(PhaseHook hook, void* ctx) {
    g_phase_hook = hook;
    g_phase_ctx = ctx;
}

void phase(const char* name, cudaStream_t s) {
    if (g_phase_hook) g_phase_hook(g_phase_ctx, name, s);
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    return GF_OK;
}

}  // namespace gfi

extern "C" {

int gf_abi_version(void) { return GF_ABI_VERSION; }
const char* gf_last_error(void) { return g_last_error.c_str(); }
uint64_t gf_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
