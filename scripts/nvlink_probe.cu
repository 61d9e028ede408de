// SPDX-License-Identifier: Apache-2.0
// NVLink peer-access microbenchmark (design probe for the K4 ring kernel).
// One process, devices 0..N-1 with peer access. Patterns (all GPUs run simultaneously):
//   read    : every GPU copies its share FROM peers into local memory (pull)
//   write   : every GPU copies local data TO peers (push)
//   mixed   : read half the bytes from peers, write half to peers
//   memcpy  : cudaMemcpyPeerAsync of the same volume
// Reports per-GPU outgoing+incoming payload GB/s per direction.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

struct Args {
    uint4* src[8];
    uint4* dst[8];
    int n, me;
    size_t vec_per_peer;  // 16-B vectors moved per peer
    int unroll;
};

template <int U>
__global__ void pull(Args a) {
    // read from each peer q: src[q][me*V ...] -> dst[me][q*V ...] (local)
    const size_t V = a.vec_per_peer;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (int qq = 1; qq < a.n; ++qq) {
        const int q = (a.me + qq) % a.n;
        const uint4* s = a.src[q] + a.me * V;
        uint4* d = a.dst[a.me] + q * V;
        for (size_t i = tid; i < V; i += stride * U) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + u * stride < V) x[u] = s[i + u * stride];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + u * stride < V) d[i + u * stride] = x[u];
        }
    }
}

template <int U>
__global__ void pull_all(Args a) {
    // interleaved: each thread loads from ALL peers before storing
    const size_t V = a.vec_per_peer;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = tid; i < V; i += stride * U) {
        uint4 x[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < a.n && q != a.me && i + u * stride < V) x[u][q] = a.src[q][a.me * V + i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < a.n && q != a.me && i + u * stride < V) a.dst[a.me][q * V + i + u * stride] = x[u][q];
    }
}

template <int U>
__global__ void push(Args a) {
    const size_t V = a.vec_per_peer;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (int qq = 1; qq < a.n; ++qq) {
        const int q = (a.me + qq) % a.n;
        const uint4* s = a.src[a.me] + q * V;
        uint4* d = a.dst[q] + a.me * V;
        for (size_t i = tid; i < V; i += stride * U) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + u * stride < V) x[u] = s[i + u * stride];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + u * stride < V) d[i + u * stride] = x[u];
        }
    }
}

template <int U>
__global__ void push_all(Args a) {
    const size_t V = a.vec_per_peer;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = tid; i < V; i += stride * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < V) x[u] = a.src[a.me][i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < a.n && q != a.me && i + u * stride < V) a.dst[q][a.me * V + i + u * stride] = x[u];
    }
}

// ring-like mix: each thread pulls one vector from every peer (its owned segment) and pushes
// one vector to every peer (the all-gather), like the K4 kernel
template <int U>
__global__ void mixed(Args a) {
    const size_t V = a.vec_per_peer;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = tid; i < V; i += stride * U) {
        uint4 x[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < a.n && i + u * stride < V) x[u][q] = a.src[q][a.me * V + i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint4 acc = x[u][0];
#pragma unroll
            for (int q = 1; q < 8; ++q)
                if (q < a.n) { acc.x ^= x[u][q].x; acc.y += x[u][q].y; }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < a.n && i + u * stride < V) a.dst[q][a.me * V + i + u * stride] = acc;
        }
    }
}

template <int U>
__global__ void pushpull(Args a) {
    // the ring kernel's pattern: owner of slot `me` loads slot me from every GPU, sums
    // (here: xor), stores the result into every GPU's slot me
    const size_t V = a.vec_per_peer;
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = tid; i < V; i += stride * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = make_uint4(0, 0, 0, 0);
        for (int q = 0; q < a.n; ++q) {
            const uint4* s = a.src[q] + a.me * V;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + u * stride < V) {
                    const uint4 y = s[i + u * stride];
                    x[u].x ^= y.x; x[u].y ^= y.y; x[u].z ^= y.z; x[u].w ^= y.w;
                }
        }
        for (int q = 0; q < a.n; ++q) {
            uint4* d = a.src[(a.me + 1 + q) % a.n] + a.me * V;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + u * stride < V) d[i + u * stride] = x[u];
        }
    }
}

// ---- TMA bulk copies (cp.async.bulk): one elected thread per CTA moves whole tiles ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(b)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

// mode 0: pull (peer -> smem -> local), 1: push (local -> smem -> peer), 2: pushpull (N loads, N stores)
constexpr int kTmaStages = 4;
template <int MODE>
__global__ void tma_copy(Args a, uint32_t tile) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[kTmaStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t V = a.vec_per_peer * 16;  // bytes per slot
    const size_t ntile = V / tile;
    const int q = (a.me + 1) % a.n;  // one peer (n == 2 probe)
    uint32_t phase[kTmaStages] = {};
    int it = 0;
    for (size_t t = blockIdx.x; t < ntile; t += gridDim.x, ++it) {
        const int s = it % kTmaStages;
        unsigned char* buf = sm + size_t(s) * tile * (MODE == 2 ? 2 : 1);
        if (it >= kTmaStages) bulk_wait_read<kTmaStages - 1>();  // stage s's stores have read smem
        const size_t off = size_t(a.me) * V + t * tile;
        if (MODE == 0) {
            mbar_expect(&bar[s], tile);
            bulk_g2s(buf, reinterpret_cast<const char*>(a.src[q]) + off, tile, &bar[s]);
            mbar_wait(&bar[s], phase[s]);
            phase[s] ^= 1;
            bulk_s2g(reinterpret_cast<char*>(a.dst[a.me]) + off, buf, tile);
        } else if (MODE == 1) {
            mbar_expect(&bar[s], tile);
            bulk_g2s(buf, reinterpret_cast<const char*>(a.src[a.me]) + off, tile, &bar[s]);
            mbar_wait(&bar[s], phase[s]);
            phase[s] ^= 1;
            bulk_s2g(reinterpret_cast<char*>(a.dst[q]) + off, buf, tile);
        } else {
            mbar_expect(&bar[s], 2 * tile);
            bulk_g2s(buf, reinterpret_cast<const char*>(a.src[a.me]) + off, tile, &bar[s]);
            bulk_g2s(buf + tile, reinterpret_cast<const char*>(a.src[q]) + off, tile, &bar[s]);
            mbar_wait(&bar[s], phase[s]);
            phase[s] ^= 1;
            bulk_s2g(reinterpret_cast<char*>(a.src[q]) + off, buf, tile);
            bulk_s2g(reinterpret_cast<char*>(a.src[a.me]) + off, buf + tile, tile);
        }
        bulk_commit();
    }
    bulk_wait_read<0>();
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 2;
    size_t mb = argc > 2 ? atoll(argv[2]) : 256;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < n) n = ndev;
    const size_t bytes = mb << 20;
    std::vector<uint4*> src(n), dst(n);
    std::vector<cudaStream_t> st(n);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < n; ++q)
            if (q != d) {
                cudaError_t pe = cudaDeviceEnablePeerAccess(q, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
                cudaGetLastError();
            }
        CK(cudaMalloc(&src[d], bytes));
        CK(cudaMalloc(&dst[d], bytes));
        CK(cudaMemset(src[d], d + 1, bytes));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    }
    const size_t V = bytes / 16 / n;  // vectors per peer slot
    const double payload = double(V) * 16 * (n - 1);  // bytes each GPU sends (or receives)
    auto run = [&](const char* name, int kind, int blocks_per_sm, int threads, int grid_override = 0) {
        std::vector<cudaEvent_t> e0(n), e1(n);
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaDeviceSynchronize());
            }
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventCreate(&e0[d]));
                CK(cudaEventCreate(&e1[d]));
                Args a{};
                for (int q = 0; q < n; ++q) { a.src[q] = src[q]; a.dst[q] = dst[q]; }
                a.n = n; a.me = d; a.vec_per_peer = V;
                CK(cudaEventRecord(e0[d], st[d]));
                dim3 g(grid_override ? grid_override : sms * blocks_per_sm);
                if (kind == 0) pull<4><<<g, threads, 0, st[d]>>>(a);
                if (kind == 1) push<4><<<g, threads, 0, st[d]>>>(a);
                if (kind == 2) pull_all<1><<<g, threads, 0, st[d]>>>(a);
                if (kind == 3) push_all<2><<<g, threads, 0, st[d]>>>(a);
                if (kind == 5) mixed<2><<<g, threads, 0, st[d]>>>(a);
                if (kind >= 10) {
                    const uint32_t tile = uint32_t(threads);  // bytes per bulk copy
                    const int mode = kind - 10;
                    const size_t smem = size_t(tile) * kTmaStages * (mode == 2 ? 2 : 1);
                    if (mode == 0) { cudaFuncSetAttribute(tma_copy<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); tma_copy<0><<<g, 32, smem, st[d]>>>(a, tile); }
                    if (mode == 1) { cudaFuncSetAttribute(tma_copy<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); tma_copy<1><<<g, 32, smem, st[d]>>>(a, tile); }
                    if (mode == 2) { cudaFuncSetAttribute(tma_copy<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); tma_copy<2><<<g, 32, smem, st[d]>>>(a, tile); }
                    CK(cudaGetLastError());
                }
                if (kind == 6) pushpull<4><<<g, threads, 0, st[d]>>>(a);
                if (kind == 7) pushpull<8><<<g, threads, 0, st[d]>>>(a);
                if (kind == 4) {
                    for (int qq = 1; qq < n; ++qq) {
                        int q = (d + qq) % n;
                        CK(cudaMemcpyPeerAsync(dst[q] + d * V, q, src[d] + q * V, d, V * 16, st[d]));
                    }
                }
                CK(cudaEventRecord(e1[d], st[d]));
            }
            float worst = 0;
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventSynchronize(e1[d]));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
                if (ms > worst) worst = ms;
            }
            if (rep > 0 && worst < best) best = worst;
        }
        printf("n=%d %-10s grid=%d thr=%d : %.3f ms  %.1f GB/s per GPU per direction\n", n, name,
               grid_override ? grid_override : sms * blocks_per_sm, threads, best, payload / (best * 1e-3) / 1e9);
    };
    if (argc > 3 && std::string(argv[3]) == "tma") {  // TMA bulk copies: tile bytes x CTAs
        for (int tile : {8192, 16384, 32768}) {
            for (int gcta : {32, 64, 148, 296}) {
                run("tma_pull", 10, 1, tile, gcta);
                run("tma_push", 11, 1, tile, gcta);
                run("tma_pp", 12, 1, tile, gcta);
            }
        }
        return 0;
    }
    if (argc > 3) {  // CTA sweep: pull / push / push-pull (the ring kernel's pattern)
        for (int gcta : {16, 32, 48, 64, 96, 148, 296}) {
            run("pull", 0, 1, 512, gcta);
            run("push", 1, 1, 512, gcta);
            run("pushpull4", 6, 1, 512, gcta);
            run("pushpull8", 7, 1, 512, gcta);
        }
        return 0;
    }
    for (int b : {1, 2}) {
        run("pull", 0, b, 512);
        run("push", 1, b, 512);
        run("pull_all", 2, b, 512);
        run("push_all", 3, b, 512);
        run("mixed(x2)", 5, b, 512);
    }
    run("memcpy", 4, 1, 1);
    return 0;
}
