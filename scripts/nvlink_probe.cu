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

#include <cstdio>
#include <cstdlib>
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
    auto run = [&](const char* name, int kind, int blocks_per_sm, int threads) {
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
                dim3 g(sms * blocks_per_sm);
                if (kind == 0) pull<4><<<g, threads, 0, st[d]>>>(a);
                if (kind == 1) push<4><<<g, threads, 0, st[d]>>>(a);
                if (kind == 2) pull_all<1><<<g, threads, 0, st[d]>>>(a);
                if (kind == 3) push_all<2><<<g, threads, 0, st[d]>>>(a);
                if (kind == 5) mixed<2><<<g, threads, 0, st[d]>>>(a);
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
        printf("n=%d %-10s blocks/SM=%d thr=%d : %.3f ms  %.1f GB/s per GPU per direction\n", n, name,
               blocks_per_sm, threads, best, payload / (best * 1e-3) / 1e9);
    };
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
