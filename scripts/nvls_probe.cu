// NVLS probe: does multimem (NVLink SHARP) work on this box, and what does a one-shot
// switch-reduced allreduce of an fp16 buffer cost? Each rank reduces its 1/N slice with
// multimem.ld_reduce (fp32 accumulation in the switch) and multicasts it with multimem.st.
// Not product code: a measurement for DESIGN.md §9.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void flag_barrier(uint32_t* const* flags, int rank, int world,
                                             uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x < world) {
    uint32_t* peer = flags[threadIdx.x] + blockIdx.x * 32 + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer), "r"(epoch) : "memory");
    uint32_t* mine = flags[rank] + blockIdx.x * 32 + threadIdx.x;
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    } while (v < epoch);
  }
  __syncthreads();
}

struct Flags { uint32_t* p[8]; };

__global__ void nvls_allreduce(uint4* mc, size_t n16, int rank, int world, Flags f,
                               uint32_t epoch, int acc32) {
  flag_barrier(f.p, rank, world, epoch * 2);
  size_t per = (n16 + world - 1) / world;
  size_t b = per * rank, e = b + per < n16 ? b + per : n16;
  for (size_t i = b + blockIdx.x * blockDim.x + threadIdx.x; i < e;
       i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a, c, d, g;
    if (acc32)
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                   : "=r"(a), "=r"(c), "=r"(d), "=r"(g) : "l"(mc + i) : "memory");
    else
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                   : "=r"(a), "=r"(c), "=r"(d), "=r"(g) : "l"(mc + i) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f16x2 [%0], {%1,%2,%3,%4};"
                 ::"l"(mc + i), "r"(a), "r"(c), "r"(d), "r"(g) : "memory");
  }
  asm volatile("fence.proxy.alias;" ::: "memory");
  flag_barrier(f.p, rank, world, epoch * 2 + 1);
}

extern "C" int nvls_run(void* mc, size_t bytes, int rank, int world, void** flags,
                        uint32_t epoch, int blocks, int acc32, void* stream) {
  Flags f{};
  for (int i = 0; i < world; ++i) f.p[i] = (uint32_t*)flags[i];
  nvls_allreduce<<<blocks, 512, 0, (cudaStream_t)stream>>>((uint4*)mc, bytes / 16, rank, world, f,
                                                           epoch, acc32);
  return (int)cudaGetLastError();
}
