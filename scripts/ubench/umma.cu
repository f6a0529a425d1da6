// Microbenchmark: tcgen05.mma issue throughput on one SM (zeros in shared
// memory, SW128 K-major descriptors): kind::tf32 / f16 (bf16) / i8 at
// M = 128 and several N; reports clocks per MMA instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/tc_kernels.cuh"
using namespace gps;

template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (KIND == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if constexpr (KIND == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND>
__global__ void k_umma(int N, int iters, long long* out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc;
    if (KIND == 0) idesc = (1u << 4) | (2u << 7) | (2u << 10);
    else if (KIND == 1) idesc = (1u << 4) | (1u << 7) | (1u << 10);
    else idesc = (2u << 4) | (1u << 7) | (1u << 10);
    idesc |= (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t da = umma_desc_sw128(smem), db = umma_desc_sw128(smem + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mma<KIND>(tm, da + 2 * k, db + 2 * k, idesc, (it | k) ? 1u : 0u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm) : "memory");
}

int main() {
  long long* out; cudaMalloc(&out, 8 * 1024);
  long long h[1024];
  const char* names[3] = {"tf32", "bf16", "i8"};
  for (int kind = 0; kind < 3; ++kind) {
    for (int N : {32, 64, 128, 256}) {
      const int iters = 4096;
      void (*kern)(int, int, long long*) = kind == 0 ? k_umma<0> : kind == 1 ? k_umma<1> : k_umma<2>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
      for (int grid : {1, 148}) {
        kern<<<grid, 128, 80 * 1024>>>(N, iters, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s N=%d: %s\n", names[kind], N, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, out, 8 * grid, cudaMemcpyDeviceToHost);
        const double clk = double(h[0]) / (iters * 4);
        const int kk = kind == 0 ? 8 : kind == 1 ? 16 : 32;
        printf("%s M=128 N=%3d K=%2d grid=%3d: %6.1f clk/MMA  %7.0f flop/clk/SM\n", names[kind], N, kk, grid, clk,
               2.0 * 128 * N * kk / clk);
      }
    }
  }
}
