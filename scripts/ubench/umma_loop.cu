// Microbenchmark: per-chunk overheads around tcgen05.mma in a producer /
// consumer loop: commits, fences and mbarrier probes per 4-MMA chunk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/tc_kernels.cuh"
using namespace gps;

__global__ void k_loop(int N, int iters, int variant, long long* out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
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
    const uint32_t idesc = umma_idesc_tf32(128, N);
    const uint64_t da = umma_desc_sw128(smem), db = umma_desc_sw128(smem + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (variant >= 4) {  // probes of a barrier that is already complete (phase 1 never reached)
        mbar_wait(&bar[7], 1u);
        mbar_wait(&bar[7], 1u);
        mbar_wait(&bar[7], 1u);
      }
      if (variant >= 3) tc_fence_after();
#pragma unroll
      for (int k = 0; k < 4; ++k) umma_tf32(tm, da + 2 * k, db + 2 * k, idesc, (it | k) ? 1u : 0u);
      if (variant >= 1) umma_commit(&bar[0]);
      if (variant >= 2) {
        umma_commit(&bar[1]);
        umma_commit(&bar[2]);
      }
      if (variant == 5 && (it & 3) == 3) {  // wait for the chunk 2 back (like tempty)
        // nothing: placeholder
      }
    }
    umma_commit(&bar[6]);
    mbar_wait(&bar[6], 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm) : "memory");
}

int main() {
  long long* out; cudaMalloc(&out, 8 * 1024);
  long long h[4];
  cudaFuncSetAttribute(k_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int N : {64, 128}) {
    for (int v = 0; v <= 4; ++v) {
      const int iters = 4096;
      k_loop<<<1, 128, 80 * 1024>>>(N, iters, v, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
      printf("N=%3d variant=%d: %7.1f clk per 4-MMA chunk\n", N, v, double(h[0]) / iters);
    }
  }
}
