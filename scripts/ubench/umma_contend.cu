// Microbenchmark: tcgen05.mma (A in TMEM, B in shared memory, N = 128 and
// N = 64 alternating like the tensor-core sweep) while other warps load the
// shared-memory port (LDS.128 streams) or TMEM (tcgen05.ld / tcgen05.st).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/tc_kernels.cuh"
using namespace gps;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ volatile int g_stop;

// mode bits: 1 = LDS streaming warps, 2 = tcgen05.st warps, 4 = tcgen05.ld warps, 8 = second MMA (N=64)
__global__ void __launch_bounds__(384, 1) k_contend(int iters, int mode, long long* out, float* sink) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    done = 0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (warp == 1) {
    const uint32_t id2 = umma_idesc_tf32(128, 128), id1 = umma_idesc_tf32(128, 64);
    const uint64_t db = umma_desc_sw128(smem + 65536);
    long long t0 = clock64();
    int slot = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (it >= 4) mbar_wait(&bar[slot], ph ^ 1u);
      tc_fence_after();
      const uint64_t b0 = db + uint64_t(slot) * 1024;
      const uint32_t a0 = tm + 256 + (slot & 1) * 64;
      const uint32_t d = tm + ((it >> 2) & 1) * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        umma_ts(d, a0 + 8 * k, b0 + 2 * k, id2, (it | k) ? 1u : 0u);
        if (mode & 8) umma_ts(d, a0 + 32 + 8 * k, b0 + 2 * k, id1, 1u);
      }
      commit_elect(&bar[slot]);
      if (++slot == 4) {
        slot = 0;
        ph ^= 1u;
      }
    }
    commit_elect(&bar[7]);
    mbar_wait(&bar[7], 0);
    long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x] = t1 - t0;
      done = 1;
    }
  } else if (warp >= 8 && (mode & 1)) {
    // LDS.128 streaming over 64 KB
    float acc = 0.f;
    const int t = threadIdx.x - 256;
    while (!done) {
      for (int i = t * 16; i < 65536; i += 128 * 16) {
        const float4 v = *reinterpret_cast<const float4*>(smem + i);
        acc += v.x + v.w;
      }
    }
    if (acc == 1.2345f) sink[0] = acc;
  } else if (warp >= 8 && (mode & 2)) {
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = i;
    const int q = warp & 3;
    while (!done) {
      tmem_st32(tm + (uint32_t(q * 32) << 16) + 384, v);
      tmem_st32(tm + (uint32_t(q * 32) << 16) + 416, v);
      tmem_wait_st();
    }
  } else if (warp >= 4 && warp < 8 && (mode & 4)) {
    const int q = warp & 3;
    float acc = 0.f;
    while (!done) {
      float v[16];
      tmem_ld16(tm + (uint32_t(q * 32) << 16) + 448, v);
      tmem_wait_ld();
      acc += v[0];
    }
    if (acc == 1.2345f) sink[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main() {
  long long* out; float* sink;
  cudaMalloc(&out, 8 * 1024); cudaMalloc(&sink, 64);
  long long h[4];
  cudaFuncSetAttribute(k_contend, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int mode : {0, 1, 2, 4, 7, 8, 9, 10, 12, 15}) {
    k_contend<<<1, 384, 140 * 1024>>>(4096, mode, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("mode=%2d (%s%s%s%s): %7.1f clk per chunk\n", mode, mode & 8 ? "2 MMAs/k " : "1 MMA/k ", mode & 1 ? "+LDS " : "",
           mode & 2 ? "+TMEM st " : "", mode & 4 ? "+TMEM ld" : "", double(h[0]) / 4096);
  }
}
