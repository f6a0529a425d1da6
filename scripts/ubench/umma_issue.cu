// Microbenchmark: single-thread vs warp-converged (elect.sync) issue of
// tcgen05.mma + commit + mbarrier probes per 4-MMA chunk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/tc_kernels.cuh"
using namespace gps;

__device__ __forceinline__ void umma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
  return e != 0;
}

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int MODE>
__global__ void k_issue(int N, int iters, int nslots, long long* out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[16];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t idesc = umma_idesc_tf32(128, N);
  const uint64_t da = umma_desc_sw128(smem), db = umma_desc_sw128(smem + 32768);
  if (MODE == 0 ? threadIdx.x == 0 : threadIdx.x < 32) {
    long long t0 = clock64();
    int slot = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      // wait for the commit of the chunk issued nslots chunks ago (ring reuse)
      if (it >= nslots) mbar_wait(&bar[slot], ph ^ 1u);
      tc_fence_after();
      const uint64_t a0 = da + uint64_t(slot) * 64, b0 = db + uint64_t(slot) * 32;
      if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_tf32(tm, a0 + 2 * k, b0 + 2 * k, idesc, (it | k) ? 1u : 0u);
        umma_commit(&bar[slot]);
      } else if (MODE == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_elect(tm, a0 + 2 * k, b0 + 2 * k, idesc, (it | k) ? 1u : 0u);
        commit_elect(&bar[slot]);
      } else if (MODE == 3) {
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_ts(tm, tm + 256 + 8 * k, b0 + 2 * k, idesc, (it | k) ? 1u : 0u);
        commit_elect(&bar[slot]);
      } else {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_tf32(tm, a0 + 2 * k, b0 + 2 * k, idesc, (it | k) ? 1u : 0u);
          umma_commit(&bar[slot]);
        }
        __syncwarp();
      }
      if (++slot == nslots) {
        slot = 0;
        ph ^= 1u;
      }
    }
    if (MODE == 0 || threadIdx.x == 0) {
      umma_commit(&bar[15]);
      mbar_wait(&bar[15], 0);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main() {
  long long* out; cudaMalloc(&out, 8 * 1024);
  long long h[4];
  void (*ks[4])(int, int, int, long long*) = {k_issue<0>, k_issue<1>, k_issue<2>, k_issue<3>};
  const char* nm[4] = {"thread0", "elect-in-asm", "if(elect)", "A-in-TMEM"};
  for (int m = 0; m < 4; ++m) cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {32, 64, 128, 256}) {
    for (int m = 1; m < 4; m += 2) {
      for (int ns : {4}) {
        const int iters = 4096;
        ks[m]<<<1, 128, 100 * 1024>>>(N, iters, ns, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d %-13s slots=%d: %7.1f clk per 4-MMA chunk (tensor floor %d)\n", N, nm[m], ns, double(h[0]) / iters,
               4 * (N <= 64 ? 48 : N / 2));
      }
    }
  }
}
