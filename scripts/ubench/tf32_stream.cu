// Experiment: can a block-sweep filter that feeds fp32 A straight from the
// TMA slot into tcgen05.mma kind::tf32 (no converter warps, no TMEM A
// stores) stream A faster than T1's fp16 path (6.6-6.9 TB/s)?  Same tile
// order and boxes as T1 (128 columns x 32 fp32 rows, SWIZZLE_128B, two boxes
// per 64-row chunk), X as fp32 boxes (N rows x 32), MMAs M = 128, K = 8,
// N = NX; the A / X slots are released by tcgen05.commit; an "epilogue"
// warp group drains the accumulator every SEG chunks (tcgen05.ld, as T1).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tf32_stream.cu -o tf32_stream -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/tc_kernels.cuh"
using namespace gps;

constexpr int kThreads = 256;

// warp-converged issue (elect.sync inside the asm, as T1 does)
__device__ __forceinline__ void umma_tf32_warp(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}  // w0 A producer, w1 MMA, w2 X producer, w4-7 epilogue

__global__ void __launch_bounds__(kThreads, 1) k_tf32(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmX, int ntiles,
                                                      int kchunks, int NX, int SA, int SX, int SEG, float* out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = 2 * 16384;         // two boxes of 128 x 128 B
  const uint32_t x_bytes = 2 * NX * 128;      // two boxes of NX x 128 B
  unsigned char* aring = smem;
  unsigned char* xring = aring + size_t(SA) * a_bytes;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(xring + size_t(SX) * x_bytes);
  uint64_t* a_empty = a_full + SA;
  uint64_t* x_full = a_empty + SA;
  uint64_t* x_empty = x_full + SX;
  uint64_t* tfull = x_empty + SX;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < SX; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int my = ntiles > int(blockIdx.x) ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int total = my * kchunks;
  if (warp == 0) {
    if (lane == 0) {
      int slot = 0; uint32_t ph = 0; int t = blockIdx.x, kc = 0;
      for (int c = 0; c < total; ++c) {
        if (c >= SA) mbar_wait(&a_empty[slot], ph ^ 1u);
        mbar_arrive_expect_tx(&a_full[slot], a_bytes);
        for (int b = 0; b < 2; ++b)
          tma_load_2d(aring + size_t(slot) * a_bytes + b * 16384, &tmA, kc * 64 + b * 32, t * 128, &a_full[slot]);
        if (++slot == SA) { slot = 0; ph ^= 1u; }
        if (++kc == kchunks) { kc = 0; t += gridDim.x; }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      int slot = 0; uint32_t ph = 0; int kc = 0;
      for (int c = 0; c < total; ++c) {
        if (c >= SX) mbar_wait(&x_empty[slot], ph ^ 1u);
        mbar_arrive_expect_tx(&x_full[slot], x_bytes);
        for (int b = 0; b < 2; ++b)
          tma_load_2d(xring + size_t(slot) * x_bytes + b * NX * 128, &tmX, kc * 64 + b * 32, 0, &x_full[slot]);
        if (++slot == SX) { slot = 0; ph ^= 1u; }
        if (++kc == kchunks) kc = 0;
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = umma_idesc_tf32(128, NX);
    int sa = 0, sx = 0; uint32_t pa = 0, px = 0; int seg = 0;
    for (int tt = 0; tt < my; ++tt)
      for (int k0 = 0; k0 < kchunks; k0 += SEG, ++seg) {
        const int b = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[b], uint32_t(((seg - 2) >> 1) & 1));
        tc_fence_after();
        const int k1 = k0 + SEG < kchunks ? k0 + SEG : kchunks;
        for (int kc = k0; kc < k1; ++kc) {
          mbar_wait(&a_full[sa], pa);
          mbar_wait(&x_full[sx], px);
          tc_fence_after();
          for (int bx = 0; bx < 2; ++bx) {
            const uint64_t da = umma_desc_sw128(aring + size_t(sa) * a_bytes + bx * 16384);
            const uint64_t dx = umma_desc_sw128(xring + size_t(sx) * x_bytes + bx * NX * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // K = 8 tf32 = 32 B per MMA
              const uint32_t acc = (kc == k0 && bx == 0 && k == 0) ? 0u : 1u;
              umma_tf32_warp(tmem + uint32_t(b * NX), da + 2 * k, dx + 2 * k, idesc, acc);
            }
          }
          umma_commit_warp(&a_empty[sa]);
          umma_commit_warp(&x_empty[sx]);
          if (kc == k1 - 1) umma_commit_warp(&tfull[b]);
          if (++sa == SA) { sa = 0; pa ^= 1u; }
          if (++sx == SX) { sx = 0; px ^= 1u; }
        }
      }
  } else if (warp >= 4) {
    const int q = warp & 3;
    float acc = 0.f;
    int seg = 0;
    for (int tt = 0; tt < my; ++tt)
      for (int k0 = 0; k0 < kchunks; k0 += SEG, ++seg) {
        const int b = seg & 1;
        mbar_wait_sleep(&tfull[b], uint32_t((seg >> 1) & 1));
        tc_fence_after();
        for (int j = 0; j < NX; j += 8) {
          float v[8];
          tmem_ld8(tmem + (uint32_t(q * 32) << 16) + uint32_t(b * NX + j), v);
          tmem_wait_ld();
          for (int u = 0; u < 8; ++u) acc += v[u];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
    if (acc == 1234.5f) out[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ld = 8192;
  const size_t n = size_t(1) << 20;  // 32 GiB fp32
  float *A, *X, *out;
  if (cudaMalloc(&A, size_t(ld) * n * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&X, size_t(ld) * 128 * 4);
  cudaMalloc(&out, 64);
  cudaMemset(A, 0, size_t(ld) * n * 4);
  cudaMemset(X, 0, size_t(ld) * 128 * 4);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &qr);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int NX : {32, 128}) {
    CUtensorMap ma, mx;
    cuuint64_t da[2] = {cuuint64_t(ld), n}, sa[1] = {cuuint64_t(ld) * 4};
    cuuint32_t ba[2] = {32, 128}, es[2] = {1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t dx[2] = {cuuint64_t(ld), cuuint64_t(NX)}, sx[1] = {cuuint64_t(ld) * 4};
    cuuint32_t bx[2] = {32, cuuint32_t(NX)};
    enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dx, sx, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int SA : {4, 5, 6}) {
      const int SX = 3, SEG = 4;
      const size_t smem = size_t(SA) * 32768 + size_t(SX) * 2 * NX * 128 + 1024 + 512;
      if (smem > 227 * 1024) continue;
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_tf32<<<sms, kThreads, smem>>>(ma, mx, int(n / 128), ld / 64, NX, SA, SX, SEG, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("NX=%3d SA=%d: %.3f ms  %7.1f GB/s  (%s)\n", NX, SA, best, size_t(ld) * n * 4 / (best * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
