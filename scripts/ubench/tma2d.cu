// Microbenchmark: HBM read bandwidth of TMA tensor (2-D / 3-D box) loads of a
// column-major fp32 matrix (ld = 8192) in the tile order of the tensor-core
// block sweep: per tile of C columns, all K chunks; boxes of 32 floats
// (128 B, SWIZZLE_128B) x C columns x KB k-blocks.  Also varies the ring depth.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/common.cuh"
using namespace gps;

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}

// map dims: (32 floats, n columns, ld/32 k-blocks); box (32, C, KB)
__global__ void __launch_bounds__(128, 1) k_tma3(const __grid_constant__ CUtensorMap map, int ntiles, int kchunks,
                                                 int C, int KB, int S, float* out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t stage = uint32_t(C) * KB * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * stage);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int my = ntiles > int(blockIdx.x) ? (ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int total = my * kchunks;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int slot = 0; uint32_t ph = 0; int t = blockIdx.x, kc = 0;
      for (int c = 0; c < total; ++c) {
        if (c >= S) mbar_wait(&empty[slot], ph ^ 1u);
        mbar_arrive_expect_tx(&full[slot], stage);
        tma3(smem + size_t(slot) * stage, &map, 0, t * C, kc * KB, &full[slot]);
        if (++slot == S) { slot = 0; ph ^= 1u; }
        if (++kc == kchunks) { kc = 0; t += gridDim.x; }
      }
    }
  } else if (warp == 1) {
    float acc = 0.f;
    int slot = 0; uint32_t ph = 0;
    for (int c = 0; c < total; ++c) {
      mbar_wait(&full[slot], ph);
      acc += reinterpret_cast<const float*>(smem + size_t(slot) * stage)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == S) { slot = 0; ph ^= 1u; }
    }
    if (acc == 12345.f) out[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ld = 8192;
  const size_t n = size_t(1) << 19;  // 16 GiB
  float* A; float* out;
  if (cudaMalloc(&A, size_t(ld) * n * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 64);
  cudaMemset(A, 0, size_t(ld) * n * 4);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_tma3, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct V { int C, KB; };
  for (V v : {V{128, 1}, V{64, 2}, V{32, 4}, V{16, 8}, V{8, 16}, V{128, 2}, V{64, 4}, V{32, 8}, V{128, 4}, V{32, 16}}) {
    CUtensorMap map;
    cuuint64_t dims[3] = {32, n, cuuint64_t(ld / 32)};
    cuuint64_t strides[2] = {cuuint64_t(ld) * 4, 128};
    cuuint32_t box[3] = {32, cuuint32_t(v.C), cuuint32_t(v.KB)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed C=%d KB=%d: %d\n", v.C, v.KB, int(r)); continue; }
    const uint32_t stage = uint32_t(v.C) * v.KB * 128;
    const int ntiles = int(n / v.C), kchunks = ld / 32 / v.KB;
    for (int S : {4, 8, 12}) {
      size_t smem = size_t(S) * stage + 16 * S + 1024;
      if (smem > 227 * 1024) continue;
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_tma3<<<sms, 128, smem>>>(map, ntiles, kchunks, v.C, v.KB, S, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("C=%3d KB=%2d (contig %5d B/col) stage=%6u S=%2d: %7.1f GB/s\n", v.C, v.KB, v.KB * 128, stage, S,
             size_t(ld) * n * 4 / (best * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
