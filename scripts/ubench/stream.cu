// Microbenchmark: HBM read bandwidth of bulk-async (TMA 1-D) streaming into an
// S-deep shared-memory ring vs plain LDG streaming, over a 16 GiB buffer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1312_6182_b200/csrc/common.cuh"
using namespace gps;

__global__ void __launch_bounds__(288, 1) k_tma(const unsigned char* A, size_t total, uint32_t stage, int S, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(S) * stage);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nst = total / stage;
  const size_t b0 = nst * blockIdx.x / gridDim.x, b1 = nst * (blockIdx.x + 1) / gridDim.x;
  const int ns = int(b1 - b0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int slot = 0; uint32_t ph = 0;
      for (int s = 0; s < ns; ++s) {
        if (s >= S) mbar_wait(&empty[slot], ph);
        mbar_arrive_expect_tx(&full[slot], stage);
        bulk_g2s(smem + size_t(slot) * stage, A + (b0 + s) * stage, stage, &full[slot], pol);
        if (++slot == S) { slot = 0; if (s >= S) ph ^= 1; }
      }
    }
    return;
  }
  float acc = 0.f;
  int slot = 0; uint32_t ph = 0;
  for (int s = 0; s < ns; ++s) {
    mbar_wait(&full[slot], ph);
    acc += reinterpret_cast<const float*>(smem + size_t(slot) * stage)[threadIdx.x];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == S) { slot = 0; ph ^= 1; }
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_ldg(const float4* A, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t j = i + size_t(u) * gridDim.x * blockDim.x;
      v[u] = j < n4 ? __ldcs(A + j) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(16) << 30;
  unsigned char* A; float* out;
  if (cudaMalloc(&A, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 64);
  cudaMemset(A, 0, total);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (uint32_t stage : {8192u, 16384u, 32768u, 65536u}) {
    for (int S : {2, 3, 4, 6, 8, 12, 16, 24}) {
      size_t smem = size_t(S) * stage + 16 * S;
      if (smem > 227 * 1024) continue;
      float best = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k_tma<<<sms, 288, smem>>>(A, total, stage, S, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("tma stage=%6u S=%2d inflight=%7zu B: %7.1f GB/s\n", stage, S, size_t(S) * stage, total / (best * 1e-3) / 1e9);
    }
  }
  for (int bpsm : {4, 8, 16}) {
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      k_ldg<<<sms * bpsm, 256>>>(reinterpret_cast<const float4*>(A), total / 16, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("ldg blocks/SM=%2d: %7.1f GB/s\n", bpsm, total / (best * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
