// Microbenchmark: issue throughput of the per-element instructions of the
// fused sweep on this B200 (F2F.F64.F32, DFMA, bit-trick conversion, FFMA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_f2f(const float* in, double* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = in[threadIdx.x * 8 + i];
  double acc[8] = {0};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += (double)v[i]; v[i] = __int_as_float(__float_as_int(v[i]) ^ 1); }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(const double* in, double* out) {
  double a[8], x = in[0];
  for (int i = 0; i < 8; ++i) a[i] = in[threadIdx.x + i];
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], x, 0.5);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ double bits_f2d(float f) {
  uint32_t u = __float_as_uint(f);
  uint32_t t = u & 0x7fffffffu;
  uint32_t hi = ((t >> 3) + 0x38000000u) | (u & 0x80000000u);
  hi = t ? hi : (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}

__global__ void k_bits(const float* in, double* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = in[threadIdx.x * 8 + i];
  double acc[8] = {0};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += bits_f2d(v[i]); v[i] = __int_as_float(__float_as_int(v[i]) ^ 1); }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_f2f_fma(const float* in, double* out) {  // F2F + DFMA per element (the sweep's inner op)
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = in[threadIdx.x * 8 + i];
  double acc[8] = {0}, x = 0.7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] = fma((double)v[i], x, acc[i]); v[i] = __int_as_float(__float_as_int(v[i]) ^ 1); }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_bits_fma(const float* in, double* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = in[threadIdx.x * 8 + i];
  double acc[8] = {0}, x = 0.7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] = fma(bits_f2d(v[i]), x, acc[i]); v[i] = __int_as_float(__float_as_int(v[i]) ^ 1); }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// no zero handling (columns flagged all-normal by the norms pass), shift+add as IMAD.HI
__device__ __forceinline__ double bits2_f2d(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t hi = (__umulhi(u & 0x7fffffffu, 1u << 29) + 0x38000000u) | (u & 0x80000000u);
  return __hiloint2double((int)hi, (int)(u << 29));
}

__global__ void k_bits2_fma(const float* in, double* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = in[threadIdx.x * 8 + i];
  double acc[8] = {0}, x = 0.7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] = fma(bits2_f2d(v[i]), x, acc[i]); v[i] = __int_as_float(__float_as_int(v[i]) ^ 1); }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the elements through F2F (XU pipe), half through the integer trick
__global__ void k_mix_fma(const float* in, double* out) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = in[threadIdx.x * 8 + i];
  double acc[8] = {0}, x = 0.7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double d = (i & 1) ? bits2_f2d(v[i]) : (double)v[i];
      acc[i] = fma(d, x, acc[i]);
      v[i] = __int_as_float(__float_as_int(v[i]) ^ 1);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename T>
void run(const char* name, void (*kern)(const T*, double*), const void* in, double* out, int threads, int sms,
         double ops_per_thread_iter) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<<<sms * 2, threads>>>((const T*)in, out);
  cudaEventRecord(a);
  kern<<<sms * 2, threads>>>((const T*)in, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = double(sms) * 2 * threads * ITERS * ops_per_thread_iter;
  printf("%-10s %8.3f ms  %8.1f Gop/s  %6.1f op/clk/SM (at %d MHz)\n", name, ms, ops / ms / 1e6,
         ops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* fin; double* din; double* out;
  cudaMalloc(&fin, 1 << 20); cudaMalloc(&din, 1 << 20); cudaMalloc(&out, 1 << 24);
  cudaMemset(fin, 0, 1 << 20); cudaMemset(din, 0, 1 << 20);
  for (int threads : {256, 512, 1024}) {
    printf("threads/CTA=%d, 2 CTAs/SM\n", threads);
    run("F2F", k_f2f, fin, out, threads, sms, 8);
    run("DFMA", k_dfma, din, out, threads, sms, 8);
    run("bits", k_bits, fin, out, threads, sms, 8);
    run("F2F+DFMA", k_f2f_fma, fin, out, threads, sms, 8);
    run("bits+DFMA", k_bits_fma, fin, out, threads, sms, 8);
    run("bits2+DFMA", k_bits2_fma, fin, out, threads, sms, 8);
    run("mix+DFMA", k_mix_fma, fin, out, threads, sms, 8);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
