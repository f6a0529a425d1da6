// Phase timing of the one-CTA polar stage pieces (m = 64, 1024 threads) with
// clock64 stamps instead of printf: mm_small, the Newton-Schulz loop, and the
// pieces of chol_stage_kernel are timed in isolation on a synthetic
// well-conditioned upper-triangular R.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I ../../paper_1312_6182_b200/csrc polar_ns.cu -o polar_ns
#include <cstdio>
#include <vector>

#define GPS_POLAR_STAMPS
#include "polar_kernels.cuh"

using namespace gps;

__global__ void __launch_bounds__(kPolarThreads) probe(const double* Rin, int m, long long* stamps, double* out) {
  extern __shared__ double sm[];
  const int ld = ns_ld(m);
  double* X = sm;  // row stride ld for the products, m for newton_schulz_polar
  double* T = X + m * ld;
  double* U = T + m * ld;
  double* ws = U + m * ld;
  __shared__ double red[40];
  const int tid = threadIdx.x;
  for (int e = tid; e < m * m; e += blockDim.x) X[(e / m) * ld + e % m] = Rin[e];
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < 10; ++r) {
    mm_small(X, X, T, m, ld, true);
    __syncthreads();
  }
  long long t1 = clock64();
  for (int r = 0; r < 10; ++r) {
    mm_small(X, T, U, m, ld, false);
    __syncthreads();
  }
  long long t2 = clock64();
  double d = 0.0;
  for (int r = 0; r < 10; ++r) d += block_sum_any(double(tid), red);
  long long t3 = clock64();
  for (int e = tid; e < m * m; e += blockDim.x) X[e] = Rin[e];
  __syncthreads();
  long long t4 = clock64();
  const bool ok = newton_schulz_polar(X, ws, red, m, 100);
  __syncthreads();
  long long t5 = clock64();
  if (tid == 0) {
    stamps[0] = t1 - t0;
    stamps[1] = t2 - t1;
    stamps[2] = t3 - t2;
    stamps[3] = t5 - t4;
    stamps[4] = ok;
    out[0] = d;
  }
}

int main() {
  const int m = 64;
  std::vector<double> R(m * m, 0.0);
  unsigned s = 12345;
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) {
      s = s * 1664525u + 1013904223u;
      R[i * m + j] = (i == j) ? 1.0 + 0.1 * i : 0.05 * (double(s >> 8) / double(1 << 24) - 0.5);
    }
  double *dR, *dout;
  long long* dst;
  cudaMalloc(&dR, m * m * 8);
  cudaMalloc(&dout, 8);
  cudaMalloc(&dst, 8 * 8);
  cudaMemcpy(dR, R.data(), m * m * 8, cudaMemcpyHostToDevice);
  const int smem = 6 * m * ns_ld(m) * 8;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<<<1, kPolarThreads, smem>>>(dR, m, dst, dout);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long st[5];
    cudaMemcpy(st, dst, sizeof(st), cudaMemcpyDeviceToHost);
    printf("kernel %.1f us | mm_small(ta) %lld clk, mm_small %lld clk, block_sum %lld clk (per call), NS %lld clk ok=%lld\n",
           ms * 1e3, st[0] / 10, st[1] / 10, st[2] / 10, st[3], st[4]);
  }
  // the real stage kernels on the Gram R'R (nparts = 1), event-timed
  std::vector<double> Gm(m * m, 0.0);
  for (int a = 0; a < m; ++a)
    for (int c = 0; c < m; ++c) {
      double t = 0.0;
      for (int k = 0; k < m; ++k) t += R[k * m + a] * R[k * m + c];
      Gm[a * m + c] = t;
    }
  double *dG, *dR1, *dS;
  PolarCtl* pc;
  cudaMalloc(&dG, m * m * 8);
  cudaMalloc(&dR1, m * m * 8);
  cudaMalloc(&dS, m * m * 8);
  cudaMalloc(&pc, sizeof(PolarCtl));
  cudaMemcpy(dG, Gm.data(), m * m * 8, cudaMemcpyHostToDevice);
  // stage 2 factors the Gram of Q1 = G R1^-1, I + E with |E| ~ kappa^2 u
  std::vector<double> G2(m * m, 0.0);
  for (int a = 0; a < m; ++a)
    for (int c = a; c < m; ++c) {
      s = s * 1664525u + 1013904223u;
      const double e = 1e-7 * (double(s >> 8) / double(1 << 24) - 0.5);
      G2[a * m + c] += e;
      if (c != a) G2[c * m + a] += e;
    }
  for (int a = 0; a < m; ++a) G2[a * m + a] += 1.0;
  double* dG2;
  cudaMalloc(&dG2, m * m * 8);
  cudaMemcpy(dG2, G2.data(), m * m * 8, cudaMemcpyHostToDevice);
  const int ssm = int(chol_smem_bytes(m));
  cudaFuncSetAttribute(chol_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm);
  for (int rep = 0; rep < 3; ++rep)
    for (int stage = 1; stage <= 2; ++stage) {
      PolarCtl h{1, 0, 0, 0};
      cudaMemcpy(pc, &h, sizeof(h), cudaMemcpyHostToDevice);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      chol_stage_kernel<<<1, kPolarThreads, ssm>>>(stage == 1 ? dG : dG2, 1, m, 8192, stage, dR1, dS, pc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(&h, pc, sizeof(h), cudaMemcpyDeviceToHost);
      long long ps[8];
      cudaMemcpyFromSymbol(ps, g_polar_stamps, sizeof(ps));
      printf("chol_stage %d: %.1f us fallback=%d rank=%d | partials %lld, cholesky %lld, inverse %lld clk", stage, ms * 1e3,
             h.fallback, h.rank, ps[1] - ps[0], ps[2] - ps[1], ps[3] - ps[2]);
      if (stage == 2) printf(", R2R1 %lld, NS %lld clk", ps[4] - ps[3], ps[5] - ps[4]);
      printf(", tail %lld, total %lld clk", ps[6] - (stage == 2 ? ps[5] : ps[3]), ps[6] - ps[0]);
      if (stage == 1) printf(" (kappa %lld)", ps[7] - ps[3]);
      printf("\n");
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
