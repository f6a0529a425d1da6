// Wide-p fallback for the sweeps: any p (the fused kernels keep a column's
// rows in registers and cover p <= 8192 fp32 / 4096 fp64).  Two passes
// with the SAME outputs as K1 / K1b (part_g, part_s, c / w):
//   W1: warp per column, fp64 dots against x (or the MG components of X)
//       read through L1/L2, threshold / objective, weights to a scratch
//       vector; per-CTA scalar partials in a fixed order.
//   W2: for every column with a nonzero weight, all threads of a CTA add
//       w * a_i over a 2048-row chunk into register-resident fp64 partials.
// A is read once by W1 plus once more for the ACTIVE columns only.
#pragma once

#include "su_kernels.cuh"

namespace gps {

constexpr int kWideThreads = 256;
constexpr int kWideRows = 2048;  // row chunk of W2 (8 rows per thread)

// W1 for up to MG components; comp_stride: distance between components in
// X / W / wbuf (MG == 1 is the single-unit case with gamma[0], mu[0] = 1).
struct WideParams {
  double gamma[4];
  double mu[4];
  BandLog* band;  // near-threshold log (kFused loops), component index comp0 + j
  int comp0;
};

template <typename TA, int MG>
__global__ void __launch_bounds__(kWideThreads) wide_dots_kernel(
    const TA* __restrict__ A, int64_t n, int ld, int p, int mode, int penalty, const double* __restrict__ X,
    int64_t x_cstride, const double* __restrict__ coef, int coef_threshold, const WideParams prm,
    double* __restrict__ wbuf, double* __restrict__ c_out, double* __restrict__ w_out, int64_t w_cstride,
    double* __restrict__ part_s, const GpsCtl* ctl, int64_t x_par_stride, int64_t w_par_stride) {
  const double* gamma = prm.gamma;
  const double* mu = prm.mu;
  __shared__ double sred[kWideThreads / 32][3];
  if (ctl != nullptr && ctl->done) return;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const double* Xp = X + parity * x_par_stride;
  double* wo = w_out != nullptr ? w_out + parity * w_par_stride : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  double f_acc = 0.0, nnz_acc = 0.0, s2_acc = 0.0;
  for (int64_t col = c0 + warp; col < c1; col += kWideThreads / 32) {
    double c[MG];
    if (mode == kCoef) {
      c[0] = coef[col];
    } else {
      const TA* a = A + col * ld;
#pragma unroll
      for (int j = 0; j < MG; ++j) c[j] = 0.0;
      for (int r = lane; r < p; r += 32) {
        const double v = static_cast<double>(a[r]);
#pragma unroll
        for (int j = 0; j < MG; ++j) c[j] = fma(v, Xp[j * x_cstride + r], c[j]);
      }
#pragma unroll
      for (int j = 0; j < MG; ++j) c[j] = warp_sum(c[j]);
    }
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      double w;
      if (mode == kCoef) {
        w = coef_threshold ? threshold_weight(c[0], gamma[0], penalty) : c[0];
      } else {
        const double s = mu[j] * c[j];
        if (mode == kFused && lane == 0) band_note(prm.band, parity, col, prm.comp0 + j, s, gamma[j], penalty);
        f_acc += objective_term(s, gamma[j], penalty);
        w = mode == kFused ? threshold_weight(s, gamma[j], penalty) : 0.0;
      }
      if (w != 0.0) {
        nnz_acc += 1.0;
        s2_acc = fma(w, w, s2_acc);
      }
      if (lane == 0) {
        wbuf[j * w_cstride + col] = w;
        if (c_out != nullptr && j == 0 && mode != kCoef) c_out[col] = c[0];
        if (wo != nullptr) wo[j * w_cstride + col] = w;
      }
      if (mode == kCoef) break;
    }
  }
  if (lane == 0) {
    sred[warp][0] = f_acc;
    sred[warp][1] = nnz_acc;
    sred[warp][2] = s2_acc;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < kWideThreads / 32; ++w) t += sred[w][threadIdx.x];
    part_s[size_t(blockIdx.x) * 4 + threadIdx.x] = t;
  }
}

// W2: grid (G, ceil(ld / kWideRows)); CTA (b, y) owns the columns of W1's CTA
// b and the rows [y*kWideRows, ...) of part_g[b] ([MG][ld] per CTA).
template <typename TA, int MG>
__global__ void __launch_bounds__(kWideThreads) wide_accum_kernel(const TA* __restrict__ A, int64_t n, int ld,
                                                                  const double* __restrict__ wbuf, int64_t w_cstride,
                                                                  double* __restrict__ part_g, const GpsCtl* ctl) {
  constexpr int RPT = kWideRows / kWideThreads;
  if (ctl != nullptr && ctl->done) return;
  const int64_t c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  const int r0 = blockIdx.y * kWideRows;
  double g[MG][RPT];
#pragma unroll
  for (int j = 0; j < MG; ++j)
#pragma unroll
    for (int k = 0; k < RPT; ++k) g[j][k] = 0.0;
  for (int64_t col = c0; col < c1; ++col) {
    double w[MG];
    bool any = false;
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      w[j] = wbuf[j * w_cstride + col];
      any |= w[j] != 0.0;
    }
    if (!any) continue;
    const TA* a = A + col * ld;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = r0 + k * kWideThreads + threadIdx.x;
      const double v = r < ld ? static_cast<double>(a[r]) : 0.0;
#pragma unroll
      for (int j = 0; j < MG; ++j) g[j][k] = fma(w[j], v, g[j][k]);
    }
  }
  double* pg = part_g + size_t(blockIdx.x) * MG * ld;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = r0 + k * kWideThreads + threadIdx.x;
    if (r < ld)
#pragma unroll
      for (int j = 0; j < MG; ++j) pg[size_t(j) * ld + r] = g[j][k];
  }
}

}  // namespace gps
