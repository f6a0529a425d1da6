// Multi-CTA polar step for large p * m (block.py:135-149 at C3 / C4 sizes).
//
// The one-CTA Householder + Jacobi polar (bk_kernels.cuh) is exact to LAPACK
// grade but latency-bound at p = 8192, m = 64 (tens of ms).  Here the O(p m^2)
// work is spread over the GPU with CholeskyQR2:
//   G = Q1 R1 (Gram of G on many CTAs, m x m Cholesky on one CTA, Q1 = G R1^-1),
//   Q1 = Q R2 (same again), R = R2 R1 = U S V' (one-sided Jacobi on one CTA),
//   X = Q U V' = Q1 (R2^-1 U V').
// The singular values of R carry the rank test of the reference.  When a
// Cholesky breaks down or cond(R) > 1e7 (where CholeskyQR2 would lose the
// accuracy the rank rule needs) the step falls back to the Householder path
// on one CTA, so results keep LAPACK-grade rank decisions in every case.
// All kernels read a device control block; nothing is decided on the host,
// so an iteration stays CUDA-graph capturable.
#pragma once

#include "bk_kernels.cuh"

namespace gps {

struct PolarCtl {
  int active;    // this iteration computes a polar step
  int fallback;  // CholeskyQR2 unusable -> Householder path
  int rank;
  int pad;
};

constexpr int kMaxGramM = 64;
constexpr int kGramBlocks = 64;
constexpr int kGramThreads = 256;
constexpr int kGramRows = 32;  // rows staged in smem per pass

// Head of the block step: history and stopping rule (block.py:211-226).
__global__ void bk_head_kernel(const double* __restrict__ exch, int ng, int mg, int ld, double* __restrict__ hist,
                               GpsCtl* ctl, double tol, int max_iter, PolarCtl* pc, int m) {
  if (threadIdx.x != 0) return;
  if (ctl->done) {
    pc->active = 0;
    return;
  }
  const int k = ctl->iter;
  const size_t gstride = size_t(mg) * ld + 4;
  double f = 0.0;
  for (int g = 0; g < ng; ++g) f += exch[g * gstride + size_t(mg) * ld];
  hist[k] = f;
  const double f_prev = ctl->f_prev;
  int d = 0;
  if (k >= 1 && fabs(f - f_prev) < tol * fmax(fabs(f_prev), 1e-30)) d = 1;
  else if (k >= max_iter) d = 2;
  ctl->f_prev = f;
  if (d != 0) {
    ctl->done = 1;
    ctl->converged = d == 1;
    pc->active = 0;
    return;
  }
  pc->active = 1;
  pc->fallback = 0;
  pc->rank = m;
}

// G[j][r] = 2 mu_j * (reduced sweep partial)  (block.py:119-120)
__global__ void bk_assemble_kernel(const double* __restrict__ exch, int mg, int ld, int m,
                                   const double* __restrict__ mu, double* __restrict__ G, const PolarCtl* pc) {
  if (!pc->active) return;
  const size_t gstride = size_t(mg) * ld + 4;
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < size_t(m) * ld;
       e += size_t(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / ld), r = static_cast<int>(e % ld);
    G[e] = 2.0 * mu[j] * exch[(j / mg) * gstride + size_t(j % mg) * ld + r];
  }
}

// Partial Gram matrices of Y ([m][ld], rows >= p_true zero): block b covers
// a contiguous row range; part[b][a*m + c].  Fixed summation order.
__global__ void __launch_bounds__(kGramThreads) gram_partial_kernel(const double* __restrict__ Y, int ld, int p_true,
                                                                   int m, double* __restrict__ part,
                                                                   const PolarCtl* pc) {
  __shared__ double tile[kGramRows][kMaxGramM + 1];
  if (!pc->active || pc->fallback) return;
  const int rows_per = (p_true + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per;
  const int r1 = min(p_true, r0 + rows_per);
  constexpr int EPT = (kMaxGramM * kMaxGramM + kGramThreads - 1) / kGramThreads;
  double acc[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) acc[i] = 0.0;
  for (int rb = r0; rb < r1; rb += kGramRows) {
    const int nr = min(kGramRows, r1 - rb);
    for (int e = threadIdx.x; e < kGramRows * m; e += kGramThreads) {
      const int rr = e % kGramRows, j = e / kGramRows;
      tile[rr][j] = rr < nr ? Y[size_t(j) * ld + rb + rr] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = threadIdx.x + i * kGramThreads;
      if (e < m * m) {
        const int a = e / m, c = e % m;
        double t = acc[i];
        for (int rr = 0; rr < kGramRows; ++rr) t = fma(tile[rr][a], tile[rr][c], t);
        acc[i] = t;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * kGramThreads;
    if (e < m * m) part[size_t(blockIdx.x) * m * m + e] = acc[i];
  }
}

// In-place Gauss-Jordan inverse with partial pivoting of the m x m
// row-major A (destroyed) into B; fcol: m scratch.  One CTA of 1024 threads,
// m <= 64: thread (i, g) = (tid / 16, tid % 16) owns row i, columns
// g, g + 16, g + 32, g + 48 of both A and B.  Returns false on an exactly
// singular pivot.
__device__ bool gj_inverse(double* A, double* B, double* fcol, int m) {
  const int tid = threadIdx.x;
  const int i = tid >> 4, g = tid & 15;
  __shared__ int s_piv;
  if (i < m)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = g + 16 * k;
      if (c < m) B[i * m + c] = (i == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (tid < 32) {  // pivot: largest |A[r][j]|, r >= j (lowest index on ties)
      double best = -1.0;
      int bi = j;
      for (int r = j + tid; r < m; r += 32) {
        const double v = fabs(A[r * m + j]);
        if (v > best) {
          best = v;
          bi = r;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (tid == 0) s_piv = best > 0.0 ? bi : -1;
    }
    __syncthreads();
    const int pv = s_piv;
    if (pv < 0) return false;
    if (pv != j && tid < 2 * m) {  // swap rows j and pv
      double* X = tid < m ? A : B;
      const int c = tid < m ? tid : tid - m;
      const double t = X[j * m + c];
      X[j * m + c] = X[pv * m + c];
      X[pv * m + c] = t;
    }
    __syncthreads();
    if (tid < m) fcol[tid] = A[tid * m + j];
    __syncthreads();
    const double inv = 1.0 / fcol[j];
    if (tid < 2 * m) {  // normalise the pivot row
      if (tid < m)
        A[j * m + tid] *= inv;
      else
        B[j * m + tid - m] *= inv;
    }
    __syncthreads();
    if (i < m && i != j) {
      const double f = fcol[i];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = g + 16 * k;
        if (c < m) {
          A[i * m + c] = fma(-f, A[j * m + c], A[i * m + c]);
          B[i * m + c] = fma(-f, B[j * m + c], B[i * m + c]);
        }
      }
    }
    __syncthreads();
  }
  return true;
}

// Polar factor of the m x m row-major R by the Frobenius-scaled Newton
// iteration X <- (z X + X^-T / z) / 2 (quadratic convergence; scaling
// dropped once the step is small).  X holds the result; W, Y, fcol, red are
// scratch.  Returns the Frobenius condition estimate |R|_F |R^-1|_F of the
// first step (0 if R is singular).
__device__ double newton_polar(const double* R, double* X, double* W, double* Y, double* fcol, double* red, int m) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < m * m; e += nt) X[e] = R[e];
  __syncthreads();
  double kappa = 0.0;
  bool scale = true;
  for (int it = 0; it < 30; ++it) {
    for (int e = tid; e < m * m; e += nt) W[e] = X[e];
    __syncthreads();
    if (!gj_inverse(W, Y, fcol, m)) return 0.0;  // Y = X^-1
    double a = 0.0, b = 0.0;
    for (int e = tid; e < m * m; e += nt) {
      a = fma(X[e], X[e], a);
      b = fma(Y[e], Y[e], b);
    }
    const double nx = sqrt(block_sum_any(a, red)), ny = sqrt(block_sum_any(b, red));
    if (it == 0) kappa = nx * ny;
    const double z = scale ? sqrt(ny / nx) : 1.0;
    double d = 0.0;
    for (int e = tid; e < m * m; e += nt) {  // X_new = (z X + Y^T / z) / 2
      const int r = e / m, c = e % m;
      const double xn = 0.5 * (z * X[e] + Y[c * m + r] / z);
      d = fma(xn - X[e], xn - X[e], d);
      W[e] = xn;
    }
    const double dn = sqrt(block_sum_any(d, red));
    for (int e = tid; e < m * m; e += nt) X[e] = W[e];
    __syncthreads();
    const double rel = dn / sqrt(double(m));  // |X| -> sqrt(m) at convergence
    if (rel < 1e-2) scale = false;
    if (rel < 1e-14) break;
  }
  return kappa;
}

// Sum the Gram partials (fixed order), Cholesky G'G = R'R (upper R), and
// invert R.  stage 1: R1 -> Rs (R1), Rinv (R1^-1).  stage 2: R2 with R = R2 R1,
// one-sided Jacobi SVD of R, rank, then S = R2^-1 U V' (the right factor of
// X = Q1 S) or the fallback flag.  One CTA; small m x m work in smem.
__global__ void __launch_bounds__(kPolarThreads) chol_stage_kernel(const double* __restrict__ part, int nparts, int m,
                                                                  int p_true, int stage, double* __restrict__ R1g,
                                                                  double* __restrict__ Sg, PolarCtl* pc) {
  extern __shared__ double psm[];
  if (!pc->active || pc->fallback) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* M = psm;              // m*m (row-major a*m+c)
  double* R = psm + m * m;      // m*m upper, row-major R[i*m+j]
  double* Ri = R + m * m;       // m*m inverse
  double* W = Ri + m * m;       // m*m scratch
  double* V = W + m * m;        // m*m scratch
  __shared__ int bad;
  for (int e = tid; e < m * m; e += nt) {
    double t = 0.0;
    for (int b = 0; b < nparts; ++b) t += part[size_t(b) * m * m + e];
    M[e] = t;
    R[e] = 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  double dmax = 0.0;
  for (int j = 0; j < m; ++j) dmax = fmax(dmax, M[j * m + j]);
  for (int j = 0; j < m; ++j) {
    if (tid == 0) {
      const double d = M[j * m + j];
      if (!(d > 1e-28 * dmax) || !(d > 0.0)) bad = 1;
      R[j * m + j] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    if (bad) break;
    const double piv = R[j * m + j];
    for (int c = j + 1 + tid; c < m; c += nt) R[j * m + c] = M[j * m + c] / piv;
    __syncthreads();
    for (int e = tid; e < m * m; e += nt) {
      const int a = e / m, c = e % m;
      if (a > j && c >= a) {
        M[a * m + c] -= R[j * m + a] * R[j * m + c];
        M[c * m + a] = M[a * m + c];
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) pc->fallback = 1;
    return;
  }
  // Ri = R^-1 (upper): column c by back substitution, columns in parallel
  for (int c = tid; c < m; c += nt) {
    for (int i = m - 1; i >= 0; --i) {
      double t = (i == c) ? 1.0 : 0.0;
      for (int k = i + 1; k <= c; ++k) t -= R[i * m + k] * Ri[k * m + c];
      Ri[i * m + c] = (i <= c) ? t / R[i * m + i] : 0.0;
    }
  }
  __syncthreads();
  if (stage == 1) {
    for (int e = tid; e < m * m; e += nt) {
      R1g[e] = R[e];
      Sg[e] = Ri[e];  // apply: Q1 = G R1^-1
    }
    return;
  }
  // stage 2: R = R2 R1 (upper, row-major in W), its polar factor P by the
  // scaled Newton iteration (the CholeskyQR2 path only runs for condition
  // numbers far below the rank cutoff max(p, m) eps, so rank = m here), then
  // S = R2^-1 P, the right factor of X = Q1 S.
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    double t = 0.0;
    for (int k = i; k <= j; ++k) t += R[i * m + k] * R1g[k * m + j];
    W[e] = (i <= j) ? t : 0.0;
  }
  __syncthreads();
  __shared__ double red[40];
  __shared__ double fcol[kMaxGramM];
  // M (m*m) receives P; V and R serve as scratch (R2 itself is no longer
  // needed: Ri = R2^-1 is kept)
  const double kappa = newton_polar(W, M, V, R, fcol, red, m);
  __syncthreads();
  if (!(kappa > 0.0) || kappa > 1e7 * sqrt(double(m))) {  // CholeskyQR2 too inaccurate: exact path decides
    if (tid == 0) pc->fallback = 1;
    return;
  }
  if (tid == 0) pc->rank = m;
  for (int e = tid; e < m * m; e += nt) {  // S = Ri (R2^-1) * P
    const int r = e / m, c = e % m;
    double t = 0.0;
    for (int k = r; k < m; ++k) t += Ri[r * m + k] * M[k * m + c];
    Sg[e] = t;
  }
}

// Out[j][r] = sum_b In[b][r] * S[b][j]   (In, Out: [m][ld]; S row-major m x m)
__global__ void __launch_bounds__(256) apply_right_kernel(const double* __restrict__ In, const double* __restrict__ S,
                                                          int ld, int m, double* Out, const PolarCtl* pc,
                                                          const GpsCtl* ctl, int64_t out_par_stride) {
  __shared__ double s[kMaxGramM * kMaxGramM];
  if (!pc->active || pc->fallback) return;
  double* O = Out + (ctl != nullptr ? ((ctl->iter + 1) & 1) * out_par_stride : 0);
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) s[e] = S[e];
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < ld; r += gridDim.x * blockDim.x) {
    double in[kMaxGramM];
    for (int b = 0; b < m; ++b) in[b] = In[size_t(b) * ld + r];
    for (int j = 0; j < m; ++j) {
      double t = 0.0;
      for (int b = 0; b < m; ++b) t = fma(in[b], s[b * m + j], t);
      O[size_t(j) * ld + r] = t;
    }
  }
}

// Fallback (exact Householder + Jacobi, one CTA) and the step's finish:
// rank failure stops the loop (block.py:215-218), else the iterate advances.
__global__ void __launch_bounds__(kPolarThreads) bk_finish_kernel(double* G, double* Xbuf, int64_t x_stride, int ld,
                                                                 int p_true, int m, GpsCtl* ctl, PolarCtl* pc,
                                                                 int* rank_out) {
  extern __shared__ double psm[];
  if (!pc->active) return;
  const int k = ctl->iter;
  int rank = pc->rank;
  if (pc->fallback) rank = polar_device(G, Xbuf + ((k + 1) & 1) * x_stride, ld, p_true, m, polar_scratch(psm, m));
  if (threadIdx.x == 0) {
    if (rank < m) {
      ctl->done = 1;
      ctl->converged = 0;
      ctl->status = 2;
      *rank_out = rank;
    } else {
      ctl->iter = k + 1;
    }
  }
}

__host__ __device__ inline size_t chol_smem_bytes(int m) { return size_t(5) * m * m * sizeof(double) + 64; }

}  // namespace gps
