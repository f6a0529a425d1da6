// Multi-CTA polar step for large p * m (block.py:135-149 at C3 / C4 sizes).
//
// The one-CTA Householder + Jacobi polar (bk_kernels.cuh) is exact to LAPACK
// grade but latency-bound at p = 8192, m = 64 (tens of ms).  Here the O(p m^2)
// work is spread over the GPU with CholeskyQR2:
//   G = Q1 R1 (Gram of G on many CTAs, m x m Cholesky on one CTA, Q1 = G R1^-1),
//   Q1 = Q R2 (same again), R = R2 R1 = U S V' (one-sided Jacobi on one CTA),
//   X = Q U V' = Q1 (R2^-1 U V').
// The singular values of R carry the rank test of the reference.  When a
// Cholesky breaks down, kappa_F(R1) > 1e5, R2 strays from I, or the new
// iterate misses the Stiefel tolerance (checked on its Gram), the step falls
// back to the Householder path on one CTA, so results keep LAPACK-grade rank
// decisions and every kept iterate is a valid StiefelPoint.
// All kernels read a device control block; nothing is decided on the host,
// so an iteration stays CUDA-graph capturable.
#pragma once

#include "bk_kernels.cuh"

namespace gps {

// Phase clock stamps of chol_stage_kernel for scripts/ubench (diagnostics
// builds only).
#ifdef GPS_POLAR_STAMPS
__device__ long long g_polar_stamps[8];
#define GPS_STAMP(i)                                   \
  do {                                                 \
    if (threadIdx.x == 0) g_polar_stamps[i] = clock64(); \
  } while (0)
#else
#define GPS_STAMP(i) \
  do {               \
  } while (0)
#endif

struct PolarCtl {
  int active;       // this iteration computes a polar step
  int fallback;     // CholeskyQR2 unusable -> Householder path
  int rank;
  int exact_steps;  // diagnostics: steps the exact path took (cumulative)
  int ns_iters;     // diagnostics: Newton-Schulz iterations of the CholeskyQR2 path (cumulative)
};

constexpr int kMaxGramM = 64;
constexpr int kGramBlocks = 64;
constexpr int kGramThreads = 256;
constexpr int kGramRows = 32;  // rows staged in smem per pass
// CholeskyQR2 trust region: kappa_F(R1) = |R1|_F |R1^-1|_F <= 1e5 keeps the
// first pass's loss of orthogonality (~kappa^2 u) near 1e-6, which the
// second pass removes; beyond it, or when R2 strays from I by more than
// 1e-4 (stage 2), the exact Householder + Jacobi path takes the step.
constexpr double kCholQr2MaxKappa = 1e5;
constexpr double kCholQr2MaxR2Dev = 1e-4;

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
  // grid (row blocks of 4 x blockDim, components): no index division per element
  const int j = blockIdx.y;
  if (j >= m) return;
  const double s = 2.0 * mu[j];
  const double* src = exch + (j / mg) * gstride + size_t(j % mg) * ld;
  double* dst = G + size_t(j) * ld;
  const int r0 = blockIdx.x * 4 * blockDim.x + threadIdx.x;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r0 + u * blockDim.x;
    if (r < ld) dst[r] = s * src[r];
  }
}

// Partial Gram matrices of Y ([m][ld], rows >= p_true zero): block b covers
// a contiguous row range; part[b][a*m + c].  On the fp64 tensor cores: the
// CTA stages 32 rows of all components at a time (k-contiguous, row stride
// 36 = 4 mod 16 doubles: conflict-free stores and fragment loads; the next
// stage's loads are issued before the current stage's DMMAs) and warp w
// accumulates output tile row w (components 8w .. 8w + 7) against every tile
// column with m8n8k4 DMMA.  Fixed summation order.
// With ctl given, Y is the parity slot the step is writing (X_{k+1}).
constexpr int kGramKS = kGramRows + 4;
__global__ void __launch_bounds__(kGramThreads) gram_partial_kernel(const double* __restrict__ Y, int ld, int p_true,
                                                                   int m, double* __restrict__ part,
                                                                   const PolarCtl* pc, const GpsCtl* ctl = nullptr,
                                                                   int64_t par_stride = 0) {
  __shared__ double tile[2][kMaxGramM * kGramKS];
  if (!pc->active || pc->fallback) return;
  if (ctl != nullptr) Y += ((ctl->iter + 1) & 1) * par_stride;
  const int rows_per = (p_true + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per;
  const int r1 = min(p_true, r0 + rows_per);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int nt = (m + 7) >> 3;  // 8 x 8 tiles per dimension
  constexpr int EPT = kGramRows * kMaxGramM / kGramThreads;  // staged values per thread
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  double rv[EPT];
  auto load = [&](int rb) {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = tid + kGramThreads * i, rr = e % kGramRows, j = e / kGramRows;
      rv[i] = (rb + rr < r1 && j < m) ? Y[size_t(j) * ld + rb + rr] : 0.0;
    }
  };
  if (r0 < r1) load(r0);
  int buf = 0;
  for (int rb = r0; rb < r1; rb += kGramRows, buf ^= 1) {
    double* tl = tile[buf];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int e = tid + kGramThreads * i, rr = e % kGramRows, j = e / kGramRows;
      tl[j * kGramKS + rr] = rv[i];
    }
    __syncthreads();
    if (rb + kGramRows < r1) load(rb + kGramRows);
    if (warp < nt) {
#pragma unroll
      for (int k0 = 0; k0 < kGramRows; k0 += 4) {
        const double a = tl[(warp * 8 + g) * kGramKS + k0 + t];
#pragma unroll
        for (int tj = 0; tj < 8; ++tj)
          if (tj < nt) {
            const double b = tl[(tj * 8 + g) * kGramKS + k0 + t];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[tj][0]), "+d"(acc[tj][1])
                         : "d"(a), "d"(b));
          }
      }
    }
    // no trailing barrier: buffer buf is rewritten two stages later, after
    // the next stage's barrier
  }
  if (warp < nt) {
    const int a_row = warp * 8 + g;
#pragma unroll
    for (int tj = 0; tj < 8; ++tj) {
      const int c = tj * 8 + 2 * t;
      if (tj < nt && a_row < m) {
        if (c < m) part[size_t(blockIdx.x) * m * m + a_row * m + c] = acc[tj][0];
        if (c + 1 < m) part[size_t(blockIdx.x) * m * m + a_row * m + c + 1] = acc[tj][1];
      }
    }
  }
}

// Row stride of the Newton-Schulz working matrices: ld = 4 (mod 16) doubles
// puts the 8 rows x 4 k of an m8n8k4 fragment load in distinct banks (two
// wavefronts per warp load, the minimum for 256 bytes); a row stride of
// m = 64 would put all 8 rows of an A fragment in one bank (8 wavefronts).
__host__ __device__ inline int ns_ld(int m) { return ((m + 15) & ~15) + 4; }

// C = op(A) B for m x m row-major smem matrices with row stride ld (op =
// transpose when ta) on the fp64 tensor cores: mma.sync m8n8k4 f64, a warp
// owns two horizontally adjacent 8 x 8 tiles of C at a time so each A
// fragment feeds two DMMAs (fragments: A[lane/4][lane%4], B[lane%4][lane/4],
// C[lane/4][2 (lane%4) + {0,1}]), k ascending in two chains (even / odd
// 4-blocks) per tile.  m <= 64, any blockDim.
__device__ void mm_small(const double* A, const double* B, double* C, int m, int ld, bool ta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int tiles = (m + 7) >> 3, pairs = (tiles + 1) >> 1;
  const int ar = lane >> 2, ak = lane & 3;  // A fragment (row, k); B fragment is (k, col) = (ak, ar)
  for (int u = warp; u < tiles * pairs; u += nw) {
    const int ti = u / pairs, tj = (u % pairs) * 2;
    const int r = ti * 8 + ar, cb = tj * 8 + ar, cb2 = cb + 8;
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;  // tile tj
    double f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;  // tile tj + 1
    for (int k0 = 0; k0 < m; k0 += 8) {
      const int k = k0 + ak, kk = k + 4;
      const double a = (r < m && k < m) ? (ta ? A[k * ld + r] : A[r * ld + k]) : 0.0;
      const double a2 = (r < m && kk < m) ? (ta ? A[kk * ld + r] : A[r * ld + kk]) : 0.0;
      const double b = (k < m && cb < m) ? B[k * ld + cb] : 0.0;
      const double b2 = (kk < m && cb < m) ? B[kk * ld + cb] : 0.0;
      const double bb = (k < m && cb2 < m) ? B[k * ld + cb2] : 0.0;
      const double bb2 = (kk < m && cb2 < m) ? B[kk * ld + cb2] : 0.0;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c0), "+d"(c1)
                   : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(f0), "+d"(f1)
                   : "d"(a), "d"(bb));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(e0), "+d"(e1)
                   : "d"(a2), "d"(b2));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(g0), "+d"(g1)
                   : "d"(a2), "d"(bb2));
    }
    c0 += e0;
    c1 += e1;
    f0 += g0;
    f1 += g1;
    const int cr = ti * 8 + (lane >> 2), cc = tj * 8 + 2 * (lane & 3), cc2 = cc + 8;
    if (cr < m) {
      if (cc < m) C[cr * ld + cc] = c0;
      if (cc + 1 < m) C[cr * ld + cc + 1] = c1;
      if (cc2 < m) C[cr * ld + cc2] = f0;
      if (cc2 + 1 < m) C[cr * ld + cc2 + 1] = f1;
    }
  }
}

// Polar factor of the well-conditioned m x m R (row-major, row stride m, in
// X on entry, the result on exit) by the Newton-Schulz iteration
// X <- 1.5 X - 0.5 X (X'X) from X0 = R / sqrt(|R|_1 |R|_inf) (all singular values in
// (0, 1], so it converges; quadratically once X'X ~ I).  ws: 3 m ns_ld(m)
// doubles of scratch (the iterate and two products at row stride ns_ld(m)).
// Returns false if it has not converged in max_it steps.
__device__ bool newton_schulz_polar(double* X, double* ws, double* red, int m, int max_it, int* iters = nullptr,
                                    bool sigma_ge_one = false) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ld = ns_ld(m);
  double* Xp = ws;
  double* T = ws + m * ld;
  double* U = T + m * ld;
  // X0 = R / sqrt(|R|_1 |R|_inf) (>= |R|_2, and closer to it than |R|_F)
  __shared__ double s_norm1, s_norminf;
  if (tid < 32) {
    double c1 = 0.0, ci = 0.0;
    for (int j = tid; j < m; j += 32) {
      double cs = 0.0, rs = 0.0;
      for (int i = 0; i < m; ++i) {
        cs += fabs(X[i * m + j]);
        rs += fabs(X[j * m + i]);
      }
      c1 = fmax(c1, cs);
      ci = fmax(ci, rs);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      c1 = fmax(c1, __shfl_xor_sync(0xffffffffu, c1, o));
      ci = fmax(ci, __shfl_xor_sync(0xffffffffu, ci, o));
    }
    if (tid == 0) {
      s_norm1 = c1;
      s_norminf = ci;
    }
  }
  __syncthreads();
  const double inv = 1.0 / sqrt(s_norm1 * s_norminf);
  for (int e = tid; e < m * m; e += nt) Xp[(e / m) * ld + e % m] = X[e] * inv;
  __syncthreads();
  // With every singular value of X known to be >= 1 (the scaled Newton step
  // guarantees it), X0's lie in [l, 1], l = inv: the first steps use the
  // cubic scaled to that interval, X <- (3 a X - a^3 X X'X) / 2 with
  // a = sqrt(3 / (1 + l + l^2)) (the image of [l, 1] is [f(a l), 1], so the
  // bound stays valid: l <- (3 a l - a^3 l^3) / 2), until l > 0.99; plain
  // Newton-Schulz (a = 1) finishes.  Same fixed point, fewer steps.
  double lb = sigma_ge_one ? inv : 1.0;
  bool ok = false;
  for (int it = 0; it < max_it && !ok; ++it) {
    const bool scaled = lb < 0.99;
    const double al = scaled ? sqrt(3.0 / (1.0 + lb + lb * lb)) : 1.0;
    const double c1 = 1.5 * al, c3 = 0.5 * al * al * al;
    if (scaled) lb = 0.5 * (3.0 * al * lb - al * al * al * lb * lb * lb);
    mm_small(Xp, Xp, T, m, ld, true);  // T = X'X
    __syncthreads();
    mm_small(Xp, T, U, m, ld, false);  // U = X T
    __syncthreads();
    double d = 0.0;
    for (int e = tid; e < m * m; e += nt) {
      const int o = (e / m) * ld + e % m;
      const double xn = scaled ? fma(-c3, U[o], c1 * Xp[o]) : fma(-0.5, U[o], 1.5 * Xp[o]);
      d = fma(xn - Xp[o], xn - Xp[o], d);
      Xp[o] = xn;
    }
    const double dn = sqrt(block_sum_any(d, red));  // (syncs)
#ifdef GPS_POLAR_DEBUG
    if (tid == 0) printf("newton-schulz it %d step %.3e\n", it, dn);
#endif
    ok = !scaled && dn < 1e-15 * sqrt(double(m));
    if (iters != nullptr && threadIdx.x == 0) *iters += 1;
  }
  if (ok)
    for (int e = tid; e < m * m; e += nt) X[e] = Xp[(e / m) * ld + e % m];
  __syncthreads();
  return ok;
}

// part[0][e] = sum_b part[b][e] in a fixed order, many CTAs (the one-CTA
// stage kernel then reads a single Gram).
// 256 threads = 8 slices of the partials x 32 elements: warp s sums slice s
// (its eight-or-so partials' loads in flight) for 32 consecutive elements,
// then the slices are added in order -- deterministic, one load round.
__global__ void __launch_bounds__(256) gram_reduce_kernel(double* __restrict__ part, int nparts, int mm,
                                                          const PolarCtl* pc) {
  __shared__ double red[8][32];
  if (!pc->active || pc->fallback) return;
  const int sl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * 32 + lane;
  const int b0 = nparts * sl / 8, b1 = nparts * (sl + 1) / 8;
  double t = 0.0;
  if (e < mm) {
#pragma unroll 8
    for (int b = b0; b < b1; ++b) t += part[size_t(b) * mm + e];
  }
  red[sl][lane] = t;
  __syncthreads();
  if (sl == 0 && e < mm) {
    double u = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) u += red[k][lane];
    part[e] = u;
  }
}

// Sum the Gram partials (fixed order), Cholesky G'G = R'R (upper R), and
// invert R.  stage 1: R1 -> Rs (R1), Rinv (R1^-1), or the fallback flag when
// kappa_F(R1) > kCholQr2MaxKappa.  stage 2: R2 with R = R2 R1, the polar factor
// P of R by Newton-Schulz, then S = R2^-1 P (the right factor of X = Q1 S).
// One CTA; small m x m work in smem.
__global__ void __launch_bounds__(kPolarThreads) chol_stage_kernel(const double* __restrict__ part, int nparts, int m,
                                                                  int p_true, int stage, double* __restrict__ R1g,
                                                                  double* __restrict__ Sg, PolarCtl* pc) {
  extern __shared__ double psm[];
  if (!pc->active || pc->fallback) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* M = psm;              // m*m (row-major a*m+c)
  double* Ri = psm + m * m;     // m*m inverse
  double* R = Ri + m * m;       // m*m upper, row-major R[i*m+j]
  double* W = R + m * m;        // m*m scratch
  // R, W and the rest of the allocation (3 m ns_ld(m) doubles from R) are
  // the Newton-Schulz workspace in stage 2
  GPS_STAMP(0);
#ifdef GPS_POLAR_DEBUG
  if (tid == 0) printf("chol stage %d start %lld\n", stage, clock64());
#endif
  __shared__ int bad;
  __shared__ double red[40];
  // Gram = sum of the partials in a fixed order (8 independent loads in
  // flight per thread)
  for (int e = tid; e < m * m; e += nt) {
    double t = 0.0;
    int b = 0;
    for (; b + 8 <= nparts; b += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[size_t(b + u) * m * m + e];
      t += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    }
    for (; b < nparts; ++b) t += part[size_t(b) * m * m + e];
    M[e] = t;
    R[e] = 0.0;
    Ri[e] = 0.0;
  }
  GPS_STAMP(1);
#ifdef GPS_POLAR_DEBUG
  if (tid == 0) printf("chol stage %d partials loaded %lld\n", stage, clock64());
#endif
  if (tid == 0) bad = 0;
  __syncthreads();
  if (stage == 2) {
    // Stage 2 factors the Gram of Q1 = G R1^-1, I + E with |E| ~ kappa^2 u
    // (<= 1e-6 inside the trust region), without the 64-step pivot chain:
    // R2 = I + U with U upper triangular solving U + U' + U'U = E, by the
    // fixed point U <- Phi(E - U'U) (Phi: strict upper part plus half the
    // diagonal; each step multiplies the error by ~|E|, from |E|^2 at U0),
    // and R2^-1 = sum_k (-U)^k (Horner).  Both are the Cholesky factor and
    // its inverse to rounding; the step counts follow |E| (typically one
    // and two mm_small, ~6.5K clocks each at m = 64, against 63.5K + 23.7K
    // for the pivot loop and the back substitution).  |E| > 1e-3 means |R2 - I| far
    // beyond the trust region below: the exact path takes the step.
    double t = 0.0;
    for (int e = tid; e < m * m; e += nt) {
      if (e / m == e % m) M[e] -= 1.0;  // M := E
      t = fma(M[e], M[e], t);
    }
    const double eps = sqrt(block_sum_any(t, red));
    if (!(eps <= 1e-3)) {
      if (tid == 0) pc->fallback = 1;
      return;
    }
    // the series and the rest of stage 2 run at the Newton-Schulz row
    // stride L (conflict-free mm_small fragments; at stride m = 64 every A
    // fragment row hits one bank): U, a product and R2^-1 in the padded
    // buffers after R (chol_smem_bytes), E in M
    const int L = ns_ld(m);
    double* Up = R;
    double* Wp = R + m * L;
    double* Rp = R + 2 * m * L;
    auto phi = [&](int i, int j, double v) { return i < j ? v : (i == j ? 0.5 * v : 0.0); };
    for (int e = tid; e < m * m; e += nt) Up[(e / m) * L + e % m] = phi(e / m, e % m, M[e]);  // U0 = Phi(E)
    int k_fp = 0;
    for (double err = eps * eps; err > 1e-18 && k_fp < 4; err *= eps) ++k_fp;
    for (int k = 0; k < k_fp; ++k) {
      __syncthreads();
      mm_small(Up, Up, Wp, m, L, true);  // U'U
      __syncthreads();
      for (int e = tid; e < m * m; e += nt) {
        const int i = e / m, j = e % m;
        Up[i * L + j] = phi(i, j, M[e] - Wp[i * L + j]);
      }
    }
    int k_neu = 1;
    for (double term = eps * eps; term > 1e-18 && k_neu < 6; term *= eps) ++k_neu;
    for (int e = tid; e < m * m; e += nt) Rp[(e / m) * L + e % m] = (e / m == e % m) ? 1.0 : 0.0;
    for (int k = 0; k < k_neu; ++k) {
      __syncthreads();
      mm_small(Up, Rp, Wp, m, L, false);  // U R2^-1 (partial sum)
      __syncthreads();
      for (int e = tid; e < m * m; e += nt) {
        const int i = e / m, j = e % m;
        Rp[i * L + j] = (i == j ? 1.0 : 0.0) - Wp[i * L + j];
      }
    }
    __syncthreads();
  }
  double dmax = 0.0;
  for (int j = 0; j < m; ++j) dmax = fmax(dmax, M[j * m + j]);
  // Right-looking Cholesky of the upper triangle, two barriers per step:
  // every thread derives the pivot itself; thread (a, g) = (tid / 16,
  // tid % 16) updates row a, columns g, g + 16, ... of the trailing block.
  // (A blocked variant -- 8 x 8 diagonal blocks factored by one warp, block
  // row solves, rank-8 trailing updates, 24 barriers instead of 128 --
  // measured slower: 78K vs 63.5K clocks at m = 64, scripts/ubench/polar_ns.cu;
  // the per-pivot chain stays, serialised in one warp.  So did 32 x 32
  // blocks with the panel factored by one warp: 25K clocks per 32-step
  // panel with the columns in registers (fully unrolled, instruction-fetch
  // bound), 40K with them in shared memory, i.e. ~1000 clocks per pivot
  // either way -- the pivot chain's fp64 latency, not the barriers.)
  if (stage == 1) {  // (stage 2 factored above)
    const int ta = tid >> 4, tg = tid & 15;
    for (int j = 0; j < m; ++j) {
      const double d = M[j * m + j];
      if (!(d > 1e-28 * dmax) || !(d > 0.0)) {
        if (tid == 0) bad = 1;
        break;  // uniform: every thread reads the same d
      }
      const double rp = rsqrt(d);  // one reciprocal square root instead of sqrt + divisions
      for (int c = j + tid; c < m; c += nt) R[j * m + c] = (c == j) ? d * rp : M[j * m + c] * rp;
      __syncthreads();
      if (ta > j && ta < m) {
        const double rja = R[j * m + ta];
        for (int c = ta + tg; c < m; c += 16) M[ta * m + c] = fma(-rja, R[j * m + c], M[ta * m + c]);
      }
      __syncthreads();
    }
    __syncthreads();
    GPS_STAMP(2);
#ifdef GPS_POLAR_DEBUG
    if (tid == 0) printf("chol stage %d cholesky done %lld\n", stage, clock64());
#endif
    if (bad) {
      if (tid == 0) pc->fallback = 1;
      return;
    }
    // Ri = R^-1 (upper) by back substitution, one thread per column c (a
    // column needs only its own rows below, so no barrier per row), times
    // the diagonal reciprocals formed in parallel first.  Every lane of a
    // warp walks the same rows i and the same k range (up to the warp's last
    // column; entries below a column's diagonal are zero), so the R reads are
    // broadcasts and the Ri reads are conflict-free.  Measured at m = 64
    // (scripts/ubench/polar_ns.cu, whole stage-1 kernel): 75 us, against 95 us
    // with a half-warp per column and shuffle sums, 100 us with one block
    // barrier per row.
    // For m > 32 the two 32-column diagonal blocks are inverted at the same
    // time (warp 0: rows / columns 0 .. 31, warp 1: 32 .. m-1) and the
    // off-diagonal block follows as Ri12 = -Ri11 R12 Ri22 over all threads:
    // the thread-per-column walk of the whole triangle made warp 1 (columns
    // 32 .. 63, rows 63 .. 0) ~2.5x longer than warp 0 (~60K clocks).
    if (tid < m) W[tid] = 1.0 / R[tid * m + tid];
    __syncthreads();
    if (tid < ((m + 31) & ~31)) {
      const int lo = m > 32 ? (tid & ~31) : 0;  // first row / column of this warp's diagonal block
      const int c = tid, cr = min(c, m - 1), cw = min((tid | 31), m - 1);  // cr: lanes past m read a live column
      for (int i = cw; i >= lo; --i) {
        double t0 = 0.0, t1 = 0.0;
        int k = i + 1;
        for (; k + 1 <= cw; k += 2) {
          t0 = fma(R[i * m + k], Ri[k * m + cr], t0);
          t1 = fma(R[i * m + k + 1], Ri[(k + 1) * m + cr], t1);
        }
        if (k <= cw) t0 = fma(R[i * m + k], Ri[k * m + cr], t0);
        if (c < m && i <= c) Ri[i * m + c] = ((i == c ? 1.0 : 0.0) - (t0 + t1)) * W[i];
      }
    }
    __syncthreads();
    if (m > 32) {
      const int n2 = m - 32;
      double* T = W + m;  // T = R12 Ri22 (32 x n2), after the diagonal reciprocals
      for (int e = tid; e < 32 * n2; e += nt) {
        const int i = e / n2, c = 32 + e % n2;
        double t = 0.0;
        for (int k = 32; k <= c; ++k) t = fma(R[i * m + k], Ri[k * m + c], t);
        T[e] = t;
      }
      __syncthreads();
      for (int e = tid; e < 32 * n2; e += nt) {
        const int i = e / n2, c = e % n2;
        double t = 0.0;
        for (int k = i; k < 32; ++k) t = fma(Ri[i * m + k], T[k * n2 + c], t);
        Ri[i * m + 32 + c] = -t;
      }
      __syncthreads();
    }
    GPS_STAMP(3);
#ifdef GPS_POLAR_DEBUG
    if (tid == 0) printf("chol stage %d inverse done %lld\n", stage, clock64());
#endif
  }
  if (stage == 1) {
    // kappa_F(R1) = |R1|_F |R1^-1|_F ~ kappa(G): beyond kCholQr2MaxKappa the
    // CholeskyQR2 result is not trusted and the exact path decides (rank too)
    double a = 0.0, b = 0.0;
    for (int e = tid; e < m * m; e += nt) {
      a = fma(R[e], R[e], a);
      b = fma(Ri[e], Ri[e], b);
    }
    const double kap = sqrt(block_sum_any(a, red)) * sqrt(block_sum_any(b, red));
    GPS_STAMP(7);
    if (!(kap <= kCholQr2MaxKappa)) {
      if (tid == 0) pc->fallback = 1;
      return;
    }
    for (int e = tid; e < m * m; e += nt) {
      R1g[e] = R[e];
      Sg[e] = Ri[e];  // apply: Q1 = G R1^-1
    }
    GPS_STAMP(6);
    return;
  }
  // stage 2: Q1 = G R1^-1 is orthonormal to ~kappa^2 u when stage 1 was
  // accurate, so R2 ~ I; a larger departure means stage 1 lost accuracy and
  // the exact path takes the step.
  const int L = ns_ld(m);
  double* Up = R;  // padded m x L buffers (see the series above)
  double* Wp = R + m * L;
  double* Rp = R + 2 * m * L;
  double* Xp = R + 3 * m * L;
  {
    double t = 0.0;
    for (int e = tid; e < m * m; e += nt) {
      const double d = Up[(e / m) * L + e % m];  // R2 - I = U
      t = fma(d, d, t);
    }
    if (!(sqrt(block_sum_any(t, red)) <= kCholQr2MaxR2Dev)) {
      if (tid == 0) pc->fallback = 1;
      return;
    }
  }
  // stage 2: R = R2 R1, its polar factor P, then S = R2^-1 P, the right
  // factor of X = Q1 S (the CholeskyQR2 path only runs for condition numbers
  // far below the rank cutoff max(p, m) eps -- stage 1 checked -- so rank =
  // m here).  P comes from one scaled Newton step, which the triangular
  // factors make cheap because R^-1 = R1^-1 R2^-1 is at hand (R1^-1 from
  // stage 1 in Sg),
  //   M = (zeta R + zeta^-1 R^-T) / 2,  zeta = sqrt(|R^-1|_F / |R|_F)
  // (same singular vectors as R; the singular values move into
  // [1, (sqrt(k) + 1 / sqrt(k)) / 2] for kappa k), followed by the
  // Newton-Schulz iteration on M, which then starts well inside its
  // quadratic region (~20 -> ~7 steps at kappa ~ 100).  Every product on
  // the fp64 tensor cores at the padded stride (mm_small over the full
  // m x m operands; zero lower triangles keep the triangular products
  // upper).
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    Up[i * L + j] += (i == j) ? 1.0 : 0.0;  // R2 = I + U
    Wp[i * L + j] = R1g[e];                 // R1
    Ri[e] = Rp[i * L + j];                  // R2^-1 (stride m: Rp is Newton-Schulz workspace below)
  }
  __syncthreads();
  mm_small(Up, Wp, Xp, m, L, false);  // R = R2 R1
  __syncthreads();
  for (int e = tid; e < m * m; e += nt) Wp[(e / m) * L + e % m] = Sg[e];  // R1^-1
  __syncthreads();
  mm_small(Wp, Rp, Up, m, L, false);  // R^-1 = R1^-1 R2^-1
  __syncthreads();
  GPS_STAMP(4);
#ifdef GPS_POLAR_DEBUG
  if (tid == 0) printf("chol stage %d R2R1 done %lld\n", stage, clock64());
#endif
  {
    double a = 0.0, b = 0.0;
    for (int e = tid; e < m * m; e += nt) {
      const int i = e / m, j = e % m;
      a = fma(Xp[i * L + j], Xp[i * L + j], a);
      b = fma(Up[i * L + j], Up[i * L + j], b);
    }
    const double fa = sqrt(block_sum_any(a, red)), fb = sqrt(block_sum_any(b, red));
    const double zeta = sqrt(fb / fa);
    for (int e = tid; e < m * m; e += nt) {
      const int i = e / m, j = e % m;
      M[e] = 0.5 * (zeta * Xp[i * L + j] + Up[j * L + i] / zeta);
    }
  }
  __syncthreads();
  if (!newton_schulz_polar(M, R, red, m, 100, &pc->ns_iters, true)) {  // not converged: exact path decides
    if (tid == 0) pc->fallback = 1;
    return;
  }
  GPS_STAMP(5);
#ifdef GPS_POLAR_DEBUG
  if (tid == 0) printf("chol stage %d NS done %lld\n", stage, clock64());
#endif
  if (tid == 0) pc->rank = m;
  for (int e = tid; e < m * m; e += nt) {  // S = R2^-1 P
    const int i = e / m, j = e % m;
    Xp[i * L + j] = Ri[e];
    Wp[i * L + j] = M[e];
  }
  __syncthreads();
  mm_small(Xp, Wp, Up, m, L, false);
  __syncthreads();
  for (int e = tid; e < m * m; e += nt) Sg[e] = Up[(e / m) * L + e % m];
  GPS_STAMP(6);
}

// Out[j][r] = sum_b In[b][r] * S[b][j]   (In, Out: [m][ld]; S row-major m x m)
// on the fp64 tensor cores: CTA b owns rows [64 b, 64 b + 64); In's rows and
// S are staged in shared memory k-contiguous (row stride 68 = 4 mod 16
// doubles, zero-padded to 64 components), and warp w computes rows
// 16 (w % 4) .. + 16 (2 m-tiles) x components 32 (w / 4) .. + 32 (4 n-tiles)
// with m8n8k4 DMMA.  (A thread per (row, 8 components) with FMAs: 21 us at
// p = 8192, m = 64; a thread per row with an m-long register array: 197 us.)
constexpr int kPolarApplyRows = 64;
constexpr int kPolarApplyStride = kMaxGramM + 4;
__host__ __device__ constexpr size_t apply_smem_bytes() {
  return size_t(2) * kMaxGramM * kPolarApplyStride * sizeof(double);
}
__global__ void __launch_bounds__(256) apply_right_kernel(const double* __restrict__ In, const double* __restrict__ S,
                                                          int ld, int m, double* Out, const PolarCtl* pc,
                                                          const GpsCtl* ctl, int64_t out_par_stride) {
  extern __shared__ __align__(16) double apply_smem[];
  if (!pc->active || pc->fallback) return;
  double* O = Out + (ctl != nullptr ? ((ctl->iter + 1) & 1) * out_par_stride : 0);
  double* sI = apply_smem;                          // [b][row]  (k = b)
  double* sS = apply_smem + kMaxGramM * kPolarApplyStride;  // [b][j]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int r0 = blockIdx.x * kPolarApplyRows;
  const int kp = (m + 3) & ~3;  // k rounded up to the DMMA k-step (zero rows beyond m)
  for (int e = tid; e < kMaxGramM * kMaxGramM; e += blockDim.x) {
    const int b = e / kMaxGramM, j = e % kMaxGramM;
    sS[b * kPolarApplyStride + j] = (b < m && j < m) ? S[b * m + j] : 0.0;
  }
  for (int e = tid; e < kMaxGramM * kPolarApplyRows; e += blockDim.x) {
    const int b = e / kPolarApplyRows, rr = e % kPolarApplyRows;
    sI[b * kPolarApplyStride + rr] = (b < m && r0 + rr < ld) ? In[size_t(b) * ld + r0 + rr] : 0.0;
  }
  __syncthreads();
  const int rg = warp & 3, cg = warp >> 2;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;
  const int jn = (m + 7) >> 3;  // valid n-tiles
  for (int k0 = 0; k0 < kp; k0 += 4) {
    double a[2], bf[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) a[mt] = sI[(k0 + t) * kPolarApplyStride + rg * 16 + mt * 8 + g];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = sS[(k0 + t) * kPolarApplyStride + cg * 32 + nt * 8 + g];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        if (cg * 4 + nt < jn)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                       : "d"(a[mt]), "d"(bf[nt]));
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int r = r0 + rg * 16 + mt * 8 + g;
    if (r < ld)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int j = cg * 32 + nt * 8 + 2 * t;
        if (j < m) O[size_t(j) * ld + r] = acc[mt][nt][0];
        if (j + 1 < m) O[size_t(j + 1) * ld + r] = acc[mt][nt][1];
      }
  }
}

// Fallback (exact Householder + Jacobi, one CTA) and the step's finish.
// On the CholeskyQR2 path `gram` holds X_{k+1}'X_{k+1} (the Gram kernels
// ran on the new iterate): an error above the reference's Stiefel
// tolerance (core.py:22) sends the step to the exact path as well, so a
// CholeskyQR2 result is only ever kept when it is a valid StiefelPoint.
// Rank failure stops the loop (block.py:215-218), else the iterate
// advances (bk_advance).
__global__ void __launch_bounds__(kPolarThreads) bk_finish_kernel(double* G, double* Xbuf, int64_t x_stride, int ld,
                                                                 int p_true, int m, GpsCtl* ctl, PolarCtl* pc,
                                                                 int* rank_out, const double* __restrict__ gram,
                                                                 BandLog* band, double* __restrict__ stiefel) {
  extern __shared__ double psm[];
  __shared__ double red[40];
  if (!pc->active) return;
  const int k = ctl->iter;
  double* Xn = Xbuf + ((k + 1) & 1) * x_stride;
  int rank = pc->rank;
  bool exact = pc->fallback != 0;
  double err = 0.0;
  if (!exact) {
    err = gram_error_from(gram, m, red);
    exact = !(err <= kStiefelTol);
  }
  if (exact) {
    rank = polar_device(G, Xn, ld, p_true, m, polar_scratch(psm, m));
    if (rank == m) err = stiefel_error(Xn, ld, m, psm);
  }
  if (threadIdx.x == 0) {
    if (exact) {
      pc->fallback = 1;
      pc->exact_steps += 1;
    }
    bk_advance(ctl, k, m, rank, err, rank_out, band, stiefel);
  }
}

// M, Ri, then four padded m x ns_ld(m) buffers from R (the Newton-Schulz
// workspace is the first three; stage 2's products use all four)
__host__ __device__ inline size_t chol_smem_bytes(int m) {
  return (size_t(2) * m * m + size_t(4) * m * ns_ld(m)) * sizeof(double) + 64;
}

}  // namespace gps
