// Recognition path: the kernels behind project /
// explained_variance (pca.py:57-103) and knn_classify (datasets.py:223-275).
//
// R1 block_apply:  Y = A C for m coefficient vectors at once (A p x n
//                  column-major, C n x m): one pass over the columns whose
//                  coefficient row is nonzero (sparse loadings touch few),
//                  fp64 accumulation, per-CTA partials reduced in a fixed
//                  order by su_reduce_kernel.
// R2 knn_dist:     d(t, s) = (|t|^2 - 2 t.s) + |s|^2, clamped at 0 -- the
//                  reference's expansion and evaluation order
//                  (datasets.py:213-220) -- for a chunk of test rows against
//                  all train rows, fp64.
// R3 row_argmin:   first minimal distance per test row (np.argmin: ties go
//                  to the lowest train index).
#pragma once

#include "su_kernels.cuh"

namespace gps {

constexpr int kApplyRows = 1024;  // rows per CTA (4 per thread)
constexpr int kApplyComps = 8;    // components per CTA
constexpr int kApplyGX = 32;      // column groups (partials)

// colmask[i] = any_j C[j][i] != 0   (C component-major: C[j * n + i])
__global__ void coef_mask_kernel(const double* __restrict__ C, int64_t n, int m, unsigned char* __restrict__ mask) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    bool any = false;
    for (int j = 0; j < m && !any; ++j) any = C[size_t(j) * n + i] != 0.0;
    mask[i] = any ? 1 : 0;
  }
}

// grid (GX, ceil(ld / kApplyRows), ceil(m / kApplyComps)); CTA (b, y, z)
// owns columns [b n / GX, (b+1) n / GX), rows [y*1024, +1024) and
// components [8z, 8z+8) of part[b] ([m_pad][ld]).
template <typename TA>
__global__ void __launch_bounds__(256) block_apply_kernel(const TA* __restrict__ A, int64_t n, int ld, int m,
                                                          const unsigned char* __restrict__ mask,
                                                          const double* __restrict__ C, int m_pad,
                                                          double* __restrict__ part) {
  constexpr int RPT = kApplyRows / 256;
  const int64_t c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  const int r0 = blockIdx.y * kApplyRows;
  const int j0 = blockIdx.z * kApplyComps;
  double g[kApplyComps][RPT];
#pragma unroll
  for (int j = 0; j < kApplyComps; ++j)
#pragma unroll
    for (int k = 0; k < RPT; ++k) g[j][k] = 0.0;
  __shared__ unsigned char flags[256];
  for (int64_t base = c0; base < c1; base += 256) {
    const int64_t mine = base + threadIdx.x;
    const unsigned char f = mine < c1 ? mask[mine] : 0;
    if (!__syncthreads_or(f)) continue;  // no active column in this chunk
    flags[threadIdx.x] = f;
    __syncthreads();
    const int cnt = (c1 - base) < 256 ? static_cast<int>(c1 - base) : 256;
    for (int k = 0; k < cnt; ++k) {
      if (!flags[k]) continue;
      const int64_t col = base + k;
      double w[kApplyComps];
#pragma unroll
      for (int j = 0; j < kApplyComps; ++j) w[j] = (j0 + j < m) ? C[size_t(j0 + j) * n + col] : 0.0;
      const TA* ac = A + col * ld;
#pragma unroll
      for (int kk = 0; kk < RPT; ++kk) {
        const int r = r0 + kk * 256 + threadIdx.x;
        const double v = r < ld ? static_cast<double>(ac[r]) : 0.0;
#pragma unroll
        for (int j = 0; j < kApplyComps; ++j) g[j][kk] = fma(w[j], v, g[j][kk]);
      }
    }
    __syncthreads();
  }
  double* pg = part + size_t(blockIdx.x) * m_pad * ld;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = r0 + k * 256 + threadIdx.x;
    if (r < ld)
#pragma unroll
      for (int j = 0; j < kApplyComps; ++j)
        if (j0 + j < m_pad) pg[size_t(j0 + j) * ld + r] = g[j][k];
  }
}

// Squared row norms of a row-major rows x dim matrix (fixed order).
__global__ void row_sqnorm_kernel(const double* __restrict__ X, int64_t rows, int dim, double* __restrict__ out) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    const double* x = X + r * dim;
    double t = 0.0;
    for (int k = 0; k < dim; ++k) t = fma(x[k], x[k], t);
    out[r] = t;
  }
}

constexpr int kKnnTileT = 16;   // test rows per CTA
constexpr int kKnnTileR = 256;  // train rows per CTA (one per thread)
constexpr int kKnnDimChunk = 64;

// dist[t][r] for t in [0, T), r in [0, R): grid (ceil(R / 256), ceil(T / 16)).
// Train rows are read column-major (trainT[k * R + r], coalesced); the CTA's
// test rows are staged in shared memory dim-chunk by dim-chunk.
__global__ void __launch_bounds__(kKnnTileR) knn_dist_kernel(const double* __restrict__ test, int64_t T,
                                                             const double* __restrict__ trainT, int64_t R, int dim,
                                                             const double* __restrict__ tt,
                                                             const double* __restrict__ ss,
                                                             double* __restrict__ dist) {
  __shared__ double st[kKnnTileT][kKnnDimChunk];
  const int64_t r = int64_t(blockIdx.x) * kKnnTileR + threadIdx.x;
  const int64_t t0 = int64_t(blockIdx.y) * kKnnTileT;
  double acc[kKnnTileT];
#pragma unroll
  for (int i = 0; i < kKnnTileT; ++i) acc[i] = 0.0;
  for (int k0 = 0; k0 < dim; k0 += kKnnDimChunk) {
    const int kc = min(kKnnDimChunk, dim - k0);
    for (int e = threadIdx.x; e < kKnnTileT * kKnnDimChunk; e += kKnnTileR) {
      const int i = e / kKnnDimChunk, k = e % kKnnDimChunk;
      st[i][k] = (t0 + i < T && k < kc) ? test[(t0 + i) * dim + k0 + k] : 0.0;
    }
    __syncthreads();
    if (r < R)
      for (int k = 0; k < kc; ++k) {
        const double s = trainT[size_t(k0 + k) * R + r];
#pragma unroll
        for (int i = 0; i < kKnnTileT; ++i) acc[i] = fma(st[i][k], s, acc[i]);
      }
    __syncthreads();
  }
  if (r < R) {
    const double sr = ss[r];
#pragma unroll
    for (int i = 0; i < kKnnTileT; ++i)
      if (t0 + i < T) {
        const double d = (tt[t0 + i] - 2.0 * acc[i]) + sr;
        dist[(t0 + i) * R + r] = d > 0.0 ? d : 0.0;
      }
  }
}

// First minimal entry of each row of dist (T x R): one CTA per row.
__global__ void __launch_bounds__(256) row_argmin_kernel(const double* __restrict__ dist, int64_t R,
                                                         int64_t* __restrict__ out) {
  __shared__ double sd[8];
  __shared__ int64_t si[8];
  const double* d = dist + int64_t(blockIdx.x) * R;
  double best = 1.0 / 0.0;
  int64_t bi = R;
  for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
    const double v = d[r];
    if (v < best) {  // strided ascending scan: the first minimum of this thread
      best = v;
      bi = r;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob < best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sd[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x >> 5); ++k)
      if (sd[k] < best || (sd[k] == best && si[k] < bi)) {
        best = sd[k];
        bi = si[k];
      }
    out[blockIdx.x] = bi;
  }
}

// k smallest entries of each row of dist (T x R) in (distance, index) order:
// np.argsort(d, kind="stable")[:, :k] (datasets.py:258).  One CTA per row;
// round j selects the lexicographic successor of round j - 1's (d, index),
// so equal distances come out in index order.  O(k R) per row: k is a
// k-NN neighbour count.
__global__ void __launch_bounds__(256) row_topk_kernel(const double* __restrict__ dist, int64_t R, int k,
                                                       int64_t* __restrict__ out) {
  __shared__ double sd[8];
  __shared__ int64_t si[8];
  __shared__ double s_prev_d;
  __shared__ int64_t s_prev_i;
  const double* d = dist + int64_t(blockIdx.x) * R;
  double prev_d = -1.0 / 0.0;
  int64_t prev_i = -1;
  for (int j = 0; j < k; ++j) {
    double best = 1.0 / 0.0;
    int64_t bi = R;
    for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
      const double v = d[r];
      const bool after = v > prev_d || (v == prev_d && r > prev_i);
      if (after && (v < best || (v == best && r < bi))) {
        best = v;
        bi = r;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      sd[w] = best;
      si[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < int(blockDim.x >> 5); ++q)
        if (sd[q] < best || (sd[q] == best && si[q] < bi)) {
          best = sd[q];
          bi = si[q];
        }
      out[int64_t(blockIdx.x) * k + j] = bi;
      s_prev_d = best;
      s_prev_i = bi;
    }
    __syncthreads();
    prev_d = s_prev_d;
    prev_i = s_prev_i;
  }
}

// ---- thin SVD by one-sided (Hestenes) Jacobi, many CTAs: the dense PCA
// baseline (pca.py:37-54) without a LAPACK / cuSOLVER call.  The k columns
// of Y are orthogonalised pairwise; tournament round `step` of a sweep
// rotates the mp / 2 disjoint pairs (mp = k rounded up to even), one CTA per
// pair, and V (k x k, optional) accumulates the rotations.  At convergence
// Y = U diag(s) (columns) and, for Y = M, M = U diag(s) V'.
__global__ void __launch_bounds__(256) jacobi_step_kernel(double* __restrict__ Y, int64_t ldy, int64_t rows,
                                                          double* __restrict__ V, int64_t ldv, int k, int step,
                                                          double tol, int* rotated) {
  __shared__ double red[3][8];
  __shared__ double cs[2];
  const int mp = (k + 1) & ~1;
  const int i = blockIdx.x;
  int p = (i == 0) ? 0 : 1 + (i - 1 + step) % (mp - 1);
  int q = 1 + (mp - 2 - i + step) % (mp - 1);
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
  if (q >= k) return;
  double* yp = Y + int64_t(p) * ldy;
  double* yq = Y + int64_t(q) * ldy;
  double a = 0.0, b = 0.0, g = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    const double u = yp[r], v = yq[r];
    a = fma(u, u, a);
    b = fma(v, v, b);
    g = fma(u, v, g);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  g = warp_sum(g);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = a;
    red[1][w] = b;
    red[2][w] = g;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0, sg = 0.0;
    for (int q2 = 0; q2 < int(blockDim.x >> 5); ++q2) {
      sa += red[0][q2];
      sb += red[1][q2];
      sg += red[2][q2];
    }
    double c = 1.0, s = 0.0;
    if (sg != 0.0 && fabs(sg) > tol * sqrt(sa * sb)) {
      const double zeta = (sb - sa) / (2.0 * sg);
      const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      c = 1.0 / sqrt(1.0 + t * t);
      s = c * t;
      *rotated = 1;
    }
    cs[0] = c;
    cs[1] = s;
  }
  __syncthreads();
  const double c = cs[0], s = cs[1];
  if (s == 0.0) return;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    const double u = yp[r], v = yq[r];
    yp[r] = c * u - s * v;
    yq[r] = s * u + c * v;
  }
  if (V != nullptr) {
    double* vp = V + int64_t(p) * ldv;
    double* vq = V + int64_t(q) * ldv;
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
      const double u = vp[r], v = vq[r];
      vp[r] = c * u - s * v;
      vq[r] = s * u + c * v;
    }
  }
}

// column norms of Y ([k][ld] fp64), warp per column, fixed order
__global__ void col_norms_f64_kernel(const double* __restrict__ Y, int64_t ld, int64_t rows, int k,
                                     double* __restrict__ out) {
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= k) return;
  const double* y = Y + warp * ld;
  double t = 0.0;
  for (int64_t r = lane; r < rows; r += 32) t = fma(y[r], y[r], t);
  t = warp_sum(t);
  if (lane == 0) out[warp] = sqrt(t);
}

// Y[j][r] = (double) A[r][j] for the transposed working copy (A: [n][lda]).
template <typename TA>
__global__ void transpose_widen_kernel(const TA* __restrict__ A, int64_t lda, int64_t p, int64_t n,
                                       double* __restrict__ Y, int64_t ldy) {
  __shared__ double tile[32][33];
  const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    tile[j][threadIdx.x] = (c < n && r < p) ? static_cast<double>(A[c * lda + r]) : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < p && c < n) Y[r * ldy + c] = tile[threadIdx.x][j];
  }
}

template <typename TA>
__global__ void widen_copy_kernel(const TA* __restrict__ A, int64_t n_elems, double* __restrict__ Y) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n_elems; e += int64_t(gridDim.x) * blockDim.x)
    Y[e] = static_cast<double>(A[e]);
}

}  // namespace gps
