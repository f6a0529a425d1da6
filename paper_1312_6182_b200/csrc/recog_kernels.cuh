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

}  // namespace gps
