// Single-unit GP-SPCA kernels: the fused column sweep (K1), the
// deterministic cross-CTA reduction (K2), the power step (K3) and the
// column-norm pass (K0).
//
// Reference loop being replaced (single_unit.py:160-181, parallel.py:85-142):
//     c = A'x ; f = obj(c) ; g = 2 sum_i w(c_i) a_i ; x = g/||g||
// which reads A twice per iteration through chunked dgemv calls.  The fused
// sweep reads every column once: the column tile lands in shared memory by a
// bulk-async copy, each thread group forms a_i'x from registers (x lives in
// registers, fp64), applies the threshold, and -- while the tile is still on
// chip -- accumulates w_i a_i into a register-resident fp64 partial of g.
#pragma once

#include "common.cuh"

namespace gps {

struct alignas(16) GpsCtl {
  int iter;       // index k of the current iterate x_k
  int done;       // 1 once the loop has stopped (all kernels early-exit)
  int converged;  // reference semantics: tol met or zero gradient
  int status;
  double f_prev;  // f_{k-1}
  double gnorm;   // ||g|| of the last step (diagnostic)
};

enum SweepMode : int { kFused = 0, kDotOnly = 1, kCoef = 2 };

template <typename TA>
struct Vec16;
template <>
struct Vec16<float> {
  using T = float4;
  static constexpr int N = 4;
  __device__ static void unpack(const T& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct Vec16<double> {
  using T = double2;
  static constexpr int N = 2;
  __device__ static void unpack(const T& v, double* o) { o[0] = v.x; o[1] = v.y; }
};

struct SweepArgs {
  const void* A;      // column-major, leading dimension ld (zero-padded rows)
  int64_t n;          // columns
  int ld;             // padded rows (multiple of 32)
  int penalty;        // 0 = l1, 1 = l0
  double gamma;
  const double* x;    // iterate base (ld entries, zero padded)
  int64_t x_stride;   // stride between the two parity slots (ctl != null)
  const double* coef; // kCoef: per-column coefficients (n)
  int coef_threshold; // kCoef: apply the threshold (1) or use coef as is (0)
  double* part_g;     // [gridDim.x][ld] per-CTA partial of sum w_i a_i
  double* part_s;     // [gridDim.x][4]: f, nnz, sum w^2, unused
  double* c_out;      // optional: c = A'x (n)
  double* w_out;      // optional: thresholded weights (n), parity slot
  int64_t w_stride;
  const GpsCtl* ctl;  // optional loop control (early exit + parity)
  int cols_per_stage; // T
  int num_stages;     // smem ring depth S
  int64_t total_stages;
};

constexpr int kSweepThreads = 256;
constexpr int kColsPerGroup = 2;  // K: columns a group handles per stage

template <int GS>
__host__ __device__ constexpr int sweep_groups() { return kSweepThreads / GS; }

// Shared memory layout: S stages | reduction scratch | mbarriers.
__host__ __device__ inline size_t sweep_red_bytes(int ng, int gs) {
  const int per_group = (gs / 32) * kColsPerGroup > 4 ? (gs / 32) * kColsPerGroup : 4;
  return size_t(ng) * per_group * sizeof(double);
}

template <typename TA, int RV, int GS, int MODE>
__global__ void __launch_bounds__(kSweepThreads, 1) su_sweep_kernel(const SweepArgs a) {
  constexpr int NT = kSweepThreads;
  constexpr int NG = NT / GS;
  constexpr int NW = GS / 32;  // warps per group
  constexpr int K = kColsPerGroup;
  constexpr int VN = Vec16<TA>::N;
  constexpr int R = RV * VN;  // rows owned by one thread
  using V = typename Vec16<TA>::T;

  extern __shared__ __align__(128) unsigned char smem[];

  if (a.ctl != nullptr && a.ctl->done) return;
  const int parity = a.ctl != nullptr ? (a.ctl->iter & 1) : 0;

  const int tid = threadIdx.x;
  const int grp = tid / GS;
  const int gt = tid % GS;
  const int wig = gt / 32;
  const int lane = tid & 31;
  const int S = a.num_stages;
  const int T = a.cols_per_stage;
  const int ld = a.ld;
  const size_t col_bytes = size_t(ld) * sizeof(TA);
  const size_t stage_bytes = size_t(T) * col_bytes;
  unsigned char* ring = smem;
  double* red = reinterpret_cast<double*>(smem + size_t(S) * stage_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(red) + sweep_red_bytes(NG, GS));

  const int64_t s_begin = a.total_stages * blockIdx.x / gridDim.x;
  const int64_t s_end = a.total_stages * (blockIdx.x + 1) / gridDim.x;
  const int64_t ns = s_end - s_begin;
  const unsigned char* Abytes = static_cast<const unsigned char*>(a.A);

  // Iterate rows owned by this thread: vectors gt, gt+GS, ... of the column.
  double xr[R];
  double gr[R];
  if (MODE != kCoef) {
    const double* x = a.x + parity * a.x_stride;
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      const int r0 = (gt + v * GS) * VN;
#pragma unroll
      for (int e = 0; e < VN; ++e) xr[v * VN + e] = (r0 + e < ld) ? x[r0 + e] : 0.0;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) gr[r] = 0.0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t s) {
    const int64_t col0 = (s_begin + s) * T;
    const int64_t ncols = (a.n - col0) < T ? (a.n - col0) : int64_t(T);
    const uint32_t bytes = static_cast<uint32_t>(ncols * col_bytes);
    const int slot = static_cast<int>(s % S);
    mbar_arrive_expect_tx(&bars[slot], bytes);
    bulk_g2s(ring + slot * stage_bytes, Abytes + col0 * col_bytes, bytes, &bars[slot], pol);
  };
  if (tid == 0) {
    const int64_t pre = ns < S ? ns : int64_t(S);
    for (int64_t s = 0; s < pre; ++s) issue(s);
  }

  double f_acc = 0.0, nnz_acc = 0.0, s2_acc = 0.0;

  for (int64_t s = 0; s < ns; ++s) {
    const int slot = static_cast<int>(s % S);
    const uint32_t phase = static_cast<uint32_t>((s / S) & 1);
    const int64_t col0 = (s_begin + s) * T;
    mbar_wait(&bars[slot], phase);
    const TA* tile = reinterpret_cast<const TA*>(ring + slot * stage_bytes);

    TA av[K][R];
    double dot[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = k * NG + grp;
      const bool valid = col0 + j < a.n && j < T;
      dot[k] = 0.0;
      if (MODE != kCoef) {
#pragma unroll
        for (int v = 0; v < RV; ++v) {
          const int r0 = (gt + v * GS) * VN;
          V q;
          if (valid && r0 < ld) {
            q = *reinterpret_cast<const V*>(tile + size_t(j) * ld + r0);
          } else {
            q = V{};
          }
          Vec16<TA>::unpack(q, &av[k][v * VN]);
        }
        double d = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) d = fma(static_cast<double>(av[k][r]), xr[r], d);
        dot[k] = d;
      }
    }

    if (MODE != kCoef) {
#pragma unroll
      for (int k = 0; k < K; ++k) dot[k] = warp_sum(dot[k]);
      if (NW > 1) {
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < K; ++k) red[(grp * NW + wig) * K + k] = dot[k];
        }
        if (NG == 1) {
          __syncthreads();
        } else {
          named_bar_sync(1 + grp, GS);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) t += red[(grp * NW + w) * K + k];
          dot[k] = t;
        }
      }
    }

#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = k * NG + grp;
      const int64_t col = col0 + j;
      const bool valid = col < a.n && j < T;
      if (!valid) continue;
      double c;
      double w;
      if (MODE == kCoef) {
        c = a.coef[col];
        w = a.coef_threshold ? threshold_weight(c, a.gamma, a.penalty) : c;
      } else {
        c = dot[k];
        f_acc += objective_term(c, a.gamma, a.penalty);
        w = (MODE == kFused) ? threshold_weight(c, a.gamma, a.penalty) : 0.0;
      }
      if (gt == 0) {
        if (a.c_out != nullptr) a.c_out[col] = c;
        if (a.w_out != nullptr) a.w_out[parity * a.w_stride + col] = w;
      }
      if (MODE != kDotOnly && w != 0.0) {
        nnz_acc += 1.0;
        s2_acc = fma(w, w, s2_acc);
        if (MODE == kCoef) {
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            const int r0 = (gt + v * GS) * VN;
            V q = (r0 < ld) ? *reinterpret_cast<const V*>(tile + size_t(j) * ld + r0) : V{};
            Vec16<TA>::unpack(q, &av[k][v * VN]);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) gr[r] = fma(w, static_cast<double>(av[k][r]), gr[r]);
      }
    }

    __syncthreads();  // ring slot and reduction scratch are free again
    if (tid == 0 && s + S < ns) issue(s + S);
  }

  // ---- epilogue: fixed-order reduction of the NG group partials ----
  double* pg = a.part_g + size_t(blockIdx.x) * ld;
  if (MODE != kDotOnly) {
    if (NG == 1) {
#pragma unroll
      for (int v = 0; v < RV; ++v) {
        const int r0 = (gt + v * GS) * VN;
#pragma unroll
        for (int e = 0; e < VN; ++e)
          if (r0 + e < ld) pg[r0 + e] = gr[v * VN + e];
      }
    } else {
      double* scratch = reinterpret_cast<double*>(ring);  // pipeline drained
#pragma unroll
      for (int v = 0; v < RV; ++v) {
        const int r0 = (gt + v * GS) * VN;
#pragma unroll
        for (int e = 0; e < VN; ++e)
          if (r0 + e < ld) scratch[size_t(grp) * ld + r0 + e] = gr[v * VN + e];
      }
      __syncthreads();
      for (int r = tid; r < ld; r += NT) {
        double t = 0.0;
#pragma unroll
        for (int g = 0; g < NG; ++g) t += scratch[size_t(g) * ld + r];
        pg[r] = t;
      }
    }
  }
  // scalar partials (every thread of a group holds identical values)
  __syncthreads();
  double* sc = red;  // reuse: NG * 3 doubles <= reduction scratch
  if (gt == 0) {
    sc[grp * 3 + 0] = f_acc;
    sc[grp * 3 + 1] = nnz_acc;
    sc[grp * 3 + 2] = s2_acc;
  }
  __syncthreads();
  if (tid < 3) {
    double t = 0.0;
    for (int g = 0; g < NG; ++g) t += sc[g * 3 + tid];
    a.part_s[size_t(blockIdx.x) * 4 + tid] = t;
  }
}

// K2: sum the per-CTA partials in CTA order (deterministic), into
// exch = [g (ld) | f | nnz | sum w^2 | 0].  Row blocks + one scalar block.
__global__ void __launch_bounds__(256) su_reduce_kernel(const double* __restrict__ part_g,
                                                        const double* __restrict__ part_s, int nparts,
                                                        int ld, double* __restrict__ exch,
                                                        const GpsCtl* ctl) {
  if (ctl != nullptr && ctl->done) return;
  const int row_blocks = (ld + 255) / 256;
  if (blockIdx.x < row_blocks) {
    const int r = blockIdx.x * 256 + threadIdx.x;
    if (r >= ld) return;
    double t = 0.0;
    const double* p = part_g + r;
#pragma unroll 8
    for (int b = 0; b < nparts; ++b) t += p[size_t(b) * ld];
    exch[r] = t;
  } else if (threadIdx.x < 4) {
    double t = 0.0;
    for (int b = 0; b < nparts; ++b) t += part_s[size_t(b) * 4 + threadIdx.x];
    exch[ld + threadIdx.x] = t;
  }
}

// K3: one power step (single_unit.py:167-180) on the reduced exchange
// vector: history, the relative-change stopping rule, the zero-gradient
// fixed point, and x_{k+1} = g / ||g|| into the other parity slot.  With
// defl_k > 0 the gradient is first projected off the previous components
// (implicit deflation, single_unit.py:287-296: g = (I - x_l x_l') ... g in
// component order), so A is never rewritten.
constexpr int kStepThreads = 1024;
constexpr int kStepRows = 8;  // ld <= kStepThreads * kStepRows

__device__ __forceinline__ double block_sum_1024(double v, double* red) {
  v = warp_sum(v);
  const int tid = threadIdx.x;
  __syncthreads();  // red reuse
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double u = tid < 32 ? red[tid] : 0.0;
  if (tid < 32) u = warp_sum(u);
  if (tid == 0) red[32] = u;
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(kStepThreads) su_step_kernel(const double* __restrict__ exch, int ld,
                                                              double* __restrict__ xbuf, int64_t x_stride,
                                                              double* __restrict__ hist, GpsCtl* ctl,
                                                              double tol, int max_iter,
                                                              const double* __restrict__ defl_X, int defl_k) {
  __shared__ double red[33];
  __shared__ int decision;
  if (ctl->done) return;
  const int k = ctl->iter;
  const double f = exch[ld];
  const double f_prev = ctl->f_prev;
  const int tid = threadIdx.x;
  if (tid == 0) {
    hist[k] = f;
    int d = 0;  // 0 continue, 1 converged, 2 max_iter
    if (k >= 1 && fabs(f - f_prev) < tol * fmax(fabs(f_prev), 1e-30)) d = 1;
    else if (k >= max_iter) d = 2;
    decision = d;
  }
  __syncthreads();
  if (decision != 0) {
    if (tid == 0) {
      ctl->done = 1;
      ctl->converged = decision == 1;
    }
    return;
  }
  double g[kStepRows];
#pragma unroll
  for (int j = 0; j < kStepRows; ++j) {
    const int r = tid + j * kStepThreads;
    g[j] = r < ld ? exch[r] : 0.0;
  }
  for (int l = 0; l < defl_k; ++l) {
    const double* xl = defl_X + size_t(l) * ld;
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < kStepRows; ++j) {
      const int r = tid + j * kStepThreads;
      if (r < ld) t = fma(xl[r], g[j], t);
    }
    const double d = block_sum_1024(t, red);
#pragma unroll
    for (int j = 0; j < kStepRows; ++j) {
      const int r = tid + j * kStepThreads;
      if (r < ld) g[j] = fma(-d, xl[r], g[j]);
    }
  }
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < kStepRows; ++j) t = fma(g[j], g[j], t);
  const double nrm = sqrt(block_sum_1024(t, red));
  if (nrm == 0.0) {
    if (tid == 0) {
      ctl->done = 1;
      ctl->converged = 1;
      ctl->gnorm = 0.0;
    }
    return;
  }
  double* xn = xbuf + ((k + 1) & 1) * x_stride;
#pragma unroll
  for (int j = 0; j < kStepRows; ++j) {
    const int r = tid + j * kStepThreads;
    if (r < ld) xn[r] = g[j] / nrm;
  }
  if (tid == 0) {
    ctl->f_prev = f;
    ctl->gnorm = nrm;
    ctl->iter = k + 1;
  }
}

// K0: column norms ||a_i|| with fp64 accumulation plus a non-finite flag
// (core.py:36-47 finiteness check, core.py:243-246 norms).  Warp per column.
template <typename TA>
__global__ void __launch_bounds__(256) column_norms_kernel(const TA* __restrict__ A, int64_t n, int ld,
                                                           double* __restrict__ norms, int* nonfinite) {
  constexpr int VN = Vec16<TA>::N;
  using V = typename Vec16<TA>::T;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int nv = ld / VN;
  int bad = 0;
  for (int64_t col = warp; col < n; col += nwarps) {
    const V* cp = reinterpret_cast<const V*>(A + col * ld);
    double acc = 0.0;
#pragma unroll 4
    for (int v = lane; v < nv; v += 32) {
      V q = __ldcs(cp + v);
      TA e[VN];
      Vec16<TA>::unpack(q, e);
#pragma unroll
      for (int u = 0; u < VN; ++u) {
        const double d = static_cast<double>(e[u]);
        bad |= !isfinite(d);
        acc = fma(d, d, acc);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) norms[col] = sqrt(acc);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
}

}  // namespace gps
