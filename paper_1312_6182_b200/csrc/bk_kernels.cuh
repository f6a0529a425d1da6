// Block GP-SPCA kernels (reference block.py): the fused block sweep over a
// group of MG components, the device polar retraction (Gram + one-CTA
// Jacobi eigensolver + Newton-Schulz polish), the block power step, and the
// CholeskyQR2 initialisation.
//
// Reference per iteration (block.py:211-226): C = A'X (m reads of A),
// G_j = 2 mu_j sum_i w(mu_j c_ij, gamma_j) a_i (m more reads), X = polar(G)
// by LAPACK SVD on the host.  Here one fused sweep per group of MG
// components reads A once (dots, threshold, objective and the rank-MG update
// of the register-resident partial of G), so an iteration costs ceil(m/MG)
// reads of A, and the polar step runs on the device.
#pragma once

#include "su_kernels.cuh"

namespace gps {

struct BlockSweepArgs {
  const void* A;
  int64_t n;
  int ld;
  int penalty;
  double gamma[4];     // this group's gamma_j (padded components: +0, X = 0)
  double mu[4];        // this group's mu_j
  const double* X;     // [MG][ld] components of this group (parity slot 0)
  int64_t x_stride;    // parity stride of the X buffer
  double* part_g;      // [grid][MG][ld]  per-CTA partial of sum_i w_ij a_i
  double* part_s;      // [grid][4]: f, nnz, 0, 0
  double* w_out;       // optional [MG][n] weights (parity slot 0)
  int64_t w_stride;    // parity stride of the W buffer
  int64_t w_cstride;   // stride between components in W
  const GpsCtl* ctl;
  BandLog* band;       // optional near-threshold log; components comp0 + j
  int comp0;
  int cols_per_stage;
  int num_stages;
  int64_t total_stages;
};

// Generic warp reduce-scatter of V = 2^v <= 32 partials: round r (offset
// 16 >> r) keeps the half selected by lane bit (16 >> r); after log2(V)
// rounds each lane holds one fully reduced value (index bk_owner_index),
// the remaining rounds finish the butterfly.  Commutative adds keep all
// holders of a value bitwise identical.
template <int V, typename T>
__device__ __forceinline__ T warp_reduce_scatter_v(T (&v)[V], int lane) {
  int c = V;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (c > 1) {
      const bool hi = (lane & o) != 0;
      const int h = c / 2;
#pragma unroll
      for (int i = 0; i < V / 2; ++i) {
        if (i < h) {
          const T send = hi ? v[i] : v[i + h];
          const T keep = hi ? v[i + h] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      c = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  return v[0];
}
template <int V>
__device__ __forceinline__ int bk_owner_index(int lane) {
  int idx = 0;
  int c = V, o = 16;
  while (c > 1) {
    c >>= 1;
    if (lane & o) idx += c;
    o >>= 1;
  }
  return idx;
}

__host__ __device__ constexpr int bk_cols_per_group(int) { return 2; }

__host__ __device__ inline size_t bk_red_bytes(int ng, int gs, int k, int mg) {
  return (size_t(kSweepD) * ng * k * mg * (gs / 32) + size_t(kSweepD) * ng * k * mg + 32 * 2) * sizeof(double);
}

// K1b: fused block sweep for MG components (same warp-specialised skeleton
// as su_sweep_kernel).  TC is the arithmetic type of the dots and of the
// register-resident G partial (fp32 for fp32 storage per the north star,
// fp64 for fp64 storage); column sums, thresholds and the objective are fp64.
template <typename TA, typename TC, int RV, int GS, int MG>
__global__ void __launch_bounds__(kSweepThreads, 1) bk_sweep_kernel(const BlockSweepArgs a) {
  constexpr int NG = kSweepWorkers / GS;
  constexpr int NW = GS / 32;
  constexpr int K = bk_cols_per_group(RV);
  constexpr int KM = K * MG;  // values per worker per stage
  constexpr int D = kSweepD;
  constexpr int L = kSweepLag;
  constexpr int VN = Vec16<TA>::N;
  constexpr int R = RV * VN;
  using V = typename Vec16<TA>::T;
  static_assert(KM <= 32 && (KM & (KM - 1)) == 0, "K*MG must be a power of two <= 32");

  extern __shared__ __align__(128) unsigned char smem[];
  if (a.ctl != nullptr && a.ctl->done) return;
  const int parity = a.ctl != nullptr ? (a.ctl->iter & 1) : 0;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int S = a.num_stages;
  const int T = a.cols_per_stage;
  const int ld = a.ld;
  const size_t col_bytes = size_t(ld) * sizeof(TA);
  const size_t stage_bytes = size_t(T) * col_bytes;
  const size_t pad = sweep_pad_bytes(ld, GS * RV * VN, sizeof(TA));
  unsigned char* ring = smem;
  double* red = reinterpret_cast<double*>(smem + size_t(S) * stage_bytes + pad);
  double* wsm = red + D * NG * KM * NW;
  double* sc = wsm + D * NG * KM;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(red) + bk_red_bytes(NG, GS, K, MG));
  uint64_t* empty = full + S;
  uint64_t* pfull = empty + S;
  uint64_t* wready = pfull + D;

  const int64_t s_begin = a.total_stages * blockIdx.x / gridDim.x;
  const int64_t s_end = a.total_stages * (blockIdx.x + 1) / gridDim.x;
  const int ns = static_cast<int>(s_end - s_begin);

  {
    const size_t nbytes = size_t(S) * stage_bytes + pad;
    for (size_t off = size_t(tid) * 16; off < nbytes; off += size_t(kSweepThreads) * 16)
      *reinterpret_cast<uint4*>(ring + off) = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kSweepWorkers / 32);
    }
    for (int i = 0; i < D; ++i) {
      mbar_init(&pfull[i], kSweepWorkers / 32);
      mbar_init(&wready[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kSweepWorkers / 32 + 1) {
    // ------------------------------------------------------ producer warp
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const unsigned char* Abytes = static_cast<const unsigned char*>(a.A);
      int slot = 0;
      uint32_t ephase = 0;
      for (int s = 0; s < ns; ++s) {
        if (s >= S) mbar_wait_sleep(&empty[slot], ephase);
        const int64_t col0 = (s_begin + s) * T;
        const int64_t ncols = (a.n - col0) < T ? (a.n - col0) : int64_t(T);
        const uint32_t bytes = static_cast<uint32_t>(ncols * col_bytes);
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + slot * stage_bytes, Abytes + col0 * col_bytes, bytes, &full[slot], pol);
        if (++slot == S) {
          slot = 0;
          if (s >= S) ephase ^= 1u;
          else ephase = 0;
        }
      }
    }
    return;
  }

  if (warp == kSweepWorkers / 32) {
    // ------------------------------------------------------- reducer warp
    constexpr int ITEMS = NG * KM;
    double f_acc = 0.0, nnz_acc = 0.0;
    double* wbase = a.w_out != nullptr ? a.w_out + parity * a.w_stride : nullptr;
    for (int s = 0; s < ns; ++s) {
      const int d = s & (D - 1);
      mbar_wait_sleep(&pfull[d], static_cast<uint32_t>((s / D) & 1));
      for (int it = lane; it < ITEMS; it += 32) {
        const int grp = it / KM;
        const int k = (it % KM) / MG;
        const int j = it % MG;
        const int64_t col = (s_begin + s) * T + k * NG + grp;
        const double* q = red + ((d * NG + grp) * KM + k * MG + j) * NW;
        double c = 0.0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) c += q[ww];
        const double sj = a.mu[j] * c;
        double w = threshold_weight(sj, a.gamma[j], a.penalty);
        if (col < a.n) {
          band_note(a.band, parity, col, a.comp0 + j, sj, a.gamma[j], a.penalty);
          f_acc += objective_term(sj, a.gamma[j], a.penalty);
          if (w != 0.0) nnz_acc += 1.0;
          if (wbase != nullptr) wbase[j * a.w_cstride + col] = w;
        } else {
          w = 0.0;
        }
        wsm[((d * NG + grp) * K + k) * MG + j] = w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&wready[d]);
    }
    sc[lane * 2 + 0] = f_acc;
    sc[lane * 2 + 1] = nnz_acc;
    __syncwarp();
    if (lane < 2) {
      double t = 0.0;
      for (int l = 0; l < 32; ++l) t += sc[l * 2 + lane];
      a.part_s[size_t(blockIdx.x) * 4 + lane] = t;
    }
    return;
  }

  // ---------------------------------------------------------- worker warps
  const int grp = tid / GS;
  const int gt = tid % GS;
  const int wig = gt / 32;

  TC xr[R][MG];
  TC gr[R][MG];
  {
    const double* X = a.X + parity * a.x_stride;
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      const int r0 = (gt + v * GS) * VN;
#pragma unroll
      for (int e = 0; e < VN; ++e)
#pragma unroll
        for (int j = 0; j < MG; ++j) {
          xr[v * VN + e][j] = (r0 + e < ld) ? static_cast<TC>(X[size_t(j) * ld + r0 + e]) : TC(0);
          gr[v * VN + e][j] = TC(0);
        }
    }
  }

  int fslot = 0, uslot = 0;
  uint32_t fphase = 0;
  for (int t = 0; t < ns + L; ++t) {
    if (t < ns) {
      const int slot = fslot;
      mbar_wait(&full[slot], fphase);
      if (++fslot == S) {
        fslot = 0;
        fphase ^= 1u;
      }
      const TA* tile = reinterpret_cast<const TA*>(ring + slot * stage_bytes);
      TC acc[KM];
#pragma unroll
      for (int i = 0; i < KM; ++i) acc[i] = TC(0);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const TA* colp = tile + size_t(k * NG + grp) * ld;
#pragma unroll
        for (int v = 0; v < RV; ++v) {
          const V q = *reinterpret_cast<const V*>(colp + (gt + v * GS) * VN);
          TA e[VN];
          Vec16<TA>::unpack(q, e);
#pragma unroll
          for (int u = 0; u < VN; ++u)
#pragma unroll
            for (int j = 0; j < MG; ++j)
              acc[k * MG + j] = fma(static_cast<TC>(e[u]), xr[v * VN + u][j], acc[k * MG + j]);
        }
      }
      double dv[KM];
#pragma unroll
      for (int i = 0; i < KM; ++i) dv[i] = static_cast<double>(acc[i]);
      const double f = warp_reduce_scatter_v<KM>(dv, lane);
      if ((lane & (32 / KM - 1)) == 0)
        red[(((t & (D - 1)) * NG + grp) * KM + bk_owner_index<KM>(lane)) * NW + wig] = f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[t & (D - 1)]);
    }
    if (t >= L) {
      const int u = t - L;
      const int d = u & (D - 1);
      mbar_wait(&wready[d], static_cast<uint32_t>((u / D) & 1));
      const TA* ptile = reinterpret_cast<const TA*>(ring + uslot * stage_bytes);
      const double* wp = wsm + (d * NG + grp) * KM;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        TC wk[MG];
        bool any = false;
#pragma unroll
        for (int j = 0; j < MG; ++j) {
          wk[j] = static_cast<TC>(wp[k * MG + j]);
          any |= wp[k * MG + j] != 0.0;
        }
        if (any) {
          const TA* colp = ptile + size_t(k * NG + grp) * ld;
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            const V q = *reinterpret_cast<const V*>(colp + (gt + v * GS) * VN);
            TA e[VN];
            Vec16<TA>::unpack(q, e);
#pragma unroll
            for (int uu = 0; uu < VN; ++uu)
#pragma unroll
              for (int j = 0; j < MG; ++j)
                gr[v * VN + uu][j] = fma(wk[j], static_cast<TC>(e[uu]), gr[v * VN + uu][j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[uslot]);
      if (++uslot == S) uslot = 0;
    }
  }

  // ---- epilogue: per-CTA partial G, layout [MG][ld] ----
  double* pg = a.part_g + size_t(blockIdx.x) * MG * ld;
  if (NG == 1) {
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      const int r0 = (gt + v * GS) * VN;
#pragma unroll
      for (int e = 0; e < VN; ++e)
        if (r0 + e < ld)
#pragma unroll
          for (int j = 0; j < MG; ++j) pg[size_t(j) * ld + r0 + e] = static_cast<double>(gr[v * VN + e][j]);
    }
  } else {
    named_bar_sync(1, kSweepWorkers);
    double* scratch = reinterpret_cast<double*>(ring);  // [NG][MG][ld]
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      const int r0 = (gt + v * GS) * VN;
#pragma unroll
      for (int e = 0; e < VN; ++e)
        if (r0 + e < ld)
#pragma unroll
          for (int j = 0; j < MG; ++j)
            scratch[(size_t(grp) * MG + j) * ld + r0 + e] = static_cast<double>(gr[v * VN + e][j]);
    }
    named_bar_sync(1, kSweepWorkers);
    for (int r = tid; r < MG * ld; r += kSweepWorkers) {
      double t = 0.0;
#pragma unroll
      for (int g = 0; g < NG; ++g) t += scratch[size_t(g) * MG * ld + r];
      pg[r] = t;
    }
  }
}

// ------------------------------------------------------------- polar step

constexpr int kPolarThreads = 1024;

// ---- accurate polar factor: Householder QR of G, one-sided Jacobi SVD of
// the m x m R, X = Q (U_r V_r').  Singular values carry LAPACK-grade
// absolute accuracy (eps * s_0), so the reference rank rule
// s > s_0 max(p, m) eps (block.py:145-147) decides like dgesdd does; no
// Gram matrix is formed (it would square the condition number).

struct PolarScratch {
  double* R;    // m*m  column-major (R[c*m + r])
  double* Vr;   // m*m  right singular vectors
  double* tau;  // m    Householder scalars
  double* red;  // 64   block-reduction scratch
  double* cs;   // 2*32 rotation (c, s) per pair
  int* pairs;   // 2*32
};

__host__ __device__ inline size_t polar_smem_bytes(int m) {
  return (size_t(2) * m * m + m + 64 + 64) * sizeof(double) + 64 * sizeof(int) + 64;
}

// Block-wide sum (any blockDim multiple of 32, <= 1024), fixed order.
__device__ double block_sum_any(double v, double* red) {
  v = warp_sum(v);
  const int tid = threadIdx.x, nw = blockDim.x >> 5;
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid < 32) {
    double u = tid < nw ? red[tid] : 0.0;
    u = warp_sum(u);
    if (tid == 0) red[32] = u;
  }
  __syncthreads();
  return red[32];
}

// In-place Householder QR of H ([m][ld], rows >= p_true are zero): on exit
// R (m x m) in smem, reflectors v_j stored in H[j][j..], tau_j in smem.
__device__ void householder_qr(double* H, int ld, int p_true, int m, PolarScratch sp) {
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int i = tid; i < m * m; i += nt) sp.R[i] = 0.0;
  for (int j = 0; j < m; ++j) {
    double* hj = H + size_t(j) * ld;
    double t = 0.0;
    for (int r = j + tid; r < p_true; r += nt) t = fma(hj[r], hj[r], t);
    const double nrm2 = block_sum_any(t, sp.red);
    const double x0 = hj[j];
    const double nrm = sqrt(nrm2);
    double alpha = 0.0, tauj = 0.0;
    if (nrm > 0.0) {
      alpha = x0 >= 0.0 ? -nrm : nrm;
      const double v0 = x0 - alpha;
      // v = [v0, x_1..]; tau = 2 / (v'v), v'v = nrm2 - x0^2 + v0^2
      const double vtv = nrm2 - x0 * x0 + v0 * v0;
      tauj = vtv > 0.0 ? 2.0 / vtv : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
      hj[j] = x0 - alpha;  // v0 (v stored unnormalised)
      sp.tau[j] = tauj;
      sp.R[j * m + j] = (nrm > 0.0) ? alpha : x0;
    }
    __syncthreads();
    // apply H_j to the trailing columns c > j
    for (int c = j + 1 + warp; c < m; c += nw) {
      double* hc = H + size_t(c) * ld;
      double w = 0.0;
      for (int r = j + lane; r < p_true; r += 32) w = fma(hj[r], hc[r], w);
      w = warp_sum(w) * tauj;
      for (int r = j + lane; r < p_true; r += 32) hc[r] = fma(-w, hj[r], hc[r]);
    }
    __syncthreads();
    for (int c = j + 1 + tid; c < m; c += nt) sp.R[c * m + j] = H[size_t(c) * ld + j];
    __syncthreads();
  }
}

// One-sided Jacobi SVD of R (m x m column-major in smem): rotates column
// pairs until mutually orthogonal; Vr accumulates the rotations.  Returns
// with R's columns = U_r * diag(s).
__device__ void onesided_jacobi(int m, PolarScratch sp, int max_sweeps) {
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int i = tid; i < m * m; i += nt) sp.Vr[i] = (i / m == i % m) ? 1.0 : 0.0;
  const int mp = (m + 1) & ~1;
  __shared__ int s_rot;
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int step = 0; step < mp - 1; ++step) {
      for (int i = warp; i < mp / 2; i += nw) {
        int p = (i == 0) ? 0 : 1 + (i - 1 + step) % (mp - 1);
        int q = 1 + (mp - 2 - i + step) % (mp - 1);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= m) continue;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int r = lane; r < m; r += 32) {
          const double rp = sp.R[p * m + r], rq = sp.R[q * m + r];
          a = fma(rp, rp, a);
          b = fma(rq, rq, b);
          g = fma(rp, rq, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        // rotate unless the pair is orthogonal to working precision (the
        // computed g carries ~m eps sqrt(ab) of rounding itself; a tighter
        // test never converges and runs every sweep to max_sweeps)
        if (g != 0.0 && fabs(g) > double(m) * 2.220446049250313e-16 * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < m; r += 32) {
            const double rp = sp.R[p * m + r], rq = sp.R[q * m + r];
            sp.R[p * m + r] = c * rp - s * rq;
            sp.R[q * m + r] = s * rp + c * rq;
            const double vp = sp.Vr[p * m + r], vq = sp.Vr[q * m + r];
            sp.Vr[p * m + r] = c * vp - s * vq;
            sp.Vr[q * m + r] = s * vp + c * vq;
          }
          if (lane == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    if (s_rot == 0) break;
    __syncthreads();
  }
  __syncthreads();
}

// X = polar(G).  G is destroyed (holds the reflectors).  Returns the rank.
__device__ int polar_device(double* G, double* X, int ld, int p_true, int m, PolarScratch sp) {
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  householder_qr(G, ld, p_true, m, sp);
  onesided_jacobi(m, sp, 60);
  __shared__ int s_rank;
  if (tid == 0) {
    double smax = 0.0;
    for (int j = 0; j < m; ++j) {
      double t = 0.0;
      for (int r = 0; r < m; ++r) t += sp.R[j * m + r] * sp.R[j * m + r];
      smax = fmax(smax, sqrt(t));
    }
    const double cutoff = smax * double(p_true > m ? p_true : m) * 2.220446049250313e-16;
    int rank = 0;
    if (smax > 0.0)
      for (int j = 0; j < m; ++j) {
        double t = 0.0;
        for (int r = 0; r < m; ++r) t += sp.R[j * m + r] * sp.R[j * m + r];
        rank += sqrt(t) > cutoff;
      }
    s_rank = rank;
  }
  __syncthreads();
  const int rank = s_rank;
  if (rank < m) return rank;
  // U_r = R / s (column-wise), Y = U_r V_r' stored in R's place via X rows 0..m-1
  for (int j = warp; j < m; j += nw) {
    double t = 0.0;
    for (int r = lane; r < m; r += 32) t = fma(sp.R[j * m + r], sp.R[j * m + r], t);
    t = sqrt(warp_sum(t));
    for (int r = lane; r < m; r += 32) sp.R[j * m + r] /= t;
  }
  __syncthreads();
  // X[:, c] = Q [Y[:, c]; 0],  Y[r][c] = sum_k U[r][k] V[c][k]
  for (size_t e = tid; e < size_t(m) * ld; e += nt) {
    const int c = static_cast<int>(e / ld), r = static_cast<int>(e % ld);
    double y = 0.0;
    if (r < m)
      for (int k = 0; k < m; ++k) y = fma(sp.R[k * m + r], sp.Vr[k * m + c], y);
    X[e] = y;
  }
  __syncthreads();
  for (int j = m - 1; j >= 0; --j) {
    const double* hj = G + size_t(j) * ld;
    const double tj = sp.tau[j];
    for (int c = warp; c < m; c += nw) {
      double* xc = X + size_t(c) * ld;
      double w = 0.0;
      for (int r = j + lane; r < p_true; r += 32) w = fma(hj[r], xc[r], w);
      w = warp_sum(w) * tj;
      for (int r = j + lane; r < p_true; r += 32) xc[r] = fma(-w, hj[r], xc[r]);
    }
    __syncthreads();
  }
  return rank;
}

__device__ inline PolarScratch polar_scratch(double* psm, int m) {
  PolarScratch sp;
  sp.R = psm;
  sp.Vr = psm + m * m;
  sp.tau = psm + 2 * m * m;
  sp.red = sp.tau + m;
  sp.cs = sp.red + 64;
  sp.pairs = reinterpret_cast<int*>(sp.cs + 64);
  return sp;
}

// ||X'X - I||_F of the device iterate X ([m][ld], zero rows >= p) by one CTA
// (fixed order; M: m*m doubles of shared scratch).  The reference builds a
// StiefelPoint -- ||X'X - I||_F <= 1e-10 (core.py:113-129) -- from every
// polar output (block.py:149); the loops record this per iteration.
__device__ double gram_error_from(const double* M, int m, double* red) {
  double t = 0.0;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const double d = M[e] - ((e / m == e % m) ? 1.0 : 0.0);
    t = fma(d, d, t);
  }
  return sqrt(block_sum_any(t, red));
}
__device__ void gram_mm(const double* P, const double* Q, int ld, int m, double* M, bool symmetric);
__device__ double stiefel_error(const double* X, int ld, int m, double* M) {
  __shared__ double red[40];
  __syncthreads();
  gram_mm(X, X, ld, m, M, true);
  __syncthreads();
  return gram_error_from(M, m, red);
}

constexpr double kStiefelTol = 1e-10;  // core.py:22 STIEFEL_TOL

// End of a block step (thread 0): rank loss stops the loop with status 2
// (block.py:144-148, RankDeficiencyError); an iterate off the Stiefel
// manifold stops it with status 3 (the reference's StiefelPoint raises
// ValueError); otherwise the error is recorded, the loop advances and the
// near-threshold list of the next sweep is cleared.
__device__ void bk_advance(GpsCtl* ctl, int k, int m, int rank, double err, int* rank_out, BandLog* band,
                           double* stiefel) {
  if (rank < m) {
    ctl->done = 1;
    ctl->converged = 0;
    ctl->status = 2;
    *rank_out = rank;
    return;
  }
  if (stiefel != nullptr) stiefel[k + 1] = err;
  if (!(err <= kStiefelTol)) {
    ctl->done = 1;
    ctl->converged = 0;
    ctl->status = 3;
    return;
  }
  if (band != nullptr) band->count[(k + 1) & 1] = 0;
  ctl->iter = k + 1;
}

// ||M - I||_F of a reduced m x m Gram (one CTA).
__global__ void gram_error_kernel(const double* __restrict__ M, int m, double* out) {
  __shared__ double red[40];
  const double e = gram_error_from(M, m, red);
  if (threadIdx.x == 0) *out = e;
}

// One-CTA record of X_0's Stiefel error (init; block.py:202).
__global__ void __launch_bounds__(kPolarThreads) stiefel_error_kernel(const double* X, int ld, int m,
                                                                      double* out) {
  extern __shared__ double psm[];
  const double e = stiefel_error(X, ld, m, psm);
  if (threadIdx.x == 0) *out = e;
}

// Block power step (block.py:211-226) on the reduced exchange vectors of the
// ng groups: exch layout [ng][MG*ld + 4].  History, stopping rule, then
// G_j = 2 mu_j sum(...) and X_{k+1} = polar(G); rank loss stops the loop with
// status 2 and the rank in ctl->gnorm's slot (as int via status field).
__global__ void __launch_bounds__(kPolarThreads) bk_step_kernel(const double* __restrict__ exch, int ng, int mg,
                                                               int ld, int p_true, int m, const double* __restrict__ mu,
                                                               double* __restrict__ Xbuf, int64_t x_stride,
                                                               double* __restrict__ Gbuf, double* __restrict__ Tbuf,
                                                               double* __restrict__ hist, GpsCtl* ctl, double tol,
                                                               int max_iter, int* rank_out, BandLog* band,
                                                               double* __restrict__ stiefel) {
  extern __shared__ double psm[];
  __shared__ int decision;
  if (ctl->done) return;
  const int k = ctl->iter;
  const int tid = threadIdx.x;
  const size_t gstride = size_t(mg) * ld + 4;
  if (tid == 0) {
    double f = 0.0;
    for (int g = 0; g < ng; ++g) f += exch[g * gstride + size_t(mg) * ld];
    hist[k] = f;
    const double f_prev = ctl->f_prev;
    int d = 0;
    if (k >= 1 && fabs(f - f_prev) < tol * fmax(fabs(f_prev), 1e-30)) d = 1;
    else if (k >= max_iter) d = 2;
    decision = d;
    ctl->f_prev = f;
  }
  __syncthreads();
  if (decision != 0) {
    if (tid == 0) {
      ctl->done = 1;
      ctl->converged = decision == 1;
    }
    return;
  }
  // assemble G (m x ld) with the 2 mu_j factor (block.py:119-120)
  for (size_t e = tid; e < size_t(m) * ld; e += blockDim.x) {
    const int j = static_cast<int>(e / ld), r = static_cast<int>(e % ld);
    const int g = j / mg, jj = j % mg;
    Gbuf[e] = 2.0 * mu[j] * exch[g * gstride + size_t(jj) * ld + r];
  }
  __syncthreads();
  double* Xn = Xbuf + ((k + 1) & 1) * x_stride;
  const int rank = polar_device(Gbuf, Xn, ld, p_true, m, polar_scratch(psm, m));
  const double err = rank < m ? 0.0 : stiefel_error(Xn, ld, m, psm);
  if (tid == 0) bk_advance(ctl, k, m, rank, err, rank_out, band, stiefel);
}

// One-shot polar (block.py:135-149 polar_projection) on device buffers.
__global__ void __launch_bounds__(kPolarThreads) polar_kernel(double* G, double* X, int ld, int p_true, int m,
                                                              int* rank_out) {
  extern __shared__ double psm[];
  const int rank = polar_device(G, X, ld, p_true, m, polar_scratch(psm, m));
  if (threadIdx.x == 0) *rank_out = rank;
}

// M[a][b] = sum_r P[a][r] * Q[b][r] for a, b < m (both [m][ld]); warp-per-
// entry dot products in a fixed lane order.  M is m x m in shared memory.
__device__ void gram_mm(const double* P, const double* Q, int ld, int m, double* M, bool symmetric) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = warp; e < m * m; e += nw) {
    const int a = e / m, b = e % m;
    if (symmetric && b < a) continue;
    double t = 0.0;
    for (int r = lane; r < ld; r += 32) t = fma(P[size_t(a) * ld + r], Q[size_t(b) * ld + r], t);
    t = warp_sum(t);
    if (lane == 0) {
      M[a * m + b] = t;
      if (symmetric) M[b * m + a] = t;
    }
  }
}

// CholeskyQR2 (block.py:152-171 init): Q = M R^{-1} with R from the Cholesky
// factor of M'M, applied twice; R has a positive diagonal, so Q equals the
// reference's sign-fixed Householder Q.  status_out: 0 ok, 1 not decided
// here (Cholesky breakdown or r_jj spread > 1e6): the caller runs the
// Householder QR, which applies the reference's rank rule.
__global__ void __launch_bounds__(kPolarThreads) cholqr2_kernel(double* Mbuf, double* Q, int ld, int m,
                                                                int* status_out) {
  extern __shared__ double psm[];
  double* Gm = psm;          // m*m Gram, then R (upper)
  double* Rt = psm + m * m;  // accumulated R of pass 1 (for the rank test)
  const int tid = threadIdx.x;
  __shared__ int bad;
  for (int pass = 0; pass < 2; ++pass) {
    const double* src = pass == 0 ? Mbuf : Q;
    gram_mm(src, src, ld, m, Gm, true);
    __syncthreads();
    if (tid == 0) {
      bad = 0;
      // in-place Cholesky: Gm = R' R, R upper stored in Gm[i][j] (i <= j)
      for (int j = 0; j < m && !bad; ++j) {
        double d = Gm[j * m + j];
        for (int k = 0; k < j; ++k) d -= Gm[k * m + j] * Gm[k * m + j];
        if (!(d > 0.0)) {
          bad = 1;
          break;
        }
        const double rjj = sqrt(d);
        Gm[j * m + j] = rjj;
        for (int c = j + 1; c < m; ++c) {
          double t = Gm[j * m + c];
          for (int k = 0; k < j; ++k) t -= Gm[k * m + j] * Gm[k * m + c];
          Gm[j * m + c] = t / rjj;
        }
      }
      if (!bad && pass == 0) {
        // trust the Gram-based factor only well inside Cholesky's range:
        // near kappa(M) ~ 1e8 rounding can make a pivot of an exactly
        // rank-deficient M positive, so r_jj spread beyond 1e6 hands the
        // decision to the Householder path (hh_init_kernel)
        double mx = 0.0, mn = INFINITY;
        for (int j = 0; j < m; ++j) {
          mx = fmax(mx, fabs(Gm[j * m + j]));
          mn = fmin(mn, fabs(Gm[j * m + j]));
        }
        if (!(mn > 1e-6 * mx)) bad = 1;
      }
      for (int i = 0; i < m * m; ++i) Rt[i] = Gm[i];
    }
    __syncthreads();
    if (bad) {
      if (tid == 0) *status_out = 1;
      return;
    }
    // Q[:, j] = (src[:, j] - sum_{k<j} Q[:, k] R[k][j]) / R[j][j]  (row-parallel forward substitution)
    for (int r = tid; r < ld; r += blockDim.x) {
      double qv[64];
      for (int j = 0; j < m; ++j) {
        double t = src[size_t(j) * ld + r];
        for (int k = 0; k < j; ++k) t -= qv[k] * Rt[k * m + j];
        qv[j] = t / Rt[j * m + j];
      }
      for (int j = 0; j < m; ++j) Q[size_t(j) * ld + r] = qv[j];
    }
    __syncthreads();
  }
  if (tid == 0) *status_out = 0;
}

// Householder QR initialisation (block.py:162-170 exactly): R's diagonal
// decides rank deficiency by the reference rule |r_jj| <= m eps
// max(1, max_i |r_ii|) (status 1 -> ValueError), otherwise
// Q = H_1 ... H_m [I; 0] diag(sign r_jj), the reference's sign-fixed Q.
// Used when CholeskyQR2 breaks down or misses the Stiefel tolerance
// (kappa(M) beyond ~1e8), where the Gram-based rank test would reject
// matrices the reference accepts.  M is destroyed (reflectors).
__global__ void __launch_bounds__(kPolarThreads) hh_init_kernel(double* M, double* Q, int ld, int p_true, int m,
                                                                int* status_out) {
  extern __shared__ double psm[];
  PolarScratch sp = polar_scratch(psm, m);
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  householder_qr(M, ld, p_true, m, sp);
  __shared__ int bad;
  if (tid == 0) {
    double mx = 1.0;
    for (int j = 0; j < m; ++j) mx = fmax(mx, fabs(sp.R[j * m + j]));
    int b = 0;
    for (int j = 0; j < m; ++j)
      if (fabs(sp.R[j * m + j]) <= m * 2.220446049250313e-16 * mx) b = 1;
    bad = b;
    *status_out = b;
  }
  __syncthreads();
  if (bad) return;
  for (size_t e = tid; e < size_t(m) * ld; e += nt) {
    const int c = static_cast<int>(e / ld), r = static_cast<int>(e % ld);
    const double d = sp.R[c * m + c];
    Q[e] = (r == c) ? (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) : 0.0;
  }
  __syncthreads();
  for (int j = m - 1; j >= 0; --j) {
    const double* hj = M + size_t(j) * ld;
    const double tj = sp.tau[j];
    for (int c = warp; c < m; c += nw) {
      double* qc = Q + size_t(c) * ld;
      double w = 0.0;
      for (int r = j + lane; r < p_true; r += 32) w = fma(hj[r], qc[r], w);
      w = warp_sum(w) * tj;
      for (int r = j + lane; r < p_true; r += 32) qc[r] = fma(-w, hj[r], qc[r]);
    }
    __syncthreads();
  }
}

}  // namespace gps
