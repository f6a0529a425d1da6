// Block GP-SPCA on the 5th-generation tensor cores (sm_100a tcgen05), for
// m >= 16 components (p = 8192, m = 64) where the CUDA-core
// block sweep would need ceil(m/MG) reads of A per iteration.
//
// T0 split_x:   X (fp64) -> X_hi = tf32(X), X_lo = tf32(X - X_hi)  (fp32, [m_pad][ld])
// T1 tc_dots:   persistent; per tile of 128 columns the correlations
//               C_tile = A_tile' X (M = 128 columns, N = m_pad, K = p) are
//               accumulated in TMEM by tcgen05.mma kind::tf32 in 3xTF32
//               form (A_hi X_hi + A_hi X_lo + A_lo X_hi, ~fp32 accuracy);
//               A and X chunks arrive by TMA (2-D tensor maps, 128-byte
//               swizzle), A_lo is split in shared memory by converter warps,
//               and the epilogue warps read TMEM (tcgen05.ld), apply mu_j,
//               the threshold and the objective in fp64, write W and a per-
//               column activity flag.  A is read from HBM once.
// T2 tc_update: G_j = sum over ACTIVE columns of w_ij a_i (fp64), row chunks
//               x component groups; reads only the active columns again.
// Roles of T1 (12 warps): w0 TMA producer, w1 MMA issuer (+TMEM owner),
// w4-7 epilogue (warp % 4 selects the TMEM lane quarter), w8-11 converters.
#pragma once

#include <cuda.h>

#include "su_kernels.cuh"

namespace gps {

constexpr int kTcTileM = 128;    // columns of A per tile (MMA M)
constexpr int kTcKChunk = 32;    // rows of A per stage (128 bytes of fp32)
constexpr int kTcStages = 4;
constexpr int kTcThreads = 384;  // 12 warps
constexpr int kTcMaxN = 64;
constexpr int kTcMinM = 16;      // block solves with m >= 16 (fp32 A) take this path
constexpr int kTcConvThreads = 128;  // converter warps 8-11
constexpr int kTcSegChunks = 2;  // TMEM accumulation segment: 2 chunks = 64 rows, drained to fp64

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 bytes (SBO), version 1 (Blackwell).
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem_ptr) {
  const uint32_t addr = smem_u32(smem_ptr);
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);          // start address
  d |= uint64_t(1) << 16;                       // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;               // SBO = 1024 B
  d |= uint64_t(1) << 46;                       // version
  d |= uint64_t(2) << 61;                       // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// T0: X (fp64 [m][ld], parity slot) -> X_hi / X_lo (fp32 [n_pad][ld], zero
// padded components).
__global__ void tc_split_x_kernel(const double* __restrict__ X, int64_t x_par_stride, int m, int n_pad, int ld,
                                  float* __restrict__ xhi, float* __restrict__ xlo, const GpsCtl* ctl) {
  if (ctl != nullptr && ctl->done) return;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const double* Xp = X + parity * x_par_stride;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < int64_t(n_pad) * ld;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / ld);
    const double x = j < m ? Xp[e] : 0.0;
    const float xf = static_cast<float>(x);
    const float hi = __uint_as_float(__float_as_uint(xf) & 0xFFFFE000u);
    const float lo = static_cast<float>(x - static_cast<double>(hi));
    xhi[e] = hi;
    xlo[e] = lo;
  }
}

struct TcDotsArgs {
  int64_t n;
  int ld;
  int m;       // real components
  int n_pad;   // MMA N (multiple of 16)
  int penalty;
  const double* gamma;  // m
  const double* mu;     // m
  double* w_out;        // [m_pad][n] parity slots (may be null)
  int64_t w_stride;
  unsigned char* colmask;  // n: 1 if any w_ij != 0
  double* part_s;          // [grid][4]
  const GpsCtl* ctl;
  int num_tiles;
};

__host__ __device__ inline size_t tc_stage_bytes(int n_pad) {
  return size_t(2) * kTcTileM * kTcKChunk * 4 + size_t(2) * n_pad * kTcKChunk * 4;
}
__host__ __device__ inline size_t tc_smem_bytes(int n_pad) {
  return 1024 /*align slack*/ + kTcStages * tc_stage_bytes(n_pad) + 4096 /*barriers, params*/;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_dots_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
                   const __grid_constant__ CUtensorMap tmXl, const TcDotsArgs a) {
  extern __shared__ unsigned char smem_raw[];
  if (a.ctl != nullptr && a.ctl->done) return;
  const int parity = a.ctl != nullptr ? (a.ctl->iter & 1) : 0;
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NP = a.n_pad;
  const size_t a_bytes = size_t(kTcTileM) * kTcKChunk * 4;   // 16 KB
  const size_t x_bytes = size_t(NP) * kTcKChunk * 4;
  const size_t stage_bytes = 2 * a_bytes + 2 * x_bytes;
  unsigned char* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * stage_bytes);
  uint64_t* conv = full + kTcStages;
  uint64_t* empty = conv + kTcStages;
  uint64_t* tfull = empty + kTcStages;  // 2 accumulator buffers
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  double* sgam = reinterpret_cast<double*>(tmem_base_slot + 4);
  double* smu = sgam + kTcMaxN;
  double* sred = smu + kTcMaxN;  // 128 x 2 scalars (f, nnz)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kchunks = a.ld / kTcKChunk;
  const uint32_t idesc = umma_idesc_tf32(kTcTileM, NP);

  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], 4);   // 4 converter warps
      mbar_init(&empty[i], 1);  // tcgen05.commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);   // tcgen05.commit
      mbar_init(&tempty[i], 4);  // 4 epilogue warps
    }
    fence_mbar_init();
  }
  for (int j = tid; j < a.m; j += blockDim.x) {
    sgam[j] = a.gamma[j];
    smu[j] = a.mu[j];
  }
  if (warp == 1) {
    // 2 accumulator buffers of NP columns; allocation is a power of two >= 32
    const uint32_t cols = (2 * NP <= 32) ? 32 : (2 * NP <= 64) ? 64 : 128;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmXh);
    tma_prefetch(&tmXl);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  // my tiles: blockIdx.x, blockIdx.x + grid, ...
  const int my_tiles = a.num_tiles > int(blockIdx.x) ? (a.num_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int total_chunks = my_tiles * kchunks;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int c = 0; c < total_chunks; ++c) {
        if (c >= kTcStages) mbar_wait_sleep(&empty[stage], ph ^ 1u);
        const int t = int(blockIdx.x) + (c / kchunks) * int(gridDim.x);
        const int kc = c % kchunks;
        unsigned char* st = stages + stage * stage_bytes;
        mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(a_bytes + 2 * x_bytes));
        tma_load_2d(st, &tmA, kc * kTcKChunk, t * kTcTileM, &full[stage]);
        tma_load_2d(st + 2 * a_bytes, &tmXh, kc * kTcKChunk, 0, &full[stage]);
        tma_load_2d(st + 2 * a_bytes + x_bytes, &tmXl, kc * kTcKChunk, 0, &full[stage]);
        if (++stage == kTcStages) {
          stage = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // Accumulate kTcSegChunks chunks (256 rows of A) per TMEM segment; the
    // epilogue drains each segment into fp64, so the tensor core's fp32
    // accumulation never spans more than 256 rows.
    int stage = 0;
    uint32_t ph = 0;
    int seg = 0;
    for (int tt = 0; tt < my_tiles; ++tt) {
      for (int k0 = 0; k0 < kchunks; k0 += kTcSegChunks, ++seg) {
        const int b = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[b], static_cast<uint32_t>(((seg - 2) >> 1) & 1));
        tc_fence_after();
        const uint32_t dtm = tmem_base + uint32_t(b * NP);
        const int k1 = (k0 + kTcSegChunks < kchunks) ? k0 + kTcSegChunks : kchunks;
        for (int kc = k0; kc < k1; ++kc) {
          mbar_wait(&conv[stage], ph);
          tc_fence_after();
          unsigned char* st = stages + stage * stage_bytes;
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < kTcKChunk / 8; ++k) {
              const uint64_t ah = umma_desc_sw128(st) + uint64_t((k * 32) >> 4);
              const uint64_t al = umma_desc_sw128(st + a_bytes) + uint64_t((k * 32) >> 4);
              const uint64_t bh = umma_desc_sw128(st + 2 * a_bytes) + uint64_t((k * 32) >> 4);
              const uint64_t bl = umma_desc_sw128(st + 2 * a_bytes + x_bytes) + uint64_t((k * 32) >> 4);
              const uint32_t first = (kc == k0 && k == 0) ? 0u : 1u;
              umma_tf32(dtm, al, bh, idesc, first);
              umma_tf32(dtm, ah, bl, idesc, 1u);
              umma_tf32(dtm, ah, bh, idesc, 1u);
            }
            umma_commit(&empty[stage]);
            if (kc == k1 - 1) umma_commit(&tfull[b]);
          }
          __syncwarp();
          if (++stage == kTcStages) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------- converter warps
    const int ct = tid - 8 * 32;  // 0..127
    int stage = 0;
    uint32_t ph = 0;
    for (int c = 0; c < total_chunks; ++c) {
      mbar_wait(&full[stage], ph);
      // The MMA reads tf32 operands by dropping the low 13 mantissa bits, so
      // A itself serves as A_hi; A_lo = A - trunc_tf32(A) is exact in fp32
      // (two integer/FP ops per element, no conversion-pipe traffic).
      const float* Ah = reinterpret_cast<const float*>(stages + stage * stage_bytes);
      float* Al = reinterpret_cast<float*>(stages + stage * stage_bytes) + kTcTileM * kTcKChunk;
#pragma unroll 4
      for (int i = ct * 4; i < kTcTileM * kTcKChunk; i += kTcConvThreads * 4) {
        const float4 v = *reinterpret_cast<const float4*>(Ah + i);
        float4 l;
        l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        *reinterpret_cast<float4*>(Al + i) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[stage]);
      if (++stage == kTcStages) {
        stage = 0;
        ph ^= 1u;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------ epilogue warps
    const int q = warp & 3;  // TMEM lane quarter
    const int et = tid - 4 * 32;
    double f_acc = 0.0, nnz_acc = 0.0;
    double* wbase = a.w_out != nullptr ? a.w_out + parity * a.w_stride : nullptr;
    int seg = 0;
    for (int tt = 0; tt < my_tiles; ++tt) {
      const int t = int(blockIdx.x) + tt * int(gridDim.x);
      double c[kTcMaxN];
#pragma unroll
      for (int j = 0; j < kTcMaxN; ++j) c[j] = 0.0;
      for (int k0 = 0; k0 < kchunks; k0 += kTcSegChunks, ++seg) {
        const int b = seg & 1;
        mbar_wait(&tfull[b], static_cast<uint32_t>((seg >> 1) & 1));
        tc_fence_after();
#pragma unroll
        for (int j0 = 0; j0 < kTcMaxN; j0 += 16) {
          if (j0 < NP) {
            float v[16];
            tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(b * NP + j0), v);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 16; ++u) c[j0 + u] += static_cast<double>(v[u]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
      const int64_t col = int64_t(t) * kTcTileM + q * 32 + lane;
      if (col < a.n) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < kTcMaxN; ++j) {
          if (j >= a.m) break;
          const double sj = smu[j] * c[j];
          const double w = threshold_weight(sj, sgam[j], a.penalty);
          f_acc += objective_term(sj, sgam[j], a.penalty);
          if (w != 0.0) {
            nnz_acc += 1.0;
            any = true;
          }
          if (wbase != nullptr) wbase[size_t(j) * a.n + col] = w;
        }
        a.colmask[col] = any ? 1 : 0;
      }
    }
    sred[et * 2 + 0] = f_acc;
    sred[et * 2 + 1] = nnz_acc;
  }
  __syncthreads();
  if (tid < 2) {
    double t = 0.0;
    for (int i = 0; i < 128; ++i) t += sred[i * 2 + tid];
    a.part_s[size_t(blockIdx.x) * 4 + tid] = t;
  }
  if (warp == 1) {
    const uint32_t cols = (2 * NP <= 32) ? 32 : (2 * NP <= 64) ? 64 : 128;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(cols) : "memory");
  }
}

// T2: sparse rank-m update on the ACTIVE columns (colmask), fp64.
// grid (GX, ceil(ld / 1024), ceil(m / 8)); CTA (b, y, z) owns columns
// [b n / GX, (b+1) n / GX), rows [y*1024, +1024) and components [8z, 8z+8)
// of part_g[b] ([m_pad][ld]).
constexpr int kTcUpdRows = 1024;
constexpr int kTcUpdComps = 8;
__global__ void __launch_bounds__(256) tc_update_kernel(const float* __restrict__ A, int64_t n, int ld, int m,
                                                        const unsigned char* __restrict__ colmask,
                                                        const double* __restrict__ W, int64_t w_par_stride,
                                                        int m_pad, double* __restrict__ part_g, const GpsCtl* ctl) {
  constexpr int RPT = kTcUpdRows / 256;
  if (ctl != nullptr && ctl->done) return;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const double* Wp = W + parity * w_par_stride;
  const int64_t c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  const int r0 = blockIdx.y * kTcUpdRows;
  const int j0 = blockIdx.z * kTcUpdComps;
  double g[kTcUpdComps][RPT];
#pragma unroll
  for (int j = 0; j < kTcUpdComps; ++j)
#pragma unroll
    for (int k = 0; k < RPT; ++k) g[j][k] = 0.0;
  __shared__ unsigned char flags[256];
  for (int64_t base = c0; base < c1; base += 256) {
    // cheap skip of fully inactive 256-column chunks (the common case)
    const int64_t mine = base + threadIdx.x;
    const unsigned char f = mine < c1 ? colmask[mine] : 0;
    if (!__syncthreads_or(f)) continue;
    flags[threadIdx.x] = f;
    __syncthreads();
    const int cnt = (c1 - base) < 256 ? static_cast<int>(c1 - base) : 256;
    for (int k = 0; k < cnt; ++k) {
      if (!flags[k]) continue;
      const int64_t col = base + k;
      double w[kTcUpdComps];
#pragma unroll
      for (int j = 0; j < kTcUpdComps; ++j) w[j] = (j0 + j < m) ? Wp[size_t(j0 + j) * n + col] : 0.0;
      const float* ac = A + col * ld;
#pragma unroll
      for (int kk = 0; kk < RPT; ++kk) {
        const int r = r0 + kk * 256 + threadIdx.x;
        const double v = r < ld ? static_cast<double>(ac[r]) : 0.0;
#pragma unroll
        for (int j = 0; j < kTcUpdComps; ++j) g[j][kk] = fma(w[j], v, g[j][kk]);
      }
    }
    __syncthreads();
  }
  double* pg = part_g + size_t(blockIdx.x) * m_pad * ld;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = r0 + k * 256 + threadIdx.x;
    if (r < ld)
#pragma unroll
      for (int j = 0; j < kTcUpdComps; ++j)
        if (j0 + j < m_pad) pg[size_t(j0 + j) * ld + r] = g[j][k];
  }
}

}  // namespace gps
