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
// Roles of T1 (12 warps): w0 A producer (TMA), w1 MMA issuer (+TMEM owner),
// w2 X producer (TMA), w4-7 epilogue (warp % 4 selects the TMEM lane quarter), w8-11 converters.
#pragma once

#include <cuda.h>

#include "su_kernels.cuh"

namespace gps {

constexpr int kTcTileM = 128;    // columns of A per tile (MMA M)
constexpr int kTcKChunk = 32;    // rows of A per stage (128 bytes of fp32)
constexpr int kTcAStages = 10;  // default A ring depth (HBM stream)
constexpr int kTcLoStages = 2;  // default TMEM A_hi / A_lo slots (converter output)
constexpr int kTcXStages = 3;   // default X_hi | X_lo ring depth (L2-resident)
constexpr int kTcMaxStages = 16;
constexpr int kTcThreads = 384;  // 12 warps
constexpr int kTcMaxN = 64;
constexpr int kTcMinM = 5;       // block solves with m >= 5 (fp32 A) take this path (one A read vs ceil(m/4))
constexpr int kTcConvThreads = 128;  // converter warps 8-11
constexpr int kTcSegChunks = 4;  // TMEM accumulation segment: 4 chunks = 128 rows, drained to fp64

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

// Warp-converged forms: every lane executes the call with identical
// operands and elect.sync picks the issuing lane inside the asm, so the
// compiler keeps descriptors in uniform registers (a single-thread branch
// instead costs a per-instruction R2UR + waterfall loop, ~90 clocks/MMA).
__device__ __forceinline__ void umma_tf32_warp(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
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
  int a_stages, lo_stages, x_stages;  // ring depths (<= kTcMaxStages)
  int seg_chunks;                     // chunks per TMEM accumulation segment
  int probe;  // timing experiments: 1 no A_lo, 2 one MMA, 4 no TMEM drain, 8 no X loads,
              // 16 no update, 32 no TMEM stores, 64 cycle accounting
};

// Operand staging of T1.  Shared memory is the scarce resource (every
// tcgen05.mma operand read from shared memory, every TMA write and every
// converter access share its ~128 B/clock), so A passes through it once:
//   A ring    SA x 16 KB in shared memory (TMA, evict-first) -> converters
//   A_hi/A_lo SL slots x 64 TMEM columns, written by the converters with
//             tcgen05.st, read by the MMAs as the TMEM-resident A operand
//   X ring    SX x (X_hi | X_lo) chunk in shared memory (TMA, evict-last)
// TMEM: columns [0, 4 NP) = 2 accumulator buffers of [A X_hi | A_hi X_lo],
// columns [256, 256 + 64 SL) = the A_hi / A_lo slots; 512 columns allocated.
constexpr uint32_t kTcTmemCols = 512;
constexpr uint32_t kTcTmemAOff = 256;
__host__ __device__ inline size_t tc_a_bytes() { return size_t(kTcTileM) * kTcKChunk * 4; }
__host__ __device__ inline size_t tc_x_bytes(int n_pad) { return size_t(n_pad) * kTcKChunk * 4; }
__host__ __device__ inline size_t tc_smem_bytes(int n_pad, int sa, int sl, int sx) {
  (void)sl;
  return 1024 /*align slack*/ + sa * tc_a_bytes() + sx * 2 * tc_x_bytes(n_pad) + 4096 /*barriers, params*/;
}

__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
      : "memory");
}

// tcgen05.mma with the A operand in TMEM (M = 128 lanes, K = 8 columns).
__device__ __forceinline__ void umma_tf32_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Optional per-role cycle accounting (tuning diagnostics, TcDotsArgs::probe & 64).
__device__ unsigned long long g_tc_prof[16];
struct TcProf {
  bool on;
  long long t;
  __device__ __forceinline__ void start() {
    if (on) t = clock64();
  }
  __device__ __forceinline__ void stop(unsigned long long& acc) {
    if (on) acc += static_cast<unsigned long long>(clock64() - t);
  }
};

// Ring cursor: slot index and the phase parity of its current use.
struct TcRing {
  int slot = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_dots_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
                   const __grid_constant__ CUtensorMap tmXl, const TcDotsArgs a) {
  extern __shared__ unsigned char smem_raw[];
  if (a.ctl != nullptr && a.ctl->done) return;
  const int parity = a.ctl != nullptr ? (a.ctl->iter & 1) : 0;
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NP = a.n_pad;
  const int SA = a.a_stages, SL = a.lo_stages, SX = a.x_stages;
  const int SEG = a.seg_chunks;
  const size_t a_bytes = tc_a_bytes();  // 16 KB
  const size_t x_bytes = tc_x_bytes(NP);
  unsigned char* aring = smem;
  unsigned char* xring = aring + SA * a_bytes;  // [stage][hi | lo]
  uint64_t* a_full = reinterpret_cast<uint64_t*>(xring + SX * 2 * x_bytes);
  uint64_t* a_empty = a_full + SA;
  uint64_t* lo_full = a_empty + SA;  // TMEM A_hi / A_lo slots
  uint64_t* lo_empty = lo_full + SL;
  uint64_t* x_full = lo_empty + SL;
  uint64_t* x_empty = x_full + SX;
  uint64_t* tfull = x_empty + SX;  // 2 accumulator buffers
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  double* sgam = reinterpret_cast<double*>(tmem_base_slot + 4);
  double* smu = sgam + kTcMaxN;
  double* sred = smu + kTcMaxN;  // 128 x 2 scalars (f, nnz)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kchunks = a.ld / kTcKChunk;
  // MMA 1: A_hi [X_hi | X_lo] (N = 2 NP, the X slot holds X_hi rows then X_lo rows);
  // MMA 2: A_lo X_hi (N = NP) accumulating into the first NP columns.
  const uint32_t idesc2 = umma_idesc_tf32(kTcTileM, 2 * NP);
  const uint32_t idesc1 = umma_idesc_tf32(kTcTileM, NP);

  if (tid == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 4);  // 4 converter warps have read the slot
    }
    for (int i = 0; i < SL; ++i) {
      mbar_init(&lo_full[i], 4);  // 4 converter warps stored their TMEM lanes
      mbar_init(&lo_empty[i], 1);  // tcgen05.commit
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "r"(kTcTmemCols)
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
    // ---------------------------------------------------------- A producer
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      TcRing r;
      TcProf pf{(a.probe & 64) != 0, 0};
      unsigned long long w0 = 0;
      int t = int(blockIdx.x), kc = 0;
      for (int c = 0; c < total_chunks; ++c) {
        pf.start();
        if (c >= SA) mbar_wait_sleep(&a_empty[r.slot], r.ph ^ 1u);
        pf.stop(w0);
        mbar_arrive_expect_tx(&a_full[r.slot], static_cast<uint32_t>(a_bytes));
        tma_load_2d_hint(aring + r.slot * a_bytes, &tmA, kc * kTcKChunk, t * kTcTileM, &a_full[r.slot], policy);
        r.next(SA);
        if (++kc == kchunks) {
          kc = 0;
          t += int(gridDim.x);
        }
      }
      if (pf.on) atomicAdd(&g_tc_prof[1], w0);
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------- X producer
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
      TcRing r;
      TcProf pf{(a.probe & 64) != 0, 0};
      unsigned long long w0 = 0;
      int kc = 0;
      for (int c = 0; c < total_chunks; ++c) {
        pf.start();
        if (c >= SX) mbar_wait_sleep(&x_empty[r.slot], r.ph ^ 1u);
        pf.stop(w0);
        const bool lx = !(a.probe & 8) || c < SX;
        unsigned char* st = xring + r.slot * 2 * x_bytes;
        mbar_arrive_expect_tx(&x_full[r.slot], static_cast<uint32_t>(lx ? 2 * x_bytes : 0));
        if (lx) {
          tma_load_2d_hint(st, &tmXh, kc * kTcKChunk, 0, &x_full[r.slot], policy);
          tma_load_2d_hint(st + x_bytes, &tmXl, kc * kTcKChunk, 0, &x_full[r.slot], policy);
        }
        r.next(SX);
        if (++kc == kchunks) kc = 0;
      }
      if (pf.on) atomicAdd(&g_tc_prof[2], w0);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp runs the loop (uniform control flow and operands);
    // elect.sync inside the asm issues each MMA / commit once.  Each TMEM
    // segment accumulates kTcSegChunks chunks (128 rows of A); the epilogue
    // drains it into fp64, so the tensor core's fp32 accumulation never
    // spans more than 128 rows.
    const uint64_t dx = umma_desc_sw128(xring);
    const uint64_t x_step = (2 * x_bytes) >> 4;
    TcRing rl, rx;
    TcProf pf{(a.probe & 64) != 0, 0};
    unsigned long long w3 = 0, w4 = 0, w5 = 0;
    const long long t_role = clock64();
    int seg = 0;
    for (int tt = 0; tt < my_tiles; ++tt) {
      for (int k0 = 0; k0 < kchunks; k0 += SEG, ++seg) {
        const int b = seg & 1;
        pf.start();
        if (seg >= 2) mbar_wait(&tempty[b], static_cast<uint32_t>(((seg - 2) >> 1) & 1));
        pf.stop(w3);
        tc_fence_after();
        const uint32_t dtm = tmem_base + uint32_t(b * 2 * NP);
        const int k1 = (k0 + SEG < kchunks) ? k0 + SEG : kchunks;
        for (int kc = k0; kc < k1; ++kc) {
          pf.start();
          mbar_wait(&lo_full[rl.slot], rl.ph);
          pf.stop(w4);
          pf.start();
          mbar_wait(&x_full[rx.slot], rx.ph);
          pf.stop(w5);
          tc_fence_after();
          const uint32_t th = tmem_base + kTcTmemAOff + uint32_t(rl.slot) * 64;  // A_hi; A_lo at +32
          const uint64_t bx = dx + uint64_t(rx.slot) * x_step;
#pragma unroll
          for (int k = 0; k < kTcKChunk / 8; ++k) {
            const uint32_t first = (kc == k0 && k == 0) ? 0u : 1u;
            umma_tf32_ts_warp(dtm, th + 8 * k, bx + 2 * k, idesc2, first);
            if (!(a.probe & 2)) umma_tf32_ts_warp(dtm, th + 32 + 8 * k, bx + 2 * k, idesc1, 1u);
          }
          umma_commit_warp(&lo_empty[rl.slot]);
          umma_commit_warp(&x_empty[rx.slot]);
          if (kc == k1 - 1) umma_commit_warp(&tfull[b]);
          rl.next(SL);
          rx.next(SX);
        }
      }
    }
    if (pf.on && lane == 0) {
      atomicAdd(&g_tc_prof[3], w3);
      atomicAdd(&g_tc_prof[4], w4);
      atomicAdd(&g_tc_prof[5], w5);
      atomicAdd(&g_tc_prof[6], static_cast<unsigned long long>(clock64() - t_role));
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------- converter warps
    // Thread r owns tile row r (one column of A, TMEM lane r): it reads its
    // 128-byte row out of the 128-byte-swizzled A slot (16-byte chunk c sits
    // at c ^ (r & 7)), splits A = A_hi + A_lo with A_hi = trunc_tf32(A)
    // (A_lo exact in fp32) and stores both halves to its TMEM lane.
    const int q = warp & 3;
    const int r = q * 32 + lane;
    TcRing ra, rl;
    TcProf pf{(a.probe & 64) != 0 && warp == 8, 0};
    unsigned long long w7 = 0, w8 = 0, w9 = 0;
    const long long t_role = clock64();
    for (int c = 0; c < total_chunks; ++c) {
      pf.start();
      mbar_wait(&a_full[ra.slot], ra.ph);
      pf.stop(w7);
      const unsigned char* row = aring + ra.slot * a_bytes + r * 128;
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const float4 v = *reinterpret_cast<const float4*>(row + ((cc ^ (r & 7)) << 4));
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t h = __float_as_uint(e[u]) & 0xFFFFE000u;
          hi[cc * 4 + u] = h;
          lo[cc * 4 + u] = (a.probe & 1) ? 0u : __float_as_uint(e[u] - __uint_as_float(h));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_empty[ra.slot]);  // the slot's bytes are in registers
      pf.start();
      if (c >= SL) mbar_wait(&lo_empty[rl.slot], rl.ph ^ 1u);
      pf.stop(w8);
      tc_fence_after();
      const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16) + kTcTmemAOff + uint32_t(rl.slot) * 64;
      pf.start();
      if (!(a.probe & 32)) {
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_wait_st();
      }
      pf.stop(w9);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lo_full[rl.slot]);
      ra.next(SA);
      rl.next(SL);
    }
    if (pf.on && lane == 0) {
      atomicAdd(&g_tc_prof[7], w7);
      atomicAdd(&g_tc_prof[8], w8);
      atomicAdd(&g_tc_prof[9], w9);
      atomicAdd(&g_tc_prof[10], static_cast<unsigned long long>(clock64() - t_role));
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------ epilogue warps
    const int q = warp & 3;  // TMEM lane quarter
    const int et = tid - 4 * 32;
    double f_acc = 0.0, nnz_acc = 0.0;
    double* wbase = a.w_out != nullptr ? a.w_out + parity * a.w_stride : nullptr;
    TcProf pf{(a.probe & 64) != 0 && warp == 4, 0};
    unsigned long long w11 = 0, w12 = 0;
    const long long t_role = clock64();
    int seg = 0;
    for (int tt = 0; tt < my_tiles; ++tt) {
      const int t = int(blockIdx.x) + tt * int(gridDim.x);
      double c[kTcMaxN];
#pragma unroll
      for (int j = 0; j < kTcMaxN; ++j) c[j] = 0.0;
      for (int k0 = 0; k0 < kchunks; k0 += SEG, ++seg) {
        const int b = seg & 1;
        pf.start();
        mbar_wait(&tfull[b], static_cast<uint32_t>((seg >> 1) & 1));
        pf.stop(w11);
        pf.start();
        tc_fence_after();
#pragma unroll
        for (int j0 = 0; j0 < kTcMaxN; j0 += 16) {
          if (j0 < NP && !(a.probe & 4)) {
            float v[16], vl[16];
            const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(b * 2 * NP + j0);
            tmem_ld16(ta, v);
            tmem_ld16(ta + uint32_t(NP), vl);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 16; ++u) c[j0 + u] += static_cast<double>(v[u] + vl[u]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        pf.stop(w12);
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
    if (pf.on && lane == 0) {
      atomicAdd(&g_tc_prof[11], w11);
      atomicAdd(&g_tc_prof[12], w12);
      atomicAdd(&g_tc_prof[13], static_cast<unsigned long long>(clock64() - t_role));
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcTmemCols)
                 : "memory");
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
