// Block GP-SPCA on the 5th-generation tensor cores (sm_100a tcgen05) for
// m >= 2 components (m = 10, C4: p = 8192, m = 64), fp32 or fp64
// storage, where the CUDA-core block sweep needs ceil(m/4) (fp32) or
// ceil(m/2) (fp64) reads of A.  The tensor cores FILTER columns; the results
// are fp64 arithmetic on every column that can be active.
//
// Filter arithmetic: column i of A is scaled by s_i = 2^e_i (max |a_ji| s_i
// in [2^14, 2^15)) and rounded to fp16, A1 = fp16(a s_i) (11 significant
// bits); X is rounded to fp16 with the common scale 2^14 (its columns are
// unit vectors), X1 = fp16(x 2^14).  One tensor-core MMA per 16 rows forms,
// with fp32 accumulation (kind::f16), D = A1 X1 and c~_ij = 2^-(e_i + 14) D.
// The rounding of A is bounded per column exactly (||a_i - a1_i||,
// tc_col_delta_kernel), that of X by |a_i| (2^-11 + 2^-39 sqrt(p)), the rest
// by 2^-16 |a_i|; T1 flags a column when any component can reach
// its threshold within that margin.  (GPSPCA_TC_XTERMS=2: the two-term split
// x 2^14 = X1 + 2^-11 X2, D = [A1 X1 | A1 X2], c~ from D0 + 2^-11 D1, and
// no X term in the margin.)
//
// T0 split_x:   X (fp64) -> X1 (and X2) (fp16, [n_pad][ld])
// T1 tc_dots:   persistent; per tile of 128 columns accumulates D in TMEM
//               over 64-row chunks: A arrives by TMA (128-byte swizzle),
//               converter warps scale and round it into TMEM (tcgen05.st),
//               the MMAs read A from TMEM and X from shared memory; epilogue
//               warps drain TMEM segments and flag the columns that can
//               reach a threshold within the margin.  A is read from HBM once.
// T1x tc_refine: the flagged columns again, in fp64: c, thresholds, the
//               objective, nnz, W and the activity mask; its CTAs' leftover
//               lists (< 64 columns each) go to T1s.
// T1s tc_refine_split: the leftover lists grouped across CTAs, rows split
//               over a persistent grid, same epilogue.
// T2 tc_update: G_j = sum over ACTIVE columns of w_ij a_i (fp64), row chunks
//               x component groups; reads only the active columns again.
// Roles of T1 (12 warps): w0 A producer (TMA), w1 MMA issuer (+TMEM owner),
// w2 X producer (TMA), w4-7 epilogue (warp % 4 selects the TMEM lane
// quarter) and w12-15 (second component half), w8-11 converters.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "su_kernels.cuh"

namespace gps {

constexpr int kTcTileM = 128;    // columns of A per tile (MMA M)
constexpr int kTcKChunk = 64;    // rows of A per chunk (two 32-row fp32 TMA boxes; one 128-byte fp16 row)
constexpr int kTcBoxBytes = 128; // inner extent of an A TMA box: 32 fp32 / 16 fp64 rows
constexpr int kTcAStages = 5;    // default A ring depth (32 KB stages, HBM stream)
#ifndef GPS_TC_LO_STAGES
#define GPS_TC_LO_STAGES 2
#endif
constexpr int kTcLoStages = GPS_TC_LO_STAGES;  // TMEM A1 slots (converter output; <= 4: columns 256..511)
constexpr int kTcXStages = 3;    // default X ring depth (X1, or X1 | X2; L2-resident)
constexpr int kTcMaxStages = 8;
constexpr int kTcThreads = 512;  // 16 warps
constexpr int kTcMaxN = 64;
constexpr int kTcMinM = 2;       // fp32 block solves with m >= 2 take this path (one A read, exact fp64 results)
constexpr int kTcSegChunks = 2;  // TMEM accumulation segment: 2 chunks = 128 rows, drained to fp64
constexpr int kTcXScaleExp = 14; // |x| <= 1 -> |x 2^14| <= 2^14
constexpr int kTcMarginExp = 13; // candidate margin 2^-13 ||a_i|| (16x the error bound)

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

// tf32 instruction descriptor and single-thread issue: used by the
// microbenchmarks in scripts/ubench (the sweep itself runs kind::f16).
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

// Warp-converged commit: every lane executes the call with identical
// operands and elect.sync picks the issuing lane inside the asm, so the
// compiler keeps operands in uniform registers (a single-thread branch
// instead costs a per-instruction R2UR + waterfall loop, ~90 clocks/MMA).
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
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// C0, once per matrix: the candidate margin of T1,
//   delta_i = ||a_i - a1_i||_2 + 2^-kTcMarginExp ||a_i||_2     (rounded up)
// where a1_i = 2^-e_i fp16(fp32(a_i 2^e_i)) is exactly the operand the tensor
// cores see (the converters' rounding, reproduced here) and e_i = 14 -
// floor(log2 max_j |a_ji|) (0 for an all-zero column, clamped to
// [-126, 126]) comes from the matrix's norms pass (column_norms_kernel).
// With unit x_j, |a1_i'x_j - a_i'x_j| <= ||a_i - a1_i|| (Cauchy-Schwarz) and
// the rest of T1's error (the 2-term split of X, fp32 accumulation) is
// < 2^-17 ||a_i||, 16x inside the second term.  Warp per column.
template <typename TA>
__global__ void tc_col_delta_kernel(const TA* __restrict__ A, int64_t n, int ld, int p,
                                    const int* __restrict__ col_exp, float* __restrict__ col_delta) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t col = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; col < n; col += warps) {
    const TA* a = A + col * ld;
    const int e = col_exp[col];
    const float sc = __int_as_float((127 + e) << 23);
    const double unsc = ldexp(1.0, -e);
    double ss = 0.0, rr = 0.0;
    for (int r = lane; r < p; r += 32) {
      const TA v = a[r];
      const float y = (sizeof(TA) == 4) ? static_cast<float>(v) * sc
                                        : __double2float_rn(static_cast<double>(v) * static_cast<double>(sc));
      const double d = static_cast<double>(v) - static_cast<double>(__half2float(__float2half_rn(y))) * unsc;
      ss = fma(static_cast<double>(v), static_cast<double>(v), ss);
      rr = fma(d, d, rr);
    }
    ss = warp_sum(ss);
    rr = warp_sum(rr);
    if (lane == 0) {
      col_delta[col] = __double2float_ru((sqrt(rr) + ldexp(sqrt(ss), -kTcMarginExp)) * (1.0 + 0x1p-40));
      col_delta[n + col] = __double2float_ru(sqrt(ss) * (1.0 + 0x1p-40));  // |a_i| (one-term X margin)
    }
  }
}

// T0: X (fp64 [m][ld], parity slot) -> X1 / X2 (fp16 [n_pad][ld], zero
// padded components): x 2^14 = X1 + 2^-11 X2 (X1 alone when x2 is null:
// the one-term filter).
__global__ void tc_split_x_kernel(const double* __restrict__ X, int64_t x_par_stride, int m, int n_pad, int ld,
                                  __half* __restrict__ x1, __half* __restrict__ x2, const GpsCtl* ctl,
                                  unsigned int* __restrict__ act_count) {
  if (ctl != nullptr && ctl->done) return;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *act_count = 0;  // this sweep's active columns (T1x / T1s count, T2 reads)
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const double* Xp = X + parity * x_par_stride;
  // grid (row blocks of 4 x blockDim, padded components): no index division per element
  const int j = blockIdx.y;
  const double* xs = Xp + size_t(j) * ld;
  const size_t o = size_t(j) * ld;
  const int r0 = blockIdx.x * 4 * blockDim.x + threadIdx.x;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r0 + u * blockDim.x;
    if (r >= ld) break;
    const double y = j < m ? xs[r] * double(1 << kTcXScaleExp) : 0.0;
    const __half h = __double2half(y);
    x1[o + r] = h;
    if (x2 != nullptr) x2[o + r] = __double2half((y - static_cast<double>(__half2float(h))) * 2048.0);
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
  const int* col_exp;   // n: scale exponents of the columns
  const float* col_delta;  // n: candidate margins (tc_col_delta_kernel)
  double* w_out;        // [m_pad][n] parity slots (unused by T1: tc_mask_w_kernel zeroes filtered columns)
  int64_t w_stride;
  unsigned char* colmask;  // [2][n]: 1 if column i is a candidate (one row per epilogue group)
  unsigned char* tflag;    // [tiles][8]: any candidate in (tile, group, lane quarter)
  const GpsCtl* ctl;
  int num_tiles;
  int a_stages, x_stages;  // ring depths (<= kTcMaxStages)
  int seg_chunks;          // chunks per TMEM accumulation segment
  int x_terms;  // fp16 terms of X in the MMA: 2 (x 2^14 = X1 + 2^-11 X2) or 1 (X1 only, wider margin)
  float x_err;  // one-term X: bound on |x_j - 2^-14 X1_j|_2 (unit x_j), times |a_i| added to the margin
  int probe;  // timing experiments: 4 no TMEM drain, 8 no X loads, 16 no update, 128 A loads with the
              // evict_first hint,
              // 32 no TMEM stores, 64 cycle accounting
};

// Operand staging of T1.  Shared memory is the scarce resource (tcgen05.mma
// shared-memory operands, TMA writes and converter reads share its ~128
// B/clock), so A passes through it once:
//   A ring    SA x 32 KB in shared memory (TMA, evict-first) -> converters
//   A1        2 slots x 64 TMEM columns (32 packed fp16 pairs used), written
//             by the converters with tcgen05.st, read by the MMAs as the
//             TMEM-resident A operand
//   X ring    SX x (X1 | X2) chunk slots in shared memory (TMA, evict-last;
//             X1 only with the one-term filter)
// TMEM: columns [0, 4 NP) = 2 accumulator buffers of [D0 | D1] (2 NP
// each), columns [256, 384) = the two A1 slots.
constexpr uint32_t kTcTmemCols = 512;
constexpr uint32_t kTcTmemAOff = 256;
// A ring stage: one 64-row chunk of a 128-column tile (32 KB fp32, 64 KB fp64)
__host__ __device__ inline size_t tc_a_bytes(int esz) { return size_t(kTcTileM) * kTcKChunk * esz; }
__host__ __device__ inline size_t tc_x_bytes(int n_pad) { return size_t(n_pad) * kTcKChunk * 2; }
__host__ __device__ inline size_t tc_smem_bytes(int n_pad, int sa, int sx, int esz) {
  return 1024 /*align slack*/ + sa * tc_a_bytes(esz) + sx * 2 * tc_x_bytes(n_pad) + 4096 /*barriers, params*/;
}

__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// Instruction descriptor: D f32, A/B f16, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// tcgen05.mma kind::f16 with the A operand in TMEM (M = 128 lanes, K = 16 =
// 8 columns of packed pairs), warp-converged issue.
__device__ __forceinline__ void umma_f16_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                                 uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Optional per-role cycle accounting (tuning diagnostics: build with
// -DGPS_TC_PROFILE and run with TcDotsArgs::probe & 64).
#ifdef GPS_TC_PROFILE
constexpr bool kTcProfile = true;
#else
constexpr bool kTcProfile = false;
#endif
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

__device__ __forceinline__ double2 lds_d2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// Round two floats to fp16 and pack them (k in the low half, k + 1 high).
__device__ __forceinline__ uint32_t pack_f16x2(float k0, float k1) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(k1), "f"(k0));
  return d;
}

template <typename TA>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_dots_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX1,
                   const __grid_constant__ CUtensorMap tmX2, const TcDotsArgs a) {
  extern __shared__ unsigned char smem_raw[];
  if (a.ctl != nullptr && a.ctl->done) return;
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NP = a.n_pad;
  const int SA = a.a_stages, SL = kTcLoStages, SX = a.x_stages;
  const int SEG = a.seg_chunks;
  constexpr int kBoxK = kTcBoxBytes / int(sizeof(TA));  // rows per A box
  constexpr int kBoxes = kTcKChunk / kBoxK;              // boxes per 64-row chunk (2 fp32, 4 fp64)
  const size_t a_bytes = tc_a_bytes(sizeof(TA));         // kBoxes boxes of 16 KB
  const size_t x_bytes = tc_x_bytes(NP);
  unsigned char* aring = smem;
  unsigned char* xring = aring + SA * a_bytes;  // [stage][X1 | X2]
  uint64_t* a_full = reinterpret_cast<uint64_t*>(xring + SX * 2 * x_bytes);
  uint64_t* a_empty = a_full + SA;
  uint64_t* lo_full = a_empty + SA;  // TMEM A1 slots
  uint64_t* lo_empty = lo_full + SL;
  uint64_t* x_full = lo_empty + SL;
  uint64_t* x_empty = x_full + SX;
  uint64_t* tfull = x_empty + SX;  // 2 accumulator buffers
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  double* sgam = reinterpret_cast<double*>(tmem_base_slot + 4);
  double* smu = sgam + kTcMaxN;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kchunks = (a.ld + kTcKChunk - 1) / kTcKChunk;
  // one MMA per 16 rows: A1 [X1 | X2] (N = 2 NP; the X slot holds X1 rows then X2 rows), or A1 X1 (N = NP)
  const uint32_t idesc2 = umma_idesc_f16(kTcTileM, a.x_terms * NP);

  if (tid == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 4);  // 4 converter warps have read the slot
    }
    for (int i = 0; i < SL; ++i) {
      mbar_init(&lo_full[i], 4);   // 4 converter warps stored their TMEM lanes
      mbar_init(&lo_empty[i], 1);  // tcgen05.commit
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);   // tcgen05.commit
      mbar_init(&tempty[i], 8);  // 8 epilogue warps
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
    tma_prefetch(&tmX1);
    tma_prefetch(&tmX2);
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
      TcProf pf{kTcProfile && (a.probe & 64) != 0, 0};
      unsigned long long w0 = 0;
      int t = int(blockIdx.x), kc = 0;
      for (int c = 0; c < total_chunks; ++c) {
        pf.start();
        if (c >= SA) mbar_wait_sleep(&a_empty[r.slot], r.ph ^ 1u);  // (a pure spin measured the same)
        pf.stop(w0);
        unsigned char* st = aring + r.slot * a_bytes;
        mbar_arrive_expect_tx(&a_full[r.slot], static_cast<uint32_t>(a_bytes));
#pragma unroll
        for (int b = 0; b < kBoxes; ++b) {
          // no L2 cache hint: evict_first on these 2-D boxes measured 2.5-3.5 % slower at
          // C3 / C4 (probe 128 restores it for experiments)
          if (a.probe & 128)
            tma_load_2d_hint(st + b * (a_bytes / kBoxes), &tmA, kc * kTcKChunk + b * kBoxK, t * kTcTileM,
                             &a_full[r.slot], policy);
          else
            tma_load_2d(st + b * (a_bytes / kBoxes), &tmA, kc * kTcKChunk + b * kBoxK, t * kTcTileM, &a_full[r.slot]);
        }
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
      TcProf pf{kTcProfile && (a.probe & 64) != 0, 0};
      unsigned long long w0 = 0;
      int kc = 0;
      for (int c = 0; c < total_chunks; ++c) {
        pf.start();
        if (c >= SX) mbar_wait_sleep(&x_empty[r.slot], r.ph ^ 1u);
        pf.stop(w0);
        const bool lx = !(a.probe & 8) || c < SX;
        unsigned char* st = xring + r.slot * 2 * x_bytes;
        mbar_arrive_expect_tx(&x_full[r.slot], static_cast<uint32_t>(lx ? a.x_terms * x_bytes : 0));
        if (lx) {
          tma_load_2d_hint(st, &tmX1, kc * kTcKChunk, 0, &x_full[r.slot], policy);
          if (a.x_terms == 2) tma_load_2d_hint(st + x_bytes, &tmX2, kc * kTcKChunk, 0, &x_full[r.slot], policy);
        }
        r.next(SX);
        if (++kc == kchunks) kc = 0;
      }
      if (pf.on) atomicAdd(&g_tc_prof[2], w0);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp runs the loop (uniform control flow and operands);
    // elect.sync inside the asm issues each MMA / commit once.  A TMEM
    // segment accumulates SEG chunks (128 rows) before the epilogue drains
    // it into fp64.
    const uint64_t dx = umma_desc_sw128(xring);
    const uint64_t x_step = (2 * x_bytes) >> 4;
    TcRing rl, rx;
    TcProf pf{kTcProfile && (a.probe & 64) != 0, 0};
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
          const uint32_t ta = tmem_base + kTcTmemAOff + uint32_t(rl.slot) * 64;  // A1
          const uint64_t bx = dx + uint64_t(rx.slot) * x_step;
#pragma unroll
          for (int k = 0; k < kTcKChunk / 16; ++k) {
            const uint32_t first = (kc == k0 && k == 0) ? 0u : 1u;
            umma_f16_ts_warp(dtm, ta + 8 * k, bx + 2 * k, idesc2, first);
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
  } else if (warp >= 8 && warp < 12) {
    // ---------------------------------------------------- converter warps
    // Thread r owns tile row r (one column of A, TMEM lane r): it reads its
    // two 128-byte rows out of the 128-byte-swizzled A slot (16-byte chunk c
    // of row r sits at c ^ (r & 7)), scales by 2^e_i, rounds to fp16 (A1) and
    // stores the packed pairs to its TMEM lane.
    const int q = warp & 3;
    const int r = q * 32 + lane;
    TcRing ra, rl;
    TcProf pf{kTcProfile && (a.probe & 64) != 0 && warp == 8, 0};
    unsigned long long w7 = 0, w8 = 0, w9 = 0;
    const long long t_role = clock64();
    int tt = 0, kc = 0;
    // scale 2^e of my column (e in [-126, 126]); the next tile's exponent is
    // loaded one chunk into the current tile, so the global-load latency is
    // not paid on the converters' critical path at every tile start
    auto col_scale = [&](int tile) {
      const int64_t col = int64_t(int(blockIdx.x) + tile * int(gridDim.x)) * kTcTileM + r;
      return col < a.n ? a.col_exp[col] : 0;
    };
    int e_next = my_tiles > 0 ? col_scale(0) : 0;
    float sc = 1.f;
    for (int c = 0; c < total_chunks; ++c) {
      if (kc == 0) sc = __int_as_float((127 + e_next) << 23);
      if (kc == (kchunks > 1 ? 1 : 0) && tt + 1 < my_tiles) e_next = col_scale(tt + 1);
      pf.start();
      mbar_wait(&a_full[ra.slot], ra.ph);
      pf.stop(w7);
      pf.start();
      if (c >= SL) mbar_wait(&lo_empty[rl.slot], rl.ph ^ 1u);
      pf.stop(w8);
      tc_fence_after();
      const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16) + kTcTmemAOff + uint32_t(rl.slot) * 64;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // rows 32 h .. 32 h + 31 (one fp32 / two fp64 TMA boxes)
        uint32_t p1[16];
        // A1 = fp16(y), y = a 2^e (fp64 storage: y rounded to fp32 first);
        // tc_col_delta_kernel reproduces exactly this rounding for the margin.
        if constexpr (sizeof(TA) == 4) {
          const uint32_t row_s = smem_u32(aring + ra.slot * a_bytes + h * (a_bytes / 2) + r * 128);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const float4 v = lds_f4(row_s + ((cc ^ (r & 7)) << 4));
            p1[cc * 2] = pack_f16x2(v.x * sc, v.y * sc);  // packed column (row / 2) within the half
            p1[cc * 2 + 1] = pack_f16x2(v.z * sc, v.w * sc);
          }
        } else {
          const double scd = static_cast<double>(sc);
#pragma unroll
          for (int bq = 0; bq < 2; ++bq) {  // 16-row box 2 h + bq
            const uint32_t row_s = smem_u32(aring + ra.slot * a_bytes + (2 * h + bq) * (a_bytes / 4) + r * 128);
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {  // 16-byte chunk = rows 2 cc, 2 cc + 1 of the box
              const double2 v = lds_d2(row_s + ((cc ^ (r & 7)) << 4));
              p1[bq * 8 + cc] = pack_f16x2(__double2float_rn(v.x * scd), __double2float_rn(v.y * scd));
            }
          }
        }
        pf.start();
        if (!(a.probe & 32)) tmem_st16(ta + 16 * h, p1);
        pf.stop(w9);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_empty[ra.slot]);  // the slot's bytes have been read
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lo_full[rl.slot]);
      ra.next(SA);
      rl.next(SL);
      if (++kc == kchunks) {
        kc = 0;
        ++tt;
      }
    }
    if (pf.on && lane == 0) {
      atomicAdd(&g_tc_prof[7], w7);
      atomicAdd(&g_tc_prof[8], w8);
      atomicAdd(&g_tc_prof[9], w9);
      atomicAdd(&g_tc_prof[10], static_cast<unsigned long long>(clock64() - t_role));
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 12) {
    // ------------------------------------------------------ epilogue warps
    // Two groups of 4 warps (warp % 4 selects the TMEM lane quarter = 32
    // columns of the tile); group g owns components [32 g, 32 g + 32).
    const int q = warp & 3;
    const int g = warp >= 12 ? 1 : 0;
    const int jbase = g * 32;
    TcProf pf{kTcProfile && (a.probe & 64) != 0 && warp == 4, 0};
    unsigned long long w11 = 0, w12 = 0;
    const long long t_role = clock64();
    int seg = 0;
    for (int tt = 0; tt < my_tiles; ++tt) {
      const int t = int(blockIdx.x) + tt * int(gridDim.x);
      // the column's scale exponent and margin, loaded at the tile start so
      // the candidate test at its end does not wait on global memory
      const int64_t col_t = int64_t(t) * kTcTileM + q * 32 + lane;
      const int e_col = col_t < a.n ? a.col_exp[col_t] : 0;
      const float d_col = col_t < a.n ? (a.x_terms == 2 ? a.col_delta[col_t]
                                                       : __fmaf_ru(a.col_delta[a.n + col_t], a.x_err, a.col_delta[col_t]))
                                      : 0.f;
      // per-tile sums with Kahan compensation in fp32 (full-rate fp32 ops
      // instead of fp64 conversions and adds)
      float ch[32], cl[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) ch[j] = cl[j] = 0.f;
      for (int k0 = 0; k0 < kchunks; k0 += SEG, ++seg) {
        const int b = seg & 1;
        pf.start();
        mbar_wait_sleep(&tfull[b], static_cast<uint32_t>((seg >> 1) & 1));  // off the converters' issue slots
        pf.stop(w11);
        pf.start();
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int j0 = jbase + 8 * h;
          if (j0 < NP && !(a.probe & 4)) {
            float v0[8], v1[8];
            const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(b * 2 * NP + j0);
            tmem_ld8(ta, v0);
            if (a.x_terms == 2) {
              tmem_ld8(ta + uint32_t(NP), v1);
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u) v1[u] = 0.f;
            }
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              // Kahan step: ch + cl carries the running sum, cl the (negated) compensation
              const float yk = __fsub_rn(fmaf(v1[u], 1.f / 2048.f, v0[u]), cl[8 * h + u]);
              const float tk = __fadd_rn(ch[8 * h + u], yk);
              cl[8 * h + u] = __fsub_rn(__fsub_rn(tk, ch[8 * h + u]), yk);
              ch[8 * h + u] = tk;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        pf.stop(w12);
      }
      const int64_t col = int64_t(t) * kTcTileM + q * 32 + lane;
      bool cand = false;
      if (col < a.n) {
        // Candidate filter.  The exact c_ij (fp64) is within delta_i of this
        // estimate (tc_col_delta_kernel; ||x_j|| = 1), so a column
        // none of whose components can reach the threshold with that margin
        // is inactive (w = 0, objective term 0) for certain; every other
        // column is recomputed exactly by T1x.
        const double unscale = ldexp(1.0, -(e_col + kTcXScaleExp));
        const double delta = static_cast<double>(d_col);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int j = jbase + jj;
          if (j >= a.m) continue;
          const double s = smu[j] * (fabs((static_cast<double>(ch[jj]) - static_cast<double>(cl[jj])) * unscale) + delta);
          cand |= (a.penalty == 0) ? (s >= sgam[j]) : (s * s >= sgam[j]);
        }
        // W is NOT zeroed here for non-candidates (1 GB of writes per C4
        // iteration competing with the A stream): the loadings read W of the
        // final sweep through tc_mask_w_kernel, which zeroes every column
        // the final activity mask leaves inactive.
        a.colmask[size_t(g) * a.n + col] = cand ? 1 : 0;
      }
      // per (tile, group, lane quarter) flag: T1x skips tiles with none
      const unsigned any = __ballot_sync(0xffffffffu, cand);
      if (lane == 0) a.tflag[size_t(t) * 8 + g * 4 + q] = any != 0u ? 1 : 0;
    }
    if (pf.on && lane == 0) {
      atomicAdd(&g_tc_prof[11], w11);
      atomicAdd(&g_tc_prof[12], w12);
      atomicAdd(&g_tc_prof[13], static_cast<unsigned long long>(clock64() - t_role));
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcTmemCols)
                 : "memory");
  }
}

// fp64 tensor-core MMA (DMMA): D(8x8) += A(8x4, row-major) B(4x8, col-major).
// Fragments: lane l holds A[l / 4][l % 4], B[l % 4][l / 4] and
// D[l / 4][2 (l % 4) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr int kTcRefItem = 256;
constexpr int kTcRefBatch = 64;
constexpr int kTcRefRows = 32;
constexpr int kRefKS = kTcRefRows + 4;  // k-contiguous row stride of the DMMA tiles (= 4 mod 16 doubles)
constexpr int kTcSplitMax = 8;          // row splits (work units per leftover list) of T1s
constexpr int kTcLeftMaxGrid = 1024;  // T1x grid bound of T1s's in-CTA scan (4 x 148 SMs fits)
__host__ __device__ constexpr size_t tc_refine_smem(int nj) {
  return (size_t(2) * kTcRefBatch * kRefKS + size_t(2) * nj * kRefKS) * sizeof(double);
}

// C (nb <= 64 candidate columns x NJ = 16 NT components) = A_cand' X over
// rows [r_lo, r_hi) (multiples of 32) on the fp64 tensor cores (DMMA
// m8n8k4, fp64 in, fp64 accumulate), 32 rows at a time.  Per chunk warp w
// stages columns 8w .. 8w + 7 (lane = row, widened to fp64 once) and
// components 8w .. 8w + 7 of X (lane = row) into double-buffered shared
// tiles stored k-contiguous (row stride kRefKS = 36 = 4 mod 16 doubles:
// stores and fragment loads are conflict-free), the next chunk's loads are
// issued before the current chunk's DMMAs, one barrier per chunk.  Warp w
// owns columns 16 (w % 4) .. + 16 (2 m-tiles) and components 8 NT (w / 4)
// .. + 8 NT (NT n-tiles); on return lane holds
// C[column 16 (w % 4) + 8 mt + lane / 4][component 8 NT (w / 4) + 8 nt + 2 (lane % 4) + h]
// in acc[mt][nt][h].  256 threads; ends with a block barrier.
template <typename TA, int NT>
__device__ __forceinline__ void ref_batch_dots(const TA* __restrict__ A, int ld, const double* __restrict__ Xp,
                                               const int64_t* cand, int nb, int r_lo, int r_hi, double* sA,
                                               double* sX, double (&acc)[2][NT][2]) {
  constexpr int NJ = 16 * NT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3, mg = warp & 3, ng = warp >> 2;
  // two accumulator sets (even / odd k-steps): 4 NT independent DMMA
  // chains per warp instead of 2 NT, so the pipe's latency is covered
  // (ncu: "wait" was 27 % of the stall samples with one set)
  double acc2[2][NT][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int u = 0; u < NT; ++u) acc[i][u][0] = acc[i][u][1] = acc2[i][u][0] = acc2[i][u][1] = 0.0;
  TA ra[8];
  double rx[8];
  auto load = [&](int r0) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int bc = warp * 8 + c;
      ra[c] = bc < nb ? A[cand[bc] * ld + r0 + lane] : TA(0);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = warp * 8 + c;
      rx[c] = j < NJ ? Xp[size_t(j) * ld + r0 + lane] : 0.0;
    }
  };
  if (r_lo < r_hi) load(r_lo);
  int buf = 0;
  for (int r0 = r_lo; r0 < r_hi; r0 += kTcRefRows, buf ^= 1) {
    double* a_s = sA + buf * kTcRefBatch * kRefKS;
    double* x_s = sX + buf * NJ * kRefKS;
#pragma unroll
    for (int c = 0; c < 8; ++c) a_s[(warp * 8 + c) * kRefKS + lane] = static_cast<double>(ra[c]);
    if (warp * 8 < NJ)
#pragma unroll
      for (int c = 0; c < 8; ++c) x_s[(warp * 8 + c) * kRefKS + lane] = rx[c];
    __syncthreads();
    if (r0 + kTcRefRows < r_hi) load(r0 + kTcRefRows);
#pragma unroll
    for (int ks = 0; ks < kTcRefRows; ks += 8) {
      double a[2], b[NT], a2[2], b2[NT];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        a[mt] = a_s[(mg * 16 + mt * 8 + g) * kRefKS + ks + t];
        a2[mt] = a_s[(mg * 16 + mt * 8 + g) * kRefKS + ks + 4 + t];
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        b[nt] = x_s[(ng * 8 * NT + nt * 8 + g) * kRefKS + ks + t];
        b2[nt] = x_s[(ng * 8 * NT + nt * 8 + g) * kRefKS + ks + 4 + t];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
        if (mg * 16 + mt * 8 < nb)  // warp-uniform: m-tiles without a column are skipped
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            dmma_8x8x4(acc[mt][nt], a[mt], b[nt]);
            dmma_8x8x4(acc2[mt][nt], a2[mt], b2[nt]);
          }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      acc[i][u][0] += acc2[i][u][0];
      acc[i][u][1] += acc2[i][u][1];
    }
}

// T1x: exact fp64 recomputation of the candidate columns T1 flagged.
// Work items are 256-column ranges (two T1 tiles), assigned to CTAs
// round-robin (item b, b + grid, ...) so contiguous runs of active columns
// spread over the grid; an item whose two tiles carry no candidate flag is
// skipped without reading its columns.  The candidates of a CTA's items are
// compacted in column order into one list (across items), and every 64 of
// them are processed as a batch: C_batch = A_batch' X, 32 rows at a time, on
// the fp64 tensor cores (ref_batch_dots: DMMA m8n8k4; A and X through shared
// memory).  The weights also go to Wt (column-major by component: one
// contiguous row of NJ doubles per column) for T2's gathers.  The final
// partial list (< 64 candidates; at C4 the whole workload: 1-2 per CTA) is
// left in `left` for T1s, which spreads its rows over a cluster of CTAs (one
// CTA streaming all p rows of X per leftover list took ~70 us per column).
// fp32 a_ri is exact in fp64, so c_ij is an fp64 dot product.  Then, per
// (column, component): s = mu_j c_ij, w_ij = threshold(s, gamma_j) (the
// reference's parallel.py:117-128 / block.py:80-89 rules), the objective
// term and nnz, W written for every component of the column, the final
// activity mask (colmask[0][i] = any w_ij != 0, colmask[1][i] = 0) and the
// per-item activity flag item_act for T2.  f and nnz are summed per thread in
// a fixed order and reduced per CTA in a fixed order into part_s[blockIdx.x]
// (deterministic run to run); part_s[gridDim.x + 4 blockIdx.x + i], i < 4,
// are T1s's group slots (zeroed here, written by T1s for existing groups).
template <typename TA, int JPT>
__global__ void __launch_bounds__(256, 2) tc_refine_kernel(const TA* __restrict__ A, int64_t n, int ld, int m,
                                                           const double* __restrict__ X, int64_t x_par_stride,
                                                           const double* __restrict__ mu,
                                                           const double* __restrict__ gamma, int penalty,
                                                           unsigned char* __restrict__ colmask,
                                                           const unsigned char* __restrict__ tflag,
                                                           unsigned char* __restrict__ item_act,
                                                           double* __restrict__ W, int64_t w_par_stride,
                                                           double* __restrict__ Wt, double* __restrict__ part_s,
                                                           const GpsCtl* ctl, BandLog* band,
                                                           int64_t* __restrict__ left, int* __restrict__ left_n,
                                                           unsigned int* __restrict__ act_count) {
  constexpr int NJ = 8 * JPT;  // padded components (X is zero beyond m)
  constexpr int NT = NJ / 16;  // DMMA n-tiles per warp (two component halves)
  if (ctl != nullptr && ctl->done) return;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const double* Xp = X + parity * x_par_stride;
  double* Wp = W + parity * w_par_stride;
  extern __shared__ __align__(16) double ref_smem[];
  double* sA = ref_smem;                                   // [2][64 columns][kRefKS] fp64
  double* sX = ref_smem + 2 * kTcRefBatch * kRefKS;        // [2][NJ components][kRefKS]
  __shared__ int64_t cand[kTcRefItem + kTcRefBatch];
  __shared__ int ilist[256];
  __shared__ int wcnt[8];
  __shared__ unsigned char act[kTcRefBatch];
  __shared__ double smu[NJ], sgam[NJ];
  __shared__ double red[2][8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int j = tid; j < NJ; j += 256) {
    smu[j] = j < m ? mu[j] : 1.0;
    sgam[j] = j < m ? gamma[j] : 0.0;
  }
  double f_acc = 0.0, nnz_acc = 0.0;
  const int64_t items = (n + kTcRefItem - 1) / kTcRefItem;
  const int64_t G = gridDim.x;

  // block-wide order-preserving compaction: returns the count, pos = my slot
  auto compact = [&](bool flag, int& pos) {
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    __syncthreads();  // previous readers of wcnt / the lists are done
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      off += (w < warp) ? wcnt[w] : 0;
      total += wcnt[w];
    }
    pos = off + __popc(bal & ((1u << lane) - 1u));
    return total;
  };
  // final activity of column c: mask for T2, item flag (benign: writers store 1)
  auto publish = [&](int64_t c, bool any) {
    colmask[c] = any ? 1 : 0;
    colmask[n + c] = 0;
    if (any) item_act[c / kTcRefItem] = 1;
  };

  // batch mode: candidates cand[b0 .. b0 + nb), nb <= 64, on the fp64
  // tensor cores over all rows
  auto batch = [&](int b0, int nb) {
    const int g = lane >> 2, t = lane & 3, mg = warp & 3, ng = warp >> 2;
    double acc[2][NT][2];
    if (tid < kTcRefBatch) act[tid] = 0;
    ref_batch_dots<TA, NT>(A, ld, Xp, cand + b0, nb, 0, ld, sA, sX, acc);
    // epilogue: lane holds C[column mg 16 + mt 8 + g][component ng 8 NT + nt 8 + 2 t + {0, 1}]
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int bc = mg * 16 + mt * 8 + g;
      if (bc < nb) {
        const int64_t c = cand[b0 + bc];
        bool any = false;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int j0 = ng * 8 * NT + nt * 8 + 2 * t;
          double wv[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = j0 + h;
            wv[h] = 0.0;
            if (j < m) {
              const double sj = smu[j] * acc[mt][nt][h];
              const double w = threshold_weight(sj, sgam[j], penalty);
              band_note(band, parity, c, j, sj, sgam[j], penalty);
              f_acc += objective_term(sj, sgam[j], penalty);
              if (w != 0.0) {
                nnz_acc += 1.0;
                any = true;
              }
              Wp[size_t(j) * n + c] = w;
              wv[h] = w;
            }
          }
          *reinterpret_cast<double2*>(Wt + c * NJ + j0) = make_double2(wv[0], wv[1]);
        }
        if (any) act[bc] = 1;  // benign: every writer stores 1
      }
    }
    __syncthreads();
    if (tid < nb) publish(cand[b0 + tid], act[tid] != 0);
    const int nact = __syncthreads_count(tid < nb && act[tid] != 0);
    if (tid == 0 && nact > 0) atomicAdd(act_count, static_cast<unsigned int>(nact));
  };

  int pending = 0;  // candidates in cand[0 .. pending) (block-uniform)
  for (int64_t kb = 0; int64_t(blockIdx.x) + kb * G < items; kb += 256) {
    // my items kb .. kb + 255 (item = blockIdx.x + k G): keep the flagged ones
    const int64_t it = int64_t(blockIdx.x) + (kb + tid) * G;
    bool ne = false;
    if (it < items) {
      const uint4 f = *reinterpret_cast<const uint4*>(tflag + it * 16);
      ne = (f.x | f.y | f.z | f.w) != 0u;
      item_act[it] = 0;  // set to 1 when one of its candidates turns out active
    }
    int pos;
    const int nitems = compact(ne, pos);
    if (ne) ilist[pos] = tid;
    __syncthreads();
    for (int ii = 0; ii < nitems; ++ii) {
      const int64_t item = int64_t(blockIdx.x) + (kb + ilist[ii]) * G;
      const int64_t col = item * kTcRefItem + tid;
      const bool flag = col < n && (colmask[col] | colmask[n + col]);
      const int total = compact(flag, pos);
      if (flag) cand[pending + pos] = col;
      pending += total;
      __syncthreads();
      if (pending >= kTcRefBatch) {
        const int full = pending / kTcRefBatch * kTcRefBatch;
        for (int b0 = 0; b0 < full; b0 += kTcRefBatch) batch(b0, kTcRefBatch);
        // move the remainder (< 64) to the front
        const int64_t keep = tid < pending - full ? cand[full + tid] : 0;
        __syncthreads();
        if (tid < pending - full) cand[tid] = keep;
        pending -= full;
        __syncthreads();
      }
    }
  }
  // the leftover list (< 64) goes to T1s, which groups the lists of all
  // CTAs (in CTA order) and splits their rows over many CTAs; this CTA
  // zeroes T1s's f / nnz slots [4 b, 4 b + 4) (T1s writes one per group)
  if (tid < pending) left[size_t(blockIdx.x) * kTcRefBatch + tid] = cand[tid];
  if (tid == 0) left_n[blockIdx.x] = pending;
  if (tid < 16) part_s[(G + 4 * blockIdx.x) * 4 + tid] = 0.0;
  f_acc = warp_sum(f_acc);
  nnz_acc = warp_sum(nnz_acc);
  __syncthreads();
  if (lane == 0) {
    red[0][warp] = f_acc;
    red[1][warp] = nnz_acc;
  }
  __syncthreads();
  if (tid < 4) {
    double t = 0.0;
    if (tid < 2)
      for (int w = 0; w < 8; ++w) t += red[tid][w];
    part_s[size_t(blockIdx.x) * 4 + tid] = t;
  }
}

// Small lists (nb <= 16 columns, two m-tiles): C = A_cand' X over rows
// [r_lo, r_hi) with the rows split over the 8 warps (split-k), fragments
// loaded straight from global memory (L1 / L2: one 16-byte segment per
// column and 4-row k-step) -- no shared staging, no block barrier per step.
// Warp w owns rows r_lo + w R8 .. + R8 (R8 = (r_hi - r_lo) / 8 rounded up to
// 4) and every component (NJ / 8 n-tiles); the 8 warp partials are summed
// in warp order through shared memory into part[bc NJ + j] (bc < 16).
template <typename TA, int NJ>
__device__ __forceinline__ void ref_small_dots(const TA* __restrict__ A, int ld, const double* __restrict__ Xp,
                                               const int64_t* cand, int nb, int r_lo, int r_hi, double* part) {
  constexpr int NTT = NJ / 8;  // n-tiles (all components)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rw = (((r_hi - r_lo + 7) / 8) + 3) & ~3;
  const int k_lo = min(r_hi, r_lo + warp * rw), k_hi = min(r_hi, k_lo + rw);
  double acc[2][NTT][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const TA* ac0 = A + cand[min(g, nb - 1)] * ld;
  const TA* ac1 = A + cand[min(8 + g, nb - 1)] * ld;
  const bool two = nb > 8;  // warp-uniform
  // k-steps in flight per warp: the loop is latency-bound (L2 / HBM loads),
  // so unroll as far as registers allow (NTT + 2 operands per k-step)
  constexpr int KU = NTT <= 2 ? 8 : (NTT <= 4 ? 4 : 2);
#pragma unroll KU
  for (int k = k_lo; k < k_hi; k += 4) {
    const double a0 = g < nb ? static_cast<double>(ac0[k + t]) : 0.0;
    const double a1 = 8 + g < nb ? static_cast<double>(ac1[k + t]) : 0.0;
    double b[NTT];
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt) b[nt] = Xp[size_t(nt * 8 + g) * ld + k + t];
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt) dmma_8x8x4(acc[0][nt], a0, b[nt]);
    if (two)
#pragma unroll
      for (int nt = 0; nt < NTT; ++nt) dmma_8x8x4(acc[1][nt], a1, b[nt]);
  }
  // warp partials [8][16][NJ] in shared memory, then the fixed-order sum
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) part[(warp * 16 + mt * 8 + g) * NJ + nt * 8 + 2 * t + h] = acc[mt][nt][h];
  __syncthreads();
  for (int e = tid; e < 16 * NJ; e += 256) {
    double v = part[e];
#pragma unroll
    for (int w = 1; w < 8; ++w) v += part[w * 16 * NJ + e];
    part[e] = v;
  }
  __syncthreads();
}

// T1s: the leftover candidate lists of T1x (< 64 columns per T1x CTA).
// Every CTA scans the list lengths in T1x-CTA order, so the candidates get a
// deterministic global order; groups of GS consecutive candidates (16 when
// they total <= 256, else 64) times RS row splits form the work units of a
// persistent grid.  Unit (group q, rs) forms the partial C over rows
// [rs R, rs R + R) (ref_small_dots for 16 columns, else ref_batch_dots) and
// stores it to lpart (group q's slab at its first candidate); the last of
// the RS units to finish (counter
// lcnt[q], reset by it) sums the RS partials in rs order (deterministic) and
// runs T1x's per-(column, component) epilogue: threshold, band log,
// objective, nnz, W, Wt, the final activity mask and item flag; f and nnz go
// to part_s[q] in a fixed order.  Grouping across lists reads X once per
// group instead of once per list.  (Per-list units measured 66-74 us at C4
// -- ~60 lists of 1-2 columns each re-reading all of X -- and a
// thread-block-cluster version reducing over distributed shared memory 78.)
template <typename TA, int JPT>
__global__ void __launch_bounds__(256) tc_refine_split_kernel(
    const TA* __restrict__ A, int64_t n, int ld, int m, const double* __restrict__ X, int64_t x_par_stride,
    const double* __restrict__ mu, const double* __restrict__ gamma, int penalty, unsigned char* __restrict__ colmask,
    unsigned char* __restrict__ item_act, double* __restrict__ W, int64_t w_par_stride, double* __restrict__ Wt,
    double* __restrict__ part_s, const GpsCtl* ctl, BandLog* band, const int64_t* __restrict__ left,
    const int* __restrict__ left_n, int nlists, int RS, int rows_per_split, double* __restrict__ lpart,
    unsigned int* __restrict__ lcnt, unsigned int* __restrict__ act_count) {
  constexpr int NJ = 8 * JPT;
  constexpr int NT = NJ / 16;
  if (ctl != nullptr && ctl->done) return;
  extern __shared__ __align__(16) double ref_smem[];
  double* sA = ref_smem;
  double* sX = ref_smem + 2 * kTcRefBatch * kRefKS;
  __shared__ int64_t cand[kTcRefBatch];
  __shared__ unsigned char act[kTcRefBatch];
  __shared__ double smu[NJ], sgam[NJ];
  __shared__ double red[2][8];
  __shared__ int s_last;
  __shared__ int pre[kTcLeftMaxGrid + 1];  // exclusive prefix of the list lengths
  __shared__ int wsum[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const double* Xp = X + parity * x_par_stride;
  double* Wp = W + parity * w_par_stride;
  for (int j = tid; j < NJ; j += 256) {
    smu[j] = j < m ? mu[j] : 1.0;
    sgam[j] = j < m ? gamma[j] : 0.0;
  }
  // block-wide exclusive scan of left_n[0 .. nlists) (4 lists per thread)
  {
    int v[4], t = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = tid * 4 + u;
      v[u] = b < nlists ? left_n[b] : 0;
      t += v[u];
    }
    int incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    int run = off + incl - t;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = tid * 4 + u;
      if (b <= kTcLeftMaxGrid) pre[b] = run;
      run += v[u];
    }
    __syncthreads();
  }
  const int total = pre[nlists];
  const int GS = total <= 256 ? 16 : kTcRefBatch;
  const int groups = (total + GS - 1) / GS;
  for (int u = blockIdx.x; u < groups * RS; u += gridDim.x) {
  const int q = u / RS, rs = u % RS;
  const int g0 = q * GS, nb = min(GS, total - g0);
  __syncthreads();  // the previous unit's readers of cand / act / part are done
  if (tid < nb) {
    // list of global candidate g0 + tid: the last b with pre[b] <= g0 + tid
    const int gi = g0 + tid;
    int lo = 0, hi = nlists - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= gi) lo = mid;
      else hi = mid - 1;
    }
    cand[tid] = left[size_t(lo) * kTcRefBatch + (gi - pre[lo])];
  }
  if (tid < kTcRefBatch) act[tid] = 0;
  __syncthreads();
  const int r_lo = min(ld, rs * rows_per_split), r_hi = min(ld, r_lo + rows_per_split);
  // this unit's partial C [nb][NJ] (shared memory), then to lpart[q][rs]
  double* part = sA;
  if (nb <= 16) {
    ref_small_dots<TA, NJ>(A, ld, Xp, cand, nb, r_lo, r_hi, part);
  } else {
    double acc[2][NT][2];
    ref_batch_dots<TA, NT>(A, ld, Xp, cand, nb, r_lo, r_hi, sA, sX, acc);  // the A tiles are done after it
    const int g = lane >> 2, t = lane & 3, mg = warp & 3, ng = warp >> 2;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          part[(mg * 16 + mt * 8 + g) * NJ + ng * 8 * NT + nt * 8 + 2 * t + h] = acc[mt][nt][h];
    __syncthreads();
  }
  double* slab = lpart + size_t(g0) * RS * NJ;  // [RS][GS][NJ] per group
  for (int e = tid; e < nb * NJ; e += 256) __stcg(slab + size_t(rs) * GS * NJ + e, part[e]);
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    s_last = atomicAdd(&lcnt[q], 1u) == unsigned(RS - 1);
    if (s_last) lcnt[q] = 0;  // for the next sweep (stream order)
  }
  __syncthreads();
  if (!s_last) continue;
  __threadfence();
  for (int e = tid; e < nb * NJ; e += 256) {
    double v = __ldcg(slab + e);
    for (int r = 1; r < RS; ++r) v += __ldcg(slab + size_t(r) * GS * NJ + e);
    part[e] = v;
  }
  __syncthreads();
  double f_acc = 0.0, nnz_acc = 0.0;
  for (int e = tid; e < nb * NJ; e += 256) {
    const int bc = e / NJ, j = e % NJ;
    const int64_t c = cand[bc];
    double w = 0.0;
    if (j < m) {
      const double sj = smu[j] * part[e];
      w = threshold_weight(sj, sgam[j], penalty);
      band_note(band, parity, c, j, sj, sgam[j], penalty);
      f_acc += objective_term(sj, sgam[j], penalty);
      if (w != 0.0) {
        nnz_acc += 1.0;
        act[bc] = 1;  // benign: every writer stores 1
      }
      Wp[size_t(j) * n + c] = w;
    }
    Wt[c * NJ + j] = w;  // padded components 0 (T2 reads whole rows)
  }
  const int nact = __syncthreads_count(tid < nb && act[tid] != 0);
  if (tid == 0 && nact > 0) atomicAdd(act_count, static_cast<unsigned int>(nact));
  if (tid < nb) {
    const int64_t c = cand[tid];
    colmask[c] = act[tid];
    colmask[n + c] = 0;
    if (act[tid]) item_act[c / kTcRefItem] = 1;
  }
  f_acc = warp_sum(f_acc);
  nnz_acc = warp_sum(nnz_acc);
  if (lane == 0) {
    red[0][warp] = f_acc;
    red[1][warp] = nnz_acc;
  }
  __syncthreads();
  if (tid < 2) {
    double t = 0.0;
    for (int w8 = 0; w8 < 8; ++w8) t += red[tid][w8];
    part_s[size_t(q) * 4 + tid] = t;
  }
  }  // units
}

// T2: sparse rank-m update on the ACTIVE columns (colmask), fp64 on the
// fp64 tensor cores: G_partial[b] = A_act W_act for the active columns of
// column range b -- a DGEMM with A's columns gathered on the fly (k = the
// gathered column, m = the row, n = the component).
// grid (GX, ceil(ld / 128)); CTA (b, y) owns the 512-column blocks
// [b B / GX, (b+1) B / GX) (B = ceil(n / 512), two T1x items each), rows
// [128 y, 128 y + 128) and all NJ = 16 NT components.  Warp w owns rows
// 32 (w % 4) .. + 32 (4 m-tiles) and components 8 NT (w / 4) .. + 8 NT (NT
// n-tiles): 4 NT accumulator fragments.  Blocks without an active item are
// skipped 256 at a time; the active columns of consecutive blocks are
// compacted in column order into a list of up to 512, consumed 16 at a time:
// the A tile (16 columns x 128 rows, widened to fp64 once) and the W tile
// (16 columns x NJ, from the column-major copy Wt written by T1x, one
// contiguous 8 NJ-byte row per column) are staged in shared memory (row
// strides = 4 mod 16 doubles: fragment loads are conflict-free), the next
// tile's loads are issued before the current tile's 4 x 4 NT DMMAs per warp
// and k-step.  Every A element is read and converted once per CTA; sums run
// in column order (deterministic run to run).
constexpr int kTcUpdBlock = 512;
constexpr int kUpdR = 128;          // rows per CTA
constexpr int kUpdKT = 16;          // list columns per staged tile
constexpr int kUpdAS = kUpdR + 4;   // sA row stride (doubles), = 4 mod 16
__host__ __device__ constexpr int upd_ws(int nj) { return nj + 4; }  // sW row stride, = 4 mod 16
__host__ __device__ constexpr size_t tc_update_smem(int nj) {
  return (size_t(2) * kUpdKT * kUpdAS + size_t(2) * kUpdKT * upd_ws(nj)) * sizeof(double);
}
constexpr unsigned int kUpdColsPerRange = 8;  // active columns per T2 column range (partial), at least
template <typename TA, int NT>
__global__ void __launch_bounds__(256, 2) tc_update_kernel(const TA* __restrict__ A, int64_t n, int ld, int m,
                                                           const unsigned char* __restrict__ colmask,
                                                           const unsigned char* __restrict__ item_act,
                                                           const double* __restrict__ Wt,
                                                           double* __restrict__ part_g, const GpsCtl* ctl,
                                                           unsigned char* __restrict__ part_nz,
                                                           const unsigned int* __restrict__ act_count) {
  constexpr int NJ = 16 * NT;
  constexpr int WS = upd_ws(NJ);
  constexpr int VN = 16 / sizeof(TA);                     // elements per 16-byte A load
  constexpr int AV = kUpdKT * kUpdR / VN / 256;           // A vectors per thread per tile
  constexpr int WV = (kUpdKT * NJ / 2 + 255) / 256;       // W double2 per thread per tile
  static_assert(AV >= 1 && kUpdKT * kUpdR % (VN * 256) == 0, "A tile mapping");
  using V = typename Vec16<TA>::T;
  if (ctl != nullptr && ctl->done) return;
  extern __shared__ __align__(16) double upd_smem[];
  double* sA = upd_smem;                        // [2][KT][AS]
  double* sW = upd_smem + 2 * kUpdKT * kUpdAS;  // [2][KT][WS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // column ranges in use: one per kUpdColsPerRange active columns (this
  // sweep's count from T1x / T1s), at most gridDim.x -- a sparse sweep sums
  // its few columns in a few partials instead of writing (and K2
  // re-reading) 32 mostly-zero p x m partials.  (One range for < 2048
  // active columns measured slower at C4: 64 CTAs each scanning all 4096
  // block flags, 69 us against 50.)
  const unsigned int want = (*act_count + kUpdColsPerRange - 1) / kUpdColsPerRange;
  const int gxe = static_cast<int>(want < 1u ? 1u : (want > gridDim.x ? gridDim.x : want));
  if (static_cast<int>(blockIdx.x) >= gxe) {
    if (blockIdx.y == 0 && tid == 0) part_nz[blockIdx.x] = 0;
    return;
  }
  const int64_t nblk = (n + kTcUpdBlock - 1) / kTcUpdBlock;
  const int64_t b0 = nblk * blockIdx.x / gxe, b1 = nblk * (blockIdx.x + 1) / gxe;
  const int r0 = blockIdx.y * kUpdR;
  const int g = lane >> 2, t = lane & 3;
  const int rg = warp & 3, cg = warp >> 2;
  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int u = 0; u < NT; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;
  __shared__ int blist[256];
  __shared__ int wcnt[8];
  __shared__ int64_t alist[kTcUpdBlock];
  int acc_n = 0;  // entries in alist (block-uniform)
  int seen = 0;   // active columns of this column range (block-uniform; the same for every row block)

  // block-wide exclusive scan of a per-thread count (fixed order)
  auto scan = [&](int v, int& total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __syncthreads();  // previous readers of wcnt are done
    if (lane == 31) wcnt[warp] = x;
    __syncthreads();
    int off = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      off += (w < warp) ? wcnt[w] : 0;
      total += wcnt[w];
    }
    return off + x - v;
  };
  // A tile vector e: list column e / (R / VN), rows VN (e % (R / VN)) ..;
  // W tile double2 e: list column e / (NJ / 2), components 2 (e % (NJ / 2))
  V ra[AV];
  double2 rw[WV];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < AV; ++i) {
      const int e = tid + 256 * i, kk = e / (kUpdR / VN), r = r0 + VN * (e % (kUpdR / VN));
      V v{};
      if (k0 + kk < acc_n && r < ld) v = *reinterpret_cast<const V*>(A + alist[k0 + kk] * ld + r);
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < WV; ++i) {
      const int e = tid + 256 * i, kk = e / (NJ / 2), j2 = e % (NJ / 2);
      double2 w = make_double2(0.0, 0.0);
      if (e < kUpdKT * NJ / 2 && k0 + kk < acc_n) w = *reinterpret_cast<const double2*>(Wt + alist[k0 + kk] * NJ + 2 * j2);
      rw[i] = w;
    }
  };
  auto flush = [&]() {
    if (acc_n == 0) return;
    load(0);
    int buf = 0;
    for (int k0 = 0; k0 < acc_n; k0 += kUpdKT, buf ^= 1) {
      double* a_s = sA + buf * kUpdKT * kUpdAS;
      double* w_s = sW + buf * kUpdKT * WS;
#pragma unroll
      for (int i = 0; i < AV; ++i) {
        const int e = tid + 256 * i, kk = e / (kUpdR / VN), r = VN * (e % (kUpdR / VN));
        TA el[VN];
        Vec16<TA>::unpack(ra[i], el);
#pragma unroll
        for (int u = 0; u < VN; ++u) a_s[kk * kUpdAS + r + u] = static_cast<double>(el[u]);
      }
#pragma unroll
      for (int i = 0; i < WV; ++i) {
        const int e = tid + 256 * i, kk = e / (NJ / 2), j2 = e % (NJ / 2);
        if (e < kUpdKT * NJ / 2) *reinterpret_cast<double2*>(w_s + kk * WS + 2 * j2) = rw[i];
      }
      __syncthreads();
      if (k0 + kUpdKT < acc_n) load(k0 + kUpdKT);
#pragma unroll
      for (int ks = 0; ks < kUpdKT; ks += 4) {
        double a[4], b[NT];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = a_s[(ks + t) * kUpdAS + rg * 32 + mt * 8 + g];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = w_s[(ks + t) * WS + cg * 8 * NT + nt * 8 + g];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], a[mt], b[nt]);
      }
      // no barrier: buffer buf is refilled two tiles later, after the next
      // tile's barrier, which every warp reaches only once done with buf
    }
    acc_n = 0;
  };

  for (int64_t bb = b0; bb < b1; bb += 256) {
    const int64_t blk = bb + tid;
    const bool ne = blk < b1 && (item_act[2 * blk] | (2 * blk + 1 < (n + kTcRefItem - 1) / kTcRefItem
                                                          ? item_act[2 * blk + 1] : 0)) != 0;
    int nblocks;
    const int bpos = scan(ne ? 1 : 0, nblocks);
    if (ne) blist[bpos] = tid;
    __syncthreads();
    for (int ii = 0; ii < nblocks; ++ii) {
      // this thread's two columns of the block
      const int64_t c0 = (bb + blist[ii]) * kTcUpdBlock + 2 * tid;
      const bool f0 = c0 < n && colmask[c0] != 0;
      const bool f1 = c0 + 1 < n && colmask[c0 + 1] != 0;
      int total;
      const int off = scan(int(f0) + int(f1), total);
      if (acc_n + total > kTcUpdBlock) flush();  // block-uniform
      if (f0) alist[acc_n + off] = c0;
      if (f1) alist[acc_n + off + int(f0)] = c0 + 1;
      acc_n += total;
      seen += total;
    }
    __syncthreads();  // blist reuse
  }
  __syncthreads();
  // A column range without an active column leaves its partial unwritten
  // and flags it empty: K2 skips it (at C4 with 64 active columns nearly
  // every range is empty, and writing and re-reading their zeros cost
  // 2 x 134 MB per iteration).
  if (blockIdx.y == 0 && tid == 0) part_nz[blockIdx.x] = seen > 0 ? 1 : 0;
  if (seen == 0) return;
  flush();
  double* pg = part_g + size_t(blockIdx.x) * NJ * ld;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int r = r0 + rg * 32 + mt * 8 + g;
    if (r < ld)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j = cg * 8 * NT + nt * 8 + 2 * t;
        pg[size_t(j) * ld + r] = acc[mt][nt][0];
        pg[size_t(j + 1) * ld + r] = acc[mt][nt][1];
      }
  }
}

// Loadings of the tensor-core path: W[j][col] of the final sweep is valid
// where T1x processed the column (every candidate, with W = 0 for an
// inactive one); the filtered-out columns still hold older values, so they
// are zeroed here by the final activity mask (colmask[col] = 0).
// Grid (column blocks, components), grid-stride over the columns.
__global__ void tc_mask_w_kernel(double* __restrict__ W, int64_t n, int m, const unsigned char* __restrict__ colmask) {
  double* w = W + int64_t(blockIdx.y) * n;
  for (int64_t col = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; col < n; col += int64_t(gridDim.x) * blockDim.x)
    if (colmask[col] == 0) w[col] = 0.0;
}

}  // namespace gps
