// Shared device helpers for the GP-SPCA engine (sm_100a only).
//
// Bulk-async copies (cp.async.bulk, SASS UBLKCP) with mbarrier completion
// are the only way A enters shared memory: a stage of T columns of the
// column-major matrix is ONE contiguous byte range, so the 1-D bulk form of
// the TMA engine moves it without a tensor map.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1312_6182_b200 is built for sm_100a only"
#endif

namespace gps {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Make mbarrier initialisation visible to the async (bulk-copy) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// Plain arrive (release semantics at CTA scope): producer/consumer hand-off
// between warp roles without a CTA-wide barrier.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Arrive on behalf of `count` arrivals (one thread releasing a hand-off that
// normally collects one arrival per warp).
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Same, for helper warps whose spinning would steal issue slots from the
// compute warps sharing their SM sub-partition: back off between probes.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(40);
}

// Tensor-core filter scale: column i is scaled by 2^e_i with max|a_i| 2^e_i in
// [2^14, 2^15) (the norms pass computes e_i, tc_kernels.cuh uses it).
constexpr int kTcAScaleExp = 14;

// L2 policy: A is streamed exactly once per sweep and is far larger than L2,
// so it is marked evict-first to keep partials / iterates resident.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
#ifdef GPS_STREAM_EVICT_NORMAL  // diagnostics build: A-stream experiments
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}

// global -> shared bulk copy, completion signalled on `bar` (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Thresholds of the reference (parallel.py:117-128):
//   l1: sign(c) * max(|c| - g, 0)      l0: c if c*c > g else 0 (tie inactive)
template <typename T>
__device__ __forceinline__ T threshold_weight(T c, T gamma, int penalty) {
  if (penalty == 0) {
    T t = fabs(c) - gamma;
    return t > T(0) ? copysign(t, c) : T(0);
  }
  return (c * c > gamma) ? c : T(0);
}

// Objective term (single_unit.py:44-48): (|c|-g)_+^2 or (c^2-g)_+
template <typename T>
__device__ __forceinline__ T objective_term(T c, T gamma, int penalty) {
  if (penalty == 0) {
    T t = fabs(c) - gamma;
    return t > T(0) ? t * t : T(0);
  }
  T t = c * c - gamma;
  return t > T(0) ? t : T(0);
}

// Near-threshold log (the band `north_star` asks to be logged): every
// (column, component) whose scaled correlation s = mu_j c_ij lies within
// 1e-6 gamma_j of the threshold -- ||s| - gamma| <= 1e-6 gamma (l1),
// |s^2 - gamma| <= 1e-6 gamma (l0) -- is appended as col * 64 + j to the
// list of the sweep's parity (the loops double-buffer by iteration parity
// like W, and the step kernel that advances to iteration k + 1 clears the
// list that sweep k + 1 fills).  At gamma = 0 there is no band: a zero
// correlation gives w = 0 on either side of the threshold.
struct BandLog {
  unsigned int count[2];  // entries appended per parity (may exceed cap)
  unsigned int cap;       // capacity per parity
  unsigned int pad;
  long long* entries;     // [2][cap]
};
constexpr double kBandRel = 1e-6;
constexpr int kBandMaxComponents = 64;

__device__ __forceinline__ void band_note(BandLog* b, int parity, int64_t col, int j, double s, double gamma,
                                          int penalty) {
  if (b == nullptr || !(gamma > 0.0)) return;
  const double d = penalty == 0 ? fabs(fabs(s) - gamma) : fabs(s * s - gamma);
  if (d <= kBandRel * gamma) {
    const unsigned int pos = atomicAdd(&b->count[parity], 1u);
    if (pos < b->cap) b->entries[size_t(parity) * b->cap + pos] = col * kBandMaxComponents + j;
  }
}

}  // namespace gps
