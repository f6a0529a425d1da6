// Peer-memory all-reduce for the sharded loops: the one exchange
// per power iteration -- the sum over ranks of [g | f | nnz | ...] (single
// unit, ld + 4 doubles) or of the block G partials -- done by one kernel per
// rank over NVLink peer memory instead of an NCCL call.
//
// Every rank owns a symmetric buffer (cudaMalloc + CUDA IPC, opened by every
// peer):
//   slots  [2][world][count] doubles   (parity of the epoch x source rank)
//   flags  [world][nchunks]  uint64    (epoch at which source rank's chunk
//                                       landed here)
//   state  {epoch, done_ctas}
// Launch e of the kernel (epoch e = previous + 1, parity e & 1) runs one CTA
// per chunk of kPxChunk doubles.  CTA c of rank r
//   1. stores its chunk of the local vector into slots[e&1][r] of EVERY rank
//      (P2P stores), fences (system scope) and release-stores flags[r][c] = e
//      at every rank;
//   2. acquire-spins until flags[q][c] >= e for all q at its own rank;
//   3. sums slots[e&1][0 .. world) in RANK ORDER (identical on every rank, so
//      the step that follows is identical everywhere, and bitwise
//      reproducible run to run) back into the local vector.
// Parity double-buffering makes the slot reuse safe: rank r can only reach
// epoch e + 2 (the next writer of parity e & 1) after its epoch e + 1
// all-reduce, which needs every peer's epoch e + 1 push, which each peer
// issues only after finishing its own epoch e sums.
#pragma once

#include "su_kernels.cuh"

namespace gps {

constexpr int kPxMaxWorld = 8;
constexpr int kPxChunk = 4096;  // doubles per CTA (32 KB)

struct PxState {
  unsigned long long epoch;
  unsigned int done_ctas;
  unsigned int error;  // 1: a wait timed out (a peer stopped, died or diverged)
};

// One rank's view of the symmetric buffers: base pointers of every rank's
// buffer as mapped into this process (peer q: IPC-opened; q == rank: local).
struct PxView {
  double* slots[kPxMaxWorld];
  unsigned long long* flags[kPxMaxWorld];
  PxState* state;  // this rank's
  int world;
  int rank;
  int64_t count;
  int nchunks;
  unsigned long long timeout_ns;  // bound on every flag wait (globaltimer)
};

// Loop status written by a timed-out exchange (GpsCtl::status): the loop
// stops and the host raises instead of every GPU spinning forever.
constexpr int kStatusExchangeTimeout = 4;

__device__ __forceinline__ unsigned long long px_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__host__ __device__ inline size_t px_slots_bytes(int world, int64_t count) {
  return size_t(2) * world * count * sizeof(double);
}
__host__ __device__ inline size_t px_flags_bytes(int world, int nchunks) {
  return size_t(world) * nchunks * sizeof(unsigned long long);
}
// flag slots per rank: the uniform chunks of px_allreduce_kernel, plus one
// (the fused reduction's scalar chunk)
__host__ __device__ inline int px_nchunks(int64_t count) { return int((count + kPxChunk - 1) / kPxChunk) + 1; }
__host__ __device__ inline int px_uniform_chunks(int64_t count) { return int((count + kPxChunk - 1) / kPxChunk); }

__device__ __forceinline__ void px_store_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long px_load_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Publish chunk c of this rank's epoch-e data: fence (system scope) and
// release-store flags[rank][c] = e at every rank.
__device__ __forceinline__ void px_signal(const PxView& v, int c, unsigned long long e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < v.world; ++q) px_store_release_sys(v.flags[q] + size_t(v.rank) * v.nchunks + c, e);
  }
}
// Wait until every rank published chunk c at this rank, then write the
// rank-order sum of elements [lo, hi) into vec.  Every wait is bounded by
// v.timeout_ns: on expiry the error flag is raised and false returned
// (vec untouched), so a rank that stopped, died or launched a different
// number of exchanges cannot hang its peers.
__device__ __forceinline__ bool px_gather(const PxView& v, double* vec, int c, int64_t lo, int64_t hi,
                                          unsigned long long e) {
  __shared__ int s_timeout;
  const int par = static_cast<int>(e & 1ull);
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
  if (threadIdx.x < v.world) {
    const unsigned long long* f = v.flags[v.rank] + size_t(threadIdx.x) * v.nchunks + c;
    const unsigned long long t0 = px_now_ns();
    while (px_load_acquire_sys(f) < e) {
      if (px_now_ns() - t0 > v.timeout_ns) {
        s_timeout = 1;
        atomicExch(&v.state->error, 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (s_timeout) return false;
  // fixed rank-order sum (L2 loads: the slots are written by peers)
  const double* own = v.slots[v.rank] + size_t(par) * v.world * v.count;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double s = __ldcg(own + i);
    for (int q = 1; q < v.world; ++q) s += __ldcg(own + size_t(q) * v.count + i);
    vec[i] = s;
  }
  return true;
}
// Element i of this rank's epoch-e vector into slots[e&1][rank][i] at every rank.
__device__ __forceinline__ void px_put(const PxView& v, int64_t i, double x, unsigned long long e) {
  const int par = static_cast<int>(e & 1ull);
  for (int q = 0; q < v.world; ++q) v.slots[q][(size_t(par) * v.world + v.rank) * v.count + i] = x;
}

// The two halves of every exchange launch.  Production launches run both
// (kPxBoth); the cross-process test on ONE GPU runs them as two launches per
// rank with a host barrier between (every rank pushes, then every rank
// gathers flags that are already set), so no rank's kernel ever waits on a
// kernel of another process sharing the GPU.
constexpr int kPxPush = 1;    // put + signal
constexpr int kPxGather = 2;  // wait + rank-order sum + epoch publication
constexpr int kPxBoth = kPxPush | kPxGather;

// CTA body: chunk c of rank v.rank at epoch e; vec is the rank's local vector.
__device__ __forceinline__ void px_chunk(const PxView& v, double* vec, int c, unsigned long long e,
                                         int phases = kPxBoth) {
  const int64_t lo = int64_t(c) * kPxChunk;
  const int64_t hi = lo + kPxChunk < v.count ? lo + kPxChunk : v.count;
  if (phases & kPxPush) {
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) px_put(v, i, vec[i], e);
    px_signal(v, c, e);
  }
  if (phases & kPxGather) px_gather(v, vec, c, lo, hi, e);  // a timeout is reported through v.state->error
}

// Epoch bookkeeping: every CTA reads the epoch before it finishes; the last
// CTA to finish publishes it for the next launch (stream order).  Returns
// true (block-uniform) in the last CTA, after a fence that makes every other
// CTA's writes of this launch visible to it.
__device__ __forceinline__ bool px_finish(PxState* st, unsigned long long e) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = 0;
    if (atomicAdd(&st->done_ctas, 1u) == gridDim.x - 1u) {
      st->epoch = e;
      st->done_ctas = 0;
      __threadfence();
      s_last = 1;
    }
  }
  __syncthreads();
  return s_last != 0;
}

__global__ void __launch_bounds__(256) px_allreduce_kernel(const PxView v, double* vec, int phases) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&v.state->epoch) + 1ull;
  px_chunk(v, vec, blockIdx.x, e, phases);
  if (phases & kPxGather) px_finish(v.state, e);  // a push-only launch leaves the epoch to its gather
}

// Test emulation of `world` ranks on ONE device as ONE cooperative kernel
// (blocks wait on one another, so they must be co-resident): block (c, r)
// runs rank r's CTA c with rank r's view; vecs[r] is rank r's vector.
struct PxEmu {
  PxView view[kPxMaxWorld];
  double* vecs[kPxMaxWorld];
};
__global__ void __launch_bounds__(256) px_emulate_kernel(const PxEmu emu) {
  const PxView& v = emu.view[blockIdx.y];
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&v.state->epoch) + 1ull;
  px_chunk(v, emu.vecs[blockIdx.y], blockIdx.x, e);
  px_finish(v.state, e);
}

// ---- K2 fused with the exchange: the cross-CTA reduction of one rank's
// sweep partials (su_reduce_kernel's rows and scalars, in the same fixed
// order) written straight into every rank's slots, then the rank-order sum
// into the local exchange vector -- compute and collective in one kernel.
// Chunk c < nrc: rows [c kPxChunk, ...) of the `rows`-long partial vector,
// 32-row sub-blocks as in su_reduce_kernel; chunk nrc: the 4 scalars at
// offset rows.  v.count == rows + 4.
__device__ __forceinline__ bool px_reduce_chunk(const PxView& v, const double* __restrict__ part_g,
                                                const double* __restrict__ part_s, int nparts, int rows,
                                                int nparts_s, double* exch, int c, unsigned long long e,
                                                int phases = kPxBoth, const unsigned char* nz = nullptr) {
  __shared__ double part[kReduceSlices][kReduceRows];
  const int nrc = (rows + kPxChunk - 1) / kPxChunk;
  if (!(phases & kPxPush)) {  // gather half only (cross-process test)
    const int64_t lo = c < nrc ? int64_t(c) * kPxChunk : rows;
    const int64_t hi = c < nrc ? (lo + kPxChunk < rows ? lo + kPxChunk : rows) : int64_t(rows) + 4;
    return px_gather(v, exch, c, lo, hi, e);
  }
  if (c < nrc) {
    const int lo = c * kPxChunk, hi = min(rows, lo + kPxChunk);
    const int rr = threadIdx.x & (kReduceRows - 1), sl = threadIdx.x / kReduceRows;
    const int b0 = nparts * sl / kReduceSlices, b1 = nparts * (sl + 1) / kReduceSlices;
    for (int base = lo; base < hi; base += kReduceRows) {
      const int r = base + rr;
      double t = 0.0;
      if (r < hi) {
        const double* p = part_g + r;
        if (nz == nullptr) {
#pragma unroll 4
          for (int b = b0; b < b1; ++b) t += p[size_t(b) * rows];
        } else {  // as su_reduce_kernel: empty partials were not written
          for (int b = b0; b < b1; ++b)
            if (nz[b]) t += p[size_t(b) * rows];
        }
      }
      part[sl][rr] = t;
      __syncthreads();
      if (sl == 0 && r < hi) {
        double u = part[0][rr];
#pragma unroll
        for (int k = 1; k < kReduceSlices; ++k) u += part[k][rr];
        px_put(v, r, u, e);
      }
      __syncthreads();
    }
    px_signal(v, c, e);
    return (phases & kPxGather) ? px_gather(v, exch, c, lo, hi, e) : true;
  } else {
    if (threadIdx.x < 128) {
      const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
      double t = 0.0;
      for (int b = lane; b < nparts_s; b += 32) t += part_s[size_t(b) * 4 + k];
      t = warp_sum(t);
      if (lane == 0) px_put(v, rows + k, t, e);
    }
    px_signal(v, c, e);
    return (phases & kPxGather) ? px_gather(v, exch, c, rows, int64_t(rows) + 4, e) : true;
  }
}

// With step.xbuf set (single-unit loops) the last CTA to finish also runs the
// power step (K3's su_step_body, same arithmetic) on the all-reduced vector:
// sweep partials -> exchange -> step in one launch per iteration.
__global__ void __launch_bounds__(256) su_reduce_px_kernel(const double* __restrict__ part_g,
                                                           const double* __restrict__ part_s, int nparts, int rows,
                                                           double* __restrict__ exch, GpsCtl* ctl, int nparts_s,
                                                           const PxView v, const SuStepArgs step,
                                                           int phases = kPxBoth,
                                                           const unsigned char* __restrict__ nz = nullptr) {
  if (ctl != nullptr && ctl->done) return;  // identical on every rank (replicated step)
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&v.state->epoch) + 1ull;
  const bool ok = px_reduce_chunk(v, part_g, part_s, nparts, rows, nparts_s, exch, blockIdx.x, e, phases, nz);
  if (!ok && ctl != nullptr && threadIdx.x == 0) {
    ctl->status = kStatusExchangeTimeout;
    ctl->done = 1;
  }
  if (!(phases & kPxGather)) return;
  const bool last = px_finish(v.state, e);
  if (last && ctl != nullptr && step.xbuf != nullptr &&
      *reinterpret_cast<volatile unsigned int*>(&v.state->error) == 0u)
    su_step_body(exch, ctl, step);
}

// Test emulation of the fused reduction: block (c, r) runs rank r's chunk c.
struct PxReduceEmu {
  PxView view[kPxMaxWorld];
  const double* part_g[kPxMaxWorld];
  const double* part_s[kPxMaxWorld];
  double* exch[kPxMaxWorld];
};
__global__ void __launch_bounds__(256) px_reduce_emulate_kernel(const PxReduceEmu emu, int nparts, int rows,
                                                                int nparts_s) {
  const int r = blockIdx.y;
  const PxView& v = emu.view[r];
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&v.state->epoch) + 1ull;
  px_reduce_chunk(v, emu.part_g[r], emu.part_s[r], nparts, rows, nparts_s, emu.exch[r], blockIdx.x, e);
  px_finish(v.state, e);
}

}  // namespace gps
