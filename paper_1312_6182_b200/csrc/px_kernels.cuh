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

#include "common.cuh"

namespace gps {

constexpr int kPxMaxWorld = 8;
constexpr int kPxChunk = 4096;  // doubles per CTA (32 KB)

struct PxState {
  unsigned long long epoch;
  unsigned int done_ctas;
  unsigned int pad;
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
};

__host__ __device__ inline size_t px_slots_bytes(int world, int64_t count) {
  return size_t(2) * world * count * sizeof(double);
}
__host__ __device__ inline size_t px_flags_bytes(int world, int nchunks) {
  return size_t(world) * nchunks * sizeof(unsigned long long);
}
__host__ __device__ inline int px_nchunks(int64_t count) { return int((count + kPxChunk - 1) / kPxChunk); }

__device__ __forceinline__ void px_store_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long px_load_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// CTA body: chunk c of rank v.rank at epoch e; vec is the rank's local vector.
__device__ __forceinline__ void px_chunk(const PxView& v, double* vec, int c, unsigned long long e) {
  const int par = static_cast<int>(e & 1ull);
  const int64_t lo = int64_t(c) * kPxChunk;
  const int64_t hi = lo + kPxChunk < v.count ? lo + kPxChunk : v.count;
  // 1. push the chunk to every rank (self included)
  for (int q = 0; q < v.world; ++q) {
    double* dst = v.slots[q] + (size_t(par) * v.world + v.rank) * v.count;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) dst[i] = vec[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < v.world; ++q) px_store_release_sys(v.flags[q] + size_t(v.rank) * v.nchunks + c, e);
  }
  // 2. wait for every rank's chunk at this rank
  if (threadIdx.x < v.world) {
    const unsigned long long* f = v.flags[v.rank] + size_t(threadIdx.x) * v.nchunks + c;
    while (px_load_acquire_sys(f) < e) __nanosleep(64);
  }
  __syncthreads();
  // 3. fixed rank-order sum (L2 loads: the slots are written by peers)
  const double* own = v.slots[v.rank] + size_t(par) * v.world * v.count;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double s = __ldcg(own + i);
    for (int q = 1; q < v.world; ++q) s += __ldcg(own + size_t(q) * v.count + i);
    vec[i] = s;
  }
}

// Epoch bookkeeping: every CTA reads the epoch before it finishes; the last
// CTA to finish publishes it for the next launch (stream order).
__device__ __forceinline__ void px_finish(PxState* st, int nchunks, unsigned long long e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&st->done_ctas, 1u) == unsigned(nchunks) - 1u) {
      st->epoch = e;
      st->done_ctas = 0;
      __threadfence();
    }
  }
}

__global__ void __launch_bounds__(256) px_allreduce_kernel(const PxView v, double* vec) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&v.state->epoch) + 1ull;
  px_chunk(v, vec, blockIdx.x, e);
  px_finish(v.state, v.nchunks, e);
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
  px_finish(v.state, v.nchunks, e);
}

}  // namespace gps
