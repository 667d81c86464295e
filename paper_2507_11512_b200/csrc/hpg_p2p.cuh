// One-sided NVLink communication between the ranks' GPUs (no NCCL on the
// data path once enabled).
//
// Every rank owns one "symmetric" device buffer (cudaMalloc'd, exported by
// CUDA IPC and mapped by every peer):
//   [0, 32 KiB)        halo flags, one uint64 per sender rank
//   [32 KiB, 64 KiB)   all-reduce flags, one uint64 per sender rank
//   [64 KiB, ...)      all-reduce slots [2 parities][nranks senders][64] x 8 B
//   then               halo staging: per level, per neighbour (ascending rank),
//                      2 parities x count x 8 B
// Messages carry a monotonically increasing sequence number; a message with
// sequence s lands in parity s&1 and is published by st.release.sys of s into
// the receiver's flag slot for that sender, after a system-scope fence.  A
// receiver acquires (ld.acquire.sys) before reading.  Two parities suffice:
// a sender can only reach message s+2 after receiving the receiver's message
// s+1, which the receiver sends only after it consumed message s.
//
//  * k_halo_p2p: pack straight into every neighbour's staging (P2P stores over
//    NVLink), publish, wait for the neighbours' messages, unpack into the halo
//    tail -- one kernel per exchange instead of pack + NCCL group
//    (ref: comm.py:239-251).
//  * p2p_allreduce_block: every rank puts its partial vector into every peer's
//    slot, then folds all ranks' slots in ascending rank order -- the
//    reference's all_reduce_sum bit for bit on every rank (ref: comm.py:97-108).
//    Used inside the fused CGS2 kernel between its passes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hpg {

constexpr int kMaxRanks = 4096;
constexpr size_t kSymHaloFlags = 0;
constexpr size_t kSymArFlags = 32 * 1024;
constexpr size_t kSymArSlots = 64 * 1024;
constexpr int kArSlot = 64;  // values per (parity, sender)

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const uint64_t* p, uint64_t seq) {
  while (ld_acquire_sys(p) < seq) {
  }
}
// Make every store of this CTA so far visible system-wide before the caller's
// next store: the CTA barrier orders the other threads' stores before thread
// 0's system-scope fence, which is cumulative (one fence per CTA, not per thread).
__device__ __forceinline__ void cta_fence_sys() {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncthreads();
}

struct P2PAr {
  char* const* peer;  // [nranks] symmetric-buffer bases (peer[me] = own)
  int me, nranks;
};

// CTA-wide rank-ordered all-reduce of buf[0..cnt) (cnt <= 64), in place.
template <typename T>
__device__ void p2p_allreduce_block(T* buf, int cnt, const P2PAr& ar, uint64_t seq) {
  const int par = (int)(seq & 1);
  __shared__ T mine[kArSlot];
  if (threadIdx.x < cnt) {
    const T v = buf[threadIdx.x];
    mine[threadIdx.x] = v;
    for (int q = 0; q < ar.nranks; ++q) {
      if (q == ar.me) continue;
      T* slot = (T*)(ar.peer[q] + kSymArSlots) + ((size_t)par * ar.nranks + ar.me) * kArSlot;
      slot[threadIdx.x] = v;
    }
  }
  cta_fence_sys();
  if (threadIdx.x == 0) {
    for (int q = 0; q < ar.nranks; ++q)
      if (q != ar.me) st_release_sys((uint64_t*)(ar.peer[q] + kSymArFlags) + ar.me, seq);
    for (int q = 0; q < ar.nranks; ++q)
      if (q != ar.me) spin_until((const uint64_t*)(ar.peer[ar.me] + kSymArFlags) + q, seq);
  }
  __syncthreads();
  if (threadIdx.x < cnt) {
    const T* own = (const T*)(ar.peer[ar.me] + kSymArSlots);
    T acc = T(0);
    for (int q = 0; q < ar.nranks; ++q) {
      const T v = q == ar.me ? mine[threadIdx.x]
                             : __ldcg(own + ((size_t)par * ar.nranks + q) * kArSlot + threadIdx.x);
      acc = q == 0 ? v : acc + v;
    }
    buf[threadIdx.x] = acc;
  }
  __syncthreads();
}

template <typename T>
__global__ void k_p2p_allreduce(T* buf, int cnt, P2PAr ar, uint64_t seq, int sqrt_first) {
  p2p_allreduce_block<T>(buf, cnt, ar, seq);
  if (sqrt_first && threadIdx.x == 0) buf[0] = sqrt(buf[0]);
}

struct P2PNbr {
  char* remote_stage;   // my region in the neighbour's staging (2 parities x cnt x 8 B)
  char* local_stage;    // the neighbour's region in my staging
  uint64_t* remote_flag;
  const uint64_t* local_flag;
  int64_t send_off;     // into the level's concatenated send list
  int64_t cnt;
  int64_t recv_base;    // first halo slot of this neighbour in the vector
};

constexpr int kMaxNbr = 26;
struct P2PHalo {
  P2PNbr nb[kMaxNbr];
  int nn;
  int64_t total;        // sum of cnt (send == receive volume per neighbour)
};

template <typename T>
__global__ void __launch_bounds__(256) k_halo_p2p(T* v, const int32_t* __restrict__ send_idx,
                                                  const __grid_constant__ P2PHalo h, uint64_t seq,
                                                  unsigned int* done) {
  // launched with PDL: let the consumer (the next colour pass / SpMV) launch now --
  // it streams its matrix planes while the halo moves and waits for this grid
  // before it reads v -- then wait for the producer of v before packing it
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int par = (int)(seq & 1);
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  // phase 1: pack straight into the neighbours' staging over NVLink
  for (int k = 0; k < h.nn; ++k) {
    const P2PNbr& nb = h.nb[k];
    T* dst = (T*)nb.remote_stage + par * nb.cnt;
    for (int64_t e = gt; e < nb.cnt; e += gs) dst[e] = v[send_idx[nb.send_off + e]];
  }
  cta_fence_sys();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(done, 1u);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {  // every block's stores are fenced: publish
    *done = 0;
    for (int k = 0; k < h.nn; ++k) st_release_sys(h.nb[k].remote_flag, seq);
  }
  // phase 2: wait for the neighbours' messages, unpack into the halo tail
  if (threadIdx.x == 0)
    for (int k = 0; k < h.nn; ++k) spin_until(h.nb[k].local_flag, seq);
  __syncthreads();
  for (int k = 0; k < h.nn; ++k) {
    const P2PNbr& nb = h.nb[k];
    const T* src = (const T*)nb.local_stage + par * nb.cnt;
    for (int64_t e = gt; e < nb.cnt; e += gs) v[nb.recv_base + e] = __ldcg(src + e);
  }
}

}  // namespace hpg
