// One forward multicolor Gauss-Seidel sweep as ONE dataflow kernel.
//
// The per-color launches of a sweep are separated by full-grid barriers, yet a
// row of color c only depends on its 26 neighbours, which lie in the half-
// planes Z-1, Z, Z+1 of the other color blocks (color blocks are sub-lattices
// in x-fastest order, so "color c, half-plane Z" is one contiguous row range).
// Work items (c, Z, chunk) are therefore processed in wavefront order
// t = Z + 2c, and an item only waits until color c-1 has finished the three
// half-planes Z-1..Z+1:
//   * read-after-write: the new values of every color < c in those planes are
//     final (color c-1 finishing plane Z' implies color c-2 finished Z'-1..Z'+1);
//   * write-after-read: color c+1 cannot write plane Z' before color c finished
//     Z'-1..Z'+1, so every old value an item reads is still the old value.
// So each row sees exactly the values it sees in the per-color schedule: the
// result is bitwise identical (ref: smoother.py:108-112).  What changes is the
// memory traffic and the schedule: the active wavefront touches only ~20 half-
// planes of z, which stay in L2 while the matrix planes stream through once,
// and there are no grid-wide drains between colors.
//
// Items are statically dealt round-robin to a co-resident (cooperative) grid in
// wavefront order, so every item an item waits on is owned by a block that
// reaches it first: no deadlock, no ticket atomics.  Completion is counted per
// (color, plane) with release/acquire at gpu scope; gathers of z use L2 loads
// (ld.global.cg) because other CTAs wrote them during this launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hpg_kernels.cuh"

namespace hpg {

constexpr int kWaveRows = 256;  // rows per work item (one per thread)

struct WaveLevel {
  int ncolors;
  int64_t off[kMaxColors + 1];
  int planes[8];      // half-planes per color (Z extent of the color's sub-lattice)
  int64_t plane[8];   // rows per half-plane per color
  int chunks[8];      // work items per half-plane per color
  const int32_t* items;  // [nitems] packed (c << 24) | (Z << 8) | chunk, wavefront order
  int64_t nitems;
  unsigned int* done;    // [8][planes] completed chunks (monotonic across sweeps)
  unsigned int* ctl;     // [0] sweeps completed, [1] blocks exited in this sweep
  int maxplanes;
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// COH: gather z through L2 (ld.global.cg).  Without it the gathers are plain
// (L1-cached) loads; thread 0's gpu-scope acquire followed by the CTA barrier
// orders them after the producers' writes (the acquire invalidates L1).
template <typename T, bool COH>
__global__ void __launch_bounds__(kWaveRows, 3) k_gs_wave(const int32_t* __restrict__ cols,
                                                         const T* __restrict__ vals, int64_t ld,
                                                         const T* __restrict__ r, T* z,
                                                         const __grid_constant__ WaveLevel w, int zero_sweep) {
  // the sweep number comes from device memory so graph replays advance it; it
  // only moves after every block has exited (below)
  const unsigned int epoch = __ldcg(w.ctl) + 1;
  for (int64_t it = blockIdx.x; it < w.nitems; it += gridDim.x) {
    const int32_t code = w.items[it];
    const int c = code >> 24, Z = (code >> 8) & 0xffff, q = code & 0xff;
    if (c > 0 && threadIdx.x < 3) {  // wait for color c-1 on planes Z-1..Z+1 (one thread each)
      const int pc = c - 1, zz = Z - 1 + (int)threadIdx.x;
      if (zz >= 0 && zz < w.planes[pc]) {
        const unsigned int target = epoch * (unsigned int)w.chunks[pc];
        const unsigned int* f = w.done + pc * w.maxplanes + zz;
        while (ld_acquire_gpu(f) < target) {
        }
      }
    }
    __syncthreads();
    const int64_t base = w.off[c] + (int64_t)Z * w.plane[c];
    const int64_t i = base + (int64_t)q * kWaveRows + threadIdx.x;
    if (i < base + w.plane[c])
      gs_row<T, COH>(cols, vals, ld, i, r, z, zero_sweep ? w.off[c] : -1);
    __syncthreads();  // the item's rows are written ...
    if (threadIdx.x == 0) {
      __threadfence();  // ... and visible GPU-wide before the count
      atomicAdd(w.done + c * w.maxplanes + Z, 1u);
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(w.ctl + 1, 1u) == gridDim.x - 1) {  // last block out
      w.ctl[1] = 0;
      w.ctl[0] = epoch;
    }
  }
}

}  // namespace hpg
