// Persistent cooperative kernel for the coarse end of the V-cycle.
//
// Below a size threshold a GS color pass is a few microseconds of HBM/L2
// traffic but still pays a full dependent-launch gap; at 256^3 the three
// coarse levels are 40 of the ~58 launches of a V-cycle.  This kernel runs
// the whole V-cycle tail (levels lc .. L-1: pre-smooth, restrict, recurse,
// prolong, post-smooth; ref: multigrid.py:140-171) in ONE cooperative launch,
// one grid-wide barrier between dependent phases instead of one launch.
// Arithmetic per row is the same device function the per-pass kernels use,
// so results are bitwise identical; vector loads go through L2 (ld.global.cg)
// because other blocks wrote them earlier in the same launch.
#pragma once
#include <cooperative_groups.h>

#include "hpg_kernels.cuh"

namespace hpg {

template <typename T>
struct TailLevel {
  const int32_t* cols;
  const T* vals;
  const int32_t* inj;  // dst map into this level from its parent (unused for the first)
  T* z;
  T* r;
  int64_t ld, n, n_ext;
  int64_t off[9];
  int ncolors;
};

constexpr int kMaxTail = 8;

template <typename T>
struct TailParams {
  TailLevel<T> lv[kMaxTail];
  int nl, nu1, nu2, nu_c;
};

// Dependent-phase barrier: the whole (cooperative) grid, or -- when the tail
// runs as ONE thread-block cluster -- the cluster's hardware barrier
// (barrier.cluster arrive.release / wait.acquire: global writes of every CTA
// of the cluster are visible after it; the vector loads go through L2).
template <bool CLUSTER>
__device__ __forceinline__ void tail_barrier() {
  if (CLUSTER) cooperative_groups::this_cluster().sync();
  else cooperative_groups::this_grid().sync();
}

// Zero initial guess (ref: smoother.py:95-96): only the halo tail is cleared;
// every owned row is written by its color pass, which forms v * 0 for the
// colors not yet updated instead of loading zeros (known0, same arithmetic).
template <typename T, bool CLUSTER>
__device__ __forceinline__ void tail_sweep(const TailLevel<T>& L, bool zero, int64_t gt, int64_t gs) {
  if (zero && L.n_ext > L.n) {
    for (int64_t i = L.n + gt; i < L.n_ext; i += gs) L.z[i] = T(0);
    tail_barrier<CLUSTER>();
  }
  for (int c = 0; c < L.ncolors; ++c) {
    for (int64_t i = L.off[c] + gt; i < L.off[c + 1]; i += gs)
      gs_row<T, true>(L.cols, L.vals, L.ld, i, L.r, L.z, zero ? L.off[c] : -1);
    tail_barrier<CLUSTER>();
  }
}

template <typename T, bool CLUSTER>
__global__ void __launch_bounds__(256, 2) k_vcycle_tail(const __grid_constant__ TailParams<T> p) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  for (int l = 0; l < p.nl; ++l) {
    const TailLevel<T>& L = p.lv[l];
    const bool last = l == p.nl - 1;
    const int sweeps = last ? p.nu_c : p.nu1;
    for (int s = 0; s < sweeps; ++s) tail_sweep<T, CLUSTER>(L, s == 0, gt, gs);
    if (last) break;
    const TailLevel<T>& C = p.lv[l + 1];
    for (int64_t j = gt; j < C.n; j += gs) restrict_row<T, true>(L.cols, L.vals, L.ld, j, C.inj, L.r, L.z, C.r);
    tail_barrier<CLUSTER>();
  }
  for (int l = p.nl - 2; l >= 0; --l) {
    const TailLevel<T>& L = p.lv[l];
    const TailLevel<T>& C = p.lv[l + 1];
    for (int64_t j = gt; j < C.n; j += gs) L.z[j] = add_rn(__ldcg(L.z + j), __ldcg(C.z + C.inj[j]));
    tail_barrier<CLUSTER>();
    for (int s = 0; s < p.nu2; ++s) tail_sweep<T, CLUSTER>(L, false, gt, gs);
  }
}

}  // namespace hpg
