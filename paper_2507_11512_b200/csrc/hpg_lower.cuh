// Zero-initial-guess Gauss-Seidel sweep on the strictly-lower part.
//
// With z = 0 on entry (ref: smoother.py:95-96), a row of color c sees new values
// only at columns of colors < c; every other product of its 27-slot sum is
// v * 0 = +-0 (the diagonal's is 0 * z_i by the reference's zeroed offvals,
// padding is 0 * z[0]).  The accumulator starts at +0 and can never become -0
// (only -0 + -0 is -0), so adding a +-0 product never changes it: the slot-order
// sum of the lower entries alone is the full row sum BIT FOR BIT.  The sweep
// therefore streams only the lower entries (about half of the matrix, ~13 of 27
// slots per row on the 8-color lattice) plus a diagonal vector, instead of every
// slot.  The flop model is unchanged (ref: metrics.py counts the full sweep).
//
// Layout per level and color block c: slot-major ELL [W_c][ldc_c] of the row's
// lower entries in their original slot order, padded with (column 0, value 0);
// W_c = max lower count over the block.  dg = a_ii per row.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "hpg_geom.h"
#include "hpg_kernels.cuh"

namespace hpg {

struct LowerColor {
  int64_t base;  // first element of this color's [W][ldc] block
  int64_t ldc;   // row stride (rows of the color padded to 32)
  int w;         // width
};

__device__ __forceinline__ int color_of_row(const Geom& g, int64_t i) {
  int c = 0;
  while (c + 1 < g.ncolors && i >= g.off[c + 1]) ++c;
  return c;
}

__device__ __forceinline__ bool is_lower(int32_t col, double v, int64_t lim) {
  return col >= 0 && col < lim && v != 0.0;  // off-diagonal (diag is ~col), stored, earlier color
}

// W_c = max over the color block of the lower-entry count
__global__ void k_lower_count(Geom g, int64_t ld, const int32_t* __restrict__ cols, const double* __restrict__ v64,
                              int* __restrict__ width) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const int c = color_of_row(g, i);
  int k = 0;
  for (int s = 0; s < kWidth; ++s) k += is_lower(cols[s * ld + i], v64[s * ld + i], g.off[c]);
  atomicMax(width + c, k);
}

__global__ void k_lower_fill(Geom g, int64_t ld, const int32_t* __restrict__ cols, const double* __restrict__ v64,
                             const LowerColor* __restrict__ lc, int32_t* __restrict__ lcols,
                             double* __restrict__ lv64, float* __restrict__ lv32, double* __restrict__ dg64,
                             float* __restrict__ dg32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const int c = color_of_row(g, i);
  const LowerColor L = lc[c];
  const int64_t j = i - g.off[c];
  int k = 0;
  for (int s = 0; s < kWidth; ++s) {
    const int32_t col = cols[s * ld + i];
    const double v = v64[s * ld + i];
    if (col < 0) {
      dg64[i] = v;
      dg32[i] = (float)v;
    }
    if (is_lower(col, v, g.off[c])) {
      lcols[L.base + k * L.ldc + j] = col;
      lv64[L.base + k * L.ldc + j] = v;
      lv32[L.base + k * L.ldc + j] = (float)v;
      ++k;
    }
  }
  for (; k < L.w; ++k) {
    lcols[L.base + k * L.ldc + j] = 0;
    lv64[L.base + k * L.ldc + j] = 0.0;
    lv32[L.base + k * L.ldc + j] = 0.0f;
  }
}

// One color of the zero-initial-guess sweep: z_i = (r_i - sum_lower v z) / a_ii.
// WMAX >= w; the loads are predicated on the (uniform) width.
// Blocks per SM by width: narrow rows keep few loads in flight per thread, so
// they need more resident warps to cover HBM latency (Little's law); wide rows
// need the registers (3 W live values per thread, 5 W in fp64).
template <typename T, int W>
constexpr int lower_minb() {
  return sizeof(T) == 4 ? (W <= 4 ? 8 : W <= 8 ? 6 : W <= 16 ? 4 : W <= 23 ? 3 : 2)
                        : (W <= 4 ? 6 : W <= 8 ? 5 : W <= 12 ? 4 : W <= 16 ? 3 : 2);
}

// L2 evict-first hint on the lower-part planes (1: fp32 sweeps, 2: fp32 and fp64)
#ifndef HPG_LOWER_HINT
#define HPG_LOWER_HINT 1
#endif
template <typename T>
__device__ __forceinline__ constexpr bool lower_hint() {
  return HPG_LOWER_HINT == 2 || (HPG_LOWER_HINT == 1 && sizeof(T) == 4);
}

// One color of the zero-initial-guess sweep: z_i = (r_i - sum_lower v z) / a_ii,
// instantiated per exact width W (no predicated slots).
template <typename T, int W>
__global__ void __launch_bounds__(256, lower_minb<T, W>()) k_gs_lower(const int32_t* __restrict__ lcols,
                                                                       const T* __restrict__ lvals, int64_t ldc,
                                                                       int64_t row0, int64_t nrows,
                                                                       const T* __restrict__ dg,
                                                                       const T* __restrict__ r, T* z, int rev) {
  pdl_trigger();
  const int64_t blk = rev ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;  // see k_gs_pass
  const int64_t j = blk * blockDim.x + threadIdx.x;
  if (j >= nrows) return;
  const int64_t i = row0 + j;
  int32_t c[W > 0 ? W : 1];
  T v[W > 0 ? W : 1];
  if (lower_hint<T>()) {  // evict-first: keep z (gathered by every color) in L2
    const uint64_t pol = evict_first_policy();
#pragma unroll
    for (int s = 0; s < W; ++s) c[s] = ld_stream_ef(lcols + s * ldc + j, pol);
#pragma unroll
    for (int s = 0; s < W; ++s) v[s] = ld_stream_ef(lvals + s * ldc + j, pol);
  } else {
    const uint64_t pol = stream_policy();
#pragma unroll
    for (int s = 0; s < W; ++s) c[s] = ld_stream(lcols + s * ldc + j, pol);
#pragma unroll
    for (int s = 0; s < W; ++s) v[s] = ld_stream(lvals + s * ldc + j, pol);
  }
  const T d = dg[i];
  // z of the earlier colors (and r) are written by previous kernels
  if (W > 0) pdl_wait_after(v[0]);
  else pdl_wait();
  const T ri = r[i];
  T g[W > 0 ? W : 1];
#pragma unroll
  for (int s = 0; s < W; ++s) g[s] = z[c[s]];
  T acc = T(0);
#pragma unroll
  for (int s = 0; s < W; ++s) acc = add_rn(acc, mul_rn(v[s], g[s]));
  z[i] = div_rn(sub_rn(ri, acc), d);
}

// Implicit-index variant for the 8-color lattice (Stencil on, parity bits
// x->0, y->1, z->2): for a color C the lower entries of an interior row are the
// offsets whose neighbour color C ^ mask(d) is < C, in slot order -- a
// compile-time list, so W = lower_width(C) and the columns of interior rows
// follow from the row's coordinates like stencil_cols (checked at build).
// Rows on a face of the box load their lower ELL columns.
__host__ __device__ constexpr int lower_mask(int s) {
  return ((s % 3) != 1 ? 1 : 0) | (((s / 3) % 3) != 1 ? 2 : 0) | ((s / 9) != 1 ? 4 : 0);
}
__host__ __device__ constexpr int lower_width(int C) {
  int w = 0;
  for (int s = 0; s < kWidth; ++s) w += s != kDiagSlot && (C ^ lower_mask(s)) < C;
  return w;
}
__host__ __device__ constexpr int lower_dir(int C, int k) {
  for (int s = 0; s < kWidth; ++s)
    if (s != kDiagSlot && (C ^ lower_mask(s)) < C && k-- == 0) return s;
  return -1;
}

template <int C, int W>
__device__ __forceinline__ bool stencil_lower_cols(const Stencil& st, uint32_t j, int32_t (&c)[W]) {
  const uint32_t Z = st_div(j, st.hxy, st.mhxy);
  const uint32_t p = j - Z * st.hxy;
  const uint32_t Y = st_div(p, st.hx, st.mhx);
  const uint32_t X = p - Y * st.hx;
  const int x = (int)(2 * X + (C & 1)), y = (int)(2 * Y + ((C >> 1) & 1)), z = (int)(2 * Z + (C >> 2));
  if (x < 1 || x > st.lx - 2 || y < 1 || y > st.ly - 2 || z < 1 || z > st.lz - 2) return false;
  int32_t px[3], py[3], pz[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int ax = x + d - 1, ay = y + d - 1, az = z + d - 1;
    px[d] = (int32_t)((ax & 1 ? st.cx : 0u) + (uint32_t)(ax >> 1));
    py[d] = (int32_t)((ay & 1 ? st.cy : 0u) + (uint32_t)(ay >> 1) * st.hx);
    pz[d] = (int32_t)((az & 1 ? st.cz : 0u) + (uint32_t)(az >> 1) * st.hxy);
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int s = lower_dir(C, k);
    c[k] = pz[s / 9] + py[(s / 3) % 3] + px[s % 3];
  }
  return true;
}

#ifndef HPG_LOWER_BLOCK
#define HPG_LOWER_BLOCK 256  // measured level-0 zero sweep: 256 260 us, 128 269
#endif
template <typename T, int C>
__global__ void __launch_bounds__(HPG_LOWER_BLOCK, lower_minb<T, lower_width(C)>() * 256 / HPG_LOWER_BLOCK) k_gs_lower_st(
    const int32_t* __restrict__ lcols, const T* __restrict__ lvals, int64_t ldc, int64_t row0, int64_t nrows,
    const T* __restrict__ dg, const T* __restrict__ r, T* z, int rev, const Stencil st) {
  constexpr int W = lower_width(C);
  pdl_trigger();
  const int64_t blk = rev ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t j = blk * blockDim.x + threadIdx.x;
  if (j >= nrows) return;
  const int64_t i = row0 + j;
  int32_t c[W > 0 ? W : 1];
  T v[W > 0 ? W : 1];
  const uint64_t pol = lower_hint<T>() ? evict_first_policy() : stream_policy();
  if constexpr (W > 0) {
    if (!stencil_lower_cols<C>(st, (uint32_t)j, c)) {
#pragma unroll
      for (int s = 0; s < W; ++s)
        c[s] = lower_hint<T>() ? ld_stream_ef(lcols + s * ldc + j, pol) : ld_stream(lcols + s * ldc + j, pol);
    }
  }
#pragma unroll
  for (int s = 0; s < W; ++s) v[s] = lower_hint<T>() ? ld_stream_ef(lvals + s * ldc + j, pol) : ld_stream(lvals + s * ldc + j, pol);
  const T d = dg[i];
  if (W > 0) pdl_wait_after(v[0]);
  else pdl_wait();
  const T ri = r[i];
  T g[W > 0 ? W : 1];
#pragma unroll
  for (int s = 0; s < W; ++s) g[s] = z[c[s]];
  T acc = T(0);
#pragma unroll
  for (int s = 0; s < W; ++s) acc = add_rn(acc, mul_rn(v[s], g[s]));
  z[i] = div_rn(sub_rn(ri, acc), d);
}

// bad |= 1 when an interior row's closed-form lower columns differ from the
// stored lower ELL of color C (the level then keeps the index stream)
template <int C>
__global__ void k_check_lower_st(const int32_t* __restrict__ lcols, int64_t ldc, int64_t nrows, Stencil st,
                                 unsigned int* __restrict__ bad) {
  constexpr int W = lower_width(C);
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (W > 0) {
    if (j >= nrows) return;
    int32_t c[W];
    if (!stencil_lower_cols<C>(st, (uint32_t)j, c)) return;
    for (int k = 0; k < W; ++k)
      if (c[k] != lcols[k * ldc + j]) atomicOr(bad, 1u);
  }
}
__host__ inline void (*check_lower_st_kernel(int color))(const int32_t*, int64_t, int64_t, Stencil, unsigned int*) {
  void (*tab[])(const int32_t*, int64_t, int64_t, Stencil, unsigned int*) = {
      k_check_lower_st<0>, k_check_lower_st<1>, k_check_lower_st<2>, k_check_lower_st<3>,
      k_check_lower_st<4>, k_check_lower_st<5>, k_check_lower_st<6>, k_check_lower_st<7>};
  return tab[color];
}

template <typename T>
using LowerStKernel = void (*)(const int32_t*, const T*, int64_t, int64_t, int64_t, const T*, const T*, T*, int,
                               const Stencil);
template <typename T>
__host__ LowerStKernel<T> lower_st_kernel(int color) {
  LowerStKernel<T> tab[] = {k_gs_lower_st<T, 0>, k_gs_lower_st<T, 1>, k_gs_lower_st<T, 2>, k_gs_lower_st<T, 3>,
                            k_gs_lower_st<T, 4>, k_gs_lower_st<T, 5>, k_gs_lower_st<T, 6>, k_gs_lower_st<T, 7>};
  return tab[color];
}

template <typename T>
using LowerKernel = void (*)(const int32_t*, const T*, int64_t, int64_t, int64_t, const T*, const T*, T*, int);

template <typename T, int... Ws>
__host__ LowerKernel<T> lower_kernel_of(int w, std::integer_sequence<int, Ws...>) {
  LowerKernel<T> tab[] = {k_gs_lower<T, Ws>...};
  return tab[w];
}
// the kernel for width w in [0, 27]
template <typename T>
__host__ LowerKernel<T> lower_kernel(int w) {
  return lower_kernel_of<T>(w, std::make_integer_sequence<int, kWidth + 1>{});
}

}  // namespace hpg
