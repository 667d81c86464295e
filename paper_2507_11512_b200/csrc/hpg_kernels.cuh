// sm_100a kernels of the HPG-MxP solve path.
//
// Layout (per level):
//   cols  int32 [27][ld]  slot-major ELL ("column-major"), ld = n rounded up to 64
//   v64   f64   [27][ld]  values, compacted rows, ascending global column
//   v32   f32   [27][ld]  the same values narrowed (26 / -1 / 0 are exact)
// The diagonal slot stores ~col (negative) instead of col, so the smoother
// finds a_ii without a separate diag_pos stream; padding slots hold column 0
// and value 0 exactly like the reference's spmv_cols (ref: problem.py:59-65).
//
// Stencil kernels reproduce the reference's arithmetic bitwise: per row the
// 27 products are accumulated in slot order with separate IEEE multiply and
// add (no FMA contraction), closed by an IEEE subtract / divide
// (ref: krylov.py:76-80, smoother.py:62-75, multigrid.py:107-128).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hpg {

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// streaming loads for the matrix planes: read once, do not pollute L1, and
// (HPG_L2_HINT) mark the lines evict-first in L2 so the gathered vectors and
// the coarse levels stay resident while gigabytes of level-0 planes stream by
#ifndef HPG_L2_HINT
#define HPG_L2_HINT 0  // measured: no gain for fp32, 1.4% slower fp64 V-cycle
#endif
__device__ __forceinline__ uint64_t stream_policy() {
  uint64_t pol = 0;
#if HPG_L2_HINT
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
  int32_t v;
#if HPG_L2_HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
  float v;
#if HPG_L2_HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
#if HPG_L2_HINT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
#endif
  return v;
}

// evict-first streaming loads regardless of HPG_L2_HINT (the zero-guess sweep's
// lower-part planes: measured -5% per fp32 level-0 sweep, see hpg_lower.cuh)
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int32_t ld_stream_ef(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream_ef(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream_ef(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// Programmatic dependent launch: a kernel launched with the PDL attribute may
// start while its predecessor drains; it issues its predecessor-independent
// loads (the matrix planes) first and waits here before touching anything the
// predecessor writes or reads.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// ptxas hoists an unconditional griddepcontrol.wait above the independent
// streaming loads (SASS: ACQBULK first), which forfeits the overlap PDL is for.
// Guarding it with a test on a streamed value pins it after that load: the
// all-ones bit pattern (a NaN / -1 index pair never stored in a matrix plane)
// never occurs, so the wait always executes.
template <typename T>
__device__ __forceinline__ void pdl_wait_after(T loaded) {
  unsigned long long bits = 0;
  if (sizeof(T) == 8) memcpy(&bits, &loaded, 8);
  else {
    unsigned int b32;
    memcpy(&b32, &loaded, 4);
    bits = b32 | 0xffffffff00000000ull;
  }
  if (bits != ~0ull) pdl_wait();
}

// ------------------------------------------------------------ stencil kernels
//
// Every stencil kernel handles one row per thread and is written "all loads
// first": the 27 column indices and 27 values of the row are loaded into
// registers, then the 27 gathers are issued, then the products are summed in
// slot order.  That puts ~81 independent loads in flight per thread, which
// saturates HBM at modest occupancy on the big levels and turns the small
// (coarse) levels into ~2 memory round trips instead of 27.

// acc = sum_s vals[s] * x[col[s]] with the diagonal slot's value returned in
// *d and (when ZERO_DIAG) excluded as 0 * x[i], exactly like the reference's
// zeroed offvals (ref: smoother.py:44-46, 62-66).
// Vector loads that must see writes made by OTHER blocks earlier in the same
// kernel (the persistent coarse-level kernel): bypass L1 (ld.global.cg).
template <bool COHERENT, typename T>
__device__ __forceinline__ T ldv(const T* p) {
  if (COHERENT) return __ldcg(p);
  return *p;
}

// Implicit-index ("stencil layout") rows.  With the greedy coloring and even
// local extents every color block is an (lx/2)(ly/2)(lz/2) sub-lattice of the
// same size n8 (ref: coloring.py:78-80 order), and a row whose 27 neighbours
// all lie inside the local box has its ELL columns in closed form: slot s is
// offset (dx,dy,dz) in z-slowest order (problem.py:88-142 compaction keeps all
// 27), column = color(x+dx, y+dy, z+dz) * n8 + natural position in that
// sub-lattice.  Such rows skip the 27 column-index loads -- 4 of the 8 (fp32)
// or 12 (fp64) bytes per nonzero -- and gather exactly the columns stored in
// the ELL (checked row by row at build, k_check_stencil), so sums are bitwise
// unchanged.  Rows on a face of the box stream their ELL columns as before.
struct Stencil {
  int on;
  uint32_t n8, hx, hy, hxy;  // color block size; sub-lattice extents
  uint32_t cx, cy, cz;       // color-block offset contributed by an odd x / y / z
  int lx, ly, lz;
  int bx, by, bz;            // parity bit of each axis in the color id
  uint64_t mn8, mhxy, mhx;   // ceil(2^64 / d): q = umul64hi(i, m) == i / d exactly for i, d < 2^32
  int ifc;                   // bit 2a / 2a+1: the low / high face of axis a is a rank interface
};

#ifndef HPG_ST_MAGIC
#define HPG_ST_MAGIC 1
#endif
__device__ __forceinline__ uint32_t st_div(uint32_t a, uint32_t d, uint64_t m) {
  if (HPG_ST_MAGIC) return d == 1 ? a : (uint32_t)__umul64hi((uint64_t)a, m);
  return a / d;
}

__device__ __forceinline__ bool stencil_cols(const Stencil& st, uint32_t i, int32_t (&c)[27]) {
  const uint32_t col = st_div(i, st.n8, st.mn8);
  uint32_t pos = i - col * st.n8;
  const uint32_t Z = st_div(pos, st.hxy, st.mhxy);
  pos -= Z * st.hxy;
  const uint32_t Y = st_div(pos, st.hx, st.mhx);
  const uint32_t X = pos - Y * st.hx;
  const int x = (int)(2 * X + ((col >> st.bx) & 1));
  const int y = (int)(2 * Y + ((col >> st.by) & 1));
  const int z = (int)(2 * Z + ((col >> st.bz) & 1));
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
  for (int s = 0; s < 27; ++s) c[s] = pz[s / 9] + py[(s / 3) % 3] + px[s % 3];
  c[13] = ~c[13];
  return true;
}

// known0 >= 0: columns >= known0 are known to hold 0 (the smoother's zero
// initial guess for colors not yet updated in this sweep, and the zeroed halo):
// their products are still formed -- v * 0, the reference's arithmetic -- only
// the load of a known zero is skipped.
template <typename T, bool ZERO_DIAG, bool COHERENT = false, bool PDL = false>
__device__ __forceinline__ T row_accumulate(const int32_t* __restrict__ cols, const T* __restrict__ vals,
                                            int64_t ld, int64_t i, const T* x, T* d, int64_t known0 = -1,
                                            const Stencil st = Stencil{}) {
  int32_t c[27];
  T v[27];
  const uint64_t pol = stream_policy();
  if (!(st.on && stencil_cols(st, (uint32_t)i, c))) {
#pragma unroll
    for (int s = 0; s < 27; ++s) c[s] = ld_stream(cols + s * ld + i, pol);
  }
#pragma unroll
  for (int s = 0; s < 27; ++s) v[s] = ld_stream(vals + s * ld + i, pol);
#ifndef HPG_PIN_WAIT
#define HPG_PIN_WAIT 0
#endif
  // x may be written by the predecessor kernel
  if (PDL) {
    if (HPG_PIN_WAIT) pdl_wait_after(v[26]);
    else pdl_wait();  // (ptxas hoists it above the streams: measured better for the 27-slot kernels)
  }
  T g[27];
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    const int32_t cc = c[s] < 0 ? ~c[s] : c[s];
    g[s] = (known0 >= 0 && cc >= known0) ? T(0) : ldv<COHERENT>(x + cc);
  }
  T acc = T(0);
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    T vs = v[s];
    if (ZERO_DIAG && c[s] < 0) {
      *d = vs;
      vs = T(0);
    }
    acc = add_rn(acc, mul_rn(vs, g[s]));
  }
  return acc;
}

// y[i] = sum_s A[i,s] x[col[i,s]]  for rows [row0, row0+nrows)
// MODE 0: y = Ax.  MODE 1: y = b - Ax and per-block partial of sum y^2 (fp64 outer residual).
// skip (nullable): rows with skip[i] != 0 are left alone (interior/boundary
// split for the overlapped halo exchange); list (nullable): row t is list[t].
#ifndef HPG_SPMV_MINB
#define HPG_SPMV_MINB 4  // fp32 (r01q/r01r A/B, 128-thread blocks): 2 (80 regs) 456 us, 4 (64 regs) 444, 5 (48 + spill) 450
#endif
#ifndef HPG_SPMV_BLOCK
#define HPG_SPMV_BLOCK 128  // measured fp32 SpMV: 128 454 us, 256 466
#endif
template <typename T, int MODE, bool SPLIT = false>
__global__ void __launch_bounds__(MODE == 0 && !SPLIT ? HPG_SPMV_BLOCK : 256,
                                  (sizeof(T) == 4 ? HPG_SPMV_MINB : 2) * 256 / (MODE == 0 && !SPLIT ? HPG_SPMV_BLOCK : 256)) k_spmv(const int32_t* __restrict__ cols, const T* __restrict__ vals,
                                                 int64_t ld, int64_t row0, int64_t nrows,
                                                 const T* __restrict__ x, const T* __restrict__ b,
                                                 T* __restrict__ y, double* __restrict__ partial,
                                                 const uint8_t* __restrict__ skip, const int32_t* __restrict__ list,
                                                 const Stencil st, int ilv) {
  pdl_trigger();
  // ilv > 1: consecutive CTAs take the same chunk position in ilv
  // equal segments of the rows (the 8 color blocks), so the x lines a chunk
  // gathers from every color block are reused in L2 by its co-resident
  // siblings instead of being re-fetched once per color block
  int64_t blk = blockIdx.x;
  if (ilv > 1) blk = (int64_t)(blockIdx.x % ilv) * (gridDim.x / ilv) + blockIdx.x / ilv;
  const int64_t t = blk * blockDim.x + threadIdx.x;
  double sq = 0.0;
  int64_t i = row0 + t;
  bool active = t < nrows;
  if (SPLIT && active) {
    if (list) i = list[t];
    if (skip && skip[i]) active = false;
  }
  if (active) {
    T dd;
    const T acc = row_accumulate<T, false, false, MODE == 0>(cols, vals, ld, i, x, &dd, -1, st);
    if (MODE == 0) {
      y[i] = acc;
    } else {
      const T r = sub_rn(b[i], acc);
      y[i] = r;
      sq = (double)r * (double)r;
    }
  }
  if (MODE == 1) {
    // deterministic block reduction of the squared residual
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
      // indexed by the row chunk, so the fold order is independent of ilv
      if (blk * blockDim.x < nrows) partial[blk] = a;
    }
  }
}

// One color pass of forward Gauss-Seidel over rows [row0, row0+nrows):
//   z_i = (r_i - sum_{s != diag} A[i,s] z[col]) / a_ii
template <typename T, bool COHERENT = false, bool PDL = false>
__device__ __forceinline__ void gs_row(const int32_t* __restrict__ cols, const T* __restrict__ vals, int64_t ld,
                                       int64_t i, const T* __restrict__ r, T* z, int64_t known0 = -1,
                                       const Stencil st = Stencil{}) {
  T d = T(0);
  const T acc = row_accumulate<T, true, COHERENT, PDL>(cols, vals, ld, i, z, &d, known0, st);
  z[i] = div_rn(sub_rn(ldv<COHERENT>(r + i), acc), d);
}

// SPLIT: rows may be skipped (skip[i] != 0) or taken from a list (interior /
// boundary halves of color 0 around an overlapped exchange); the plain
// instantiation is the hot path and carries neither.
#ifndef HPG_GS_BLOCK
#define HPG_GS_BLOCK 64  // measured per level-0 fp32 sweep: 64 583 us, 128 591, 256 625, 512 800
#endif
template <typename T, int MINB = 2, bool SPLIT = false>
__global__ void __launch_bounds__(SPLIT ? 256 : HPG_GS_BLOCK, SPLIT ? MINB : MINB * 256 / HPG_GS_BLOCK) k_gs_pass(const int32_t* __restrict__ cols, const T* __restrict__ vals,
                                                    int64_t ld, int64_t row0, int64_t nrows,
                                                    const T* __restrict__ r, T* z,
                                                    const uint8_t* __restrict__ skip,
                                                    const int32_t* __restrict__ list, int64_t known0, int rev,
                                                    const Stencil st) {
  pdl_trigger();
  // rev: blocks walk the color block from its end, so a pass starts on the
  // planes the previous pass finished last (their z lines are still in L2)
  const int64_t blk = rev ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t t = blk * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  int64_t i = row0 + t;
  if (SPLIT) {
    if (list) i = list[t];
    if (skip && skip[i]) return;
  }
  gs_row<T, false, true>(cols, vals, ld, i, r, z, known0, st);
}

// Fused residual + injection: for fine color-0 row j < nc,
//   rc[dst[j]] = r[j] - (A z)[j]     (ref: multigrid.py:107-128)
template <typename T, bool COHERENT = false, bool PDL = false>
__device__ __forceinline__ void restrict_row(const int32_t* __restrict__ cols, const T* __restrict__ vals,
                                             int64_t ld, int64_t j, const int32_t* __restrict__ dst,
                                             const T* __restrict__ r, const T* z, T* __restrict__ rc,
                                             const Stencil st = Stencil{}) {
  T dd;
  const T acc = row_accumulate<T, false, COHERENT, PDL>(cols, vals, ld, j, z, &dd, -1, st);
  rc[dst[j]] = sub_rn(ldv<COHERENT>(r + j), acc);
}

template <typename T>
__global__ void __launch_bounds__(256, 2) k_restrict(const int32_t* __restrict__ cols, const T* __restrict__ vals,
                                                     int64_t ld, int64_t nc, const int32_t* __restrict__ dst,
                                                     const T* __restrict__ r, const T* __restrict__ z,
                                                     T* __restrict__ rc, const Stencil st) {
  pdl_trigger();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  restrict_row<T, false, true>(cols, vals, ld, j, dst, r, z, rc, st);
}

// Injection transpose: z[j] += zc[dst[j]]  (ref: multigrid.py:131-137)
template <typename T>
__global__ void k_prolong(int64_t nc, const int32_t* __restrict__ dst, T* __restrict__ z,
                          const T* __restrict__ zc) {
  pdl_trigger();
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  z[j] = add_rn(z[j], zc[dst[j]]);
}

// z[0, n) = 0 (the smoother's zero initial guess, ref: smoother.py:95-96)
template <typename T>
__global__ void k_zero(T* __restrict__ z, int64_t n) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 4 <= n && ((uintptr_t)(z + i) & 15) == 0) {
    if (sizeof(T) == 4) *(float4*)(z + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    else { *(double2*)(z + i) = make_double2(0., 0.); *(double2*)(z + i + 2) = make_double2(0., 0.); }
  } else {
    for (int64_t k = i; k < i + 4 && k < n; ++k) z[k] = T(0);
  }
}

// ---------------------------------------------------------- halo pack

template <typename T>
__global__ void k_pack(const T* __restrict__ v, const int32_t* __restrict__ idx, int64_t cnt,
                       T* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < cnt) out[e] = v[idx[e]];
}

// --------------------------------------------------------- Krylov vectors
// Deterministic two-stage reductions: every kernel writes one partial per
// block (fixed grid), a single-block fold sums them in a fixed tree order.

// Partials are stored j-major: partial[j * nb + block], so the fold reads
// them coalesced.  Each block owns one contiguous chunk of rows (good DRAM
// page locality for the kb concurrent Q streams).
template <int KB, typename T>
__device__ __forceinline__ void block_reduce_store(T (&acc)[KB], int kb, T* out, int nb) {
  __shared__ T red[8][KB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    T a = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp][j] = a;
  }
  __syncthreads();
  if (threadIdx.x < kb) {
    T a = red[0][threadIdx.x];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a += red[w][threadIdx.x];
    out[(int64_t)threadIdx.x * nb + blockIdx.x] = a;
  }
}

// rows of block b: [lo, hi)
__device__ __forceinline__ void block_chunk(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 31) & ~(int64_t)31;
  lo = (int64_t)blockIdx.x * chunk;
  hi = lo + chunk < n ? lo + chunk : n;
}

// partial[j][b] = sum_{i in chunk b} Q[j][i] * w[i],  j < kb
// (dot products accumulate in fp64 for every T; see hpg_cgs.cuh:round_dot)
template <typename T, int KB>
__global__ void __launch_bounds__(256) k_dots(const T* __restrict__ Q, int64_t ldq, int kb,
                                              const T* __restrict__ w, int64_t n, double* __restrict__ partial) {
  double acc[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) acc[j] = 0.0;
  int64_t lo, hi;
  block_chunk(n, lo, hi);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const T wi = w[i];
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < kb) acc[j] = fma((double)Q[j * ldq + i], (double)wi, acc[j]);
  }
  block_reduce_store<KB>(acc, kb, partial, gridDim.x);
}

// CGS pass-1 correction fused with the pass-2 projection:
//   w_i -= sum_j Q[j][i] h[j];  partial[j][b] = sum Q[j][i] w_i(new)
template <typename T, int KB>
__global__ void __launch_bounds__(256) k_cgs_sub_dots(const T* __restrict__ Q, int64_t ldq, int kb,
                                                      T* __restrict__ w, int64_t n, const double* __restrict__ h,
                                                      double* __restrict__ partial) {
  double acc[KB];
  T hr[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    acc[j] = 0.0;
    hr[j] = j < kb ? (T)h[j] : T(0);
  }
  int64_t lo, hi;
  block_chunk(n, lo, hi);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    T q[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) q[j] = j < kb ? Q[j * ldq + i] : T(0);
    T tsum = T(0);
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < kb) tsum = fma(q[j], hr[j], tsum);
    const T wi = w[i] - tsum;
    w[i] = wi;
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < kb) acc[j] = fma((double)q[j], (double)wi, acc[j]);
  }
  block_reduce_store<KB>(acc, kb, partial, gridDim.x);
}

// CGS pass-2 correction fused with the norm: w_i -= sum_j Q[j][i] h[j]; partial[b] = sum w_i^2
template <typename T, int KB>
__global__ void __launch_bounds__(256) k_cgs_sub_norm(const T* __restrict__ Q, int64_t ldq, int kb,
                                                      T* __restrict__ w, int64_t n, const double* __restrict__ h,
                                                      double* __restrict__ partial) {
  T hr[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) hr[j] = j < kb ? (T)h[j] : T(0);
  double acc[1] = {0.0};
  int64_t lo, hi;
  block_chunk(n, lo, hi);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    T tsum = T(0);
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < kb) tsum = fma(Q[j * ldq + i], hr[j], tsum);
    const T wi = w[i] - tsum;
    w[i] = wi;
    acc[0] = fma((double)wi, (double)wi, acc[0]);
  }
  block_reduce_store<1>(acc, 1, partial, gridDim.x);
}

// Single-block fold of j-major partials [kb][nb] into out[j], fixed order.
// kb == 1: all threads stride over the blocks, then a shared-memory tree;
// kb > 1: one warp per output, lanes stride, shuffle tree.
template <typename T>
__global__ void k_fold(const T* __restrict__ partial, int nb, int kb, T* __restrict__ out, int do_sqrt) {
  if (kb == 1) {
    __shared__ T red[1024];
    T a = T(0);  // per-thread order b = tid, tid + blockDim, ...; four loads in flight
    for (int b0 = threadIdx.x; b0 < nb; b0 += 4 * blockDim.x) {
      T v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = b0 + u * (int)blockDim.x < nb ? partial[b0 + u * blockDim.x] : T(0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (b0 + u * (int)blockDim.x < nb) a += v[u];
    }
    red[threadIdx.x] = a;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = do_sqrt ? sqrt(red[0]) : red[0];
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < kb; j += nw) {
    T a = T(0);  // per-lane order b = lane, lane + 32, ...; eight loads in flight
    const T* row = partial + (int64_t)j * nb;
    for (int b0 = lane; b0 < nb; b0 += 32 * 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = b0 + 32 * u < nb ? row[b0 + 32 * u] : T(0);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b0 + 32 * u < nb) a += v[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) out[j] = a;
  }
}

// fold over ranks in ascending rank order (ref: comm.py:97-108): out[j] = sum_r g[r*cnt+j]
template <typename T>
__global__ void k_fold_ranks(const T* __restrict__ g, int nranks, int cnt, T* __restrict__ out, int sqrt_first) {
  const int j = threadIdx.x;
  if (j >= cnt) return;
  T a = g[j];
  for (int r = 1; r < nranks; ++r) a = a + g[(int64_t)r * cnt + j];
  out[j] = (sqrt_first && j == 0) ? sqrt(a) : a;
}

template <typename T>
__global__ void k_sqrt_inplace(T* v) {
  v[0] = sqrt(v[0]);
}

// fp64-accumulated dots -> rounded to T (beta: square root in T of the rounded
// w.w), held as double (ref: krylov.py:123, 268; hpg_cgs.cuh:round_dot)
template <typename T>
__global__ void k_round_dots(double* v, int cnt, int do_sqrt) {
  const int j = threadIdx.x;
  if (j >= cnt) return;
  const T a = (T)v[j];
  v[j] = (double)(do_sqrt ? sqrt(a) : a);
}

// Q[k+1] = w / beta  (0 when beta == 0)  (ref: krylov.py:267-273)
template <typename T>
__global__ void k_scale(const T* __restrict__ w, const double* __restrict__ beta, T* __restrict__ q, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T bt = (T)*beta;
  q[i] = bt != T(0) ? div_rn(w[i], bt) : T(0);
}

// Q0 = (T)(r / rho) computed in fp64 then narrowed (ref: krylov.py:250-252)
template <typename T>
__global__ void k_scale_cast(const double* __restrict__ r, double rho, T* __restrict__ q, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) q[i] = (T)__ddiv_rn(r[i], rho);
}

// x += z (fp64 += promoted z)   (ref: krylov.py:292-293)
template <typename T>
__global__ void k_axpy_mixed(double* __restrict__ x, const T* __restrict__ z, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = __dadd_rn(x[i], (double)z[i]);
}

// partial sum of x^2 (norms of b and of arbitrary vectors)
template <typename T>
__global__ void __launch_bounds__(256) k_sumsq(const T* __restrict__ x, int64_t n, T* __restrict__ partial) {
  T acc[1] = {T(0)};
  int64_t lo, hi;
  block_chunk(n, lo, hi);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc[0] = fma(x[i], x[i], acc[0]);
  block_reduce_store<1>(acc, 1, partial, gridDim.x);
}

// -------------------------------------------------------------- setup

__global__ void k_build_level(Geom g, int64_t ld, int32_t* __restrict__ cols, double* __restrict__ v64,
                              float* __restrict__ v32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  int32_t c[27];
  double v[27];
  int diag = 0;
  const int nnz = build_row(g, i, c, v, &diag);
  for (int s = 0; s < 27; ++s) {
    int32_t cc = 0;
    double vv = 0.0;
    if (s < nnz) {
      cc = s == diag ? ~c[s] : c[s];
      vv = v[s];
    }
    cols[s * ld + i] = cc;
    v64[s * ld + i] = vv;
    v32[s * ld + i] = (float)vv;
  }
}

// General injection (any coloring): f2c[i] = fine row of coarse row i's point
// (2x, 2y, 2z) (ref: multigrid.py:87-99)
__global__ void k_build_f2c(Geom gc, Geom gf, int32_t* __restrict__ f2c) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= gc.n) return;
  int x, y, z;
  decode(gc, i, x, y, z);
  f2c[i] = (int32_t)iperm(gf, 2 * x, 2 * y, 2 * z);
}

// rc[i] = r[f2c[i]] - (A z)[f2c[i]] for any coloring (rows gathered; ref: multigrid.py:107-128)
template <typename T>
__global__ void __launch_bounds__(256, 2) k_restrict_gen(const int32_t* __restrict__ cols, const T* __restrict__ vals,
                                                         int64_t ld, int64_t nc, const int32_t* __restrict__ f2c,
                                                         const T* __restrict__ r, const T* __restrict__ z,
                                                         T* __restrict__ rc) {
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int64_t f = f2c[i];
  T dd;
  const T acc = row_accumulate<T, false, false, true>(cols, vals, ld, f, z, &dd);
  rc[i] = sub_rn(r[f], acc);
}

// z[f2c[i]] += zc[i] for any coloring (ref: multigrid.py:131-137)
template <typename T>
__global__ void k_prolong_gen(int64_t nc, const int32_t* __restrict__ f2c, T* __restrict__ z, const T* __restrict__ zc) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nc) return;
  const int64_t f = f2c[i];
  z[f] = add_rn(z[f], zc[i]);
}

// dst[j] = coarse iperm of coarse natural index j   (f2c inverse on color-0 rows)
__global__ void k_build_inject(Geom gc, int32_t* __restrict__ dst) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= gc.n) return;
  const int x = (int)(j % gc.lx);
  const int y = (int)((j / gc.lx) % gc.ly);
  const int z = (int)(j / ((int64_t)gc.lx * gc.ly));
  dst[j] = (int32_t)iperm(gc, x, y, z);
}

// bad |= 1 when an implicit-index row's closed-form columns differ from its
// stored ELL columns (the level then keeps streaming indices)
__global__ void k_check_stencil(const int32_t* __restrict__ cols, int64_t ld, int64_t n, Stencil st,
                                unsigned int* __restrict__ bad, unsigned long long* __restrict__ rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t c[27];
  if (!stencil_cols(st, (uint32_t)i, c)) return;
  atomicAdd(rows, 1ull);
  for (int s = 0; s < 27; ++s)
    if (c[s] != cols[s * ld + i]) atomicOr(bad, 1u);
}

// flag[i] = 1 when row i reads a halo slot (ref: problem.py:78-85 halo_row_split)
__global__ void k_build_halo_flags(Geom g, uint8_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < g.n) flag[i] = row_has_halo(g, i) ? 1 : 0;
}

__global__ void k_build_send(Geom g, int sx, int sy, int sz, int64_t cnt, int32_t* __restrict__ idx) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < cnt) idx[p] = (int32_t)send_row(g, sx, sy, sz, p);
}

}  // namespace hpg
