// CGS2 + norm + normalise in ONE persistent cooperative kernel.
//
// One Arnoldi step needs, for kb = k+1 basis rows Q[0..kb) of length n
// (ref: krylov.py:110-129, 266-273):
//   pass A  h1 = Q w                  (kb dots)
//   pass B  w -= Q^T h1 ; h2 = Q w    (correction fused with the 2nd projection)
//   pass C  w -= Q^T h2 ; beta^2 = w.w
//   pass D  Q[k+1] = w / beta
// i.e. three streams of the kb rows instead of the four of the textbook
// order, and one launch instead of ~8.
//
// Data movement: the CTA's 8 warps are WR row groups x WE element groups.
// Row group rg streams rows rg, rg+WR, ...; element group eg takes its own
// tiles; every lane moves 16-byte vectors, U tiles at a time, so a lane has
// U*(rows/WR + 1) independent 16 B loads in flight and a warp reads 512
// contiguous bytes of a row per load.  Small bases (kb < 8) use fewer row
// groups so every warp still streams.  (A first version staged
// the rows through shared memory with cp.async.bulk / 2-D TMA copies; its
// per-tile mbarrier round trip capped it near 3.6 TB/s.)  The correction
// sum_j Q[j][i] h[j] of passes B/C crosses the row group: each warp writes
// its partial for the tile to shared memory and every warp of the group adds
// the WR partials in warp order, so w_i is identical (and deterministic).
// Between passes: grid barrier, fixed-order fold of the per-CTA partials by
// CTA 0, grid barrier.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hpg_p2p.cuh"

namespace hpg {

template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using V = float4;
  static constexpr int N = 4;
};
template <>
struct Vec16<double> {
  using V = double2;
  static constexpr int N = 2;
};

template <typename T>
__device__ __forceinline__ T vget(const typename Vec16<T>::V& v, int c);
template <>
__device__ __forceinline__ float vget<float>(const float4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}
template <>
__device__ __forceinline__ double vget<double>(const double2& v, int c) {
  return c == 0 ? v.x : v.y;
}
template <typename T>
__device__ __forceinline__ void vset(typename Vec16<T>::V& v, int c, T x);
template <>
__device__ __forceinline__ void vset<float>(float4& v, int c, float x) {
  if (c == 0) v.x = x;
  else if (c == 1) v.y = x;
  else if (c == 2) v.z = x;
  else v.w = x;
}
template <>
__device__ __forceinline__ void vset<double>(double2& v, int c, double x) {
  if (c == 0) v.x = x;
  else v.y = x;
}

template <typename T>
struct CgsParams {
  const T* Q;      // basis, row-major, row stride ldq (multiple of 32 elements)
  T* w;            // vector being orthogonalised (length >= round_up(n, 32))
                   // n must be a multiple of the 16-byte vector width (host checks)
  T* qnext;        // Q[k+1] (NULL: skip norm/normalise)
  double* partial;  // [64][gridDim] per-CTA partials (fp64 accumulation)
  double* scal;     // [0,64) h1, [64,128) h2, [128] beta -- values rounded to T
  int64_t ldq, n;
  int kb;
  P2PAr ar;        // multi-rank: NVLink all-reduce between passes (ar.nranks == 1: none)
  uint64_t seq0;   // sequence number of the first of this call's all-reduces
  int zigzag;      // passes B and D walk each CTA's range backwards, so they start on
                   // the tiles passes A and C read last (still in L2)
  int solo_fold;   // single rank: every CTA folds the partials (one grid barrier per fold)
};

#ifndef HPG_CGS_PIPE_MIN
#define HPG_CGS_PIPE_MIN 4  // software-pipeline the passes when RPW >= this
#endif
constexpr int kCgsThreads = 256;
constexpr int kCgsWarps = kCgsThreads / 32;

// Dot products accumulate in fp64 whatever T is: an fp32 x fp32 product is
// exact in fp64, so every h / beta^2 is the exact dot up to fp64 rounding of the
// sum, and is rounded to T once, after the cross-CTA and cross-rank folds.  The
// result is (to within ~1e-16 relative) independent of the grid and of the rank
// decomposition -- the reference's fp32 OpenBLAS dots are one of many fp32
// orders, each landing within rounding noise of this value.
template <typename T>
__device__ __forceinline__ double round_dot(double a, bool do_sqrt) {
  const T v = (T)a;
  return (double)(do_sqrt ? sqrt(v) : v);  // beta = sqrt in T of the T-rounded w.w (ref: krylov.py:268)
}

// CTA 0 folds the per-CTA partials of cnt outputs into dst (fixed order); with
// several ranks it then all-reduces dst over NVLink in ascending rank order,
// then rounds to T (and takes the square root) (ref: krylov.py:123, 268;
// comm.py:97-108).
template <typename T>
__device__ __forceinline__ void cgs_fold(const double* partial, int cnt, double* dst, bool do_sqrt,
                                         const P2PAr& ar, uint64_t seq) {
  if (blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool multi = ar.nranks > 1;
  // the same per-lane order as a plain strided loop (b = lane, lane + 32, ...); two rows
  // per warp and ten partials per lane in flight at once (one L2 round trip per 320)
  constexpr int RW = 2, UL = 10;
  const int G = (int)gridDim.x;
  for (int j0 = warp; j0 < cnt; j0 += kCgsWarps * RW) {
    double a[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) a[r] = 0.0;
    for (int b0 = lane; b0 < G; b0 += 32 * UL) {
      double v[RW][UL];
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const int j = j0 + r * kCgsWarps;
        const double* row = partial + (int64_t)j * G;
#pragma unroll
        for (int u = 0; u < UL; ++u) v[r][u] = (j < cnt && b0 + 32 * u < G) ? __ldcg(row + b0 + 32 * u) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int u = 0; u < UL; ++u)
          if (b0 + 32 * u < G) a[r] += v[r][u];
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      double x = a[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      const int j = j0 + r * kCgsWarps;
      if (lane == 0 && j < cnt) dst[j] = multi ? x : round_dot<T>(x, do_sqrt);
    }
  }
  if (multi) {
    __syncthreads();
    p2p_allreduce_block<double>(dst, cnt, ar, seq);
    if (threadIdx.x < cnt) dst[threadIdx.x] = round_dot<T>(dst[threadIdx.x], do_sqrt);
  }
}

// Single rank: EVERY CTA folds the partials itself, in cgs_fold's order (so the
// values are bitwise the same), into shared memory -- one grid barrier per
// fold instead of two; CTA 0 also stores them to gdst for the host.
// Each warp takes up to 2 rows at once and issues all their loads before adding
// (one L2 round trip per 320 partials instead of one per 256 per row); the
// additions per row are in the same order as cgs_fold's.
template <typename T>
__device__ __forceinline__ void cta_fold(const double* partial, int cnt, double* sh, bool do_sqrt, double* gdst) {
  constexpr int RW = 2, UL = 10;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = (int)gridDim.x;
  for (int j0 = warp; j0 < cnt; j0 += kCgsWarps * RW) {
    double a[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) a[r] = 0.0;
    for (int b0 = lane; b0 < G; b0 += 32 * UL) {
      double v[RW][UL];
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const int j = j0 + r * kCgsWarps;
        const double* row = partial + (int64_t)j * G;
#pragma unroll
        for (int u = 0; u < UL; ++u) v[r][u] = (j < cnt && b0 + 32 * u < G) ? __ldcg(row + b0 + 32 * u) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int u = 0; u < UL; ++u)
          if (b0 + 32 * u < G) a[r] += v[r][u];
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      double x = a[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      const int j = j0 + r * kCgsWarps;
      if (lane == 0 && j < cnt) {
        const double v = round_dot<T>(x, do_sqrt);
        sh[j] = v;
        if (gdst) gdst[j] = v;
      }
    }
  }
  __syncthreads();
}
__device__ __forceinline__ double ld_h(const double* a) { return __isShared(a) ? *a : __ldcg(a); }

// Warp roles: WR warps split the rows (row group rg = warp % WR streams rows
// rg, rg+WR, ...), WE = W/WR element groups split the tiles, so small bases
// still keep every warp streaming.
// MODE 0: acc[r] += q_{j(r)} . w                       (pass A)
// MODE 1: w -= sum_j q_j h_j ; acc[r] += q_{j(r)} . w   (pass B)
// MODE 2: w -= sum_j q_j h_j ; acc[0] += w . w (rg 0)   (pass C)
// MODE 3: w  = sum_j q_j h_j                           (end-of-cycle basis combination)
template <typename T, int WR, int RPW, int U, int MODE>
struct CgsStream {
  using V = typename Vec16<T>::V;
  static constexpr int VN = Vec16<T>::N;
  static constexpr int TILE = 32 * VN;  // elements per warp-wide 512 B load
  static constexpr int WE = kCgsWarps / WR;
  static constexpr int STEP = WE * U;   // tiles per CTA iteration

  const CgsParams<T>& p;
  int lane, warp, rg, eg, kb;
  int64_t t1;
  T hr[RPW];

  __device__ __forceinline__ CgsStream(const CgsParams<T>& p_, const double* h, int64_t t1_) : p(p_), t1(t1_) {
    lane = threadIdx.x & 31;
    warp = threadIdx.x >> 5;
    rg = warp % WR;
    eg = warp / WR;
    kb = p.kb;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int j = rg + r * WR;
      hr[r] = (MODE > 0 && j < kb) ? (T)ld_h(h + j) : T(0);
    }
  }

  // issue every load of the iteration starting at tile tb (nothing is used yet)
  __device__ __forceinline__ void load(int64_t tb, V (&q)[U][RPW], V (&wv)[U]) const {
    if (tb + STEP <= t1 && (tb + STEP) * TILE <= p.n) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = (tb + eg * U + u) * TILE + lane * VN;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          // rows past kb are not loaded (warp-uniform predicate; the register is
          // pre-zeroed, so no select waits on loaded data)
          const int j = rg + r * WR;
          q[u][r] = V{};
          if (j < kb) q[u][r] = __ldcs((const V*)(p.Q + j * p.ldq + i));
        }
        if (MODE != 3) wv[u] = __ldcg((const V*)(p.w + i));
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t tile = tb + eg * U + u;
        const int64_t i = tile * TILE + lane * VN;
        const bool in = tile < t1 && i < p.n;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          const int j = rg + r * WR;
          q[u][r] = (in && j < kb) ? __ldcs((const V*)(p.Q + j * p.ldq + i)) : V{};
        }
        wv[u] = (in && MODE != 3) ? __ldcg((const V*)(p.w + i)) : V{};
      }
    }
  }

  // consume one iteration (block-uniform: contains barriers when WR > 1)
  __device__ __forceinline__ void process(int64_t tb, V (&q)[U][RPW], V (&wv)[U], double (&acc)[RPW],
                                          V* red) const {
    if (MODE > 0) {
      if (WR > 1) {
        // this warp's share of the correction, then the sum over the row group (fixed order)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          V t{};
#pragma unroll
          for (int c = 0; c < VN; ++c) {
            T s = T(0);
#pragma unroll
            for (int r = 0; r < RPW; ++r) s = fma(vget<T>(q[u][r], c), hr[r], s);
            vset<T>(t, c, s);
          }
          red[(u * kCgsWarps + warp) * 32 + lane] = t;
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        V tot;
        if (WR > 1) {
          tot = red[(u * kCgsWarps + eg * WR) * 32 + lane];
          for (int v = 1; v < WR; ++v) {
            const V x = red[(u * kCgsWarps + eg * WR + v) * 32 + lane];
#pragma unroll
            for (int c = 0; c < VN; ++c) vset<T>(tot, c, vget<T>(tot, c) + vget<T>(x, c));
          }
        } else {
#pragma unroll
          for (int c = 0; c < VN; ++c) {
            T s = T(0);
#pragma unroll
            for (int r = 0; r < RPW; ++r) s = fma(vget<T>(q[u][r], c), hr[r], s);
            vset<T>(tot, c, s);
          }
        }
        V nw;
        if (MODE == 3) {
          nw = tot;
        } else {
#pragma unroll
          for (int c = 0; c < VN; ++c) vset<T>(nw, c, vget<T>(wv[u], c) - vget<T>(tot, c));
        }
        wv[u] = nw;
        const int64_t tile = tb + eg * U + u;
        const int64_t i = tile * TILE + lane * VN;
        if (rg == 0 && tile < t1 && i < p.n) *(V*)(p.w + i) = nw;
      }
      if (WR > 1) __syncthreads();  // partials consumed before the next iteration overwrites them
    }
    if (MODE < 2) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RPW; ++r)
#pragma unroll
          for (int c = 0; c < VN; ++c)
            acc[r] = fma((double)vget<T>(q[u][r], c), (double)vget<T>(wv[u], c), acc[r]);
    } else if (MODE == 2 && rg == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < VN; ++c) acc[0] = fma((double)vget<T>(wv[u], c), (double)vget<T>(wv[u], c), acc[0]);
    }
  }
};

// One streaming pass over this CTA's contiguous range of tiles.  PIPE (wide
// bases): software pipelined, the loads of iteration i+1 are in flight while
// iteration i is consumed (two register sets, alternating); narrow bases use
// one larger register set (U tiles) instead -- measured faster for kb <= 16.
template <typename T, int WR, int RPW, int U, int MODE, bool PIPE, bool REV = false>
__device__ __forceinline__ void cgs_pass(const CgsParams<T>& p, const double* h, double (&acc)[RPW],
                                         typename Vec16<T>::V* red) {
  using S = CgsStream<T, WR, RPW, U, MODE>;
  using V = typename S::V;
  const int64_t ntiles = (p.n + S::TILE - 1) / S::TILE;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per;
  const int64_t t1 = t0 + per < ntiles ? t0 + per : ntiles;
  const S st(p, h, t1);
  // iteration b covers tiles [at(b), at(b) + STEP); rev walks the range backwards
  const int64_t nb = t1 > t0 ? (t1 - t0 + S::STEP - 1) / S::STEP : 0;
  auto at = [&](int64_t b) { return t0 + (REV ? nb - 1 - b : b) * S::STEP; };
  if (!PIPE) {  // one register set: load, then consume
    for (int64_t b = 0; b < nb; ++b) {
      V q[U][RPW], wv[U];
      st.load(at(b), q, wv);
      st.process(at(b), q, wv, acc, red);
    }
    return;
  }
  V qa[U][RPW], wa[U], qb[U][RPW], wb[U];
  if (nb > 0) st.load(at(0), qa, wa);
  for (int64_t b = 0; b < nb; b += 2) {
    if (b + 1 < nb) st.load(at(b + 1), qb, wb);
    st.process(at(b), qa, wa, acc, red);
    if (b + 1 >= nb) break;
    if (b + 2 < nb) st.load(at(b + 2), qa, wa);
    st.process(at(b + 1), qb, wb, acc, red);
  }
}

// rows -> partial[j][block]: lane reduce per warp, then element groups added in order
template <int WR, int RPW>
__device__ __forceinline__ void cgs_store_rows(const double (&acc)[RPW], int kb, double* partial, double* sacc) {
  constexpr int WE = kCgsWarps / WR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    double a = acc[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sacc[warp * RPW + r] = a;
  }
  __syncthreads();
  if (threadIdx.x < kb) {
    const int j = threadIdx.x, rg = j % WR, r = j / WR;
    double a = sacc[rg * RPW + r];
    for (int e = 1; e < WE; ++e) a += sacc[(e * WR + rg) * RPW + r];
    partial[(int64_t)j * gridDim.x + blockIdx.x] = a;
  }
  __syncthreads();
}

template <typename T, int WR, int RPW, int U, int MINB = 2>
__global__ void __launch_bounds__(kCgsThreads, MINB) k_cgs2_fused(const __grid_constant__ CgsParams<T> p) {
  namespace cg = cooperative_groups;
  using V = typename Vec16<T>::V;
  cg::grid_group grid = cg::this_grid();
  __shared__ V red[WR > 1 ? U * kCgsWarps * 32 : 1];
  __shared__ double sacc[kCgsWarps * RPW];
  // single rank: redundant per-CTA folds (cta_fold); pass B's partials go to a second
  // buffer so no CTA overwrites partials another CTA may still be folding
  __shared__ double hsh[64];
  const bool solo = p.ar.nranks <= 1 && p.solo_fold;
  double* part_b = solo ? p.partial + (int64_t)64 * gridDim.x : p.partial;
  auto fold = [&](const double* part, int cnt, int slot, bool sq, uint64_t seq) -> const double* {
    grid.sync();
    if (solo) {
      cta_fold<T>(part, cnt, hsh, sq, blockIdx.x == 0 ? p.scal + slot : nullptr);
      return hsh;
    }
    cgs_fold<T>(part, cnt, p.scal + slot, sq, p.ar, seq);
    grid.sync();
    return p.scal + slot;
  };
  {  // pass A: h1
    double acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) acc[r] = 0.0;
    cgs_pass<T, WR, RPW, U, 0, (RPW >= HPG_CGS_PIPE_MIN)>(p, nullptr, acc, red);
    cgs_store_rows<WR, RPW>(acc, p.kb, p.partial, sacc);
  }
  const double* h1 = fold(p.partial, p.kb, 0, false, p.seq0);
  {  // pass B: w -= Q^T h1 ; h2
    double acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) acc[r] = 0.0;
    if (p.zigzag) cgs_pass<T, WR, RPW, U, 1, (RPW >= HPG_CGS_PIPE_MIN), true>(p, h1, acc, red);
    else cgs_pass<T, WR, RPW, U, 1, (RPW >= HPG_CGS_PIPE_MIN)>(p, h1, acc, red);
    cgs_store_rows<WR, RPW>(acc, p.kb, part_b, sacc);
  }
  const double* h2 = fold(part_b, p.kb, 64, false, p.seq0 + 1);
  {  // pass C: w -= Q^T h2 ; beta^2 (row-group-0 warps hold the block's share)
    double acc[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) acc[r] = 0.0;
    cgs_pass<T, WR, RPW, U, 2, (RPW >= HPG_CGS_PIPE_MIN)>(p, h2, acc, red);
    cgs_store_rows<WR, RPW>(acc, 1, p.partial, sacc);
  }
  if (p.qnext == nullptr) return;
  const double* bsq = fold(p.partial, 1, 128, true, p.seq0 + 2);
  // pass D: Q[k+1] = w / beta  (ref: krylov.py:269-273), 16-byte vectors
  using VV = typename Vec16<T>::V;
  constexpr int VN = Vec16<T>::N;
  const T bt = (T)ld_h(bsq);
  const int64_t nv = p.n / VN;
  if (p.zigzag) {
    // this CTA's pass-C range, backwards (its last tiles are still in L2)
    constexpr int TILE = 32 * VN;
    const int64_t ntiles = (p.n + TILE - 1) / TILE, per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t v0 = (int64_t)blockIdx.x * per * 32, v1e = v0 + per * 32 < nv ? v0 + per * 32 : nv;
    for (int64_t v = v1e - 1 - threadIdx.x; v >= v0; v -= blockDim.x) {
      const VV x = __ldcg((const VV*)p.w + v);
      VV y;
#pragma unroll
      for (int c = 0; c < VN; ++c) vset<T>(y, c, bt != T(0) ? div_rn(vget<T>(x, c), bt) : T(0));
      ((VV*)p.qnext)[v] = y;
    }
    return;
  }
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const VV x = __ldcg((const VV*)p.w + v);
    VV y;
#pragma unroll
    for (int c = 0; c < VN; ++c) vset<T>(y, c, bt != T(0) ? div_rn(vget<T>(x, c), bt) : T(0));
    ((VV*)p.qnext)[v] = y;
  }
}

// One CGS2 pass per launch (multi-rank path: the cross-rank reduction of the
// per-CTA partials -- NCCL all-gather + rank-ordered fold -- runs between the
// passes).  MODE 0/1 write per-CTA row partials, MODE 2 the per-CTA norm share.
template <typename T, int WR, int RPW, int U, int MODE>
__global__ void __launch_bounds__(kCgsThreads, 2) k_cgs_onepass(const __grid_constant__ CgsParams<T> p,
                                                               const double* __restrict__ h) {
  using V = typename Vec16<T>::V;
  __shared__ V red[WR > 1 ? U * kCgsWarps * 32 : 1];
  __shared__ double sacc[kCgsWarps * RPW];
  double acc[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) acc[r] = 0.0;
  cgs_pass<T, WR, RPW, U, MODE, (RPW >= HPG_CGS_PIPE_MIN)>(p, h, acc, red);
  cgs_store_rows<WR, RPW>(acc, MODE == 2 ? 1 : p.kb, p.partial, sacc);
}

// out = Q[0:k]^T y (ref: krylov.py:288-289): one streaming pass over k rows,
// same warp roles as CGS2; y (narrowed to T, held as double) sits in p.scal[0..k).
template <typename T, int WR, int RPW, int U>
__global__ void __launch_bounds__(kCgsThreads, 2) k_gemv_combine(const __grid_constant__ CgsParams<T> p) {
  using V = typename Vec16<T>::V;
  __shared__ V red[WR > 1 ? U * kCgsWarps * 32 : 1];
  double acc[RPW];
  cgs_pass<T, WR, RPW, U, 3, (RPW >= HPG_CGS_PIPE_MIN)>(p, p.scal, acc, red);
}

}  // namespace hpg
