// Colour pass with BOTH operands staged by the tensor engine ("brick" pass).
//
// k_gs_pass_tma (hpg_tma.cuh) stages a tile's 27 value planes but still gathers
// the 26 neighbour z values per row from L1/L2 one load at a time; with 27 of
// them outstanding per thread the register file caps a SM at ~1024 rows in
// flight and the pass is gather-latency bound (profiles/r02_*).  Here a CTA's
// tile is a brick of the colour's sub-lattice -- ROWS = hx * BY rows: BY whole
// x-lines of one z-plane (the colour block's row order is x fastest) -- and
// every neighbour colour's z values that brick touches form one small box of
// that colour's sub-lattice: for the colour c' = c ^ (axis mask am), the box is
// the brick widened by one on each axis whose parity differs, on the side the
// row's parity selects.  Thread 0 issues
//   * one 2-D tensor copy of the 27 value planes {ROWS x 27} -- before the PDL
//     wait (the matrix does not depend on the previous pass), and
//   * after the wait, one 4-D tensor copy per neighbour colour (7 of them; the
//     z vector seen as [colour][z][y][x] sub-lattices) -- in a zero-initial-
//     guess sweep only for colours already updated (c' < c), the others are 0.
// Each thread then forms its row from shared memory alone: 27 value loads and
// 26 z loads at per-colour constant offsets (the table sconst), conflict-free,
// no register array of outstanding gathers.  The sum keeps the reference's slot
// order with separate IEEE multiply / add and the IEEE subtract / divide, so z
// is bitwise the same as every other sweep kernel (ref: smoother.py:62-75).
// Rows on a face of the local box (their neighbours leave the brick or the box)
// take the indexed path: column indices and z from global memory.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hpg_tma.cuh"

namespace hpg {

__device__ __forceinline__ void tma_g2s_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int w,
                                           uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
      : "memory");
}

struct BrickPlan {
  CUtensorMap vmap;     // value planes [27][ld], box {ROWS, 27}
  CUtensorMap zmap[8];  // z as [8 colours][hz][hy][hx], box of axis mask am (1..7)
  const int32_t* cols;  // face rows only
  int64_t ld;
  int64_t row0, nrows;  // this colour block (row0 = c * n8)
  int64_t known0;       // zero sweep: columns >= known0 are 0
  int rev, color;
  int hx, hxy;          // sub-lattice extents
  int box_x[8], box_y[8], box_z[8], box_c[8];  // box start relative to the brick origin; colour
  int box_off[8];       // element offset of each box in shared memory
  uint32_t box_bytes[8];
  uint32_t load_mask;   // boxes to load (bit am)
  int pad;              // X extent of a box whose x parity differs: hx + pad
  uint32_t xsel;        // slot s reads with row term rx + (hx + pad) * ry
  uint32_t kmask;       // slot s is known zero (zero sweep)
  int32_t sconst[27];   // slot s: shared-memory element offset beyond the row term
  Stencil st;
};

template <typename T, int ROWS>
struct BrickSmem {
  static constexpr size_t kValBytes = (size_t)27 * ROWS * sizeof(T);
};

template <typename T, int ROWS, int MINB>
__global__ void __launch_bounds__(ROWS, MINB) k_gs_pass_brick(const __grid_constant__ BrickPlan p,
                                                              const T* __restrict__ r, T* z, size_t zoff_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* sv = (T*)smem;
  T* sz = (T*)(smem + zoff_bytes);
  uint64_t* bars = (uint64_t*)(smem + zoff_bytes + p.box_off[0] * sizeof(T));  // box_off[0]: end of the boxes
  const int64_t blk = p.rev ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t t0 = blk * ROWS;  // first row of the brick within the colour block
  const int Z0 = (int)(t0 / p.hxy);
  const int Y0 = (int)((t0 - (int64_t)Z0 * p.hxy) / p.hx);
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bars, (uint32_t)BrickSmem<T, ROWS>::kValBytes);
    tma_g2s_2d(sv, &p.vmap, (int)(p.row0 + t0), 0, bars, evict_first_policy());
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();  // z and r come from the predecessors
  if (threadIdx.x == 0) {
    uint32_t bytes = 0;
#pragma unroll
    for (int am = 1; am < 8; ++am)
      if ((p.load_mask >> am) & 1u) bytes += p.box_bytes[am];
    mbar_expect_tx(bars + 1, bytes);
#pragma unroll
    for (int am = 1; am < 8; ++am)
      if ((p.load_mask >> am) & 1u)
        tma_g2s_4d(sz + p.box_off[am], &p.zmap[am], p.box_x[am], Y0 + p.box_y[am], Z0 + p.box_z[am], p.box_c[am],
                   bars + 1);
  }
  const int t = threadIdx.x;
  const int64_t i = p.row0 + t0 + t;
  if (t0 + t >= p.nrows) return;
  const T ri = __ldg(r + i);
  const T zi = (p.known0 >= 0) ? T(0) : z[i];  // the row's own (diagonal) z: 0 in a zero sweep
  const int rx = t % p.hx, ry = t / p.hx;
  const int pc = p.color;
  const int x = 2 * rx + ((pc >> p.st.bx) & 1), y = 2 * (Y0 + ry) + ((pc >> p.st.by) & 1),
            zc = 2 * Z0 + ((pc >> p.st.bz) & 1);
  const bool interior = x >= 1 && x <= p.st.lx - 2 && y >= 1 && y <= p.st.ly - 2 && zc >= 1 && zc <= p.st.lz - 2;
  T acc = T(0), d = T(0);
  if (interior) {
    const int ta = t, tb = t + p.pad * ry;  // row terms for box X extents hx and hx + pad
    mbar_wait(bars + 1, 0);
    mbar_wait(bars, 0);
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      T vs = sv[s * ROWS + t];
      T g;
      if (s == 13) {  // the diagonal slot: a_ii aside, the product formed as 0 * z_i
        d = vs;
        vs = T(0);
        g = zi;
      } else {
        g = ((p.kmask >> s) & 1u) ? T(0) : sz[(((p.xsel >> s) & 1u) ? tb : ta) + p.sconst[s]];
      }
      acc = add_rn(acc, mul_rn(vs, g));
    }
  } else {
    int32_t c[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) c[s] = __ldg(p.cols + s * p.ld + i);
    T g[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      const int32_t cc = c[s] < 0 ? ~c[s] : c[s];
      g[s] = (p.known0 >= 0 && cc >= p.known0) ? T(0) : z[cc];
    }
    mbar_wait(bars, 0);
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      T vs = sv[s * ROWS + t];
      if (c[s] < 0) {  // the diagonal slot (stored as ~col)
        d = vs;
        vs = T(0);
      }
      acc = add_rn(acc, mul_rn(vs, g[s]));
    }
  }
  z[i] = div_rn(sub_rn(ri, acc), d);
  // the z boxes land in this CTA's shared memory: it must not retire before they
  // do, even when no row of the brick is interior (thread 0 is always active)
  if (t == 0 && !interior) mbar_wait(bars + 1, 0);
}

// ---------------------------------------------------------------------------
// Pipelined brick pass (the default colour pass where the layout allows).
//
// k_gs_pass_brick exposes one round trip for its z boxes per CTA.  Here each
// CTA is persistent over its share of the pass's bricks (round-robin, so the
// grid works on one narrow window of the colour block at a time) with an
// S-stage shared-memory ring: warp 0 (one lane) issues, per brick, the 2-D
// tensor copy of the 27 value planes and the 4-D copies of the neighbour
// colours' z boxes; the value copies of the first S bricks go out before the
// PDL wait, everything else after it.  The ROWS consumer threads (one row
// each) form their rows from shared memory alone and release the stage.  With
// 3 CTAs x 3 stages per SM, nine bricks' operands are in flight per SM while
// the consumers hold no gathered values in registers.
// Face rows read their slots through the position-class table (kFaceSlots)
// from the same boxes; rows whose missing neighbours are across a rank
// interface (halo columns) take the indexed path with global gathers.
// a row whose missing neighbours lie across a rank interface: indexed columns,
// global gathers (the halo tail); out of line, so its 54 live registers do not
// weigh on the shared-memory path
template <typename T, int ROWS>
__device__ __noinline__ T brick_interface_row(const BrickPlan& p, const T* sv, int t, int64_t i, const T* z, T ri) {
  int32_t c[27];
#pragma unroll
  for (int s = 0; s < 27; ++s) c[s] = __ldg(p.cols + s * p.ld + i);
  T g[27];
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    const int32_t cc = c[s] < 0 ? ~c[s] : c[s];
    g[s] = (p.known0 >= 0 && cc >= p.known0) ? T(0) : z[cc];
  }
  T acc = T(0), d = T(0);
#pragma unroll
  for (int s = 0; s < 27; ++s) {
    T vs = sv[s * ROWS + t];
    if (c[s] < 0) {
      d = vs;
      vs = T(0);
    }
    acc = add_rn(acc, mul_rn(vs, g[s]));
  }
  return div_rn(sub_rn(ri, acc), d);
}

struct BrickPipe {
  uint32_t stage_bytes;  // one ring stage: values, z boxes, r, own z (128-byte aligned parts)
  uint32_t zoff;         // byte offset of the z boxes inside a stage
  uint32_t roff;         // byte offset of the brick's r (ROWS values), then its own z
  uint32_t vbytes;       // value bytes per brick
  int64_t ntiles;        // bricks in this colour block
};

template <typename T, int ROWS, int S>
__global__ void __launch_bounds__(32 + ROWS, 1) k_gs_brick_pp(const __grid_constant__ BrickPlan p,
                                                              const __grid_constant__ BrickPipe q,
                                                              const T* __restrict__ r, T* z) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + (size_t)S * q.stage_bytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int64_t mine = q.ntiles > blockIdx.x ? (q.ntiles - blockIdx.x + G - 1) / G : 0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) {
      mbar_init(full + k, 1);
      mbar_init(empty + k, ROWS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  uint32_t zbytes = (uint32_t)(ROWS * sizeof(T)) * (p.known0 < 0 ? 2u : 1u);  // r (+ own z)
#pragma unroll
  for (int am = 1; am < 8; ++am)
    if ((p.load_mask >> am) & 1u) zbytes += p.box_bytes[am];
  auto tile_of = [&](int64_t m) {
    const int64_t j = (int64_t)blockIdx.x + m * G;
    return p.rev ? q.ntiles - 1 - j : j;
  };
  if (warp == 0) {  // ---- producer
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      auto issue_z = [&](int64_t m) {
        const int64_t t0 = tile_of(m) * ROWS;
        const int Z0 = (int)(t0 / p.hxy), Y0 = (int)((t0 - (int64_t)Z0 * p.hxy) / p.hx);
        unsigned char* st = smem + (size_t)(m % S) * q.stage_bytes;
        T* sz = (T*)(st + q.zoff);
        // the brick's r and own z (contiguous rows) ride in the same stage
        bulk_g2s(st + q.roff, r + p.row0 + t0, ROWS * sizeof(T), full + (m % S), pol);
        if (p.known0 < 0) bulk_g2s(st + q.roff + ROWS * sizeof(T), z + p.row0 + t0, ROWS * sizeof(T), full + (m % S), pol);
#pragma unroll
        for (int am = 1; am < 8; ++am)
          if ((p.load_mask >> am) & 1u)
            tma_g2s_4d(sz + p.box_off[am], &p.zmap[am], p.box_x[am], Y0 + p.box_y[am], Z0 + p.box_z[am],
                       p.box_c[am], full + (m % S));
      };
      const int64_t first = mine < S ? mine : S;
      for (int64_t m = 0; m < first; ++m) {  // matrix planes ahead of the dependency
        mbar_expect_tx(full + m, q.vbytes + zbytes);
        tma_g2s_2d(smem + (size_t)m * q.stage_bytes, &p.vmap, (int)(p.row0 + tile_of(m) * ROWS), 0, full + m, pol);
      }
      pdl_wait();
      for (int64_t m = 0; m < first; ++m) issue_z(m);
      for (int64_t m = first; m < mine; ++m) {
        const int k = (int)(m % S);
        mbar_wait(empty + k, (uint32_t)(((m / S) - 1) & 1));
        mbar_expect_tx(full + k, q.vbytes + zbytes);
        tma_g2s_2d(smem + (size_t)k * q.stage_bytes, &p.vmap, (int)(p.row0 + tile_of(m) * ROWS), 0, full + k, pol);
        issue_z(m);
      }
    }
    return;
  }
  // ---- consumers: one row per thread per brick
  const int t = threadIdx.x - 32;
  pdl_wait();
  const T z0 = (p.known0 >= 0 && p.known0 == 0) ? T(0) : z[0];  // padding slots gather column 0
  const int rx = t % p.hx, ry = t / p.hx;
  const int pc = p.color;
  const int ta = t, tb = t + p.pad * ry;
  for (int64_t m = 0; m < mine; ++m) {
    const int k = (int)(m % S);
    const int64_t t0 = tile_of(m) * ROWS;
    const int64_t i = p.row0 + t0 + t;
    const int Z0 = (int)(t0 / p.hxy), Y0 = (int)((t0 - (int64_t)Z0 * p.hxy) / p.hx);
    const int x = 2 * rx + ((pc >> p.st.bx) & 1), y = 2 * (Y0 + ry) + ((pc >> p.st.by) & 1),
              zc = 2 * Z0 + ((pc >> p.st.bz) & 1);
    const int cx = x == 0 ? 0 : (x == p.st.lx - 1 ? 2 : 1);
    const int cy = y == 0 ? 0 : (y == p.st.ly - 1 ? 2 : 1);
    const int cz = zc == 0 ? 0 : (zc == p.st.lz - 1 ? 2 : 1);
    const int cut = (cx == 0 ? 1 : 0) | (cx == 2 ? 2 : 0) | (cy == 0 ? 4 : 0) | (cy == 2 ? 8 : 0) |
                    (cz == 0 ? 16 : 0) | (cz == 2 ? 32 : 0);
    unsigned char* st = smem + (size_t)k * q.stage_bytes;
    const T* sv = (const T*)st;
    const T* sz = (const T*)(st + q.zoff);
    mbar_wait(full + k, (uint32_t)((m / S) & 1));
    const T ri = ((const T*)(st + q.roff))[t];
    const T zi = p.known0 >= 0 ? T(0) : ((const T*)(st + q.roff))[ROWS + t];
    T out;
    if (cut & p.st.ifc) {
      out = brick_interface_row<T, ROWS>(p, sv, t, i, z, ri);
    } else {
      T acc = T(0), d = T(0);
      if (cut == 0) {  // interior: slot s is offset s
#pragma unroll
        for (int s = 0; s < 27; ++s) {
          T vs = sv[s * ROWS + t];
          T g;
          if (s == 13) {
            d = vs;
            vs = T(0);
            g = zi;
          } else {
            g = ((p.kmask >> s) & 1u) ? T(0) : sz[(((p.xsel >> s) & 1u) ? tb : ta) + p.sconst[s]];
          }
          acc = add_rn(acc, mul_rn(vs, g));
        }
      } else {  // a face row: slot k is the k-th in-box offset of its class
        const unsigned char* tab = kFaceSlots.s[cz * 9 + cy * 3 + cx];
#pragma unroll
        for (int kk = 0; kk < 27; ++kk) {
          const int s = tab[kk];
          T vs = sv[kk * ROWS + t];
          T g;
          if (s == 27) {
            g = z0;  // padding: value 0, column 0 (the reference's spmv_cols)
          } else if (s == 13) {
            d = vs;
            vs = T(0);
            g = zi;
          } else {
            g = ((p.kmask >> s) & 1u) ? T(0) : sz[(((p.xsel >> s) & 1u) ? tb : ta) + p.sconst[s]];
          }
          acc = add_rn(acc, mul_rn(vs, g));
        }
      }
      out = div_rn(sub_rn(ri, acc), d);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + k);
    z[i] = out;
  }
}

}  // namespace hpg
