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

}  // namespace hpg
