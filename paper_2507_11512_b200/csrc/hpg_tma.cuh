// Bulk-copy (TMA engine) pipelined stencil kernels for the big levels.
//
// The row-per-thread kernels of hpg_kernels.cuh keep 27 value loads + 27
// gathers in flight per thread; at the occupancy their 64-80 registers allow,
// the level-0 colour pass sits at ~54% of the HBM copy rate, stalled on
// long-scoreboard (profiles/r01g_full_k_gs_pass.md).  Here the value planes --
// 90% of the bytes -- are decoupled from the arithmetic:
//
//   * warp 0 (one elected lane) is the PRODUCER: for each tile of ROWS rows it
//     issues ONE 2-D tensor copy (cp.async.bulk.tensor, SASS UTMALDG) of the
//     {ROWS x 27 slot planes} box, into a STAGES-deep shared-memory ring guarded by mbarriers
//     (full: transaction bytes; empty: one arrival per consumer warp), with an
//     L2 evict-first policy so the gathered vector stays resident in L2;
//   * warps 1..ROWS/32 are CONSUMERS: one row per thread, the row's 27 values
//     read from shared memory (conflict-free: plane-major tile), the 27 gathers
//     from global memory through L1, the slot-ordered sum with separate IEEE
//     multiply / add, the IEEE subtract / divide -- the reference's arithmetic
//     bit for bit (ref: smoother.py:62-75, krylov.py:76-80).
//
// k_gs_sweep_tma runs ALL colour passes of one forward sweep in one persistent
// launch (2 CTAs per SM).  Colour c+1 may gather what colour c wrote, so the
// consumers of every CTA meet at a grid-wide counter between passes
// (release/acquire at gpu scope, then an L1 invalidation: fence.acq_rel.gpu),
// while the producer runs ahead across the pass boundary -- the value planes do
// not depend on z -- so HBM keeps streaming through the drain that separates
// dependent colour passes.  Tiles of a pass are dealt round-robin over the CTAs,
// so at any moment the grid works on one narrow window of the colour block and
// the other colours' z lines it gathers are shared in L2.  Odd colours walk
// their block backwards (rev), starting where the previous pass ended.
#pragma once
#include <cuda.h>  // CUtensorMap (encoded on the host through the driver entry point)
#include <cuda_runtime.h>
#include <stdint.h>

#include "hpg_kernels.cuh"

namespace hpg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  while (!mbar_try_wait(b, parity)) {
  }
}
// global -> shared bulk copy completing on an mbarrier (bytes: multiple of 16,
// both addresses 16-byte aligned), L2 cache policy attached
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// 2-D tensor copy (SASS UTMALDG): box {ROWS rows, 27 slot planes} at row x
__device__ __forceinline__ void tma_g2s_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                           uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// Spin with relaxed loads (an acquire load per iteration would invalidate the
// SM's L1 every time -- CCTL.IVALL -- under the feet of the co-resident CTA);
// one acquire fence once the count is reached.
__device__ __forceinline__ unsigned ld_relaxed_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void consumers_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// One forward sweep of one level, all colour blocks (ref: smoother.py:78-114).
struct SweepPlan {
  CUtensorMap vmap;     // the value planes [27][ld] of T as a 2-D tensor, box {ROWS, 27}
  const int32_t* cols;  // [27][ld] (face rows: implicit-index rows compute theirs)
  const void* vals;     // [27][ld] of T
  int64_t ld;
  int64_t off[kMaxColors + 1];  // colour block c = rows [off[c], off[c+1])
  int ncolors;
  int zero;             // zero initial guess: columns >= off[c] hold 0 in pass c (loads skipped,
                        // the v * 0 products are still formed -- the reference's arithmetic)
  int rev_odd;          // odd colours walk their (CTA's share of the) block backwards
  int contiguous;       // 1: CTA b owns rows [b cnt / G, (b+1) cnt / G) of every colour block --
                        // the same spatial slab in every pass, so the z lines it gathers stay
                        // in its SM's L1 / its die's L2; 0: tiles dealt round-robin
  unsigned* done;       // [kMaxColors] pass counters; the last CTA resets them
  Stencil st;
  // implicit-index rows of colour c (st.on): slot s gathers column i + doff[c][s]
  // (per-colour constants: the neighbour's colour block and sub-lattice shift),
  // and in a zero sweep skips the load when bit s of kmask[c] is set (the
  // neighbour's colour is >= c: still 0) -- only face rows read the index plane
  int32_t doff[8][27];
  uint32_t kmask[8];
};

template <typename T, int ROWS>
struct TmaTile {
  static constexpr int kBytes = 27 * ROWS * (int)sizeof(T);
};

// The tiles of colour c this CTA processes, in order: tile m starts at row0(m) and
// holds the rows [row0, end) (the producer and the consumers walk the same list).
struct TileSpan {
  int64_t lo, hi, nt, step;
  int ROWS;
  bool rev, contig;
  __device__ __forceinline__ TileSpan(const SweepPlan& p, int c, int rows_per_tile) {
    ROWS = rows_per_tile;
    const int64_t a = p.off[c], cnt = p.off[c + 1] - a;
    const int G = gridDim.x, b = blockIdx.x;
    contig = p.contiguous != 0;
    rev = p.rev_odd && (c & 1);
    if (contig) {  // slab edges on 32-row (128-byte) boundaries: tensor-copy starts stay aligned
      lo = a + ((cnt * b / G) & ~int64_t{31});
      hi = b == G - 1 ? a + cnt : a + ((cnt * (b + 1) / G) & ~int64_t{31});
      nt = (hi - lo + ROWS - 1) / ROWS;
      step = 1;
    } else {
      lo = a;
      hi = a + cnt;
      const int64_t all = (cnt + ROWS - 1) / ROWS;
      nt = all > b ? (all - b + G - 1) / G : 0;  // tiles b, b+G, ...
      step = G;
    }
  }
  __device__ __forceinline__ int64_t row0(int64_t m) const {
    if (contig) return lo + (rev ? nt - 1 - m : m) * ROWS;
    const int64_t all = (hi - lo + ROWS - 1) / ROWS;
    const int64_t j = (int64_t)blockIdx.x + m * step;
    return lo + (rev ? all - 1 - j : j) * ROWS;
  }
};

// Is row i of colour pc (of the Stencil layout) interior -- all 27 neighbours local?
__device__ __forceinline__ bool st_interior(const Stencil& st, int64_t i, int pc) {
  uint32_t pos = (uint32_t)(i - (int64_t)pc * st.n8);
  const uint32_t Z = st_div(pos, st.hxy, st.mhxy);
  pos -= Z * st.hxy;
  const uint32_t Y = st_div(pos, st.hx, st.mhx);
  const uint32_t X = pos - Y * st.hx;
  const int x = (int)(2 * X + ((pc >> st.bx) & 1));
  const int y = (int)(2 * Y + ((pc >> st.by) & 1));
  const int z = (int)(2 * Z + ((pc >> st.bz) & 1));
  return x >= 1 && x <= st.lx - 2 && y >= 1 && y <= st.ly - 2 && z >= 1 && z <= st.lz - 2;
}

// Columns of a FACE row of colour pc in closed form (the row's compacted ELL
// slots, ref: problem.py:127-138): slot k is the k-th in-box offset s of the
// row's position class (table kFaceSlots), column i + doff[s] (the same
// per-colour constants as the interior rows); slots past the row's nnz are
// padding, column 0.  Rows whose
// missing neighbours lie across a RANK INTERFACE (halo columns, numbered by the
// halo plan) return false and read the index plane.  Replaces 27 sparse 4-byte
// index loads per x-face row -- a 32-byte sector each.
// k-th in-box offset (0..26, z-slowest) of a row whose position class per axis is
// 0 (low face), 1 (interior) or 2 (high face); 27 = padding.  Built at compile time.
struct FaceSlots {
  unsigned char s[27][27];
  constexpr FaceSlots() : s() {
    for (int cls = 0; cls < 27; ++cls) {
      const int cx = cls % 3, cy = (cls / 3) % 3, cz = cls / 9;
      int k = 0;
      for (int o = 0; o < 27; ++o) {
        const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
        const bool ok = !(cx == 0 && dx < 0) && !(cx == 2 && dx > 0) && !(cy == 0 && dy < 0) &&
                        !(cy == 2 && dy > 0) && !(cz == 0 && dz < 0) && !(cz == 2 && dz > 0);
        if (ok) s[cls][k++] = (unsigned char)o;
      }
      for (; k < 27; ++k) s[cls][k] = 27;
    }
  }
};
__constant__ FaceSlots kFaceSlots = FaceSlots();

__device__ __forceinline__ bool st_face_cols(const Stencil& st, int64_t i, int pc, const int32_t* doff,
                                             int32_t (&c)[27]) {
  uint32_t pos = (uint32_t)(i - (int64_t)pc * st.n8);
  const uint32_t Z = st_div(pos, st.hxy, st.mhxy);
  pos -= Z * st.hxy;
  const uint32_t Y = st_div(pos, st.hx, st.mhx);
  const uint32_t X = pos - Y * st.hx;
  const int x = (int)(2 * X + ((pc >> st.bx) & 1));
  const int y = (int)(2 * Y + ((pc >> st.by) & 1));
  const int z = (int)(2 * Z + ((pc >> st.bz) & 1));
  const int cx = x == 0 ? 0 : (x == st.lx - 1 ? 2 : 1);
  const int cy = y == 0 ? 0 : (y == st.ly - 1 ? 2 : 1);
  const int cz = z == 0 ? 0 : (z == st.lz - 1 ? 2 : 1);
  const int cut = (cx == 0 ? 1 : 0) | (cx == 2 ? 2 : 0) | (cy == 0 ? 4 : 0) | (cy == 2 ? 8 : 0) |
                  (cz == 0 ? 16 : 0) | (cz == 2 ? 32 : 0);
  if (cut & st.ifc) return false;
  const unsigned char* tab = kFaceSlots.s[cz * 9 + cy * 3 + cx];
#pragma unroll
  for (int k = 0; k < 27; ++k) {
    const int s = tab[k];
    int32_t cc = 0;
    if (s < 27) {
      cc = (int32_t)i + doff[s];
      if (s == 13) cc = ~cc;
    }
    c[k] = cc;
  }
  return true;
}

// An x-face row (x == 0 or lx-1, y and z interior, the x face not a rank
// interface): its 18 valid offsets are, per (dy, dz) pair in order, the two dx
// on the box side -- slot k is offset 3 (k >> 1) + (k & 1) + (x == 0), a
// compile-time map per side, so the columns cost no table lookups.  Returns
// 0 (not such a row), 1 (low x face) or 2 (high x face).
__device__ __forceinline__ int st_xface(const Stencil& st, int64_t i, int pc) {
  uint32_t pos = (uint32_t)(i - (int64_t)pc * st.n8);
  const uint32_t Z = st_div(pos, st.hxy, st.mhxy);
  pos -= Z * st.hxy;
  const uint32_t Y = st_div(pos, st.hx, st.mhx);
  const uint32_t X = pos - Y * st.hx;
  const int x = (int)(2 * X + ((pc >> st.bx) & 1));
  const int y = (int)(2 * Y + ((pc >> st.by) & 1));
  const int z = (int)(2 * Z + ((pc >> st.bz) & 1));
  if (y < 1 || y > st.ly - 2 || z < 1 || z > st.lz - 2) return 0;
  if (x == 0) return (st.ifc & 1) ? 0 : 1;
  if (x == st.lx - 1) return (st.ifc & 2) ? 0 : 2;
  return 0;
}

// z_i of one row of colour pc: values from the shared-memory tile sv (plane-major,
// ROWS per plane), gathers through L1, the reference's slot-order arithmetic.
template <typename T, int ROWS>
__device__ __forceinline__ T gs_tma_row(const SweepPlan& p, const T* __restrict__ sv, int t, int64_t i,
                                        const T* __restrict__ r, const T* z, int64_t known0,
                                        const int32_t (&D)[27], uint32_t kmask, int pc) {
  const T ri = __ldg(r + i);  // issued first: its DRAM latency overlaps the gathers
  T acc = T(0), d = T(0);
  if (p.st.on && st_interior(p.st, i, pc)) {
    const T* zi = z + i;
    T g[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) g[s] = ((kmask >> s) & 1u) ? T(0) : zi[D[s]];
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      T vs = sv[s * ROWS + t];
      if (s == 13) {  // the diagonal slot: a_ii aside, the product formed as 0 * z_i
        d = vs;
        vs = T(0);
      }
      acc = add_rn(acc, mul_rn(vs, g[s]));
    }
  } else {
    int32_t c[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) c[s] = __ldg(p.cols + s * p.ld + i);
    T g[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      const int32_t cc = c[s] < 0 ? ~c[s] : c[s];
      g[s] = (known0 >= 0 && cc >= known0) ? T(0) : z[cc];
    }
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
  return div_rn(sub_rn(ri, acc), d);
}

template <typename T, int ROWS, int STAGES>
__global__ void __launch_bounds__(32 + ROWS, 2) k_gs_sweep_tma(const __grid_constant__ SweepPlan p,
                                                                const T* __restrict__ r, T* z) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kTile = TmaTile<T, ROWS>::kBytes;
  T* ring = (T*)smem;
  uint64_t* full = (uint64_t*)(smem + (size_t)STAGES * kTile);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, ROWS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  const int G = gridDim.x;
  if (warp == 0) {
    // ---------------- producer: value planes only (constant: no wait on the predecessor)
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.vmap) : "memory");
      uint32_t k = 0;
      for (int c = 0; c < p.ncolors; ++c) {
        const TileSpan sp(p, c, ROWS);
        for (int64_t m = 0; m < sp.nt; ++m, ++k) {
          const int64_t row0 = sp.row0(m);  // a short last tile reads past its rows (zero-filled past ld)
          const int s = k % STAGES;
          if (k >= STAGES) mbar_wait(empty + s, ((k / STAGES) - 1) & 1);
          mbar_expect_tx(full + s, (uint32_t)kTile);
          tma_g2s_2d(ring + (size_t)s * 27 * ROWS, &p.vmap, (int)row0, 0, full + s, pol);
        }
      }
    }
    return;
  }
  // ---------------- consumers: one row per thread
  const int t = threadIdx.x - 32;
  pdl_wait();  // r, z (and the pass counters) come from the predecessors
  uint32_t k = 0;
  for (int c = 0; c < p.ncolors; ++c) {
    if (c > 0) {
      // colour c gathers what colour c-1 wrote anywhere in the grid
      if (t == 0) {
        while (ld_relaxed_gpu_u32(p.done + c - 1) < (unsigned)G) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire; also invalidates this SM's L1 (stale z lines)
      }
      consumers_sync(ROWS);
    }
    const TileSpan sp(p, c, ROWS);
    const int64_t known0 = p.zero ? p.off[c] : -1;
    int32_t D[27];
    const int cd = c < 8 ? c : 7;
#pragma unroll
    for (int q = 0; q < 27; ++q) D[q] = p.doff[cd][q];
    const uint32_t kmask = p.zero ? p.kmask[cd] : 0u;
    for (int64_t m = 0; m < sp.nt; ++m, ++k) {
      const int64_t row0 = sp.row0(m);
      const int s = k % STAGES;
      mbar_wait(full + s, (k / STAGES) & 1);
      const int64_t i = row0 + t;
      T zi = T(0);
      const bool act = i < sp.hi;
      if (act) zi = gs_tma_row<T, ROWS>(p, ring + (size_t)s * 27 * ROWS, t, i, r, z, known0, D, kmask, c);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);  // the stage's values are consumed
      if (act) z[i] = zi;
    }
    consumers_sync(ROWS);  // every z of this CTA's tiles of colour c is written
    if (t == 0) {
      __threadfence();
      const unsigned old = atomicAdd(p.done + c, 1u);
      if (c == p.ncolors - 1 && old == (unsigned)G - 1) {
        // every CTA is past its last wait: reset the counters for the next sweep
        for (int q = 0; q < p.ncolors; ++q) p.done[q] = 0u;
        __threadfence();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// One colour pass per launch, one tile of ROWS rows per CTA (the default).
//
// The persistent sweep above keeps the value stream busy across the pass
// drains, but measured slower (2 CTAs x ROWS rows per SM in flight: too few
// outstanding z gathers; the gathers, not the value stream, bound the pass).
// Here every CTA stages ITS tile's 27 value planes with one tensor copy issued
// by thread 0 before anything else -- under programmatic dependent launch that
// is before the predecessor pass has drained, since the values do not depend
// on z -- and its threads hold only the 27 gathered z values in registers
// while the copy lands.  Rows in flight per SM rise from 768 (all 54 loads in
// registers, hpg_kernels.cuh k_gs_pass) to MINB x ROWS.
struct PassPlan {
  CUtensorMap vmap;     // value planes [27][ld] of T, box {ROWS, 27}
  const int32_t* cols;  // [27][ld]: face rows only
  int64_t ld;
  int64_t row0, nrows;  // this colour block
  int64_t known0;       // zero sweep: columns >= known0 hold 0 (loads skipped, products formed)
  int rev;              // CTAs walk the block from its end
  int color;
  uint32_t kmask;       // implicit-index rows: slot s's load skipped when bit s is set
  int32_t doff[27];     // implicit-index rows: slot s gathers column i + doff[s]
  int xface;            // x-face rows use the compile-time slot map (st_xface)
  const uint8_t* skip;  // overlapped exchange: face rows flagged here are left to a later
                        // launch (they read halo slots / are sent); interior rows never are
  Stencil st;
};

template <typename T, int ROWS, int MINB>
__global__ void __launch_bounds__(ROWS, MINB) k_gs_pass_tma(const __grid_constant__ PassPlan p,
                                                            const T* __restrict__ r, T* z) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* sv = (T*)smem;
  uint64_t* bar = (uint64_t*)(smem + (size_t)27 * ROWS * sizeof(T));
  const int64_t blk = p.rev ? (int64_t)(gridDim.x - 1 - blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t tile0 = p.row0 + blk * ROWS;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(27 * ROWS * sizeof(T)));
    tma_g2s_2d(sv, &p.vmap, (int)tile0, 0, bar, evict_first_policy());
  }
  pdl_trigger();
  __syncthreads();  // the barrier is initialised before anyone waits on it
  const int t = threadIdx.x;
  const int64_t i = tile0 + t;
  if (i >= p.row0 + p.nrows) return;
  pdl_wait();  // z (and r) come from the predecessors
  const T ri = __ldg(r + i);
  T acc = T(0), d = T(0);
  if (p.st.on && st_interior(p.st, i, p.color)) {
    const T* zi = z + i;
    T g[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) g[s] = ((p.kmask >> s) & 1u) ? T(0) : zi[p.doff[s]];
    mbar_wait(bar, 0);
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      T vs = sv[s * ROWS + t];
      if (s == 13) {  // the diagonal slot: a_ii aside, the product formed as 0 * z_i
        d = vs;
        vs = T(0);
      }
      acc = add_rn(acc, mul_rn(vs, g[s]));
    }
  } else {
    if (p.skip && p.skip[i]) {
      mbar_wait(bar, 0);  // (the tile's copy must land before the CTA may retire)
      return;
    }
    int32_t c[27];
    const int xf = (p.st.on && p.xface) ? st_xface(p.st, i, p.color) : 0;
    if (xf) {  // x-face row: compile-time slot map per side
#pragma unroll
      for (int k = 0; k < 27; ++k) {
        int32_t cc = 0;
        if (k < 18) {
          const int s_lo = 3 * (k >> 1) + (k & 1) + 1, s_hi = 3 * (k >> 1) + (k & 1);
          const int s = xf == 1 ? s_lo : s_hi;
          cc = (int32_t)i + (xf == 1 ? p.doff[s_lo] : p.doff[s_hi]);
          if (s == 13) cc = ~cc;
        }
        c[k] = cc;
      }
    } else if (!(p.st.on && st_face_cols(p.st, i, p.color, p.doff, c))) {
#pragma unroll
      for (int s = 0; s < 27; ++s) c[s] = __ldg(p.cols + s * p.ld + i);
    }
    T g[27];
#pragma unroll
    for (int s = 0; s < 27; ++s) {
      const int32_t cc = c[s] < 0 ? ~c[s] : c[s];
      g[s] = (p.known0 >= 0 && cc >= p.known0) ? T(0) : z[cc];
    }
    mbar_wait(bar, 0);
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
}

// ---------------------------------------------------------------------------
// SpMV (MODE 0: y = A x) and the fp64 outer residual (MODE 1: y = b - A x and a
// per-CTA partial of sum y^2) with the same staging as k_gs_pass_tma: one
// tensor copy of the tile's value planes before the PDL wait, the row's 27
// gathers in registers, the slot-ordered sum (ref: krylov.py:76-107, 215-226).
// ilv > 1: consecutive CTAs take the same tile position in ilv equal segments
// of the rows (the colour blocks) so the x lines they gather are shared in L2.
struct SpmvPlan {
  CUtensorMap vmap;     // value planes [27][ld] of T, box {ROWS, 27}
  const int32_t* cols;  // face rows only
  int64_t ld, n;
  int64_t n8;           // implicit-index rows: colour block size (a multiple of ROWS)
  int ilv;
  int xface;            // x-face rows use the compile-time slot map (st_xface)
  int32_t doff[8][27];  // implicit-index rows of colour c: slot s reads column i + doff[c][s]
  const uint8_t* skip;  // MODE 0, overlapped exchange: flagged (face) rows are left to a later launch
  Stencil st;
};

// MODE 2: the fused residual + injection (ref: multigrid.py:107-128): rows are the
// fine colour-0 rows [0, n), y[dst[i]] = b[i] - (A x)[i]
template <typename T, int ROWS, int MINB, int MODE>
__global__ void __launch_bounds__(ROWS, MINB) k_spmv_tma(const __grid_constant__ SpmvPlan p, const T* __restrict__ x,
                                                         const T* __restrict__ b, T* __restrict__ y,
                                                         double* __restrict__ partial,
                                                         const int32_t* __restrict__ dst = nullptr) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* sv = (T*)smem;
  uint64_t* bar = (uint64_t*)(smem + (size_t)27 * ROWS * sizeof(T));
  int64_t blk = blockIdx.x;
  if (p.ilv > 1) blk = (int64_t)(blockIdx.x % p.ilv) * (gridDim.x / p.ilv) + blockIdx.x / p.ilv;
  const int64_t tile0 = blk * ROWS;
  if (tile0 >= p.n) return;  // (grid padded to a multiple of ilv)
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(27 * ROWS * sizeof(T)));
    tma_g2s_2d(sv, &p.vmap, (int)tile0, 0, bar, evict_first_policy());
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();  // x (and b) come from the predecessors
  const int t = threadIdx.x;
  const int64_t i = tile0 + t;
  double sq = 0.0;
  bool skipped = false;
  if (i < p.n) {
    T g[27];
    const int col = p.st.on ? (int)(tile0 / p.n8) : 0;
    if (p.st.on && st_interior(p.st, i, col)) {
      const T* xi = x + i;
#pragma unroll
      for (int s = 0; s < 27; ++s) g[s] = xi[p.doff[col][s]];
    } else {
      skipped = MODE == 0 && p.skip && p.skip[i];
      int32_t cf[27];
      const int xf = (p.st.on && p.xface) ? st_xface(p.st, i, col) : 0;
      if (xf) {  // x-face row: compile-time slot map per side
#pragma unroll
        for (int k = 0; k < 27; ++k) {
          int32_t cc = 0;
          if (k < 18) {
            const int s_lo = 3 * (k >> 1) + (k & 1) + 1, s_hi = 3 * (k >> 1) + (k & 1);
            cc = (int32_t)i + (xf == 1 ? p.doff[col][s_lo] : p.doff[col][s_hi]);
          }
          cf[k] = cc;  // (no diagonal marker needed: the SpMV forms every product)
        }
      } else if (!(p.st.on && st_face_cols(p.st, i, col, p.doff[col], cf))) {
#pragma unroll
        for (int s = 0; s < 27; ++s) cf[s] = __ldg(p.cols + s * p.ld + i);
      }
#pragma unroll
      for (int s = 0; s < 27; ++s) g[s] = x[cf[s] < 0 ? ~cf[s] : cf[s]];
    }
    mbar_wait(bar, 0);
    T acc = T(0);
#pragma unroll
    for (int s = 0; s < 27; ++s) acc = add_rn(acc, mul_rn(sv[s * ROWS + t], g[s]));
    if (MODE == 0) {
      if (!skipped) y[i] = acc;
    } else if (MODE == 2) {
      y[dst[i]] = sub_rn(b[i], acc);
    } else {
      const T rr = sub_rn(b[i], acc);
      y[i] = rr;
      sq = (double)rr * (double)rr;
    }
  }
  if (MODE == 1) {  // deterministic CTA reduction, indexed by the row tile
    __shared__ double red[ROWS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((t & 31) == 0) red[t >> 5] = sq;
    __syncthreads();
    if (t == 0) {
      double a = 0.0;
      for (int w = 0; w < ROWS / 32; ++w) a += red[w];
      partial[blk] = a;
    }
  }
}

}  // namespace hpg
