// CGS2 + norm + normalise in ONE persistent cooperative kernel, with the
// basis rows streamed through shared memory by the bulk-copy (TMA) engine.
//
// One Arnoldi step needs, for kb = k+1 basis rows Q[0..kb) of length n
// (ref: krylov.py:110-129, 266-273):
//   pass A  h1 = Q w                  (kb dots)
//   pass B  w -= Q^T h1 ; h2 = Q w    (correction fused with the 2nd projection)
//   pass C  w -= Q^T h2 ; beta^2 = w.w
//   pass D  Q[k] = w / beta
// i.e. three streams of the kb rows instead of the four of the textbook
// order.  Each pass walks this CTA's contiguous range of tiles; thread 0
// issues cp.async.bulk copies of the kb row-segments (and w) of tile t+S-1
// into stage (t+S-1)%S while all threads consume tile t from shared memory,
// so the copy engine keeps ~S-1 tiles of every row in flight with no
// register cost.  Between passes one grid barrier, a fixed-order fold of the
// per-CTA partials by CTA 0, and another barrier: deterministic, and no host
// round trip until the final (h1, h2, beta) read.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hpg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 2-D tensor copy: box {tile, kb} of the basis at element (x, y) -> shared
__device__ __forceinline__ void tma_2d_g2s(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

template <typename T>
struct CgsParams {
  const T* Q;      // basis, row-major, row stride ldq
  T* w;            // vector being orthogonalised (length >= round_up(n, 32))
  T* qnext;        // Q[k+1] (NULL: skip norm/normalise)
  T* partial;      // [KBMAX][gridDim] per-CTA partials
  T* scal;         // [0,64) h1, [64,128) h2, [128] beta
  int64_t ldq, n;
  int kb, tile;    // elements per tile = boxes * box
  int box, boxes;  // TMA box inner extent (elements) and boxes per stage
  int stages;
};

constexpr int kCgsThreads = 512;

template <typename T, int KB>
__device__ __forceinline__ void cgs_block_reduce(T (&acc)[KB], int kb, T* out, T* red) {
  // red: [kCgsThreads/32][KB] in shared memory
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    T a = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) red[warp * KB + j] = a;
  }
  __syncthreads();
  if (threadIdx.x < kb) {
    T a = T(0);
    for (int w = 0; w < kCgsThreads / 32; ++w) a += red[w * KB + threadIdx.x];
    out[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = a;
  }
  __syncthreads();
}

// CTA 0 folds the per-CTA partials of cnt outputs into dst (fixed order)
template <typename T>
__device__ __forceinline__ void cgs_fold(const T* partial, int cnt, T* dst, bool do_sqrt) {
  if (blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < cnt; j += kCgsThreads / 32) {
    T a = T(0);
    for (int b = lane; b < (int)gridDim.x; b += 32) a += __ldcg(partial + (int64_t)j * gridDim.x + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) dst[j] = do_sqrt ? sqrt(a) : a;
  }
}

// MODE 0: acc[j] += q_j w            (pass A)
// MODE 1: w -= sum q_j h; acc[j] += q_j w   (pass B)
// MODE 2: w -= sum q_j h; acc[0] += w^2     (pass C)
template <typename T, int KB, int MODE>
__device__ __forceinline__ void cgs_pass(const CgsParams<T>& p, const CUtensorMap* qmap, T* sq, T* sw, T* sh,
                                         uint64_t* bars, uint32_t& phases, const T* h, T (&acc)[KB]) {
  const int64_t ntiles = (p.n + p.tile - 1) / p.tile;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per;
  const int64_t t1 = t0 + per < ntiles ? t0 + per : ntiles;
  const int S = p.stages;
  const int kb = p.kb;
  if (MODE > 0 && threadIdx.x < kb) sh[threadIdx.x] = __ldcg(h + threadIdx.x);
  __syncthreads();

  auto issue = [&](int64_t t) {
    const int st = (int)((t - t0) % S);
    const int64_t i0 = t * p.tile;
    const int64_t cnt = p.n - i0 < p.tile ? p.n - i0 : p.tile;
    const uint32_t bytes = (uint32_t)(((cnt * sizeof(T)) + 15) & ~(int64_t)15);
    T* qs = sq + (int64_t)st * kb * p.tile;
    // tensor copies always land full boxes (zero-filled past n); stage layout [box b][row j][box]
    const int nbx = (int)((cnt + p.box - 1) / p.box);
    mbar_expect_tx(&bars[st], (uint32_t)(nbx * p.box * kb * sizeof(T)) + bytes);
    for (int b = 0; b < nbx; ++b)
      tma_2d_g2s(qs + (int64_t)b * kb * p.box, qmap, (int)(i0 + (int64_t)b * p.box), 0, &bars[st]);
    bulk_g2s(sw + (int64_t)st * p.tile, p.w + i0, bytes, &bars[st]);
  };

  if (threadIdx.x == 0)
    for (int64_t t = t0; t < t1 && t < t0 + S - 1; ++t) issue(t);
  for (int64_t t = t0; t < t1; ++t) {
    if (threadIdx.x == 0 && t + S - 1 < t1) issue(t + S - 1);
    const int st = (int)((t - t0) % S);
    mbar_wait(&bars[st], (phases >> st) & 1u);
    phases ^= 1u << st;
    const T* qs = sq + (int64_t)st * kb * p.tile;
    const T* ws = sw + (int64_t)st * p.tile;
    const int64_t i0 = t * p.tile;
    const int cnt = (int)(p.n - i0 < p.tile ? p.n - i0 : p.tile);
    for (int e = threadIdx.x; e < cnt; e += kCgsThreads) {
      const T* qe = qs + (int64_t)(e / p.box) * kb * p.box + (e % p.box);  // row j at qe[j * box]
      T wi = ws[e];
      if (MODE > 0) {
        T ts = T(0);
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < kb) ts = fma(qe[j * p.box], sh[j], ts);
        wi = wi - ts;
        p.w[i0 + e] = wi;  // read back by the next pass's bulk copies (async proxy)
      }
      if (MODE < 2) {
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j < kb) acc[j] = fma(qe[j * p.box], wi, acc[j]);
      } else {
        acc[0] = fma(wi, wi, acc[0]);
      }
    }
    __syncthreads();  // stage st free for refill
  }
}

template <typename T, int KB>
__global__ void __launch_bounds__(kCgsThreads, 1) k_cgs2_fused(const __grid_constant__ CgsParams<T> p,
                                                              const __grid_constant__ CUtensorMap qmap) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sq = (T*)smem_raw;                                   // [S][kb][tile]
  T* sw = sq + (int64_t)p.stages * p.kb * p.tile;         // [S][tile]
  T* red = sw + (int64_t)p.stages * p.tile;               // [warps][KB]
  T* sh = red + (kCgsThreads / 32) * KB;                  // [KB] current h
  uint64_t* bars = (uint64_t*)(sh + KB + 2);
  bars = (uint64_t*)(((uintptr_t)bars + 7) & ~(uintptr_t)7);
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phases = 0;

  {  // pass A: h1
    T acc[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) acc[j] = T(0);
    cgs_pass<T, KB, 0>(p, &qmap, sq, sw, sh, bars, phases, nullptr, acc);
    cgs_block_reduce<T, KB>(acc, p.kb, p.partial, red);
  }
  grid.sync();
  cgs_fold(p.partial, p.kb, p.scal, false);
  grid.sync();
  {  // pass B: w -= Q^T h1 ; h2
    T acc[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) acc[j] = T(0);
    cgs_pass<T, KB, 1>(p, &qmap, sq, sw, sh, bars, phases, p.scal, acc);
    cgs_block_reduce<T, KB>(acc, p.kb, p.partial, red);
  }
  asm volatile("fence.proxy.async;" ::: "memory");  // generic w stores -> async-proxy reads
  grid.sync();
  cgs_fold(p.partial, p.kb, p.scal + 64, false);
  grid.sync();
  {  // pass C: w -= Q^T h2 ; beta^2
    T acc[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) acc[j] = T(0);
    cgs_pass<T, KB, 2>(p, &qmap, sq, sw, sh, bars, phases, p.scal + 64, acc);
    T a1[1] = {acc[0]};
    cgs_block_reduce<T, 1>(a1, 1, p.partial, red);
  }
  asm volatile("fence.proxy.async;" ::: "memory");
  if (p.qnext == nullptr) return;
  grid.sync();
  cgs_fold(p.partial, 1, p.scal + 128, true);
  grid.sync();
  // pass D: Q[k+1] = w / beta  (ref: krylov.py:269-273)
  const T bt = __ldcg(p.scal + 128);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x)
    p.qnext[i] = bt != T(0) ? div_rn(__ldcg(p.w + i), bt) : T(0);
}

}  // namespace hpg
