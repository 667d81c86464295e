// Jones-Plassmann-Luby colouring on the device, bit-identical to the
// reference's (ref: coloring.py:56-70) including its random stream.
//
// The reference draws w = rng.random(n) every round from numpy's
// default_rng(seed) -- PCG64 (128-bit LCG, XSL-RR output) and
// random() = (next_uint64 >> 11) * 2^-53.  Round r's draw i is the generator
// advanced (r n + i + 1) steps from the seeded state, so every thread jumps
// straight to its own state with the LCG power-advance (O(log) 128-bit
// multiply-adds): no sequential stream.  A row still uncoloured is selected
// when (w_i, i) beats (w_j, j) of every uncoloured in-box neighbour; selected
// rows are pairwise independent, so a second kernel gives each the smallest
// colour its coloured neighbours lack -- the reference's sequential loop
// over `selected` gives the same colours.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hpg {

struct U128 {
  uint64_t lo, hi;
};
__host__ __device__ __forceinline__ U128 u128_mul(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
  r.hi = __umul64hi(a.lo, b.lo);
#else
  r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64);
#endif
  r.hi += a.lo * b.hi + a.hi * b.lo;
  return r;
}
__host__ __device__ __forceinline__ U128 u128_add(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}
// numpy's PCG64 multiplier (PCG_DEFAULT_MULTIPLIER_128)
__host__ __device__ __forceinline__ U128 pcg_mult() { return U128{0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull}; }

// state advanced by delta steps of s <- s * MULT + inc
__host__ __device__ __forceinline__ U128 pcg_advance(U128 state, U128 inc, uint64_t delta) {
  U128 acc_mult{1, 0}, acc_plus{0, 0}, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = u128_mul(acc_mult, cur_mult);
      acc_plus = u128_add(u128_mul(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = u128_mul(u128_add(cur_mult, U128{1, 0}), cur_plus);
    cur_mult = u128_mul(cur_mult, cur_mult);
    delta >>= 1;
  }
  return u128_add(u128_mul(acc_mult, state), acc_plus);
}
// XSL-RR output of a (post-step) state
__host__ __device__ __forceinline__ uint64_t pcg_output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// w[i] = round r's i-th rng.random() draw; base = the state before the round
__global__ void k_jpl_weights(int64_t n, U128 base, U128 inc, double* __restrict__ w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const U128 s = pcg_advance(base, inc, (uint64_t)i + 1);
  w[i] = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ bool jpl_nbr(int lx, int ly, int lz, int64_t i, int q, int64_t* j) {
  const int x = (int)(i % lx), y = (int)((i / lx) % ly), z = (int)(i / ((int64_t)lx * ly));
  const int dx = q % 3 - 1, dy = (q / 3) % 3 - 1, dz = q / 9 - 1;
  const int ax = x + dx, ay = y + dy, az = z + dz;
  if (ax < 0 || ax >= lx || ay < 0 || ay >= ly || az < 0 || az >= lz) return false;
  *j = ax + (int64_t)lx * (ay + (int64_t)ly * az);
  return true;
}

// sel[i] = uncoloured row i beats every uncoloured in-box neighbour (natural order)
__global__ void k_jpl_select(int lx, int ly, int lz, const double* __restrict__ w, const int32_t* __restrict__ colors,
                             uint8_t* __restrict__ sel) {
  const int64_t n = (int64_t)lx * ly * lz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool s = colors[i] < 0;
  const double wi = w[i];
  for (int q = 0; q < 27 && s; ++q) {
    int64_t j;
    if (q == 13 || !jpl_nbr(lx, ly, lz, i, q, &j) || colors[j] >= 0) continue;
    const double wj = w[j];
    s = wi > wj || (wi == wj && i > j);
  }
  sel[i] = s ? 1 : 0;
}

// selected rows take the smallest colour their coloured neighbours lack
__global__ void k_jpl_color(int lx, int ly, int lz, const uint8_t* __restrict__ sel, int32_t* colors,
                            unsigned long long* __restrict__ count) {
  const int64_t n = (int64_t)lx * ly * lz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !sel[i]) return;
  uint32_t used = 0;
  for (int q = 0; q < 27; ++q) {
    int64_t j;
    if (q == 13 || !jpl_nbr(lx, ly, lz, i, q, &j)) continue;
    const int32_t c = colors[j];
    if (c >= 0 && c < 32) used |= 1u << c;
  }
  colors[i] = __ffs(~used) - 1;
  atomicAdd(count, 1ull);
}

}  // namespace hpg
