// Streaming microbenchmark for the slot-major value planes [27][ld] (fp32):
// how fast can a CTA ring pull {ROWS x 27} tiles into shared memory with
// 2-D tensor copies vs plain coalesced loads?  Standalone (not part of the
// library):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tma_stream tools/tma_stream.cu
//   ./tools/tma_stream
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(sa(b)), "r"(par)
                 : "memory");
}

// producer warp 0 lane 0: one 2-D box {ROWS, PLANES} per tile; consumers: sum
template <int ROWS, int PLANES, int STAGES>
__global__ void __launch_bounds__(32 + ROWS) k_tma(const __grid_constant__ CUtensorMap map, int64_t n, float* out,
                                                   int evict_first) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int TB = ROWS * 27 * 4;
  float* ring = (float*)sm;
  uint64_t* full = (uint64_t*)(sm + (size_t)STAGES * TB);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mb_init(full + s, 1);
      mb_init(empty + s, ROWS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nt = n / ROWS;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      uint64_t pol;
      if (evict_first) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      uint32_t k = 0;
      for (int64_t j = blockIdx.x; j < nt; j += gridDim.x, ++k) {
        const int s = k % STAGES;
        if (k >= STAGES) mb_wait(empty + s, ((k / STAGES) - 1) & 1);
        mb_tx(full + s, TB);
        for (int y = 0; y < 27; y += PLANES)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
              "{%2, %3}], [%4], %5;" ::"r"(sa(ring + (size_t)s * ROWS * 27 + y * ROWS)),
              "l"(&map), "r"((int)(j * ROWS)), "r"(y), "r"(sa(full + s)), "l"(pol)
              : "memory");
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;
  float acc = 0.f;
  uint32_t k = 0;
  for (int64_t j = blockIdx.x; j < nt; j += gridDim.x, ++k) {
    const int s = k % STAGES;
    mb_wait(full + s, (k / STAGES) & 1);
    const float* sv = ring + (size_t)s * ROWS * 27;
#pragma unroll
    for (int q = 0; q < 27; ++q) acc += sv[q * ROWS + t];
    __syncwarp();
    if ((t & 31) == 0) mb_arrive(empty + s);
  }
  if (acc == 12345.f) out[0] = acc;
}

// plain: one row per thread, 27 streaming loads
__global__ void __launch_bounds__(128) k_ldg(const float* __restrict__ v, int64_t ld, int64_t n, float* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float a[27];
#pragma unroll
  for (int q = 0; q < 27; ++q) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(a[q]) : "l"(v + q * ld + i));
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < 27; ++q) acc += a[q];
  if (acc == 12345.f) out[0] = acc;
}

template <int ROWS, int PLANES, int STAGES>
int run_tma(PFN_cuTensorMapEncodeTiled_v12000 enc, float* v, int64_t ld, int64_t n, float* out, int ctas_per_sm,
            int evict_first) {
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, 27};
  const cuuint64_t str[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {ROWS, PLANES};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, v, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const size_t smem = (size_t)STAGES * ROWS * 27 * 4 + 2 * STAGES * 8;
  auto fn = k_tma<ROWS, PLANES, STAGES>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 32 + ROWS, smem));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int cps = ctas_per_sm < per ? ctas_per_sm : per;
  const int grid = cps * sms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fn<<<grid, 32 + ROWS, smem>>>(map, n, out, evict_first);
  CK(cudaDeviceSynchronize());
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) fn<<<grid, 32 + ROWS, smem>>>(map, n, out, evict_first);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / reps;
  printf("tma ROWS %d PLANES/box %d STAGES %d ctas/SM %d (max %d) smem %zu ef %d: %.1f us  %.0f GB/s\n", ROWS, PLANES,
         STAGES, cps, per, smem, evict_first, us, 27.0 * n * 4 / us / 1e3);
  return 0;
}

int main() {
  const int64_t n = 256LL * 256 * 256, ld = n + 32;  // level-0 fp32 planes (1.8 GB)
  float* v;
  float* out;
  CK(cudaMalloc(&v, 27 * ld * 4));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(v, 0, 27 * ld * 4));
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_ldg<<<(n + 127) / 128, 128>>>(v, ld, n, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k_ldg<<<(n + 127) / 128, 128>>>(v, ld, n, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg row-per-thread 27 loads: %.1f us  %.0f GB/s\n", ms * 100, 27.0 * n * 4 / (ms * 100) / 1e3);
  }
  run_tma<256, 27, 4>(enc, v, ld, n, out, 2, 1);
  run_tma<256, 27, 4>(enc, v, ld, n, out, 2, 0);
  run_tma<256, 27, 4>(enc, v, ld, n, out, 1, 1);
  run_tma<256, 27, 7>(enc, v, ld, n, out, 1, 1);
  run_tma<256, 27, 2>(enc, v, ld, n, out, 3, 1);
  run_tma<128, 27, 8>(enc, v, ld, n, out, 2, 1);
  run_tma<128, 27, 4>(enc, v, ld, n, out, 4, 1);
  run_tma<256, 9, 4>(enc, v, ld, n, out, 2, 1);   // 3 boxes of 9 planes per tile
  run_tma<64, 27, 8>(enc, v, ld, n, out, 4, 1);
  return 0;
}
