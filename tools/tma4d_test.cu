// Standalone check of the 4-D tensor copies the brick colour pass uses: z as
// [8 colours][hz][hy][hx] sub-lattices, boxes widened by one on chosen axes.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tma4d_test tools/tma4d_test.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct P {
  CUtensorMap map[8];
  int bx[8], by[8], bz[8], bc[8], bytes[8], off[8];
};

__global__ void k(const __grid_constant__ P p, int am, float* out, int n) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* s = (float*)sm;
  uint64_t* bar = (uint64_t*)(sm + 32768);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(p.bytes[am]) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(sa(s)),
        "l"(&p.map[am]), "r"(p.bx[am]), "r"(p.by[am]), "r"(p.bz[am]), "r"(p.bc[am]), "r"(sa(bar))
        : "memory");
  }
  __syncthreads();
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
                 : "=r"(ok)
                 : "r"(sa(bar))
                 : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  const int hx = 128, hy = 128, hz = 128, BY = 2;
  const int pad = argc > 1 ? atoi(argv[1]) : 4;      // X widening
  const int negx = argc > 2 ? atoi(argv[2]) : 1;     // start x at -1
  const int dimpad = argc > 3 ? atoi(argv[3]) : 1;   // tensor X extent hx + pad
  const size_t n8 = (size_t)hx * hy * hz;
  float* z;
  cudaMalloc(&z, 8 * n8 * 4 + 4096);
  std::vector<float> h(8 * n8);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000003);
  cudaMemcpy(z, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  P p;
  int xe[8], ye[8], ze[8];
  for (int am = 1; am < 8; ++am) {
    xe[am] = hx + ((am & 1) ? pad : 0);
    ye[am] = BY + ((am >> 1) & 1);
    ze[am] = 1 + ((am >> 2) & 1);
    const cuuint64_t dims[4] = {(cuuint64_t)(hx + (dimpad ? pad : 0)), (cuuint64_t)hy, (cuuint64_t)hz, 8};
    const cuuint64_t str[3] = {(cuuint64_t)hx * 4, (cuuint64_t)hx * hy * 4, (cuuint64_t)n8 * 4};
    const cuuint32_t box[4] = {(cuuint32_t)xe[am], (cuuint32_t)ye[am], (cuuint32_t)ze[am], 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&p.map[am], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, z, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("am %d encode %d box %d %d %d\n", am, (int)r, xe[am], ye[am], ze[am]);
    p.bx[am] = ((am & 1) && negx) ? -1 : 0;
    p.by[am] = 5 + (((am >> 1) & 1) ? -1 : 0);
    p.bz[am] = 7 + (((am >> 2) & 1) ? -1 : 0);
    p.bc[am] = am;
    p.bytes[am] = xe[am] * ye[am] * ze[am] * 4;
  }
  float* out;
  cudaMalloc(&out, 32768);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  int bad = 0;
  for (int am = 1; am < 8; ++am) {
    const int n = xe[am] * ye[am] * ze[am];
    k<<<1, 256, 40000>>>(p, am, out, n);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("pad %d negx %d dimpad %d am %d: %s\n", pad, negx, dimpad, am, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> o(n);
    cudaMemcpy(o.data(), out, n * 4, cudaMemcpyDeviceToHost);
    for (int zz = 0; zz < ze[am]; ++zz)
      for (int yy = 0; yy < ye[am]; ++yy)
        for (int xx = 0; xx < xe[am]; ++xx) {
          const int X = p.bx[am] + xx, Y = p.by[am] + yy, Z = p.bz[am] + zz;
          float ref = 0.f;
          if (X >= 0 && X < hx + (dimpad ? pad : 0) && Y >= 0 && Y < hy && Z >= 0 && Z < hz)
            ref = h[(size_t)am * n8 + (size_t)Z * hx * hy + (size_t)Y * hx + X];
          const float got = o[(zz * ye[am] + yy) * xe[am] + xx];
          if (got != ref && bad++ < 5) printf("am %d (%d,%d,%d): got %g want %g\n", am, X, Y, Z, got, ref);
        }
  }
  printf("pad %d negx %d dimpad %d: done, %d mismatches\n", pad, negx, dimpad, bad);
  return 0;
}
