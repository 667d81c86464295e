// Does a line read by SMs of both dies come from DRAM once or twice?
// Every CTA (one per SM) reads the same BYTES-sized buffer; run under
//   ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct ./tools/l2_dup
// and compare dram__bytes_read with the buffer size (1x: one L2 for the chip,
// 2x: each die's L2 fetches its own copy).  Also records the smid of every CTA
// and the per-CTA time of a second pass (L2-resident).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/l2_dup tools/l2_dup.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_read(const float4* __restrict__ v, int64_t n4, float* out, unsigned* smid, long long* cyc) {
  float acc = 0.f;
  long long t0 = clock64();
  // every CTA walks the whole buffer, starting at a CTA-dependent offset
  const int64_t start = (int64_t)blockIdx.x * (n4 / gridDim.x);
  for (int64_t k = threadIdx.x; k < n4; k += blockDim.x) {
    int64_t i = start + k;
    if (i >= n4) i -= n4;
    const float4 x = __ldcg(v + i);
    acc += x.x + x.y + x.z + x.w;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    unsigned s;
    asm("mov.u32 %0, %%smid;" : "=r"(s));
    smid[blockIdx.x] = s;
    cyc[blockIdx.x] = t1 - t0;
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const int64_t bytes = 32ll << 20;
  const int64_t n4 = bytes / 16;
  float4* v;
  float* out;
  unsigned* smid;
  long long* cyc;
  cudaMalloc(&v, bytes);
  cudaMemset(v, 0, bytes);
  cudaMalloc(&out, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&smid, sms * 4);
  cudaMalloc(&cyc, sms * 8);
  // pass 1 (cold) and pass 2 (warm)
  for (int p = 0; p < 2; ++p) {
    k_read<<<sms, 1024>>>(v, n4, out, smid, cyc);
    cudaDeviceSynchronize();
  }
  unsigned hs[256];
  long long hc[256];
  cudaMemcpy(hs, smid, sms * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, cyc, sms * 8, cudaMemcpyDeviceToHost);
  printf("buffer %lld MB, %d CTAs\n", (long long)(bytes >> 20), sms);
  for (int b = 0; b < sms; ++b) printf("cta %d smid %u cycles %lld\n", b, hs[b], hc[b]);
  return 0;
}
