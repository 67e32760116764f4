// Microbenchmark: MUFU exp2 throughput per SM for fp32 and packed half-precision forms
// (ex2.approx.f32, ex2.approx.f16x2, ex2.approx.ftz.bf16x2): one CTA per SM, 8 warps, independent
// chains of `iters` exp2 per thread. Prints element-exp2 per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ex2_rate.cu -o ex2_rate
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256, 1) kern(int iters, float* out, long long* clk) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  uint32_t h0 = 0x3c003c00u + threadIdx.x, h1 = h0 + 7, h2 = h0 + 13, h3 = h0 + 17;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (MODE == 1) {
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
    } else {
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 256 + threadIdx.x] = a0 + a1 + a2 + a3 + (float)(h0 ^ h1 ^ h2 ^ h3);
}

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  const char* names[3] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) kern<0><<<148, 256>>>(iters, out, clk);
      if (mode == 1) kern<1><<<148, 256>>>(iters, out, clk);
      if (mode == 2) kern<2><<<148, 256>>>(iters, out, clk);
      cudaDeviceSynchronize();
    }
    long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    const double elems = 256.0 * iters * 4 * (mode == 0 ? 1 : 2);
    printf("%-24s %8.2f element-exp2/clk/SM  (%lld clk)\n", names[mode], elems / h, h);
  }
  return 0;
}
