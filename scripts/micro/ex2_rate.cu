// Microbenchmark: MUFU exp2 throughput per SM for fp32 and packed half-precision forms
// (ex2.approx.f32, ex2.approx.f16x2, ex2.approx.ftz.bf16x2): one CTA per SM, 8 warps, independent
// chains of `iters` exp2 per thread. Prints element-exp2 per clock per SM. Modes 3-5: the attention
// softmax's per-element instruction mix (FFMA + MUFU.EX2 + FADD + FMNMX + F2FP bf16x2 pack), the
// F2FP pack alone, and the same mix with the pack done by PRMT (truncation) instead of F2FP.
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
  float mx0 = 0.f, mx1 = 0.f, rs0 = 0.f, rs1 = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (MODE == 1) {
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
    } else if (MODE == 2) {
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
    } else if (MODE == 3 || MODE == 5) {
      // two element pairs per iteration: x = a*, m = running max, rs = running sum, pk = packed P
      float p0, p1, p2, p3;
      asm volatile("fma.rn.ftz.f32 %0, %1, 0.0883883, -1.5;" : "=f"(p0) : "f"(a0));
      asm volatile("fma.rn.ftz.f32 %0, %1, 0.0883883, -1.5;" : "=f"(p1) : "f"(a1));
      asm volatile("fma.rn.ftz.f32 %0, %1, 0.0883883, -1.5;" : "=f"(p2) : "f"(a2));
      asm volatile("fma.rn.ftz.f32 %0, %1, 0.0883883, -1.5;" : "=f"(p3) : "f"(a3));
      asm volatile("max.ftz.f32 %0, %0, %1;" : "+f"(mx0) : "f"(a0)); asm volatile("max.ftz.f32 %0, %0, %1;" : "+f"(mx1) : "f"(a2));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(p0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(p1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(p2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(p3));
      rs0 += p0 + p1; rs1 += p2 + p3;
      uint32_t k0, k1;
      if (MODE == 3) {
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(k0) : "f"(p1), "f"(p0));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(k1) : "f"(p3), "f"(p2));
      } else {
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(k0) : "r"(__float_as_uint(p0)), "r"(__float_as_uint(p1)));
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(k1) : "r"(__float_as_uint(p2)), "r"(__float_as_uint(p3)));
      }
      h0 ^= k0; h1 ^= k1;
      a0 += 1e-7f; a1 += 1e-7f; a2 += 1e-7f; a3 += 1e-7f;
    } else {
      uint32_t k0, k1, k2, k3;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(k0) : "f"(a1), "f"(a0));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(k1) : "f"(a3), "f"(a2));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(k2) : "f"(a0), "f"(a3));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(k3) : "f"(a2), "f"(a1));
      h0 ^= k0; h1 ^= k1; h2 ^= k2; h3 ^= k3;
      a0 += 1e-7f; a1 += 1e-7f; a2 += 1e-7f; a3 += 1e-7f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  out[blockIdx.x * 256 + threadIdx.x] = a0 + a1 + a2 + a3 + (float)(h0 ^ h1 ^ h2 ^ h3) + mx0 + mx1 + rs0 + rs1;
}

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  const char* names[6] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2",
                          "softmax mix (F2FP pack)", "cvt.rn.bf16x2 alone", "softmax mix (PRMT pack)"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) kern<0><<<148, 256>>>(iters, out, clk);
      if (mode == 1) kern<1><<<148, 256>>>(iters, out, clk);
      if (mode == 2) kern<2><<<148, 256>>>(iters, out, clk);
      if (mode == 3) kern<3><<<148, 256>>>(iters, out, clk);
      if (mode == 4) kern<4><<<148, 256>>>(iters, out, clk);
      if (mode == 5) kern<5><<<148, 256>>>(iters, out, clk);
      cudaDeviceSynchronize();
    }
    long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    if (mode == 3) {  // the same mix with one warp per SM sub-partition (4 warps per CTA)
      for (int rep = 0; rep < 2; ++rep) { kern<3><<<148, 128>>>(iters, out, clk); cudaDeviceSynchronize(); }
      long long h1; cudaMemcpy(&h1, clk, 8, cudaMemcpyDeviceToHost);
      printf("%-26s %8.2f elements/clk/SM  (%lld clk)\n", "softmax mix, 1 warp/SMSP", 128.0 * iters * 4 / h1, h1);
    }
    const double elems = 256.0 * iters * 4 * (mode == 1 || mode == 2 || mode == 4 ? 2 : 1);
    printf("%-26s %8.2f elements/clk/SM  (%lld clk)\n", names[mode], elems / h, h);
  }
  return 0;
}
