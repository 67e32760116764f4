// Microbenchmark: tcgen05.mma issue/execution rate per instruction shape (one CTA per SM, one
// warp issues `iters` MMAs back to back into TMEM, operands from shared memory). Prints cycles per
// MMA and the implied dense bf16 FLOP/clk/SM for M=128, N in {32, 64, 128, 256}, K=16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2102_07988_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "tc5.cuh"
using namespace tp::tc5;

__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}
// MODE 0: A, B K-major (smem); 1: A K-major, B MN-major; 2: both MN-major; 3: A from TMEM, B MN-major
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) kern(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint32_t a = smem_u32(smem), b = a + 16384;
    constexpr uint32_t id = idesc_bf16(128, N, MODE == 2, MODE >= 1);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = MODE == 2 ? make_desc(a + k * 2048, 8192, 1024) : make_desc(a + k * 32, 16, 1024);
        const uint64_t bd = MODE >= 1 ? make_desc(b + k * 2048, 8192, 1024) : make_desc(b + k * 32, 16, 1024);
        if (MODE == 3) mma_ts_w(tmem, tmem + 256 + k * 8, bd, id, 1);
        else mma_bf16_w(tmem, ad, bd, id, 1);
      }
    }
    mma_commit_w(&bar);
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, int MODE>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, 16);
  const int iters = 2000;
  cudaFuncSetAttribute(kern<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  kern<N, MODE><<<sms, 128, 65536>>>(iters, d);
  kern<N, MODE><<<sms, 128, 65536>>>(iters, d);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = 4.0 * iters;
  printf("mode %d M=128 N=%3d K=16: issue %.1f clk/mma, complete %.1f clk/mma -> %.0f FLOP/clk/SM (err %s)\n", MODE, N, h[0] / n,
         h[1] / n, 2.0 * 128 * N * 16 / (h[1] / n), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<32, 0>(sms); run<64, 0>(sms); run<128, 0>(sms); run<256, 0>(sms);
  run<64, 1>(sms); run<128, 1>(sms); run<64, 2>(sms); run<128, 2>(sms); run<64, 3>(sms); run<128, 3>(sms);
  return 0;
}
