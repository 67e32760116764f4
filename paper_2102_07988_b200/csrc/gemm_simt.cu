// gemm_simt.cu — SIMT FFMA GEMM with the fused epilogues of epilogue.cuh.
//
// Used (a) for TP_FP32 mode, where operands are true fp32 (tcgen05 has no fp32 kind and TF32
// cannot meet the 1e-4 bar, A-18), and (b) in TP_BF16 mode under TP_FLAG_FORCE_SIMT as
// an independent cross-check of the tcgen05 GEMM. Not a hot path in bf16 mode.
//
//   acc[m][n] = sum_k A(m, k) * B(n, k)
//   A(m, k) = A[m*lda + k] (K-major)  or  A[k*lda + m] (MN-major, A_MN)
//   B(n, k) = B[n*ldb + k] (K-major)  or  B[k*ldb + n] (MN-major, B_MN)
#include "epilogue.cuh"
#include "kernels.h"

namespace tp {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <typename T, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, const T* __restrict__ A,
                                                        int64_t lda, const T* __restrict__ B,
                                                        int64_t ldb, Epi epi) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = tid % 8, ty = tid / 8;  // cols tx*8..+7, rows ty*2..+1
  float acc[2][8] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int idx = tid + r * 256;  // 0..1023 over a 64x16 tile
      int mm, kk;
      if (A_MN) { mm = idx % BM; kk = idx / BM; } else { kk = idx % BK; mm = idx / BK; }
      const int gm = m0 + mm, gk = k0 + kk;
      float a = 0.f;
      if (gm < M && gk < K) a = to_f<T>(A_MN ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk]);
      As[kk][mm] = a;
      int nn;
      if (B_MN) { nn = idx % BN; kk = idx / BN; } else { kk = idx % BK; nn = idx / BK; }
      const int gn = n0 + nn;
      const int gk2 = k0 + kk;
      float b = 0.f;
      if (gn < N && gk2 < K) b = to_f<T>(B_MN ? B[(int64_t)gk2 * ldb + gn] : B[(int64_t)gn * ldb + gk2]);
      Bs[kk][nn] = b;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float a0 = As[kk][ty * 2], a1 = As[kk][ty * 2 + 1];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float b = Bs[kk][tx * 8 + j];
        acc[0][j] = fmaf(a0, b, acc[0][j]);
        acc[1][j] = fmaf(a1, b, acc[1][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int m = m0 + ty * 2 + i, n = n0 + tx * 8;
    if (m < M && n < N) epi_apply8<T>(epi, m, n, acc[i]);
  }
}
}  // namespace

template <typename T>
cudaError_t gemm_simt(const GemmDesc& g, const Epi& epi, cudaStream_t st) {
  if (g.M == 0 || g.N == 0) return cudaSuccess;
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM);
  const T* A = reinterpret_cast<const T*>(g.A);
  const T* B = reinterpret_cast<const T*>(g.B);
  if (!g.a_mn && !g.b_mn) gemm_simt_kernel<T, false, false><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, epi);
  else if (g.a_mn && !g.b_mn) gemm_simt_kernel<T, true, false><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, epi);
  else if (!g.a_mn && g.b_mn) gemm_simt_kernel<T, false, true><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, epi);
  else gemm_simt_kernel<T, true, true><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, epi);
  return cudaGetLastError();
}

template cudaError_t gemm_simt<float>(const GemmDesc&, const Epi&, cudaStream_t);
template cudaError_t gemm_simt<bf16>(const GemmDesc&, const Epi&, cudaStream_t);

}  // namespace tp
