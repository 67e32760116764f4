// epilogue.cuh — fused GEMM epilogues shared by the tcgen05 GEMM (gemm_sm100.cu) and the SIMT
// GEMM (gemm_simt.cu). A GEMM computes acc[m][n] = sum_k A[m][k] B[n][k] in fp32; the epilogue
// turns a run of NV consecutive columns of one row into the layer's output:
//   EPI_STORE : out[m][n] = acc + bias[n]                        (out: T or fp32)
//   EPI_RESID : out[m][n] = resid[m][n] + acc + bias[n]          (fp32 residual stream, A-23)
//   EPI_GELU  : U = acc + bias;  out = U (T);  out2 = gelu(U) (T)     (Eq. 3; A-2)
//   EPI_DGELU : out[m][n] = acc * gelu'(aux[m][n])               (dU from dG and stored U)
//   EPI_QKV   : v = acc + bias; column n -> (part = n / H, head = (n % H) / d, e = n % d);
//               part 0 -> q, 1 -> k, 2 -> v, each [seq][a][s][d] at (m % bs, row0 + m / bs): the slice's
//               queries and its K/V appended to the per-layer prefix cache
//   EPI_ACCUM : out[m][n] += acc                                (fp32 weight-gradient accumulate)
#pragma once
#include "dtypes.cuh"

namespace tp {

enum EpiKind : int { EPI_STORE = 0, EPI_RESID = 1, EPI_GELU = 2, EPI_DGELU = 3, EPI_QKV = 4, EPI_ACCUM = 5 };

struct Epi {
  int kind = EPI_STORE;
  const float* bias = nullptr;
  void* out = nullptr;        // STORE/RESID/GELU(U)/DGELU/ACCUM
  int64_t ldo = 0;
  int out_f32 = 0;            // STORE: 1 -> fp32 output, 0 -> T output
  const float* resid = nullptr;
  int64_t ldr = 0;
  void* out2 = nullptr;       // GELU: G
  int64_t ldo2 = 0;
  const void* aux = nullptr;  // DGELU: U
  int64_t ld_aux = 0;
  void* q = nullptr;          // QKV scatter targets, [a][s][d] of the current sequence
  void* k = nullptr;
  void* v = nullptr;
  int s_len = 0, head_dim = 0, hidden = 0, row0 = 0;
  int bs = 1;                 // QKV: rows m -> (sequence m % bs, position row0 + m / bs); sequences s_len*hidden apart
  int n_off = 0;              // column offset of this GEMM in the epilogue's column space (N-split launches)
  float* dbias = nullptr;     // DGELU (tcgen05 GEMM): += column sums of the output (the bias gradient of
                              // the layer whose dY this is), one 16-byte L2 reduction per warp and 8 columns
};

// tanh: exact libm form in fp32 mode; the MUFU tanh.approx (rel. err ~2^-11, below the bf16 output
// rounding of 2^-9) in bf16 mode, where the GeLU epilogue would otherwise pace the GEMM.
template <typename T> __device__ __forceinline__ float tanh_t(float x) { return tanhf(x); }
template <> __device__ __forceinline__ float tanh_t<bf16>(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <typename T>
__device__ __forceinline__ float gelu_f(float u) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * u * (1.f + tanh_t<T>(c * (u + 0.044715f * u * u * u)));
}
template <typename T>
__device__ __forceinline__ float gelu_grad_f(float u) {
  const float c = 0.7978845608028654f;
  const float t = tanh_t<T>(c * (u + 0.044715f * u * u * u));
  return 0.5f * (1.f + t) + 0.5f * u * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * u * u);
}

// The per-element input an epilogue reads besides the accumulator (RESID: the fp32 residual row,
// DGELU: the stored U), fetched ahead of time so its latency overlaps other work.
template <typename T>
__device__ __forceinline__ void epi_prefetch8(const Epi& e, int m, int n0, float (&aux)[8]) {
  if (e.kind == EPI_RESID) load8<float>(e.resid + (int64_t)m * e.ldr + n0, aux);
  else if (e.kind == EPI_DGELU) load8<T>(reinterpret_cast<const T*>(e.aux) + (int64_t)m * e.ld_aux + n0, aux);
}

// Applies the epilogue to columns [n0, n0+8) of row m; n0 % 8 == 0, caller guarantees m < M and
// n0 + 8 <= N. `aux` holds epi_prefetch8's result for the same (m, n0).
template <typename T>
__device__ __forceinline__ void epi_apply8(const Epi& e, int m, int n0, float (&v)[8], const float (&aux)[8]) {
  if (e.kind != EPI_DGELU && e.kind != EPI_ACCUM && e.bias) {
    float b[8];
    load8<float>(e.bias + n0, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += b[i];
  }
  switch (e.kind) {
    case EPI_STORE:
      if (e.out_f32) store8<float>(reinterpret_cast<float*>(e.out) + (int64_t)m * e.ldo + n0, v);
      else store8<T>(reinterpret_cast<T*>(e.out) + (int64_t)m * e.ldo + n0, v);
      break;
    case EPI_RESID: {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] += aux[i];
      store8<float>(reinterpret_cast<float*>(e.out) + (int64_t)m * e.ldo + n0, v);
      break;
    }
    case EPI_GELU: {
      // U is rounded to T first so that G = gelu(U) and gelu'(U) in backward see the same U.
      float u[8], g[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) u[i] = to_f<T>(from_f<T>(v[i]));
#pragma unroll
      for (int i = 0; i < 8; ++i) g[i] = gelu_f<T>(u[i]);
      store8<T>(reinterpret_cast<T*>(e.out) + (int64_t)m * e.ldo + n0, u);
      store8<T>(reinterpret_cast<T*>(e.out2) + (int64_t)m * e.ldo2 + n0, g);
      break;
    }
    case EPI_DGELU: {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_f<T>(aux[i]);
      store8<T>(reinterpret_cast<T*>(e.out) + (int64_t)m * e.ldo + n0, v);
      break;
    }
    case EPI_QKV: {
      const int part = n0 / e.hidden;
      const int within = n0 - part * e.hidden;
      const int head = within / e.head_dim;
      const int dd = within - head * e.head_dim;
      T* base = reinterpret_cast<T*>(part == 0 ? e.q : (part == 1 ? e.k : e.v));
      const int sq = m % e.bs, pos = e.row0 + m / e.bs;
      store8<T>(base + (int64_t)sq * e.s_len * e.hidden + ((int64_t)head * e.s_len + pos) * e.head_dim + dd, v);
      break;
    }
    case EPI_ACCUM: {
      float* o = reinterpret_cast<float*>(e.out) + (int64_t)m * e.ldo + n0;
      float r[8];
      load8<float>(o, r);
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] += v[i];
      store8<float>(o, r);
      break;
    }
  }
}

template <typename T>
__device__ __forceinline__ void epi_apply8(const Epi& e, int m, int n0, float (&v)[8]) {
  float aux[8];
  epi_prefetch8<T>(e, m, n0, aux);
  epi_apply8<T>(e, m, n0, v, aux);
}

}  // namespace tp
