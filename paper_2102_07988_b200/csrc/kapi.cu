// kapi.cu — include/tp_kernels.h: single-kernel entry points for unit tests and kernel benchmarks.
#include <cuda_runtime.h>

#include "common.h"
#include "kernels.h"
#include "tp_kernels.h"

using namespace tp;

namespace {
// grow-only device scratch (kernel-level entry points are test/benchmark plumbing; per-call
// cudaMallocAsync would put pool growth/trim inside the timed region)
float* scratch(int which, size_t n) {
  static float* buf[2] = {nullptr, nullptr};
  static size_t cap[2] = {0, 0};
  if (n > cap[which]) {
    if (buf[which]) cudaFree(buf[which]);
    buf[which] = nullptr;
    if (cudaMalloc(&buf[which], n * sizeof(float)) != cudaSuccess) { cap[which] = 0; return nullptr; }
    cap[which] = n;
  }
  return buf[which];
}
tp_status cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(TP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return TP_OK;
}
}  // namespace

extern "C" tp_status tpk_gemm(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_mn,
                              const void* B, int64_t ldb, int32_t b_mn, float* out, int64_t ldo, int32_t impl,
                              void* stream) {
  TP_CHECK_ARG(A && B && out && M >= 0 && N >= 0 && K >= 1, "tpk_gemm: bad arguments");
  TP_CHECK_ARG(N % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0 && ldo % 8 == 0, "tpk_gemm: N/lda/ldb/ldo must be multiples of 8");
  GemmDesc g;
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.a_mn = a_mn != 0; g.B = B; g.ldb = ldb; g.b_mn = b_mn != 0;
  Epi e;
  e.kind = EPI_STORE; e.out = out; e.ldo = ldo; e.out_f32 = 1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (impl == 0) {
    // fixed-size stream-K workspace of the kernel-level API (allocated once, never reallocated, so a
    // captured launch never sees a freed pointer); tickets start at zero and the last part resets them
    static float* ws = nullptr;
    static int* cnt = nullptr;
    if (!ws) {
      size_t nw = 0, nc = 0;
      gemm_sm100_workspace(&nw, &nc);
      if (cudaMalloc(&ws, nw * sizeof(float)) != cudaSuccess || cudaMalloc(&cnt, nc * sizeof(int)) != cudaSuccess ||
          cudaMemset(cnt, 0, nc * sizeof(int)) != cudaSuccess)
        return fail(TP_ENOMEM, "tpk_gemm: stream-K workspace");
    }
    g.sk_ws = ws;
    g.sk_cnt = cnt;
    if (!gemm_sm100_supported(g)) return fail(TP_EINVAL, "tpk_gemm: shape/alignment not supported by the sm100 kernel");
    return cu(gemm_sm100(g, e, st), "gemm_sm100");
  }
  return cu(gemm_simt<bf16>(g, e, st), "gemm_simt");
}

extern "C" tp_status tpk_attention_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int32_t a,
                                       int32_t s, int32_t d, int32_t c, int32_t l, int32_t impl, void* stream) {
  TP_CHECK_ARG(q && k && v && o && lse, "tpk_attention_fwd: null pointer");
  TP_CHECK_ARG(a >= 1 && d % 16 == 0 && d <= 128 && c >= 0 && l >= 0 && c + l <= s, "tpk_attention_fwd: bad shape");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bf16 *Q = (const bf16*)q, *Kp = (const bf16*)k, *Vp = (const bf16*)v;
  if (impl == 0 && attn_sm100_supported(d))
    return cu(attn_fwd_sm100(Q, Kp, Vp, (bf16*)o, (int64_t)a * d, lse, a, s, d, c, l, st), "attn_fwd_sm100");
  if (impl == 0 || impl == 2) return cu(attn_fwd_tc(Q, Kp, Vp, (bf16*)o, (int64_t)a * d, lse, a, s, d, c, l, st), "attn_fwd_tc");
  return cu(attn_fwd_simt<bf16>(Q, Kp, Vp, (bf16*)o, (int64_t)a * d, lse, a, s, d, c, l, st), "attn_fwd_simt");
}

extern "C" tp_status tpk_attention_bwd(const void* dO, const void* o, const void* q, const void* k, const void* v,
                                       const float* lse, void* dq, int64_t ldq, float* dk_acc, float* dv_acc, int32_t a,
                                       int32_t s, int32_t d, int32_t c, int32_t l, int32_t accumulate, int32_t impl,
                                       void* stream) {
  TP_CHECK_ARG(dO && o && q && k && v && lse && dq && dk_acc && dv_acc, "tpk_attention_bwd: null pointer");
  TP_CHECK_ARG(a >= 1 && d % 16 == 0 && d <= 128 && c >= 0 && l >= 1 && c + l <= s, "tpk_attention_bwd: bad shape");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  float* Dvec = scratch(0, (size_t)2 * a * (l + 64));
  if (!Dvec) return fail(TP_ENOMEM, "tpk_attention_bwd: scratch");
  tp_status r = TP_OK;
  const int64_t H = (int64_t)a * d;
  if (impl == 0 && attn_sm100_supported(d)) {
    float* dq_acc = scratch(1, (size_t)H * l);
    if (!dq_acc) return fail(TP_ENOMEM, "tpk_attention_bwd: scratch");
    r = cu(attn_bwd_sm100((const bf16*)dO, H, (const bf16*)o, H, (const bf16*)q, (const bf16*)k, (const bf16*)v, lse, Dvec,
                          dq_acc, (bf16*)dq, ldq, dk_acc, dv_acc, a, s, d, c, l, accumulate, st), "attn_bwd_sm100");
  } else if (impl == 0 || impl == 2)
    r = cu(attn_bwd_tc((const bf16*)dO, H, (const bf16*)o, H, (const bf16*)q, (const bf16*)k, (const bf16*)v, lse, Dvec,
                       (bf16*)dq, ldq, dk_acc, dv_acc, a, s, d, c, l, accumulate, st), "attn_bwd_tc");
  else
    r = cu(attn_bwd_simt<bf16>((const bf16*)dO, H, (const bf16*)o, H, (const bf16*)q, (const bf16*)k, (const bf16*)v,
                               lse, Dvec, (bf16*)dq, ldq, dk_acc, dv_acc, a, s, d, c, l, accumulate, st),
           "attn_bwd_simt");
  return r;
}

extern "C" tp_status tpk_layernorm_fwd(const float* x, const float* gamma, const float* beta, void* y, float* mean,
                                       float* rstd, int32_t rows, int32_t H, void* stream) {
  TP_CHECK_ARG(x && gamma && beta && y && mean && rstd, "tpk_layernorm_fwd: null pointer");
  TP_CHECK_ARG(rows >= 0 && H >= 8 && H % 8 == 0 && H <= 12288, "tpk_layernorm_fwd: bad shape");
  return cu(layernorm_fwd<bf16>(x, gamma, beta, (bf16*)y, mean, rstd, rows, H, reinterpret_cast<cudaStream_t>(stream)),
            "layernorm_fwd");
}

extern "C" tp_status tpk_layernorm_bwd(const void* dy, const float* x, const float* mean, const float* rstd,
                                       const float* gamma, const float* resid, float* dx_out, void* dx_copy,
                                       float* dgamma, float* dbeta, float* dbias, int32_t rows, int32_t H,
                                       void* stream) {
  TP_CHECK_ARG(dy && x && mean && rstd && gamma && dx_out && dgamma && dbeta, "tpk_layernorm_bwd: null pointer");
  TP_CHECK_ARG(rows >= 0 && H >= 8 && H % 8 == 0 && H <= 12288, "tpk_layernorm_bwd: bad shape");
  return cu(layernorm_bwd<bf16>((const bf16*)dy, x, mean, rstd, gamma, resid, dx_out, (bf16*)dx_copy, dgamma, dbeta,
                                nullptr, rows, H, reinterpret_cast<cudaStream_t>(stream), dbias),
            "layernorm_bwd");
}
