/*
 * tp_kernels.h — kernel-level entry points of libtp.so, for unit tests and per-kernel benchmarks.
 * They run ONE hot-path kernel on caller-owned DEVICE buffers, asynchronously on `stream`
 * (a cudaStream_t; NULL = legacy default stream). Same status/error conventions as tp.h.
 *
 * tpk_gemm: acc[m][n] = sum_k A(m,k) B(n,k) with bf16 operands and fp32 accumulation
 * (the projections of PAPER.md:174-178), out[m*ldo + n] = acc (fp32).
 *   A(m,k) = A[m*lda + k] if a_mn == 0 (K-major), else A[k*lda + m] (MN-major); same for B(n,k).
 *   impl: 0 = tcgen05/TMEM/TMA kernel (sm_100a), 1 = SIMT kernel. N, lda, ldb multiples of 8.
 *
 * tpk_attention_fwd / _bwd: slice-vs-prefix causal attention of one sequence (Eq. 2,
 * PAPER.md:174-177): queries are rows [c, c+l) of q[a][s][d], keys/values rows [0, c+l) of
 * k/v[a][s][d] (bf16); o[l][a*d] bf16 token-major, lse[a][s] fp32 (rows c..c+l written).
 * Backward: dO[l][a*d]; writes dq[l][a*d] (bf16, ld = ldq) and adds (accumulate=1) or writes
 * (accumulate=0) dK/dV of key rows [0, c+l) into dk_acc/dv_acc[a][s][d] fp32.
 *   impl: 0 = tensor-core kernel, 1 = SIMT kernel.
 *
 * tpk_layernorm_fwd / _bwd: the pre-LN LayerNorm of the block ("LayerNorm";
 * DESIGN.md reading A-3: fp32 statistics, eps = 1e-5) over `rows` rows of H (H % 8 == 0,
 * H <= 12288) fp32 values, all buffers row-major with ld = H, device pointers 16-byte aligned.
 * Forward: y = (x - mean) * rstd * gamma + beta as bf16, mean[r] / rstd[r] fp32.
 * Backward (dy bf16, mean / rstd from the forward): dx_out = resid + dLN/dx (fp32; resid may be
 * NULL = 0), dx_copy (bf16, may be NULL) = the same values; dgamma, dbeta and (if non-NULL) dbias
 * = column sums of dx_out are ADDED to the caller's fp32 [H] accumulators. `impl` is ignored
 * (one CUDA implementation, chosen by H; TP_LN_BULK=0 selects the register-prefetch variant).
 */
#ifndef TP_KERNELS_H_
#define TP_KERNELS_H_
#include <stdint.h>

#include "tp.h"

#ifdef __cplusplus
extern "C" {
#endif

tp_status tpk_gemm(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_mn, const void* B,
                   int64_t ldb, int32_t b_mn, float* out, int64_t ldo, int32_t impl, void* stream);

tp_status tpk_attention_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int32_t a, int32_t s,
                            int32_t d, int32_t c, int32_t l, int32_t impl, void* stream);

tp_status tpk_attention_bwd(const void* dO, const void* o, const void* q, const void* k, const void* v,
                            const float* lse, void* dq, int64_t ldq, float* dk_acc, float* dv_acc, int32_t a,
                            int32_t s, int32_t d, int32_t c, int32_t l, int32_t accumulate, int32_t impl,
                            void* stream);

tp_status tpk_layernorm_fwd(const float* x, const float* gamma, const float* beta, void* y, float* mean,
                            float* rstd, int32_t rows, int32_t H, void* stream);

tp_status tpk_layernorm_bwd(const void* dy, const float* x, const float* mean, const float* rstd, const float* gamma,
                            const float* resid, float* dx_out, void* dx_copy, float* dgamma, float* dbeta,
                            float* dbias, int32_t rows, int32_t H, void* stream);

#ifdef __cplusplus
}
#endif
#endif
