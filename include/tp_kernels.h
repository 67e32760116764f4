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

#ifdef __cplusplus
}
#endif
#endif
