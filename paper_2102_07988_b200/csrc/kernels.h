// kernels.h — host launchers of every device kernel of the hot path (all asynchronous on `st`).
// Layout conventions:
//   token-major activations  X[t][C]  (row t = position c + r of the job's slice), ld = C
//   per-sequence head-major  Q/K/V[a][s][d]   (the per-layer prefix cache, appended per slice)
//   fp32 dK/dV accumulators  [a][s][d]
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dtypes.cuh"
#include "epilogue.cuh"

namespace tp {

struct GemmDesc {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr;
  int64_t lda = 0;
  bool a_mn = false;  // false: A[m*lda + k];  true: A[k*lda + m]
  const void* B = nullptr;
  int64_t ldb = 0;
  bool b_mn = false;  // false: B[n*ldb + k];  true: B[k*ldb + n]
  bool persistent = true;  // false: one tile per CTA (lets higher-priority streams interleave)
  // stream-K workspace of the caller (gemm_sm100_workspace sizes): fp32 partial tiles + per-tile
  // tickets (zero between launches). Null: no stream-K split. One GEMM at a time may use a workspace.
  float* sk_ws = nullptr;
  int* sk_cnt = nullptr;
};

template <typename T> cudaError_t gemm_simt(const GemmDesc& g, const Epi& e, cudaStream_t st);
// tcgen05 / TMEM / TMA GEMM for sm_100a, bf16 operands, fp32 accumulation (gemm_sm100.cu).
cudaError_t gemm_sm100(const GemmDesc& g, const Epi& e, cudaStream_t st);
bool gemm_sm100_supported(const GemmDesc& g);
// Fixed stream-K workspace size that covers every launch on this device: one 128 x 512 fp32 partial
// slot per CTA of a persistent grid (floats), plus one int flag per CTA.
void gemm_sm100_workspace(size_t* ws_floats, size_t* cnt_ints);
// false when the driver's cuTensorMapEncodeTiled entry point is unavailable (no TMA descriptors)
bool tensor_maps_available();

template <typename T>
cudaError_t layernorm_fwd(const float* x, const float* gam, const float* bet, T* y, float* mean,
                          float* rstd, int rows, int H, cudaStream_t st);
template <typename T>
cudaError_t layernorm_bwd(const T* dy /* compute precision: bf16 in bf16 mode */, const float* x, const float* mean,
                          const float* rstd,
                          const float* gam, const float* resid, float* dx_out, T* dx_copy,
                          float* dgam, float* dbet, float* ws /* unused */, int rows, int H, cudaStream_t st,
                          float* dbias = nullptr /* += column sums of dx_out (the upstream bias gradient) */);

// Job rows m = 0..b*l-1 map to (sequence j = m % b, position p = c + m / b); tok points at the job's
// first sequence row of tokens[B][s+1].
cudaError_t embed_fwd(const int32_t* tok, const float* wte, const float* wpe, float* h, int c, int l, int b,
                      int s, int H, int V, cudaStream_t st);
cudaError_t embed_bwd(const int32_t* tok, const float* dh, float* gwte, float* gwpe, int c, int l, int b,
                      int s, int H, int V, cudaStream_t st);
// *bad = number of token ids outside [0, V) among tok[0..n) (device-side check of device tokens)
cudaError_t count_bad_tokens(const int32_t* tok, int64_t n, int V, int* bad, cudaStream_t st);

template <typename T>
cudaError_t ce_fwd_bwd(T* logits_inout, const int32_t* tok, int c, int b, int s, float* loss_rows,
                       float* logits_copy, int rows, int V, float scale, cudaStream_t st);
cudaError_t sum_rows(const float* x, int n, float* out, cudaStream_t st);

template <typename T>
cudaError_t attn_fwd_simt(const T* q, const T* k, const T* v, T* o, int64_t ldo, float* lse, int a,
                          int s, int d, int c, int l, cudaStream_t st);
template <typename T>
cudaError_t attn_bwd_simt(const T* dO, int64_t ld_do, const T* o, int64_t ldo, const T* q, const T* k,
                          const T* v, const float* lse, float* Dvec, T* dq, int64_t ldq, float* dk_acc,
                          float* dv_acc, int a, int s, int d, int c, int l, int accumulate, cudaStream_t st);
// Tensor-core (bf16) slice-vs-prefix attention (attn_tc.cu); same contract as the SIMT versions.
cudaError_t attn_fwd_tc(const bf16* q, const bf16* k, const bf16* v, bf16* o, int64_t ldo, float* lse, int a, int s,
                        int d, int c, int l, cudaStream_t st);
cudaError_t attn_bwd_tc(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, const bf16* q, const bf16* k,
                        const bf16* v, const float* lse, float* Dvec, bf16* dq, int64_t ldq, float* dk_acc,
                        float* dv_acc, int a, int s, int d, int c, int l, int accumulate, cudaStream_t st);
// tcgen05/TMEM attention (attn_sm100.cu), head_dim 128 only.
bool attn_sm100_supported(int d);
// nseq sequences per launch (grid.z): sequence j uses q/k/v + j*qkv_sstride, o + j*o_sstride (row r at
// + r*ldo), lse + j*lse_sstride.
cudaError_t attn_fwd_sm100(const bf16* q, const bf16* k, const bf16* v, bf16* o, int64_t ldo, float* lse, int a, int s,
                           int d, int c, int l, cudaStream_t st, int nseq = 1, int64_t qkv_sstride = 0,
                           int64_t o_sstride = 0, int64_t lse_sstride = 0);
// D[head][r] = rowsum(dO * O) per head (attn_tc.cu)
cudaError_t attn_bwd_prep(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, float* Dvec, int a, int d, int l,
                          cudaStream_t st, int nseq = 1, int64_t o_sstride = 0);
// dq_acc: fp32 scratch [l][a*d] per sequence (zeroed inside); dq: bf16 output rows (ld ldq);
// Dvec: fp32 scratch of at least nseq * a * 128 * ceil(l/64) floats (per-tile lse / D staging)
cudaError_t attn_bwd_sm100(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, const bf16* q, const bf16* k,
                           const bf16* v, const float* lse, float* Dvec, float* dq_acc, bf16* dq, int64_t ldq,
                           float* dk_acc, float* dv_acc, int a, int s, int d, int c, int l, int accumulate,
                           cudaStream_t st, int nseq = 1, int64_t qkv_sstride = 0, int64_t o_sstride = 0,
                           int64_t lse_sstride = 0, int64_t dq_sstride = 0, int64_t dkv_sstride = 0,
                           int finalize_dkv = 0 /* 1: also write the slice rows' final dK / dV (bf16) into
                                                   dq's columns [H, 3H) (row r of the slice: dq + r*ldq),
                                                   replacing attn_dkv_finalize; their fp32 accumulator
                                                   rows are then not maintained */);
template <typename T>
cudaError_t attn_dkv_finalize(const float* dk_acc, const float* dv_acc, T* dqkv, int64_t ld, int a,
                              int s, int d, int c, int l, cudaStream_t st, int nseq = 1, int64_t acc_sstride = 0,
                              int64_t out_sstride = 0);

// device-initiated p2p (p2p.cu): peer address of an NCCL symmetric window (host readback), the step
// epoch counter, and the release-store signal / acquire-spin wait on per-job flag slots
cudaError_t p2p_peer_pointer(void* window, int peer, void** host_out, cudaStream_t st);
cudaError_t p2p_epoch_inc(unsigned long long* epoch, cudaStream_t st);
cudaError_t p2p_signal(unsigned long long* remote_slot, const unsigned long long* epoch, cudaStream_t st);
cudaError_t p2p_wait(const unsigned long long* local_slot, const unsigned long long* epoch, cudaStream_t st);

template <typename T> cudaError_t convert_f32(const float* src, T* dst, int64_t n, cudaStream_t st);
template <typename T>
cudaError_t transpose_convert(const float* src, T* dst, int R, int C, cudaStream_t st);
template <typename T>
cudaError_t colsum_accum(const T* src, int64_t ld, float* out, int rows, int N, cudaStream_t st);

}  // namespace tp
