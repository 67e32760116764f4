// attn_simt.cu — slice-vs-prefix causal attention, SIMT (fp32 FFMA) version.
//
// For one job (one sequence, slice rows [c, c+l)) and each head: query at absolute position c+r
// attends keys [0, c+r] of the per-layer prefix cache (Eq. 2; dependency
// property); scale 1/sqrt(d) (reading A-1).
// Backward pushes dK/dV contributions of this slice into the fp32 accumulators of ALL prefix rows
// [0, c+l) — rows of slice j are final once every slice i >= j has run (reverse slice order).
//
// Used for TP_FP32 mode (true fp32 maths, A-18) and as the independent cross-check of the
// tensor-core attention in bf16 mode (TP_FLAG_FORCE_SIMT). One warp per (row, head); lanes split
// the head dimension (d <= 128 -> <= 4 elements per lane).
#include "kernels.h"

namespace tp {

namespace {
constexpr int WARPS = 4;

template <typename T>
__device__ __forceinline__ void load_head_row(const T* p, int d, int lane, float (&v)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < d ? to_f<T>(p[e]) : 0.f;
  }
}
__device__ __forceinline__ float dot4(const float (&a)[4], const float (&b)[4]) {
  return warp_sum(a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3]);
}

template <typename T>
__global__ void __launch_bounds__(WARPS * 32) attn_fwd_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                              const T* __restrict__ v, T* __restrict__ o, int64_t ldo,
                                                              float* __restrict__ lse, int s, int d, int c, int l) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x * WARPS + w, head = blockIdx.y;
  if (r >= l) return;
  const float scale = rsqrtf((float)d);
  const int64_t hb = (int64_t)head * s * d;
  float qv[4], acc[4] = {0.f, 0.f, 0.f, 0.f};
  load_head_row(q + hb + (int64_t)(c + r) * d, d, lane, qv);
  float m = -INFINITY, den = 0.f;
  for (int j = 0; j <= c + r; ++j) {
    float kv[4], vv[4];
    load_head_row(k + hb + (int64_t)j * d, d, lane, kv);
    load_head_row(v + hb + (int64_t)j * d, d, lane, vv);
    const float sc = dot4(qv, kv) * scale;
    const float mn = fmaxf(m, sc);
    const float corr = __expf(m - mn), p = __expf(sc - mn);
    den = den * corr + p;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = acc[i] * corr + p * vv[i];
    m = mn;
  }
  const float inv = 1.f / den;
  T* orow = o + (int64_t)r * ldo + head * d;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = lane + 32 * i;
    if (e < d) orow[e] = from_f<T>(acc[i] * inv);
  }
  if (lane == 0) lse[(int64_t)head * s + c + r] = m + logf(den);
}

// dQ (one writer per query row) and Dvec = rowsum(dO * O).
template <typename T>
__global__ void __launch_bounds__(WARPS * 32) attn_bwd_dq_kernel(const T* __restrict__ dO, int64_t ld_do,
                                                                 const T* __restrict__ o, int64_t ldo,
                                                                 const T* __restrict__ q, const T* __restrict__ k,
                                                                 const T* __restrict__ v, const float* __restrict__ lse,
                                                                 float* __restrict__ Dvec, T* __restrict__ dq,
                                                                 int64_t ldq, int s, int d, int c, int l) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x * WARPS + w, head = blockIdx.y;
  if (r >= l) return;
  const float scale = rsqrtf((float)d);
  const int64_t hb = (int64_t)head * s * d;
  float qv[4], dov[4], ov[4], acc[4] = {0.f, 0.f, 0.f, 0.f};
  load_head_row(q + hb + (int64_t)(c + r) * d, d, lane, qv);
  load_head_row(dO + (int64_t)r * ld_do + head * d, d, lane, dov);
  load_head_row(o + (int64_t)r * ldo + head * d, d, lane, ov);
  const float D = dot4(dov, ov);
  const float L = lse[(int64_t)head * s + c + r];
  for (int j = 0; j <= c + r; ++j) {
    float kv[4], vv[4];
    load_head_row(k + hb + (int64_t)j * d, d, lane, kv);
    load_head_row(v + hb + (int64_t)j * d, d, lane, vv);
    const float p = __expf(dot4(qv, kv) * scale - L);
    const float ds = p * (dot4(dov, vv) - D);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += ds * kv[i];
  }
  T* drow = dq + (int64_t)r * ldq + head * d;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = lane + 32 * i;
    if (e < d) drow[e] = from_f<T>(acc[i] * scale);
  }
  if (lane == 0) Dvec[(int64_t)head * l + r] = D;
}

// dK/dV push: one warp per (prefix key row j in [0, c+l), head), exactly one writer per row.
template <typename T>
__global__ void __launch_bounds__(WARPS * 32) attn_bwd_dkv_kernel(const T* __restrict__ dO, int64_t ld_do,
                                                                  const T* __restrict__ q, const T* __restrict__ k,
                                                                  const T* __restrict__ v, const float* __restrict__ lse,
                                                                  const float* __restrict__ Dvec, float* __restrict__ dk_acc,
                                                                  float* __restrict__ dv_acc, int s, int d, int c, int l,
                                                                  int accumulate) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.x * WARPS + w, head = blockIdx.y;
  if (j >= c + l) return;
  const float scale = rsqrtf((float)d);
  const int64_t hb = (int64_t)head * s * d;
  float kv[4], vv[4], dk[4] = {0.f, 0.f, 0.f, 0.f}, dv[4] = {0.f, 0.f, 0.f, 0.f};
  load_head_row(k + hb + (int64_t)j * d, d, lane, kv);
  load_head_row(v + hb + (int64_t)j * d, d, lane, vv);
  for (int r = max(0, j - c); r < l; ++r) {  // queries c+r >= j
    float qv[4], dov[4];
    load_head_row(q + hb + (int64_t)(c + r) * d, d, lane, qv);
    load_head_row(dO + (int64_t)r * ld_do + head * d, d, lane, dov);
    const float p = __expf(dot4(qv, kv) * scale - lse[(int64_t)head * s + c + r]);
    const float ds = p * (dot4(dov, vv) - Dvec[(int64_t)head * l + r]);
#pragma unroll
    for (int i = 0; i < 4; ++i) { dv[i] += p * dov[i]; dk[i] += ds * qv[i]; }
  }
  float* dkr = dk_acc + hb + (int64_t)j * d;
  float* dvr = dv_acc + hb + (int64_t)j * d;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = lane + 32 * i;
    if (e < d) {
      if (accumulate) { dkr[e] += dk[i] * scale; dvr[e] += dv[i]; }
      else { dkr[e] = dk[i] * scale; dvr[e] = dv[i]; }
    }
  }
}

// dQKV[r][H + i] = dK_acc[head][c + r][e], dQKV[r][2H + i] = dV_acc[...] (i = head*d + e), 8-wide.
template <typename T>
__global__ void dkv_finalize_kernel(const float* __restrict__ dk_acc, const float* __restrict__ dv_acc,
                                    T* __restrict__ dqkv, int64_t ld, int a, int s, int d, int c,
                                    int64_t acc_sstride, int64_t out_sstride) {
  const int r = blockIdx.x;
  dk_acc += blockIdx.y * acc_sstride;
  dv_acc += blockIdx.y * acc_sstride;
  dqkv += blockIdx.y * out_sstride;
  const int H = a * d;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    const int head = i / d, e = i - head * d;
    const int64_t src = ((int64_t)head * s + c + r) * d + e;
    float v[8];
    load8<float>(dk_acc + src, v);
    store8<T>(dqkv + (int64_t)r * ld + H + i, v);
    load8<float>(dv_acc + src, v);
    store8<T>(dqkv + (int64_t)r * ld + 2 * H + i, v);
  }
}
}  // namespace

template <typename T>
cudaError_t attn_fwd_simt(const T* q, const T* k, const T* v, T* o, int64_t ldo, float* lse, int a, int s, int d,
                          int c, int l, cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  dim3 grid((l + WARPS - 1) / WARPS, a);
  attn_fwd_kernel<T><<<grid, WARPS * 32, 0, st>>>(q, k, v, o, ldo, lse, s, d, c, l);
  return cudaGetLastError();
}

template <typename T>
cudaError_t attn_bwd_simt(const T* dO, int64_t ld_do, const T* o, int64_t ldo, const T* q, const T* k, const T* v,
                          const float* lse, float* Dvec, T* dq, int64_t ldq, float* dk_acc, float* dv_acc, int a,
                          int s, int d, int c, int l, int accumulate, cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  dim3 g1((l + WARPS - 1) / WARPS, a);
  attn_bwd_dq_kernel<T><<<g1, WARPS * 32, 0, st>>>(dO, ld_do, o, ldo, q, k, v, lse, Dvec, dq, ldq, s, d, c, l);
  dim3 g2((c + l + WARPS - 1) / WARPS, a);
  attn_bwd_dkv_kernel<T><<<g2, WARPS * 32, 0, st>>>(dO, ld_do, q, k, v, lse, Dvec, dk_acc, dv_acc, s, d, c, l, accumulate);
  return cudaGetLastError();
}

template <typename T>
cudaError_t attn_dkv_finalize(const float* dk_acc, const float* dv_acc, T* dqkv, int64_t ld, int a, int s, int d,
                              int c, int l, cudaStream_t st, int nseq, int64_t acc_sstride, int64_t out_sstride) {
  if (l == 0 || nseq == 0) return cudaSuccess;
  dkv_finalize_kernel<T><<<dim3(l, nseq), 256, 0, st>>>(dk_acc, dv_acc, dqkv, ld, a, s, d, c, acc_sstride, out_sstride);
  return cudaGetLastError();
}

#define TP_INST(T)                                                                                              \
  template cudaError_t attn_fwd_simt<T>(const T*, const T*, const T*, T*, int64_t, float*, int, int, int, int, int, \
                                        cudaStream_t);                                                          \
  template cudaError_t attn_bwd_simt<T>(const T*, int64_t, const T*, int64_t, const T*, const T*, const T*,         \
                                        const float*, float*, T*, int64_t, float*, float*, int, int, int, int, int, int, \
                                        cudaStream_t);                                                          \
  template cudaError_t attn_dkv_finalize<T>(const float*, const float*, T*, int64_t, int, int, int, int, int,       \
                                            cudaStream_t, int, int64_t, int64_t);
TP_INST(float)
TP_INST(bf16)
#undef TP_INST

}  // namespace tp
