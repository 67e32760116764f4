// kernels_elem.cu — the HBM-bound kernels of the hot path: LayerNorm fwd/bwd (reading A-3),
// embedding gather/scatter (A-7), fused cross-entropy fwd+bwd (Eq. 1, A-9),
// dtype conversion/transposition of parameters, bias-gradient column sums, loss reduction.
// All use 16-byte vector accesses where the row length allows (H % 8 == 0 is guaranteed).
#include "kernels.h"

namespace tp {

namespace {

// ---------------------------------------------------------------- LayerNorm
// one CTA per row; the row is staged in shared memory (H <= 16384 -> 64 KB).
template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gam,
                                                     const float* __restrict__ bet, T* __restrict__ y,
                                                     float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                     int H) {
  extern __shared__ float row[];
  __shared__ float red[8];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float* xr = x + (int64_t)r * H;
  float s = 0.f;
  for (int i = tid * 4; i < H; i += 1024) {
    float4 v = *reinterpret_cast<const float4*>(xr + i);
    *reinterpret_cast<float4*>(row + i) = v;
    s += (v.x + v.y) + (v.z + v.w);
  }
  s = warp_sum(s);
  if (lane == 0) red[wid] = s;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float mean = tot / H;
  __syncthreads();
  float q = 0.f;
  for (int i = tid; i < H; i += 256) { const float d = row[i] - mean; q += d * d; }
  q = warp_sum(q);
  if (lane == 0) red[wid] = q;
  __syncthreads();
  float var = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) var += red[w];
  var /= H;
  const float rstd = rsqrtf(var + 1e-5f);
  if (tid == 0) { mean_out[r] = mean; rstd_out[r] = rstd; }
  T* yr = y + (int64_t)r * H;
  for (int i = tid * 8; i < H; i += 2048) {
    float v[8], g[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = row[i + j];
    load8<float>(gam + i, g);
    load8<float>(bet + i, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (v[j] - mean) * rstd * g[j] + b[j];
    store8<T>(yr + i, v);
  }
}

// dx = resid + rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)),  dxhat = dy * gamma;
// dgamma += dy * xhat, dbeta += dy (fp32 atomics).
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                                     const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                                                     const float* __restrict__ gam, const float* __restrict__ resid,
                                                     float* __restrict__ dx_out, T* __restrict__ dx_copy,
                                                     float* __restrict__ dgam, float* __restrict__ dbet, int H) {
  __shared__ float red[2][8];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float mean = mean_in[r], rstd = rstd_in[r];
  const float* dyr = dy + (int64_t)r * H;
  const float* xr = x + (int64_t)r * H;
  float s1 = 0.f, s2 = 0.f;
  for (int i = tid; i < H; i += 256) {
    const float xh = (xr[i] - mean) * rstd;
    const float dxh = dyr[i] * gam[i];
    s1 += dxh;
    s2 += dxh * xh;
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) { red[0][wid] = s1; red[1][wid] = s2; }
  __syncthreads();
  float m1 = 0.f, m2 = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) { m1 += red[0][w]; m2 += red[1][w]; }
  m1 /= H;
  m2 /= H;
  for (int i = tid; i < H; i += 256) {
    const float xh = (xr[i] - mean) * rstd;
    const float d = dyr[i];
    float dx = rstd * (d * gam[i] - m1 - xh * m2);
    if (resid) dx += resid[(int64_t)r * H + i];
    dx_out[(int64_t)r * H + i] = dx;
    if (dx_copy) dx_copy[(int64_t)r * H + i] = from_f<T>(dx);
    atomicAdd(dgam + i, d * xh);
    atomicAdd(dbet + i, d);
  }
}

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ wte,
                                 const float* __restrict__ wpe, float* __restrict__ h, int c, int H, int V) {
  const int r = blockIdx.x;
  int id = tok[c + r];
  id = min(max(id, 0), V - 1);
  const float* e = wte + (int64_t)id * H;
  const float* p = wpe + (int64_t)(c + r) * H;
  float* o = h + (int64_t)r * H;
  for (int i = threadIdx.x * 4; i < H; i += blockDim.x * 4) {
    float4 a = *reinterpret_cast<const float4*>(e + i), b = *reinterpret_cast<const float4*>(p + i);
    *reinterpret_cast<float4*>(o + i) = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
}

__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ dh,
                                 float* __restrict__ gwte, float* __restrict__ gwpe, int c, int H) {
  const int r = blockIdx.x;
  const int id = tok[c + r];
  const float* g = dh + (int64_t)r * H;
  float* e = gwte + (int64_t)id * H;
  float* p = gwpe + (int64_t)(c + r) * H;  // rows c..c+l are owned by this job alone
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    const float v = g[i];
    atomicAdd(e + i, v);
    p[i] += v;
  }
}

// ---------------------------------------------------------------- cross-entropy
// per row: lse = log sum exp z; loss_row = lse - z_y; z <- (softmax(z) - onehot(y)) * scale.
template <typename T>
__global__ void __launch_bounds__(512) ce_kernel(T* __restrict__ z, const int32_t* __restrict__ tgt,
                                                 float* __restrict__ loss_rows, float* __restrict__ zcopy,
                                                 int V, float scale) {
  __shared__ float rm[16], rs[16];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  T* zr = z + (int64_t)r * V;
  float m = -INFINITY, s = 0.f;
  for (int i = tid; i < V; i += 512) {
    const float v = to_f<T>(zr[i]);
    if (zcopy) zcopy[(int64_t)r * V + i] = v;
    if (v > m) { s = s * __expf(m - v) + 1.f; m = v; }
    else s += __expf(v - m);
  }
  // combine (m, s) pairs across the block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mn = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
    m = mn;
  }
  if (lane == 0) { rm[wid] = m; rs[wid] = s; }
  __syncthreads();
  float M = -INFINITY;
  for (int w = 0; w < 16; ++w) M = fmaxf(M, rm[w]);
  float S = 0.f;
  for (int w = 0; w < 16; ++w) S += rs[w] * __expf(rm[w] - M);
  const float lse = M + logf(S);
  const int y = tgt[r];
  if (tid == 0) loss_rows[r] = lse - to_f<T>(zr[y]);
  __syncthreads();  // every thread has read z[y] (via tid 0) before it is overwritten
  for (int i = tid; i < V; i += 512) {
    const float p = __expf(to_f<T>(zr[i]) - lse);
    zr[i] = from_f<T>((p - (i == y ? 1.f : 0.f)) * scale);
  }
}

__global__ void sum_rows_kernel(const float* __restrict__ x, int n, float* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = (float)t;
  }
}

// ---------------------------------------------------------------- conversions
template <typename T>
__global__ void convert_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = from_f<T>(src[i]);
}

template <typename T>
__global__ void transpose_kernel(const float* __restrict__ src, T* __restrict__ dst, int R, int C) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[i][threadIdx.x] = src[(int64_t)r * C + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < C) dst[(int64_t)c * R + r] = from_f<T>(tile[threadIdx.x][i]);
  }
}

template <typename T>
__global__ void colsum_kernel(const T* __restrict__ src, int64_t ld, float* __restrict__ out, int rows, int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int r0 = blockIdx.y * 128, r1 = min(rows, r0 + 128);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += to_f<T>(src[(int64_t)r * ld + n]);
  atomicAdd(out + n, s);
}

}  // namespace

template <typename T>
cudaError_t layernorm_fwd(const float* x, const float* gam, const float* bet, T* y, float* mean, float* rstd,
                          int rows, int H, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  ln_fwd_kernel<T><<<rows, 256, H * sizeof(float), st>>>(x, gam, bet, y, mean, rstd, H);
  return cudaGetLastError();
}
template <typename T>
cudaError_t layernorm_bwd(const float* dy, const float* x, const float* mean, const float* rstd, const float* gam,
                          const float* resid, float* dx_out, T* dx_copy, float* dgam, float* dbet, int rows, int H,
                          cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  ln_bwd_kernel<T><<<rows, 256, 0, st>>>(dy, x, mean, rstd, gam, resid, dx_out, dx_copy, dgam, dbet, H);
  return cudaGetLastError();
}
cudaError_t embed_fwd(const int32_t* tok, const float* wte, const float* wpe, float* h, int c, int l, int H, int V,
                      cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  embed_fwd_kernel<<<l, 256, 0, st>>>(tok, wte, wpe, h, c, H, V);
  return cudaGetLastError();
}
cudaError_t embed_bwd(const int32_t* tok, const float* dh, float* gwte, float* gwpe, int c, int l, int H,
                      cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  embed_bwd_kernel<<<l, 256, 0, st>>>(tok, dh, gwte, gwpe, c, H);
  return cudaGetLastError();
}
template <typename T>
cudaError_t ce_fwd_bwd(T* logits, const int32_t* targets, float* loss_rows, float* logits_copy, int rows, int V,
                       float scale, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  ce_kernel<T><<<rows, 512, 0, st>>>(logits, targets, loss_rows, logits_copy, V, scale);
  return cudaGetLastError();
}
cudaError_t sum_rows(const float* x, int n, float* out, cudaStream_t st) {
  sum_rows_kernel<<<1, 1024, 0, st>>>(x, n, out);
  return cudaGetLastError();
}
template <typename T>
cudaError_t convert_f32(const float* src, T* dst, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  convert_kernel<T><<<blocks, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}
template <typename T>
cudaError_t transpose_convert(const float* src, T* dst, int R, int C, cudaStream_t st) {
  dim3 grid((C + 31) / 32, (R + 31) / 32), block(32, 8);
  transpose_kernel<T><<<grid, block, 0, st>>>(src, dst, R, C);
  return cudaGetLastError();
}
template <typename T>
cudaError_t colsum_accum(const T* src, int64_t ld, float* out, int rows, int N, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  dim3 grid((N + 255) / 256, (rows + 127) / 128);
  colsum_kernel<T><<<grid, 256, 0, st>>>(src, ld, out, rows, N);
  return cudaGetLastError();
}

#define TP_INST(T)                                                                                          \
  template cudaError_t layernorm_fwd<T>(const float*, const float*, const float*, T*, float*, float*, int, int, \
                                        cudaStream_t);                                                      \
  template cudaError_t layernorm_bwd<T>(const float*, const float*, const float*, const float*, const float*,   \
                                        const float*, float*, T*, float*, float*, int, int, cudaStream_t);  \
  template cudaError_t ce_fwd_bwd<T>(T*, const int32_t*, float*, float*, int, int, float, cudaStream_t);   \
  template cudaError_t convert_f32<T>(const float*, T*, int64_t, cudaStream_t);                            \
  template cudaError_t transpose_convert<T>(const float*, T*, int, int, cudaStream_t);                     \
  template cudaError_t colsum_accum<T>(const T*, int64_t, float*, int, int, cudaStream_t);
TP_INST(float)
TP_INST(bf16)
#undef TP_INST

}  // namespace tp
