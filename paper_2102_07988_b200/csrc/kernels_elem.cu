// kernels_elem.cu — the HBM-bound kernels of the hot path: LayerNorm fwd/bwd (reading A-3),
// embedding gather/scatter (A-7), fused cross-entropy fwd+bwd (Eq. 1, A-9),
// dtype conversion/transposition of parameters, bias-gradient column sums, loss reduction.
// All use 16-byte vector accesses where the row length allows (H % 8 == 0 is guaranteed).
#include <algorithm>

#include "kernels.h"
#include "tc5.cuh"

namespace tp {

template <typename T>
cudaError_t colsum_accum(const T* src, int64_t ld, float* out, int rows, int N, cudaStream_t st);

namespace {

// ---------------------------------------------------------------- LayerNorm
// Rows are held in registers: thread t owns columns (c*NT + t)*8 .. +7 for chunk c < NCH
// (16-byte vectors), H <= NT*8*NCH. Two-pass mean/variance from registers.
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red /*[NT/32]*/) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) t += red[w];
  return t;
}

// One warp per row for H <= 32 * 8 * NCW (the row in registers, shuffle reductions, no block
// barrier): 8 rows per 256-thread CTA, so many rows' loads are in flight per SM.
template <typename T, int NCW>
__global__ void __launch_bounds__(256) ln_fwd_warp_kernel(const float* __restrict__ x, const float* __restrict__ gam,
                                                          const float* __restrict__ bet, T* __restrict__ y,
                                                          float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                          int rows, int H) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* xr = x + (int64_t)r * H;
  float v[NCW][8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCW; ++c) {
    const int col = (c * 32 + lane) * 8;
    if (col < H) load8<float>(xr + col, v[c]);
    else
#pragma unroll
      for (int i = 0; i < 8; ++i) v[c][i] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[c][i];
  }
  const float mean = warp_sum(s) / H;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < NCW; ++c) {
    const int col = (c * 32 + lane) * 8;
    if (col < H)
#pragma unroll
      for (int i = 0; i < 8; ++i) { const float d = v[c][i] - mean; q += d * d; }
  }
  const float rstd = rsqrtf(warp_sum(q) / H + 1e-5f);
  if (lane == 0) { mean_out[r] = mean; rstd_out[r] = rstd; }
  T* yr = y + (int64_t)r * H;
#pragma unroll
  for (int c = 0; c < NCW; ++c) {
    const int col = (c * 32 + lane) * 8;
    if (col < H) {
      float g[8], b[8], o[8];
      load8<float>(gam + col, g);
      load8<float>(bet + col, b);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (v[c][i] - mean) * rstd * g[i] + b[i];
      store8<T>(yr + col, o);
    }
  }
}

template <typename T, int NT, int NCH>
__global__ void __launch_bounds__(NT) ln_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gam,
                                                    const float* __restrict__ bet, T* __restrict__ y,
                                                    float* __restrict__ mean_out, float* __restrict__ rstd_out, int H) {
  __shared__ float red[2][NT / 32];
  const int r = blockIdx.x, tid = threadIdx.x;
  const float* xr = x + (int64_t)r * H;
  float v[NCH][8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = (c * NT + tid) * 8;
    if (col < H) load8<float>(xr + col, v[c]);
    else
#pragma unroll
      for (int i = 0; i < 8; ++i) v[c][i] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[c][i];
  }
  const float mean = block_sum<NT>(s, red[0]) / H;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = (c * NT + tid) * 8;
    if (col < H)
#pragma unroll
      for (int i = 0; i < 8; ++i) { const float d = v[c][i] - mean; q += d * d; }
  }
  const float rstd = rsqrtf(block_sum<NT>(q, red[1]) / H + 1e-5f);
  if (tid == 0) { mean_out[r] = mean; rstd_out[r] = rstd; }
  T* yr = y + (int64_t)r * H;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = (c * NT + tid) * 8;
    if (col < H) {
      float g[8], b[8], o[8];
      load8<float>(gam + col, g);
      load8<float>(bet + col, b);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (v[c][i] - mean) * rstd * g[i] + b[i];
      store8<T>(yr + col, o);
    }
  }
}

// out[0..3] += (a, b, c, d) as one 16-byte L2 reduction (sm_90+ vector red)
__device__ __forceinline__ void red_add4(float* out, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// dx = resid + rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)),  dxhat = dy * gamma.
// A CTA handles `rpb` consecutive rows and keeps its dgamma/dbeta partial sums in registers, so the
// fp32 reductions are one per column per CTA (not per row). The next row's dy / x / stats are
// loaded before the current row's block reduction, so the HBM latency overlaps the barrier.
template <typename T, int NT, int NCH>
__global__ void __launch_bounds__(NT) ln_bwd_kernel(const T* __restrict__ dy, const float* __restrict__ x,
                                                    const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                                                    const float* __restrict__ gam, const float* __restrict__ resid,
                                                    float* __restrict__ dx_out, T* __restrict__ dx_copy,
                                                    float* __restrict__ dgam, float* __restrict__ dbet,
                                                    float* __restrict__ dbias, int rows, int H, int rpb) {
  __shared__ float red[2][2][NT / 32];
  const int tid = threadIdx.x;
  float g[NCH][8], pg[NCH][8], pb[NCH][8], pd[NCH][8];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = (c * NT + tid) * 8;
    if (col < H) load8<float>(gam + col, g[c]);
#pragma unroll
    for (int i = 0; i < 8; ++i) { pg[c][i] = 0.f; pb[c][i] = 0.f; pd[c][i] = 0.f; if (col >= H) g[c][i] = 0.f; }
  }
  const int r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  float nd[NCH][8], nx[NCH][8], nres[NCH][8], nmean = 0.f, nrstd = 0.f;  // row r+1, prefetched
  auto fetch = [&](int r) {
    if (r >= r1) return;
    nmean = mean_in[r];
    nrstd = rstd_in[r];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int col = (c * NT + tid) * 8;
      if (col < H) {
        load8<T>(dy + (int64_t)r * H + col, nd[c]);
        load8<float>(x + (int64_t)r * H + col, nx[c]);
        if (resid) load8<float>(resid + (int64_t)r * H + col, nres[c]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) { nd[c][i] = 0.f; nx[c][i] = 0.f; }
      }
    }
  };
  fetch(r0);
  for (int r = r0; r < r1; ++r) {
    const float mean = nmean, rstd = nrstd;
    float d[NCH][8], xh[NCH][8], rs[NCH][8];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int i = 0; i < 8; ++i) { d[c][i] = nd[c][i]; xh[c][i] = nx[c][i]; rs[c][i] = resid ? nres[c][i] : 0.f; }
    fetch(r + 1);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        xh[c][i] = (xh[c][i] - mean) * rstd;
        const float dxh = d[c][i] * g[c][i];
        s1 += dxh;
        s2 += dxh * xh[c][i];
        pg[c][i] += d[c][i] * xh[c][i];
        pb[c][i] += d[c][i];
      }
    }
    // two block reductions sharing one barrier; buffers alternate with the row parity
    float (*rd)[NT / 32] = red[r & 1];
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((tid & 31) == 0) { rd[0][tid >> 5] = s1; rd[1][tid >> 5] = s2; }
    __syncthreads();
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) { m1 += rd[0][w]; m2 += rd[1][w]; }
    m1 /= H;
    m2 /= H;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int col = (c * NT + tid) * 8;
      if (col < H) {
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o[i] = rstd * (d[c][i] * g[c][i] - m1 - xh[c][i] * m2) + rs[c][i];
          pd[c][i] += o[i];
        }
        store8<float>(dx_out + (int64_t)r * H + col, o);
        if (dx_copy) store8<T>(dx_copy + (int64_t)r * H + col, o);
      }
    }
  }
  // per-CTA partial dgamma / dbeta added in L2 (16-byte vector reductions; no workspace pass)
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = (c * NT + tid) * 8;
    if (col < H) {
      red_add4(dgam + col, pg[c][0], pg[c][1], pg[c][2], pg[c][3]);
      red_add4(dgam + col + 4, pg[c][4], pg[c][5], pg[c][6], pg[c][7]);
      red_add4(dbet + col, pb[c][0], pb[c][1], pb[c][2], pb[c][3]);
      red_add4(dbet + col + 4, pb[c][4], pb[c][5], pb[c][6], pb[c][7]);
      if (dbias) {
        red_add4(dbias + col, pd[c][0], pd[c][1], pd[c][2], pd[c][3]);
        red_add4(dbias + col + 4, pd[c][4], pd[c][5], pd[c][6], pd[c][7]);
      }
    }
  }
}

// Wide rows (H > 2048, e.g. 13B / 175B): the same math with more threads per row and the dgamma /
// dbeta / dbias partial sums in shared memory (thread t owns its columns' slots, no conflicts) instead
// of registers, and no prefetch buffers, so the CTA keeps <= 64-80 registers per thread and 16-24
// warps per SM are in flight (the register-resident version spilled or ran one 8-warp CTA per SM).
template <typename T, int NT, int NCH>
__global__ void __launch_bounds__(NT, 1) ln_bwd_wide_kernel(const T* __restrict__ dy, const float* __restrict__ x,
                                                            const float* __restrict__ mean_in,
                                                            const float* __restrict__ rstd_in,
                                                            const float* __restrict__ gam, const float* __restrict__ resid,
                                                            float* __restrict__ dx_out, T* __restrict__ dx_copy,
                                                            float* __restrict__ dgam, float* __restrict__ dbet,
                                                            float* __restrict__ dbias, int rows, int H, int rpb) {
  extern __shared__ float acc_s[];  // [3][NCH * NT * 8]: dgamma, dbeta, dbias partials
  __shared__ float red[2][2][NT / 32];
  const int tid = threadIdx.x;
  constexpr int W = NCH * NT * 8;
  for (int i = tid; i < 3 * W; i += NT) acc_s[i] = 0.f;
  __syncthreads();
  const int r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  for (int r = r0; r < r1; ++r) {
    const float mean = mean_in[r], rstd = rstd_in[r];
    float d[NCH][8], xh[NCH][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int col = (c * NT + tid) * 8;
      if (col < H) {
        float g[8];
        load8<T>(dy + (int64_t)r * H + col, d[c]);
        load8<float>(x + (int64_t)r * H + col, xh[c]);
        load8<float>(gam + col, g);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          xh[c][i] = (xh[c][i] - mean) * rstd;
          const float dxh = d[c][i] * g[i];
          s1 += dxh;
          s2 += dxh * xh[c][i];
          acc_s[col + i] += d[c][i] * xh[c][i];
          acc_s[W + col + i] += d[c][i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) { d[c][i] = 0.f; xh[c][i] = 0.f; }
      }
    }
    float (*rd)[NT / 32] = red[r & 1];
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((tid & 31) == 0) { rd[0][tid >> 5] = s1; rd[1][tid >> 5] = s2; }
    __syncthreads();
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) { m1 += rd[0][w]; m2 += rd[1][w]; }
    m1 /= H;
    m2 /= H;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int col = (c * NT + tid) * 8;
      if (col < H) {
        float g[8], o[8], rs[8];
        load8<float>(gam + col, g);
        if (resid) load8<float>(resid + (int64_t)r * H + col, rs);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o[i] = rstd * (d[c][i] * g[i] - m1 - xh[c][i] * m2) + (resid ? rs[i] : 0.f);
          acc_s[2 * W + col + i] += o[i];
        }
        store8<float>(dx_out + (int64_t)r * H + col, o);
        if (dx_copy) store8<T>(dx_copy + (int64_t)r * H + col, o);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = (c * NT + tid) * 8;
    if (col < H) {
      const float* a = acc_s + col;
      red_add4(dgam + col, a[0], a[1], a[2], a[3]);
      red_add4(dgam + col + 4, a[4], a[5], a[6], a[7]);
      red_add4(dbet + col, a[W], a[W + 1], a[W + 2], a[W + 3]);
      red_add4(dbet + col + 4, a[W + 4], a[W + 5], a[W + 6], a[W + 7]);
      if (dbias) {
        red_add4(dbias + col, a[2 * W], a[2 * W + 1], a[2 * W + 2], a[2 * W + 3]);
        red_add4(dbias + col + 4, a[2 * W + 4], a[2 * W + 5], a[2 * W + 6], a[2 * W + 7]);
      }
    }
  }
}

// ---- bulk-staged variants (H <= 2048): rows move HBM -> shared memory by cp.async.bulk into a
// ring of stages completing on mbarriers (thread 0 issues them), so each SM keeps ~160-190 KB of
// loads in flight (the register-prefetch kernels above: 40-128 KB, with a warp's / CTA's loads
// stalled behind its own reductions and stores). One CTA of 256 threads (8 columns each) per group
// of `rpb` consecutive rows; the block reduction's barrier doubles as the "stage consumed" signal,
// after which thread 0 refills the stage with the row LN*_STAGES ahead.
// NT threads x 8 columns per row (NT = 256 for H <= 2048, 640 for H <= 5120, e.g. 13B).
// Forward (H <= 2048): 4 stages of one row (4H bytes); 48 registers -> 5 CTAs per SM.
constexpr int LNF_STAGES = 4;
template <typename T, int NT>
__global__ void __launch_bounds__(NT) ln_fwd_bulk_kernel(const float* __restrict__ x, const float* __restrict__ gam,
                                                          const float* __restrict__ bet, T* __restrict__ y,
                                                          float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                          int rows, int H, int rpb) {
  extern __shared__ __align__(128) float lnf_ring[];  // [LNF_STAGES][H]
  __shared__ __align__(8) uint64_t full[LNF_STAGES];
  constexpr int NW = NT / 32;
  __shared__ float red[2][2][NW];
  const int tid = threadIdx.x, col = tid * 8;
  const bool act = col < H;
  const uint32_t bytes = (uint32_t)H * 4u;
  const int r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  if (tid == 0) {
#pragma unroll
    for (int d = 0; d < LNF_STAGES; ++d) tc5::mbar_init(&full[d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int d = 0; d < LNF_STAGES && r0 + d < r1; ++d) {
      tc5::mbar_expect_tx(&full[d], bytes);
      tc5::bulk_load(lnf_ring + d * H, x + (int64_t)(r0 + d) * H, bytes, &full[d]);
    }
  }
  float g[8], b[8];
  if (act) { load8<float>(gam + col, g); load8<float>(bet + col, b); }
  __syncthreads();  // barrier initialisation visible to every waiter
  for (int i = 0, r = r0; r < r1; ++i, ++r) {
    const int d = i % LNF_STAGES;
    tc5::mbar_wait(&full[d], (uint32_t)(i / LNF_STAGES) & 1u);
    float v[8];
    if (act) load8<float>(lnf_ring + d * H + col, v);
    else
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.f;
    // one-pass statistics with one block barrier: sums of (x - x0) and (x - x0)^2, x0 = the row's
    // first element (a value of the row, so E[x - x0]^2 stays of the order of the variance and the
    // difference below does not cancel catastrophically)
    const float x0 = lnf_ring[d * H];
    float s = 0.f, q = 0.f;
    if (act)
#pragma unroll
      for (int k = 0; k < 8; ++k) { const float dd = v[k] - x0; s += dd; q += dd * dd; }
    float (*rd)[NW] = red[i & 1];
    s = warp_sum(s);
    q = warp_sum(q);
    if ((tid & 31) == 0) { rd[0][tid >> 5] = s; rd[1][tid >> 5] = q; }
    __syncthreads();  // also: every thread has read stage d
    if (tid == 0 && r + LNF_STAGES < r1) {
      tc5::mbar_expect_tx(&full[d], bytes);
      tc5::bulk_load(lnf_ring + d * H, x + (int64_t)(r + LNF_STAGES) * H, bytes, &full[d]);
    }
    float m = 0.f, qq = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) { m += rd[0][w]; qq += rd[1][w]; }
    const float dm = m / H;
    const float mean = x0 + dm;
    const float rstd = rsqrtf(fmaxf(qq / H - dm * dm, 0.f) + 1e-5f);
    if (tid == 0) { mean_out[r] = mean; rstd_out[r] = rstd; }
    if (act) {
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = (v[k] - mean) * rstd * g[k] + b[k];
      store8<T>(y + (int64_t)r * H + col, o);
    }
  }
}

// Backward: the CTA-per-row-group structure of ln_bwd_kernel (256 threads x 8 columns, dgamma /
// dbeta / dbias partials in registers), with the row's x, resid and dy staged through a ring of
// LNB_STAGES shared-memory stages by thread 0. The per-row block reduction's barrier doubles as the
// "stage consumed" signal: after it, thread 0 refills the stage with row r + LNB_STAGES. The
// group's mean / rstd are read into shared memory 128 rows at a time. ~100 registers: 2 CTAs per SM
// at NT = 256 (4 stages of 20 KB), 1 at NT = 640 (3 stages of 50 KB at H = 5120).
template <typename T, int NT, int LNB_STAGES>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) ln_bwd_bulk_kernel(const T* __restrict__ dy, const float* __restrict__ x,
                                                             const float* __restrict__ mean_in,
                                                             const float* __restrict__ rstd_in,
                                                             const float* __restrict__ gam, const float* __restrict__ resid,
                                                             float* __restrict__ dx_out, T* __restrict__ dx_copy,
                                                             float* __restrict__ dgam, float* __restrict__ dbet,
                                                             float* __restrict__ dbias, int rows, int H, int rpb) {
  extern __shared__ __align__(128) uint8_t lnb_ring[];  // [LNB_STAGES][x: 4H | resid: 4H | dy: H*sizeof(T)]
  __shared__ __align__(8) uint64_t full[LNB_STAGES];
  constexpr int NW = NT / 32;
  __shared__ float red[2][2][NW];
  __shared__ float st[2][128];
  const int tid = threadIdx.x, col = tid * 8;
  const bool act = col < H;
  const size_t stage_bytes = (size_t)H * (8 + sizeof(T));
  const uint32_t row_bytes = (uint32_t)H * (resid ? 8u : 4u) + (uint32_t)(H * sizeof(T));
  const int r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  auto issue = [&](int r, int d) {
    uint8_t* sb = lnb_ring + d * stage_bytes;
    tc5::mbar_expect_tx(&full[d], row_bytes);
    tc5::bulk_load(sb, x + (int64_t)r * H, H * 4u, &full[d]);
    if (resid) tc5::bulk_load(sb + H * 4, resid + (int64_t)r * H, H * 4u, &full[d]);
    tc5::bulk_load(sb + H * 8, dy + (int64_t)r * H, (uint32_t)(H * sizeof(T)), &full[d]);
  };
  if (tid == 0) {
#pragma unroll
    for (int d = 0; d < LNB_STAGES; ++d) tc5::mbar_init(&full[d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int d = 0; d < LNB_STAGES && r0 + d < r1; ++d) issue(r0 + d, d);
  }
  float g[8], pg[8], pb[8], pd[8];
  if (act) load8<float>(gam + col, g);
#pragma unroll
  for (int i = 0; i < 8; ++i) { pg[i] = 0.f; pb[i] = 0.f; pd[i] = 0.f; if (!act) g[i] = 0.f; }
  for (int i = 0, r = r0; r < r1; ++i, ++r) {
    if ((i & 127) == 0) {  // stats of the next (up to) 128 rows of the group
      __syncthreads();     // previous chunk's readers are done (first pass: barrier init visible)
      if (tid < 128) { if (r + tid < r1) st[0][tid] = mean_in[r + tid]; }
      else if (tid < 256 && r + tid - 128 < r1) st[1][tid - 128] = rstd_in[r + tid - 128];
      __syncthreads();
    }
    const float mean = st[0][i & 127], rstd = st[1][i & 127];
    const int d = i % LNB_STAGES;
    tc5::mbar_wait(&full[d], (uint32_t)(i / LNB_STAGES) & 1u);
    const uint8_t* sb = lnb_ring + d * stage_bytes;
    float dv[8], xh[8], rs[8];
    if (act) {
      load8<float>(reinterpret_cast<const float*>(sb) + col, xh);
      load8<T>(reinterpret_cast<const T*>(sb + H * 8) + col, dv);
      if (resid) load8<float>(reinterpret_cast<const float*>(sb + H * 4) + col, rs);
      else
#pragma unroll
        for (int k = 0; k < 8; ++k) rs[k] = 0.f;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) { dv[k] = 0.f; xh[k] = 0.f; rs[k] = 0.f; }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      xh[k] = (xh[k] - mean) * rstd;
      const float dxh = dv[k] * g[k];
      s1 += dxh;
      s2 += dxh * xh[k];
      pg[k] += dv[k] * xh[k];
      pb[k] += dv[k];
    }
    float (*rd)[NW] = red[i & 1];
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((tid & 31) == 0) { rd[0][tid >> 5] = s1; rd[1][tid >> 5] = s2; }
    __syncthreads();  // also: every thread has read stage d
    if (tid == 0 && r + LNB_STAGES < r1) issue(r + LNB_STAGES, d);
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) { m1 += rd[0][w]; m2 += rd[1][w]; }
    m1 /= H;
    m2 /= H;
    if (act) {
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        o[k] = rstd * (dv[k] * g[k] - m1 - xh[k] * m2) + rs[k];
        pd[k] += o[k];
      }
      store8<float>(dx_out + (int64_t)r * H + col, o);
      if (dx_copy) store8<T>(dx_copy + (int64_t)r * H + col, o);
    }
  }
  if (act) {
    red_add4(dgam + col, pg[0], pg[1], pg[2], pg[3]);
    red_add4(dgam + col + 4, pg[4], pg[5], pg[6], pg[7]);
    red_add4(dbet + col, pb[0], pb[1], pb[2], pb[3]);
    red_add4(dbet + col + 4, pb[4], pb[5], pb[6], pb[7]);
    if (dbias) {
      red_add4(dbias + col, pd[0], pd[1], pd[2], pd[3]);
      red_add4(dbias + col + 4, pd[4], pd[5], pd[6], pd[7]);
    }
  }
}

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ wte,
                                 const float* __restrict__ wpe, float* __restrict__ h, int c, int b, int s, int H,
                                 int V) {
  const int r = blockIdx.x;
  const int j = r % b, pos = c + r / b;
  const int id = tok[(int64_t)j * (s + 1) + pos];
  // ids outside [0, V) are rejected by the step (host check, or the device count of
  // count_bad_tokens); the row is then NaN, never an out-of-range read
  const bool ok = id >= 0 && id < V;
  const float* e = wte + (int64_t)(ok ? id : 0) * H;
  const float* p = wpe + (int64_t)pos * H;
  float* o = h + (int64_t)r * H;
  for (int i = threadIdx.x * 4; i < H; i += blockDim.x * 4) {
    float4 a = ok ? *reinterpret_cast<const float4*>(e + i) : make_float4(NAN, NAN, NAN, NAN);
    float4 b = *reinterpret_cast<const float4*>(p + i);
    *reinterpret_cast<float4*>(o + i) = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
}

__global__ void embed_bwd_kernel(const int32_t* __restrict__ tok, const float* __restrict__ dh,
                                 float* __restrict__ gwte, float* __restrict__ gwpe, int c, int b, int s, int H, int V) {
  const int r = blockIdx.x;
  const int j = r % b, pos = c + r / b;
  const int id = tok[(int64_t)j * (s + 1) + pos];
  if (id < 0 || id >= V) return;  // rejected by the step; never scatter outside wte's gradient
  const float* g = dh + (int64_t)r * H;
  float* e = gwte + (int64_t)id * H;
  float* p = gwpe + (int64_t)pos * H;  // positions c..c+l are shared by the job's b sequences
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    const float v = g[i];
    atomicAdd(e + i, v);
    if (b == 1) p[i] += v;
    else atomicAdd(p + i, v);
  }
}

// ---------------------------------------------------------------- cross-entropy
// per row: lse = log sum exp z; loss_row = lse - z_y; z <- (softmax(z) - onehot(y)) * scale.
template <typename T>
__global__ void __launch_bounds__(512) ce_kernel(T* __restrict__ z, const int32_t* __restrict__ tok, int c, int b,
                                                 int seq_len, float* __restrict__ loss_rows, float* __restrict__ zcopy,
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
  int y = tok[(int64_t)(r % b) * (seq_len + 1) + c + r / b + 1];  // target = next token (A-8)
  const bool yok = y >= 0 && y < V;  // else rejected by the step: NaN loss, no read outside the row
  if (tid == 0) loss_rows[r] = yok ? lse - to_f<T>(zr[y]) : NAN;
  if (!yok) y = -1;
  __syncthreads();  // every thread has read z[y] (via tid 0) before it is overwritten
  for (int i = tid; i < V; i += 512) {
    const float p = __expf(to_f<T>(zr[i]) - lse);
    zr[i] = from_f<T>((p - (i == y ? 1.f : 0.f)) * scale);
  }
}

// Same contract for bf16 logits with 16-byte accesses (V % 8 == 0): pass 1 reads the row once from
// HBM with an online (max, sum) per thread, pass 2 re-reads it (L2-resident: one 100 KB row per CTA)
// and writes the gradient in place.
__global__ void __launch_bounds__(512) ce_vec_kernel(bf16* __restrict__ z, const int32_t* __restrict__ tok, int c,
                                                     int b, int seq_len, float* __restrict__ loss_rows,
                                                     float* __restrict__ zcopy, int V, float scale) {
  __shared__ float rm[16], rs[16];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  bf16* zr = z + (int64_t)r * V;
  const int nch = V / 8;
  float m = -INFINITY, s = 0.f;
  for (int ch = tid; ch < nch; ch += 512) {
    float v[8];
    load8<bf16>(zr + ch * 8, v);
    if (zcopy) store8<float>(zcopy + (int64_t)r * V + ch * 8, v);
    float cm = v[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) cm = fmaxf(cm, v[i]);
    const float mn = fmaxf(m, cm);
    float cs = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) cs += __expf(v[i] - mn);
    s = s * __expf(m - mn) + cs;  // m = -inf on the first chunk: exp(-inf) = 0
    m = mn;
  }
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
#pragma unroll
  for (int w = 0; w < 16; ++w) M = fmaxf(M, rm[w]);
  float S = 0.f;
#pragma unroll
  for (int w = 0; w < 16; ++w) S += rs[w] * __expf(rm[w] - M);
  const float lse = M + logf(S);
  int y = tok[(int64_t)(r % b) * (seq_len + 1) + c + r / b + 1];  // target = next token (A-8)
  const bool yok = y >= 0 && y < V;  // else rejected by the step: NaN loss, no read outside the row
  if (tid == 0) loss_rows[r] = yok ? lse - __bfloat162float(zr[y]) : NAN;
  if (!yok) y = -1;
  __syncthreads();  // z[y] read before the row is overwritten
  for (int ch = tid; ch < nch; ch += 512) {
    float v[8];
    load8<bf16>(zr + ch * 8, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (__expf(v[i] - lse) - (ch * 8 + i == y ? 1.f : 0.f)) * scale;
    store8<bf16>(zr + ch * 8, v);
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

// out[n] += sum_r src[r][n]: a CTA covers 256 columns (32 lanes x 8, 16-byte loads) and 256 rows
// (8 warps striding the rows), reduces across warps in shared memory, one atomic per column.
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ src, int64_t ld, float* __restrict__ out,
                                                     int rows, int N) {
  __shared__ float red[8][256 + 8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n0 = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * 256, r1 = min(rows, r0 + 256);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (n0 < N)
    for (int r = r0 + w; r < r1; r += 8) {
      float v[8];
      load8<T>(src + (int64_t)r * ld + n0, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[w][lane * 8 + i] = acc[i];
  __syncthreads();
  const int n = blockIdx.x * 256 + threadIdx.x;
  if (n < N) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
    atomicAdd(out + n, t);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
// TP_LN_BULK=0 selects the register-prefetch LayerNorm kernels (A/B knob)
bool ln_bulk_enabled() {
  static const bool on = !(getenv("TP_LN_BULK") && atoi(getenv("TP_LN_BULK")) == 0);
  return on;
}

}  // namespace

template <typename T>
cudaError_t layernorm_fwd(const float* x, const float* gam, const float* bet, T* y, float* mean, float* rstd,
                          int rows, int H, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  // bulk forward for H <= 2048 only: at H = 5120 the 640-thread variant measured slower than the
  // block-per-row kernel (3.45 vs 3.70 TB/s, profiles/r02_ln_bulk_ab.txt)
  if (H <= 2048 && ln_bulk_enabled() && aligned16(x) && aligned16(y)) {
    const int smem = LNF_STAGES * H * (int)sizeof(float);
    auto launch = [&](auto kern, int nt, int hmax) -> cudaError_t {
      static int per_sm[2] = {0, 0};  // resident CTAs per SM at the widest H of the variant
      int& ps = per_sm[nt > 256];
      if (!ps) {
        if (nt > 256) {
          cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               LNF_STAGES * hmax * (int)sizeof(float));
          if (e != cudaSuccess) return e;
        }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, nt, LNF_STAGES * hmax * (int)sizeof(float)) !=
            cudaSuccess || ps < 1)
          ps = 1;
      }
      const int units = std::max(1, num_sms()) * ps;
      const int rpb = std::max(4, (rows + units - 1) / units);
      kern<<<(rows + rpb - 1) / rpb, nt, smem, st>>>(x, gam, bet, y, mean, rstd, rows, H, rpb);
      return cudaSuccess;
    };
    cudaError_t e = launch(ln_fwd_bulk_kernel<T, 256>, 256, 2048);
    if (e != cudaSuccess) return e;
  } else if (H <= 2048) ln_fwd_warp_kernel<T, 8><<<(rows + 7) / 8, 256, 0, st>>>(x, gam, bet, y, mean, rstd, rows, H);
  else if (H <= 4096) ln_fwd_kernel<T, 256, 2><<<rows, 256, 0, st>>>(x, gam, bet, y, mean, rstd, H);
  else if (H <= 6144) ln_fwd_kernel<T, 256, 3><<<rows, 256, 0, st>>>(x, gam, bet, y, mean, rstd, H);
  else if (H <= 12288) ln_fwd_kernel<T, 512, 3><<<rows, 512, 0, st>>>(x, gam, bet, y, mean, rstd, H);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}
template <typename T>
cudaError_t layernorm_bwd(const T* dy, const float* x, const float* mean, const float* rstd, const float* gam,
                          const float* resid, float* dx_out, T* dx_copy, float* dgam, float* dbet, float* ws, int rows,
                          int H, cudaStream_t st, float* dbias) {
  if (rows == 0) return cudaSuccess;
  // Row groups sized for `ctas` CTAs per SM. The 112-register H <= 2048 kernel keeps 2 CTAs of 256
  // threads resident per SM, so 2 x 148 groups run as one wave (measured: LayerNorm class 10.2 -> 9.6
  // ms per step vs 4 x 148; an 80-register 3-CTA variant spilled and was slower). The wide kernels
  // keep 4 x 148 (at H = 5120, 4 vs 2 per SM measured within noise, profiles/r01_lnb_ab_13b_n4.txt).
  // TP_LNB_CTAS overrides (A/B knob, scripts/ln_ab.sh, scripts/ln_ab_13b.sh).
  static const int ctas_env = getenv("TP_LNB_CTAS") ? std::max(1, atoi(getenv("TP_LNB_CTAS"))) : 0;
  const int ctas = ctas_env ? ctas_env : (H <= 2048 ? 2 : 4);
  const int rpb = std::max(4, (rows + ctas * 148 - 1) / (ctas * 148));
  const int grid = (rows + rpb - 1) / rpb;
  (void)ws;
#define LNB(NT, NCH) ln_bwd_kernel<T, NT, NCH><<<grid, NT, 0, st>>>(dy, x, mean, rstd, gam, resid, dx_out, dx_copy, dgam, dbet, dbias, rows, H, rpb)
#define LNBW(NT, NCH)                                                                                     \
  do {                                                                                                    \
    const int smem = 3 * NCH * NT * 8 * (int)sizeof(float);                                               \
    static bool attr = false;                                                                             \
    if (!attr) {                                                                                          \
      cudaError_t e = cudaFuncSetAttribute(ln_bwd_wide_kernel<T, NT, NCH>,                                \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
      if (e != cudaSuccess) return e;                                                                     \
      attr = true;                                                                                        \
    }                                                                                                     \
    ln_bwd_wide_kernel<T, NT, NCH><<<grid, NT, smem, st>>>(dy, x, mean, rstd, gam, resid, dx_out, dx_copy, \
                                                          dgam, dbet, dbias, rows, H, rpb);               \
  } while (0)
  if (H <= 5120 && ln_bulk_enabled() && aligned16(x) && aligned16(dy) && aligned16(resid)) {
    auto launch = [&](auto kern, int nt, int stages, int ctas, int hmax) -> cudaError_t {
      static bool attr[2] = {false, false};
      if (!attr[nt > 256]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             stages * hmax * (8 + (int)sizeof(T)));
        if (e != cudaSuccess) return e;
        attr[nt > 256] = true;
      }
      const int units = std::max(1, num_sms()) * ctas;
      const int rpb2 = std::max(4, (rows + units - 1) / units);
      kern<<<(rows + rpb2 - 1) / rpb2, nt, stages * H * (8 + (int)sizeof(T)), st>>>(
          dy, x, mean, rstd, gam, resid, dx_out, dx_copy, dgam, dbet, dbias, rows, H, rpb2);
      return cudaSuccess;
    };
    cudaError_t e = H <= 2048 ? launch(ln_bwd_bulk_kernel<T, 256, 4>, 256, 4, 2, 2048)
                              : launch(ln_bwd_bulk_kernel<T, 640, 3>, 640, 3, 1, 5120);
    if (e != cudaSuccess) return e;
  } else if (H <= 2048) LNB(256, 1);
  else if (H <= 4096) LNBW(512, 1);
  else if (H <= 6144) LNBW(768, 1);
  else if (H <= 12288) LNBW(768, 2);
  else return cudaErrorInvalidValue;
#undef LNB
#undef LNBW
  return cudaGetLastError();
}
cudaError_t embed_fwd(const int32_t* tok, const float* wte, const float* wpe, float* h, int c, int l, int b, int s,
                      int H, int V, cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  embed_fwd_kernel<<<l * b, 256, 0, st>>>(tok, wte, wpe, h, c, b, s, H, V);
  return cudaGetLastError();
}
__global__ void count_bad_tokens_kernel(const int32_t* __restrict__ tok, int64_t n, int V, int* __restrict__ bad) {
  int cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cnt += (tok[i] < 0 || tok[i] >= V) ? 1 : 0;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(bad, cnt);
}
cudaError_t count_bad_tokens(const int32_t* tok, int64_t n, int V, int* bad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (e != cudaSuccess || n == 0) return e;
  const int blocks = (int)std::min<int64_t>(1024, (n + 255) / 256);
  count_bad_tokens_kernel<<<blocks, 256, 0, st>>>(tok, n, V, bad);
  return cudaGetLastError();
}

cudaError_t embed_bwd(const int32_t* tok, const float* dh, float* gwte, float* gwpe, int c, int l, int b, int s,
                      int H, int V, cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  embed_bwd_kernel<<<l * b, 256, 0, st>>>(tok, dh, gwte, gwpe, c, b, s, H, V);
  return cudaGetLastError();
}
template <typename T>
cudaError_t ce_fwd_bwd(T* logits, const int32_t* tok, int c, int b, int s, float* loss_rows, float* logits_copy,
                       int rows, int V, float scale, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  if constexpr (std::is_same<T, bf16>::value) {
    if (V % 8 == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0) {
      ce_vec_kernel<<<rows, 512, 0, st>>>(logits, tok, c, b, s, loss_rows, logits_copy, V, scale);
      return cudaGetLastError();
    }
  }
  ce_kernel<T><<<rows, 512, 0, st>>>(logits, tok, c, b, s, loss_rows, logits_copy, V, scale);
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
  dim3 grid((N + 255) / 256, (rows + 255) / 256);
  colsum_kernel<T><<<grid, 256, 0, st>>>(src, ld, out, rows, N);
  return cudaGetLastError();
}

#define TP_INST(T)                                                                                          \
  template cudaError_t layernorm_fwd<T>(const float*, const float*, const float*, T*, float*, float*, int, int, \
                                        cudaStream_t);                                                      \
  template cudaError_t layernorm_bwd<T>(const T*, const float*, const float*, const float*, const float*,       \
                                        const float*, float*, T*, float*, float*, float*, int, int, cudaStream_t,  \
                                        float*);                                                                \
  template cudaError_t ce_fwd_bwd<T>(T*, const int32_t*, int, int, int, float*, float*, int, int, float,    \
                                     cudaStream_t);                                                        \
  template cudaError_t convert_f32<T>(const float*, T*, int64_t, cudaStream_t);                            \
  template cudaError_t transpose_convert<T>(const float*, T*, int, int, cudaStream_t);                     \
  template cudaError_t colsum_accum<T>(const T*, int64_t, float*, int, int, cudaStream_t);
TP_INST(float)
TP_INST(bf16)
#undef TP_INST

}  // namespace tp
