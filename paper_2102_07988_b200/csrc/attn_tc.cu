// attn_tc.cu — slice-vs-prefix causal attention on tensor cores (bf16 operands, fp32 accumulate).
//
// One job = one sequence's slice rows [c, c+l); query at absolute position c+r attends keys
// [0, c+r] of the per-layer prefix K/V cache [a][s][d] (Eq. 2; the dependency
// property PAPER.md:180 that makes token slicing legal). Scale 1/sqrt(d) (A-1).
//
//   forward : per (64-row query tile, head): online softmax over 64-key blocks of the prefix,
//             S = Q K^T and O += P V on mma.sync m16n8k16, exp2 with the scale folded in;
//             writes O (bf16, token-major) and LSE (fp32).
//   backward: D = rowsum(dO * O); kernel dQ: per query tile, recompute P, dP = dO V^T,
//             dS = P (dP - D), dQ = scale * dS K (one writer per row, no atomics);
//             kernel dKV: per 64-key block of the prefix [0, c+l), loop over the slice's query
//             tiles that can see it: P^T, dV += P^T dO, dP^T = V dO^T, dK += scale * dS^T Q, then
//             write (first backward slice) or add into the fp32 dK/dV accumulators — each key row
//             has exactly one writer per launch, so the push into earlier slices needs no atomics.
// Key blocks are aligned to absolute multiples of 64, so only the diagonal block of a query tile
// is partially masked; K/V/Q/dO tiles are staged with 16-byte cp.async (zero-filled out of range)
// into padded shared memory (row pitch d+8 -> conflict-free ldmatrix).
//
// B200 note: this is the legacy warp-level MMA path (HMMA); the tcgen05/TMEM version is the
// next step for this kernel (DESIGN.md "Kernels" / "Next").
#include "kernels.h"

namespace tp {

namespace {

constexpr int BQ = 64, BKEY = 64, NWARP = 4;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(dst)), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Stage rows [row0, row0+64) of a [rows][ld] bf16 matrix (columns [0, D)) into smem tile [64][D+8];
// rows >= row_end are zero-filled.
template <int D>
__device__ __forceinline__ void load_tile(bf16* sm, const bf16* g, int64_t ld, int row0, int row_end) {
  constexpr int CPR = D / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < 64 * CPR; i += NWARP * 32) {
    const int r = i / CPR, ch = i - r * CPR;
    const bool ok = row0 + r < row_end;
    const bf16* src = ok ? g + (int64_t)(row0 + r) * ld + ch * 8 : g;
    cp_async16(sm + r * (D + 8) + ch * 8, src, ok);
  }
}

// A fragment (16x16, row-major smem tile with pitch P elements) at (row0, col0).
__device__ __forceinline__ void lda_frag(uint32_t (&a)[4], const bf16* sm, int P, int row0, int col0) {
  const int lane = threadIdx.x & 31, mat = lane >> 3, rr = lane & 7;
  ldsm_x4(a, saddr(sm + (row0 + (mat & 1) * 8 + rr) * P + col0 + (mat >> 1) * 8));
}
// B fragments of two 8-wide n-tiles, storage rows = n, cols = k (non-transposed).
__device__ __forceinline__ void ldb_frag_n(uint32_t (&b)[4], const bf16* sm, int P, int n0, int k0) {
  const int lane = threadIdx.x & 31, mat = lane >> 3, rr = lane & 7;
  ldsm_x4(b, saddr(sm + (n0 + (mat >> 1) * 8 + rr) * P + k0 + (mat & 1) * 8));
}
// B fragments of two 8-wide n-tiles, storage rows = k, cols = n (transposed load).
__device__ __forceinline__ void ldb_frag_t(uint32_t (&b)[4], const bf16* sm, int P, int k0, int n0) {
  const int lane = threadIdx.x & 31, mat = lane >> 3, rr = lane & 7;
  ldsm_x4_t(b, saddr(sm + (k0 + (mat & 1) * 8 + rr) * P + n0 + (mat >> 1) * 8));
}

// ======================================================================== forward
template <int D>
__global__ void __launch_bounds__(NWARP * 32) attn_fwd_tc_kernel(const bf16* __restrict__ q, const bf16* __restrict__ k,
                                                                 const bf16* __restrict__ v, bf16* __restrict__ o,
                                                                 int64_t ldo, float* __restrict__ lse, int s, int c,
                                                                 int l, float scale_log2) {
  constexpr int P = D + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Qs = reinterpret_cast<bf16*>(smem_raw);
  bf16* Ks = Qs + BQ * P;       // [2][64][P]
  bf16* Vs = Ks + 2 * BKEY * P; // [2][64][P]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int head = blockIdx.y, r0 = blockIdx.x * BQ;
  const int64_t hb = (int64_t)head * s * D;
  const int qpos_last = c + min(l, r0 + BQ) - 1;
  const int nkb = qpos_last / BKEY + 1;

  load_tile<D>(Qs, q + hb + (int64_t)c * D, D, r0, l);
  load_tile<D>(Ks, k + hb, D, 0, c + l);
  load_tile<D>(Vs, v + hb, D, 0, c + l);
  cp_commit();

  float m_i[2] = {-INFINITY, -INFINITY}, l_i[2] = {0.f, 0.f};
  float oacc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  const int qrow0 = c + r0 + warp * 16 + g;  // absolute positions of this thread's rows g, g+8

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<D>(Ks + (buf ^ 1) * BKEY * P, k + hb, D, (kb + 1) * BKEY, c + l);
      load_tile<D>(Vs + (buf ^ 1) * BKEY * P, v + hb, D, (kb + 1) * BKEY, c + l);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* Kb = Ks + buf * BKEY * P;
    const bf16* Vb = Vs + buf * BKEY * P;
    float sacc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) sacc[i][0] = sacc[i][1] = sacc[i][2] = sacc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a[4];
      lda_frag(a, Qs, P, warp * 16, kk * 16);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b[4];
        ldb_frag_n(b, Kb, P, np * 16, kk * 16);
        mma16816(sacc[2 * np], a, b[0], b[1]);
        mma16816(sacc[2 * np + 1], a, b[2], b[3]);
      }
    }
    // scale (log2 domain), causal mask on the diagonal block, online softmax
    const int key0 = kb * BKEY;
    const bool diag = key0 + BKEY - 1 > c + r0 + warp * 16;  // some key may exceed some row of this warp
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = key0 + nt * 8 + 2 * t + (e & 1);
        const int qp = qrow0 + (e >> 1) * 8;
        float x = sacc[nt][e] * scale_log2;
        if (diag && key > qp) x = -INFINITY;
        sacc[nt][e] = x;
        mx[e >> 1] = fmaxf(mx[e >> 1], x);
      }
    float corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
      const float mn = fmaxf(m_i[h], mx[h]);
      corr[h] = exp2f(m_i[h] - mn);  // m_i = -inf on the first block -> 0
      m_i[h] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(sacc[nt][e] - m_i[e >> 1]);
        sacc[nt][e] = p;
        rs[e >> 1] += p;
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 1);
      rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 2);
      l_i[h] = l_i[h] * corr[h] + rs[h];
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      oacc[i][0] *= corr[0]; oacc[i][1] *= corr[0];
      oacc[i][2] *= corr[1]; oacc[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int j = 0; j < BKEY / 16; ++j) {
      uint32_t a[4] = {pack_bf16(sacc[2 * j][0], sacc[2 * j][1]), pack_bf16(sacc[2 * j][2], sacc[2 * j][3]),
                       pack_bf16(sacc[2 * j + 1][0], sacc[2 * j + 1][1]),
                       pack_bf16(sacc[2 * j + 1][2], sacc[2 * j + 1][3])};
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t b[4];
        ldb_frag_t(b, Vb, P, j * 16, dn * 16);
        mma16816(oacc[2 * dn], a, b[0], b[1]);
        mma16816(oacc[2 * dn + 1], a, b[2], b[3]);
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's prefetch
  }
  // epilogue
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = r0 + warp * 16 + g + h * 8;
    if (r < l) {
      const float inv = 1.f / l_i[h];
      bf16* orow = o + (int64_t)r * ldo + head * D;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        *reinterpret_cast<__nv_bfloat162*>(orow + i * 8 + 2 * t) =
            __floats2bfloat162_rn(oacc[i][2 * h] * inv, oacc[i][2 * h + 1] * inv);
      }
      if (t == 0) lse[(int64_t)head * s + c + r] = (m_i[h] + log2f(l_i[h])) / LOG2E;
    }
  }
}

// ======================================================================== backward
// D[head][r] = rowsum(dO * O): one warp per row, lanes take 8-element chunks of all heads.
template <int D>
__global__ void attn_bwd_prep_kernel(const bf16* __restrict__ dO, int64_t ld_do, const bf16* __restrict__ o,
                                     int64_t ldo, float* __restrict__ Dvec, int a, int l, int64_t o_sstride) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x * 4 + w;
  dO += blockIdx.y * o_sstride;
  o += blockIdx.y * o_sstride;
  Dvec += (int64_t)blockIdx.y * a * l;
  if (r >= l) return;
  constexpr int CPH = D / 8;  // chunks per head (2..16)
  for (int base = 0; base < a * CPH; base += 32) {
    const int ch = base + lane;
    float acc = 0.f;
    if (ch < a * CPH) {
      float x[8], y[8];
      load8<bf16>(dO + (int64_t)r * ld_do + ch * 8, x);
      load8<bf16>(o + (int64_t)r * ldo + ch * 8, y);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += x[i] * y[i];
    }
    // reduce groups of CPH consecutive lanes (one head each)
#pragma unroll
    for (int off = 1; off < CPH && off < 32; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (CPH <= 32 && ch < a * CPH && (lane % CPH) == 0) Dvec[(int64_t)(ch / CPH) * l + r] = acc;
  }
}

// dQ: per (64-row query tile, head).
template <int D>
__global__ void __launch_bounds__(NWARP * 32) attn_bwd_dq_kernel(const bf16* __restrict__ dO, int64_t ld_do,
                                                                 const bf16* __restrict__ q, const bf16* __restrict__ k,
                                                                 const bf16* __restrict__ v, const float* __restrict__ lse,
                                                                 const float* __restrict__ Dvec, bf16* __restrict__ dq,
                                                                 int64_t ldq, int s, int c, int l, float scale,
                                                                 float scale_log2) {
  constexpr int P = D + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Qs = reinterpret_cast<bf16*>(smem_raw);
  bf16* dOs = Qs + BQ * P;
  bf16* Ks = dOs + BQ * P;       // [2][64][P]
  bf16* Vs = Ks + 2 * BKEY * P;  // [2][64][P]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int head = blockIdx.y, r0 = blockIdx.x * BQ;
  const int64_t hb = (int64_t)head * s * D;
  const int qpos_last = c + min(l, r0 + BQ) - 1;
  const int nkb = qpos_last / BKEY + 1;

  load_tile<D>(Qs, q + hb + (int64_t)c * D, D, r0, l);
  load_tile<D>(dOs, dO + head * D, ld_do, r0, l);
  load_tile<D>(Ks, k + hb, D, 0, c + l);
  load_tile<D>(Vs, v + hb, D, 0, c + l);
  cp_commit();

  float lrow[2], drow[2];
  const int qrow0 = c + r0 + warp * 16 + g;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = r0 + warp * 16 + g + h * 8;
    lrow[h] = r < l ? lse[(int64_t)head * s + c + r] * LOG2E : 0.f;
    drow[h] = r < l ? Dvec[(int64_t)head * l + r] : 0.f;
  }
  float dqacc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dqacc[i][0] = dqacc[i][1] = dqacc[i][2] = dqacc[i][3] = 0.f;

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<D>(Ks + (buf ^ 1) * BKEY * P, k + hb, D, (kb + 1) * BKEY, c + l);
      load_tile<D>(Vs + (buf ^ 1) * BKEY * P, v + hb, D, (kb + 1) * BKEY, c + l);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* Kb = Ks + buf * BKEY * P;
    const bf16* Vb = Vs + buf * BKEY * P;
    float sacc[8][4], pacc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) sacc[i][e] = pacc[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a[4], ad[4];
      lda_frag(a, Qs, P, warp * 16, kk * 16);
      lda_frag(ad, dOs, P, warp * 16, kk * 16);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b[4], bv[4];
        ldb_frag_n(b, Kb, P, np * 16, kk * 16);
        mma16816(sacc[2 * np], a, b[0], b[1]);
        mma16816(sacc[2 * np + 1], a, b[2], b[3]);
        ldb_frag_n(bv, Vb, P, np * 16, kk * 16);
        mma16816(pacc[2 * np], ad, bv[0], bv[1]);
        mma16816(pacc[2 * np + 1], ad, bv[2], bv[3]);
      }
    }
    const int key0 = kb * BKEY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = key0 + nt * 8 + 2 * t + (e & 1);
        const int h = e >> 1;
        const int qp = qrow0 + h * 8;
        const float p = key > qp ? 0.f : exp2f(sacc[nt][e] * scale_log2 - lrow[h]);
        sacc[nt][e] = p * (pacc[nt][e] - drow[h]);  // dS
      }
    // dQ += dS K
#pragma unroll
    for (int j = 0; j < BKEY / 16; ++j) {
      uint32_t a[4] = {pack_bf16(sacc[2 * j][0], sacc[2 * j][1]), pack_bf16(sacc[2 * j][2], sacc[2 * j][3]),
                       pack_bf16(sacc[2 * j + 1][0], sacc[2 * j + 1][1]),
                       pack_bf16(sacc[2 * j + 1][2], sacc[2 * j + 1][3])};
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t b[4];
        ldb_frag_t(b, Kb, P, j * 16, dn * 16);
        mma16816(dqacc[2 * dn], a, b[0], b[1]);
        mma16816(dqacc[2 * dn + 1], a, b[2], b[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = r0 + warp * 16 + g + h * 8;
    if (r < l) {
      bf16* drow_p = dq + (int64_t)r * ldq + head * D;
#pragma unroll
      for (int i = 0; i < D / 8; ++i)
        *reinterpret_cast<__nv_bfloat162*>(drow_p + i * 8 + 2 * t) =
            __floats2bfloat162_rn(dqacc[i][2 * h] * scale, dqacc[i][2 * h + 1] * scale);
    }
  }
}

// dK/dV: per (64-key block of the prefix [0, c+l), head).
template <int D>
__global__ void __launch_bounds__(NWARP * 32) attn_bwd_dkv_kernel(const bf16* __restrict__ dO, int64_t ld_do,
                                                                  const bf16* __restrict__ q, const bf16* __restrict__ k,
                                                                  const bf16* __restrict__ v, const float* __restrict__ lse,
                                                                  const float* __restrict__ Dvec, float* __restrict__ dk_acc,
                                                                  float* __restrict__ dv_acc, int s, int c, int l,
                                                                  float scale, float scale_log2, int accumulate) {
  constexpr int P = D + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Ks = reinterpret_cast<bf16*>(smem_raw);
  bf16* Vs = Ks + BKEY * P;
  bf16* Qs = Vs + BKEY * P;      // [2][64][P]
  bf16* dOs = Qs + 2 * BQ * P;   // [2][64][P]
  float* Ls = reinterpret_cast<float*>(dOs + 2 * BQ * P);  // [2][64] lse (log2 domain)
  float* Ds = Ls + 2 * BQ;                                  // [2][64]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int head = blockIdx.y, key0 = blockIdx.x * BKEY;
  const int64_t hb = (int64_t)head * s * D;
  const int nkeys = c + l;
  // query rows r with c + r >= key0 can see this block
  const int rs = max(0, key0 - c);
  const int qt0 = rs / BQ, nqt = (l + BQ - 1) / BQ;

  load_tile<D>(Ks, k + hb, D, key0, nkeys);
  load_tile<D>(Vs, v + hb, D, key0, nkeys);
  auto load_q = [&](int qt, int buf) {
    load_tile<D>(Qs + buf * BQ * P, q + hb + (int64_t)c * D, D, qt * BQ, l);
    load_tile<D>(dOs + buf * BQ * P, dO + head * D, ld_do, qt * BQ, l);
    for (int i = threadIdx.x; i < BQ; i += NWARP * 32) {
      const int r = qt * BQ + i;
      Ls[buf * BQ + i] = r < l ? lse[(int64_t)head * s + c + r] * LOG2E : INFINITY;
      Ds[buf * BQ + i] = r < l ? Dvec[(int64_t)head * l + r] : 0.f;
    }
  };
  if (qt0 < nqt) load_q(qt0, 0);
  cp_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int krow0 = key0 + warp * 16 + g;  // absolute key positions of this thread's rows g, g+8

  for (int qt = qt0; qt < nqt; ++qt) {
    const int buf = (qt - qt0) & 1;
    if (qt + 1 < nqt) {
      __syncthreads();  // Ls/Ds of buf^1 were last read two iterations ago
      load_q(qt + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* Qb = Qs + buf * BQ * P;
    const bf16* dOb = dOs + buf * BQ * P;
    const float* Lb = Ls + buf * BQ;
    const float* Db = Ds + buf * BQ;
    // S^T = K Q^T (rows = keys, cols = queries) and dP^T = V dO^T
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ak[4], av[4];
      lda_frag(ak, Ks, P, warp * 16, kk * 16);
      lda_frag(av, Vs, P, warp * 16, kk * 16);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b[4], bd[4];
        ldb_frag_n(b, Qb, P, np * 16, kk * 16);
        mma16816(st[2 * np], ak, b[0], b[1]);
        mma16816(st[2 * np + 1], ak, b[2], b[3]);
        ldb_frag_n(bd, dOb, P, np * 16, kk * 16);
        mma16816(dpt[2 * np], av, bd[0], bd[1]);
        mma16816(dpt[2 * np + 1], av, bd[2], bd[3]);
      }
    }
    const int qbase = c + qt * BQ;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = nt * 8 + 2 * t + e;  // query index in tile
        const float L = Lb[col], Dq = Db[col];
        const int qp = qbase + col;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kp = krow0 + h * 8;
          const float p = kp > qp ? 0.f : exp2f(st[nt][h * 2 + e] * scale_log2 - L);
          st[nt][h * 2 + e] = p;
          dpt[nt][h * 2 + e] = p * (dpt[nt][h * 2 + e] - Dq);  // dS^T
        }
      }
    // dV += P^T dO ; dK += dS^T Q
#pragma unroll
    for (int j = 0; j < BQ / 16; ++j) {
      uint32_t ap[4] = {pack_bf16(st[2 * j][0], st[2 * j][1]), pack_bf16(st[2 * j][2], st[2 * j][3]),
                        pack_bf16(st[2 * j + 1][0], st[2 * j + 1][1]), pack_bf16(st[2 * j + 1][2], st[2 * j + 1][3])};
      uint32_t as[4] = {pack_bf16(dpt[2 * j][0], dpt[2 * j][1]), pack_bf16(dpt[2 * j][2], dpt[2 * j][3]),
                        pack_bf16(dpt[2 * j + 1][0], dpt[2 * j + 1][1]),
                        pack_bf16(dpt[2 * j + 1][2], dpt[2 * j + 1][3])};
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t b[4], bq[4];
        ldb_frag_t(b, dOb, P, j * 16, dn * 16);
        mma16816(dv[2 * dn], ap, b[0], b[1]);
        mma16816(dv[2 * dn + 1], ap, b[2], b[3]);
        ldb_frag_t(bq, Qb, P, j * 16, dn * 16);
        mma16816(dk[2 * dn], as, bq[0], bq[1]);
        mma16816(dk[2 * dn + 1], as, bq[2], bq[3]);
      }
    }
  }
  // write / accumulate rows of this key block (one writer per row)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kp = krow0 + h * 8;
    if (kp < nkeys) {
      float* dkr = dk_acc + hb + (int64_t)kp * D;
      float* dvr = dv_acc + hb + (int64_t)kp * D;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        float2* pk = reinterpret_cast<float2*>(dkr + i * 8 + 2 * t);
        float2* pv = reinterpret_cast<float2*>(dvr + i * 8 + 2 * t);
        float2 nk = make_float2(dk[i][2 * h] * scale, dk[i][2 * h + 1] * scale);
        float2 nv = make_float2(dv[i][2 * h], dv[i][2 * h + 1]);
        if (accumulate) {
          const float2 ok = *pk, ov = *pv;
          nk.x += ok.x; nk.y += ok.y; nv.x += ov.x; nv.y += ov.y;
        }
        *pk = nk;
        *pv = nv;
      }
    }
  }
}

template <int D>
cudaError_t fwd_d(const bf16* q, const bf16* k, const bf16* v, bf16* o, int64_t ldo, float* lse, int a, int s, int c,
                  int l, cudaStream_t st) {
  constexpr int P = D + 8;
  const int smem = (BQ + 4 * BKEY) * P * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((l + BQ - 1) / BQ, a);
  attn_fwd_tc_kernel<D><<<grid, NWARP * 32, smem, st>>>(q, k, v, o, ldo, lse, s, c, l, rsqrtf((float)D) * LOG2E);
  return cudaGetLastError();
}

template <int D>
cudaError_t bwd_d(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, const bf16* q, const bf16* k, const bf16* v,
                  const float* lse, float* Dvec, bf16* dq, int64_t ldq, float* dk_acc, float* dv_acc, int a, int s, int c,
                  int l, int accumulate, cudaStream_t st) {
  constexpr int P = D + 8;
  const int smem_q = (2 * BQ + 4 * BKEY) * P * 2;
  const int smem_kv = (2 * BKEY + 4 * BQ) * P * 2 + 4 * BQ * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dkv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const float scale = rsqrtf((float)D);
  attn_bwd_prep_kernel<D><<<dim3((l + 3) / 4), 128, 0, st>>>(dO, ld_do, o, ldo, Dvec, a, l, 0);
  attn_bwd_dq_kernel<D><<<dim3((l + BQ - 1) / BQ, a), NWARP * 32, smem_q, st>>>(dO, ld_do, q, k, v, lse, Dvec, dq, ldq, s,
                                                                                c, l, scale, scale * LOG2E);
  attn_bwd_dkv_kernel<D><<<dim3((c + l + BKEY - 1) / BKEY, a), NWARP * 32, smem_kv, st>>>(
      dO, ld_do, q, k, v, lse, Dvec, dk_acc, dv_acc, s, c, l, scale, scale * LOG2E, accumulate);
  return cudaGetLastError();
}

}  // namespace

cudaError_t attn_bwd_prep(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, float* Dvec, int a, int d, int l,
                          cudaStream_t st, int nseq, int64_t o_sstride) {
  if (l == 0) return cudaSuccess;
  dim3 grid((l + 3) / 4, nseq);
  switch (d) {
    case 16: attn_bwd_prep_kernel<16><<<grid, 128, 0, st>>>(dO, ld_do, o, ldo, Dvec, a, l, o_sstride); break;
    case 32: attn_bwd_prep_kernel<32><<<grid, 128, 0, st>>>(dO, ld_do, o, ldo, Dvec, a, l, o_sstride); break;
    case 64: attn_bwd_prep_kernel<64><<<grid, 128, 0, st>>>(dO, ld_do, o, ldo, Dvec, a, l, o_sstride); break;
    case 128: attn_bwd_prep_kernel<128><<<grid, 128, 0, st>>>(dO, ld_do, o, ldo, Dvec, a, l, o_sstride); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t attn_fwd_tc(const bf16* q, const bf16* k, const bf16* v, bf16* o, int64_t ldo, float* lse, int a, int s,
                        int d, int c, int l, cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  switch (d) {
    case 16: return fwd_d<16>(q, k, v, o, ldo, lse, a, s, c, l, st);
    case 32: return fwd_d<32>(q, k, v, o, ldo, lse, a, s, c, l, st);
    case 64: return fwd_d<64>(q, k, v, o, ldo, lse, a, s, c, l, st);
    case 128: return fwd_d<128>(q, k, v, o, ldo, lse, a, s, c, l, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t attn_bwd_tc(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, const bf16* q, const bf16* k,
                        const bf16* v, const float* lse, float* Dvec, bf16* dq, int64_t ldq, float* dk_acc,
                        float* dv_acc, int a, int s, int d, int c, int l, int accumulate, cudaStream_t st) {
  if (l == 0) return cudaSuccess;
  switch (d) {
    case 16: return bwd_d<16>(dO, ld_do, o, ldo, q, k, v, lse, Dvec, dq, ldq, dk_acc, dv_acc, a, s, c, l, accumulate, st);
    case 32: return bwd_d<32>(dO, ld_do, o, ldo, q, k, v, lse, Dvec, dq, ldq, dk_acc, dv_acc, a, s, c, l, accumulate, st);
    case 64: return bwd_d<64>(dO, ld_do, o, ldo, q, k, v, lse, Dvec, dq, ldq, dk_acc, dv_acc, a, s, c, l, accumulate, st);
    case 128: return bwd_d<128>(dO, ld_do, o, ldo, q, k, v, lse, Dvec, dq, ldq, dk_acc, dv_acc, a, s, c, l, accumulate, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tp
