// attn_sm100.cu — slice-vs-prefix causal attention on 5th-generation tensor cores (head_dim 128).
//
// Same contract as attn_tc.cu (Eq. 2; one job = one sequence's slice rows
// [c, c+l) attending keys [0, c+r] of the per-layer prefix K/V cache [a][s][d]), for d = 128.
//
// Forward (attn_fwd2_sm100_kernel): per 256 query rows (two 128-row tiles) x head x sequence,
// heaviest tiles first; K_j / V_j 128-key blocks are TMA-loaded once per CTA for both tiles (4-D maps
// {d, c+l, a, seq}, rows past the prefix zero-filled); S_t = Q_t K_j^T and O_t += P_t V_j on tcgen05
// with P_t written back over S_t in TMEM (TS-MMA), O kept in TMEM and rescaled lazily; one thread
// per query row for the softmax (see the kernel's comment).
// Backward (attn_bwd_sm100_kernel): per 128-key block x head x sequence, software-pipelined over
// the 64-query tiles that see the block (see the kernel's comment).
// Key blocks are aligned to absolute multiples of 128; only blocks crossing a query's position are
// masked element-wise.
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "tc5.cuh"

namespace tp {

namespace {

using namespace tc5;

constexpr int AT = 128;                   // query rows per CTA, keys per block, head dim
constexpr uint32_t TILE = AT * AT * 2;    // one 128 x 128 bf16 tile (two 64-column swizzle atoms)
constexpr uint32_t HALF = TILE / 2;       // 16 KiB: second 64-column atom
constexpr float LOG2E_F = 1.4426950408889634f;

// K and V in separate rings: K_j is released as soon as S_j is computed (3 stages), V_j after
// O_j = P_j V_j (2 stages), so the loads run two key blocks ahead of the MMAs that need them.
constexpr int NKS = 3, NVS = 2;


__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]: the A operand (bf16, K packed two per 32-bit column) read from TMEM
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void mma_bf16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// byte offset of 16-byte chunk `cc` (0..7) of row `row` inside a 128B-swizzled K-major atom region
__device__ __forceinline__ uint32_t swz(int row, int cc) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((cc ^ (row & 7)) << 4));
}


// ------------------------------------------------------------------ forward, two query tiles
// Per (256 query rows = two 128-row tiles, head, sequence), LPT order. Each K_j / V_j block loaded
// once serves both tiles. TMEM: S_0 (cols 0-127), S_1 (128-255), O_0 (256-383), O_1 (384-511).
//   warp 0      TMA: Q_0, Q_1 once; K_j into a 3-deep ring, V_j into a 2-deep ring;
//   warp 1      MMA (whole warp, one elected lane): per block j, S_t = Q_t K_j^T for both tiles, then
//               O_t += P_t V_j (P_t read from TMEM where the softmax wrote it over S_t);
//   warps 2-5   softmax of tile 0, warps 6-9 of tile 1: thread = query row (its TMEM lane), all 128
//               scores of the block in registers, so the row max needs no exchange; P = exp2(S*scale
//               - m_ref) packed as bf16 into TMEM. O stays in TMEM: it is rescaled (by the owning
//               thread, warp-uniform decision) only when a row's max grows past m_ref + 8 (log2
//               units), so P <= 256 and the common case has no O traffic at all.
// Softmax inner loops, specialised on whether the block crosses the causal diagonal (the mask test
// costs two instructions per element, so the common unmasked case gets its own loop).
template <bool MASK>
__device__ __forceinline__ void row_max_chunk(const uint32_t (&r)[2][32], int col0, int nvis, float (&m4)[4]) {
#pragma unroll
  for (int u = 0; u < 64; ++u) {
    const float x = __uint_as_float(r[u >> 5][u & 31]);
    m4[u & 3] = fmaxf(m4[u & 3], MASK && col0 + u >= nvis ? -INFINITY : x);
  }
}
template <bool MASK>
__device__ __forceinline__ void exp_max_chunk(const uint32_t (&r)[32], int col0, int nvis, float scale_log2, float nm,
                                              float (&rs4)[4], float (&m4)[4], uint32_t (&pk)[64], int pk0) {
#pragma unroll
  for (int u = 0; u < 32; u += 2) {
    float x0 = __uint_as_float(r[u]), x1 = __uint_as_float(r[u + 1]);
    if (MASK) {
      x0 = col0 + u < nvis ? x0 : -INFINITY;
      x1 = col0 + u + 1 < nvis ? x1 : -INFINITY;
    }
    m4[(u >> 1) & 3] = fmaxf(m4[(u >> 1) & 3], fmaxf(x0, x1));
    const float p0 = ex2(fmaf(x0, scale_log2, nm));
    const float p1 = ex2(fmaf(x1, scale_log2, nm));
    rs4[(u >> 1) & 3] += p0 + p1;
    __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
    pk[pk0 + (u >> 1)] = *reinterpret_cast<uint32_t*>(&h);
  }
}
template <bool MASK>
__device__ __forceinline__ void exp_max_chunk16(const uint32_t (&r)[32], int col0, int nvis, float scale_log2,
                                                float nm, float (&rs4)[4], float (&m4)[4], uint32_t (&pk)[16]) {
#pragma unroll
  for (int u = 0; u < 32; u += 2) {
    float x0 = __uint_as_float(r[u]), x1 = __uint_as_float(r[u + 1]);
    if (MASK) {
      x0 = col0 + u < nvis ? x0 : -INFINITY;
      x1 = col0 + u + 1 < nvis ? x1 : -INFINITY;
    }
    const float p0 = ex2(fmaf(x0, scale_log2, nm));
    const float p1 = ex2(fmaf(x1, scale_log2, nm));
    rs4[(u >> 1) & 3] += p0 + p1;
    __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
    pk[u >> 1] = *reinterpret_cast<uint32_t*>(&h);
  }
}
constexpr int F2_THREADS = 320;
struct Fwd2Smem {
  static constexpr uint32_t Q = 0, K = 2 * TILE, V = K + NKS * TILE;
  static constexpr uint32_t BAR = V + NVS * TILE;
  static constexpr uint32_t BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "forward tile set exceeds 227 KB of shared memory");
};
constexpr float RESCALE_LOG2 = 8.f;

// TP_ATTN_TRACE: clock64 timeline of CTA (0, 0, 0), slot (role * 8 + event) * 64 + key block
#define TRF(role, ev, i)                                                                  \
  do {                                                                                    \
    if (trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 64) trace[((role) * 8 + (ev)) * 64 + (i)] = clock64(); \
  } while (0)
__global__ void __launch_bounds__(F2_THREADS, 1)
    attn_fwd2_sm100_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ o, int64_t ldo,
                           float* __restrict__ lse, int s, int c, int l, float scale_log2, int64_t o_sstride,
                           int64_t lse_sstride, long long* trace, int inorder) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc5::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Fwd2Smem::BAR);
  uint64_t* qfull = bars + 0;
  uint64_t* kfull = bars + 1;    // [3]
  uint64_t* kfree = bars + 4;    // [3]
  uint64_t* vfull = bars + 7;    // [2]
  uint64_t* vfree = bars + 9;    // [2]
  uint64_t* sfull = bars + 11;   // [2 tiles]
  uint64_t* pfull = bars + 13;   // [2 tiles] (4 warps each)
  uint64_t* ofull = bars + 15;   // [2 tiles] O_t += P_t V_j complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  // warp index through a shuffle: provably warp-uniform, so the role branches below keep the
  // uniform datapath (descriptor arithmetic in uniform registers for tcgen05.mma)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // raster: the query-tile pairs of one (head, sequence) are consecutive CTAs (heaviest first), so
  // they run concurrently and read that head's K / V blocks from L2 instead of DRAM
  const int head = blockIdx.y, sq = blockIdx.z, r0 = (gridDim.x - 1 - blockIdx.x) * 2 * AT;
  o += sq * o_sstride;
  lse += sq * lse_sstride;
  // key blocks of each tile: tile t covers rows [r0 + t*128, +128) of the slice (absolute c + ...)
  const int ntiles = r0 + AT < l ? 2 : 1;
  // key blocks per tile as scalars (a dynamically indexed array would live in local memory and its
  // values would not be provably warp-uniform in the MMA warp)
  const int nkb0 = (c + min(l, r0 + AT) - 1) / AT + 1, nkb1 = (c + min(l, r0 + 2 * AT) - 1) / AT + 1;
  auto nkb = [&](int t) { return t ? nkb1 : nkb0; };
  const int nkbmax = ntiles > 1 ? nkb1 : nkb0;

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int i = 0; i < NKS; ++i) { mbar_init(kfull + i, 1); mbar_init(kfree + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(vfull + i, 1); mbar_init(vfree + i, 1);
      mbar_init(sfull + i, 1); mbar_init(pfull + i, 4); mbar_init(ofull + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
    // ---------------- TMA producer
    mbar_expect_tx(qfull, 2 * TILE);
    for (int t = 0; t < 2; ++t) {
      tma_load_4d(sm + Fwd2Smem::Q + t * TILE, &tmQ, 0, c + r0 + t * AT, head, sq, qfull);
      tma_load_4d(sm + Fwd2Smem::Q + t * TILE + HALF, &tmQ, 64, c + r0 + t * AT, head, sq, qfull);
    }
    for (int j = 0; j < nkbmax; ++j) {
      const int bk = j % NKS, bv = j & 1;
      if (j >= NKS) mbar_wait(kfree + bk, ((j / NKS) - 1) & 1);
      uint8_t* kd = sm + Fwd2Smem::K + bk * TILE;
      mbar_expect_tx(kfull + bk, TILE);
      tma_load_4d(kd, &tmK, 0, j * AT, head, sq, kfull + bk);
      tma_load_4d(kd + HALF, &tmK, 64, j * AT, head, sq, kfull + bk);
      if (j >= NVS) mbar_wait(vfree + bv, ((j >> 1) - 1) & 1);
      uint8_t* vd = sm + Fwd2Smem::V + bv * TILE;
      mbar_expect_tx(vfull + bv, TILE);
      tma_load_4d(vd, &tmV, 0, j * AT, head, sq, vfull + bv);
      tma_load_4d(vd + HALF, &tmV, 64, j * AT, head, sq, vfull + bv);
    }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idO = idesc_bf16(128, 128, false, true);
    // Issue order O_0 += P_0 V_j, S_0 = Q_0 K_{j+1}^T, O_1 += P_1 V_j, S_1 = Q_1 K_{j+1}^T: the two
    // tiles' softmaxes alternate (ping-pong), each running while the tensor pipe works on the other
    // tile's MMAs.
    auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T (K_j resident)
      const uint32_t k_base = smem_u32(sm + Fwd2Smem::K + (j % NKS) * TILE);
      const uint32_t q_base = smem_u32(sm + Fwd2Smem::Q + t * TILE);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk) {
        const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
        mma_bf16_w(tmem + t * 128, make_desc(q_base + off, 16, 1024), make_desc(k_base + off, 16, 1024), idS, kk > 0);
      }
      mma_commit_w(sfull + t);
      if (lane == 0) TRF(1, 1 + t, j);
    };
    mbar_wait(qfull, 0);
    mbar_wait(kfull, 0);
    if (lane == 0) TRF(1, 0, 0);
    for (int t = 0; t < ntiles; ++t) issue_s(t, 0);
    mma_commit_w(kfree);
    for (int j = 0; j < nkbmax; ++j) {
      const int bv = j & 1;
      const bool next_k = j + 1 < nkbmax;
      bool k_waited = false;
      mbar_wait(vfull + bv, (j >> 1) & 1);
      const uint32_t v_base = smem_u32(sm + Fwd2Smem::V + bv * TILE);
      for (int t = 0; t < ntiles; ++t) {
        if (j >= nkb(t)) continue;
        mbar_wait(pfull + t, j & 1);
        if (lane == 0) TRF(1, 3 + t, j);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT / 16; ++kk)
          mma_bf16_ts_w(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, make_desc(v_base + kk * 2048, HALF, 1024), idO,
                        (j | kk) != 0);
        mma_commit_w(ofull + t);
        if (lane == 0) TRF(1, 5 + t, j);
        if (j + 1 < nkb(t)) {
          if (!k_waited) { mbar_wait(kfull + (j + 1) % NKS, ((j + 1) / NKS) & 1); k_waited = true; }
          if (lane == 0) TRF(1, 0, j + 1);
          // S_t's columns hold P_t, read by O_t += P_t V_j just issued. tcgen05.mma instructions of
          // one thread execute in issue order, so S_{j+1} (issued after it) cannot overwrite P_t
          // before that MMA has read it: no completion wait, the MMA warp goes straight on to the
          // other tile (inorder = 0, TP_ATTN_INORDER=0: wait for O_t += P_t V_j to complete first)
          if (!inorder) mbar_wait(ofull + t, j & 1);
          issue_s(t, j + 1);
        }
      }
      mma_commit_w(vfree + bv);
      if (next_k) mma_commit_w(kfree + (j + 1) % NKS);
    }
  } else if (warp >= 2) {
    // ---------------- softmax: tile t = (warp - 2) / 4, thread = query row of the tile
    const int t = (warp - 2) >> 2, q = warp & 3, row = q * 32 + lane;
    if (t < ntiles) {
      const int qabs = c + r0 + t * AT + row;
      const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
      const uint32_t s_col = t * 128, o_col = 256 + t * 128;
      float m_ref = -INFINITY, lsum = 0.f;
      for (int j = 0; j < nkb(t); ++j) {
        mbar_wait(sfull + t, j & 1);
        if (row == 0) TRF(2 + t, 0, j);
        tc_fence_after();
        const int nvis = qabs - j * AT + 1;  // keys j*128 .. qabs of this block are visible
        // only blocks crossing some row's diagonal need the element mask (warp-uniform branch)
        const bool diag = __any_sync(0xffffffffu, nvis < AT);
        // One pass over the block's 128 scores: P = exp2(S * scale_log2 - m_ref) into registers (packed
        // bf16) while tracking the row max. P is written to TMEM (over S) only after the whole row is
        // read, so the rare case where the max outgrew m_ref + 8 (and always the first block) can
        // rescale O and recompute P from the intact S.
        float rs4[4] = {0.f, 0.f, 0.f, 0.f}, m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        uint32_t pk[64];
        const float nm = -m_ref;
        if (j > 0) {
          // software-pipelined TMEM loads: chunk ch + 1 is in flight while chunk ch is exponentiated
          // (one load latency per block instead of four)
          uint32_t ra[32], rb[32];
          tmem_ld32_nowait(lane_base + s_col, ra);
          tmem_wait_ld();
#pragma unroll
          for (int ch = 0; ch < AT / 32; ch += 2) {
            tmem_ld32_nowait(lane_base + s_col + (ch + 1) * 32, rb);
            if (diag) exp_max_chunk<true>(ra, ch * 32, nvis, scale_log2, nm, rs4, m4, pk, ch * 16);
            else exp_max_chunk<false>(ra, ch * 32, nvis, scale_log2, nm, rs4, m4, pk, ch * 16);
            tmem_wait_ld();
            if (ch + 2 < AT / 32) tmem_ld32_nowait(lane_base + s_col + (ch + 2) * 32, ra);
            if (diag) exp_max_chunk<true>(rb, (ch + 1) * 32, nvis, scale_log2, nm, rs4, m4, pk, (ch + 1) * 16);
            else exp_max_chunk<false>(rb, (ch + 1) * 32, nvis, scale_log2, nm, rs4, m4, pk, (ch + 1) * 16);
            if (ch + 2 < AT / 32) tmem_wait_ld();
          }
        } else {
          // first block: only the max (m_ref = -inf would make every P infinite)
#pragma unroll
          for (int ch = 0; ch < AT / 32; ch += 2) {
            uint32_t r[2][32];
            tmem_ld32_nowait(lane_base + s_col + ch * 32, r[0]);
            tmem_ld32_nowait(lane_base + s_col + ch * 32 + 32, r[1]);
            tmem_wait_ld();
            if (diag) row_max_chunk<true>(r, ch * 32, nvis, m4);
            else row_max_chunk<false>(r, ch * 32, nvis, m4);
          }
        }
        if (row == 0) TRF(2 + t, 1, j);
        const float m_blk = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;  // scale > 0
        // lazy rescale: move the reference max only when it grew by more than 2^8
        const bool grow = m_blk > m_ref + RESCALE_LOG2;
        if (__any_sync(0xffffffffu, grow)) {
          const float m_new = grow ? m_blk : m_ref;
          const float f = ex2(m_ref - m_new);  // 0 on the first block (m_ref = -inf), 1 if unchanged
          if (j >= 1) {
            // O_t += P_t V_{j-1} must be complete before O is rewritten
            mbar_wait(ofull + t, (j - 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int ch = 0; ch < AT / 32; ++ch) {
              uint32_t r[32];
              tmem_ld32_nowait(lane_base + o_col + ch * 32, r);
              tmem_wait_ld();
#pragma unroll
              for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * f);
              tmem_st32(lane_base + o_col + ch * 32, r);
            }
            tmem_wait_st();
          }
          lsum *= f;
          m_ref = m_new;
          // recompute P with the new reference
          const float nm2 = -m_ref;
#pragma unroll
          for (int i = 0; i < 4; ++i) rs4[i] = 0.f;
#pragma unroll
          for (int ch = 0; ch < AT / 32; ++ch) {
            uint32_t r[32];
            tmem_ld32_nowait(lane_base + s_col + ch * 32, r);
            tmem_wait_ld();
            uint32_t pk16[16];
            float mm[4];
            exp_max_chunk16<true>(r, ch * 32, nvis, scale_log2, nm2, rs4, mm, pk16);
#pragma unroll
            for (int u = 0; u < 16; ++u) pk[ch * 16 + u] = pk16[u];
          }
        }
        const float rs = (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
        // P (bf16, two per column) over S_t's first 64 columns
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t pk16[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) pk16[u] = pk[ch * 16 + u];
          tmem_st16(lane_base + s_col + ch * 16, pk16);
        }
        lsum += rs;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfull + t);
        if (row == 0) TRF(2 + t, 2, j);
      }
      // epilogue: O / lsum -> bf16 rows, lse
      mbar_wait(ofull + t, (nkb(t) - 1) & 1);
      tc_fence_after();
      const int r = r0 + t * AT + row;
      const float inv = 1.f / lsum;
      bf16* orow = o + (int64_t)r * ldo + head * AT;
#pragma unroll 1
      for (int ch = 0; ch < AT / 32; ++ch) {
        uint32_t rr[32];
        tmem_ld32_nowait(lane_base + o_col + ch * 32, rr);
        tmem_wait_ld();
        if (r < l) {
#pragma unroll
          for (int u = 0; u < 32; u += 8) {
            float v8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v8[e] = __uint_as_float(rr[u + e]) * inv;
            store8<bf16>(orow + ch * 32 + u, v8);
          }
        }
      }
      if (r < l) lse[(int64_t)head * s + c + r] = (m_ref + log2f(lsum)) / LOG2E_F;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ forward, one query tile per CTA
// Per (128 query rows, head, sequence), heaviest first. TMEM: S_0 (cols 0-127), S_1 (128-255), O
// (256-383): S is double-buffered, so S_{j+1} = Q K_{j+1}^T is computed while the softmax works on
// S_j — the two-tile kernel above must wait for O += P_j V_j before it can reuse S (P lives in S's
// columns), which serialises softmax -> PV -> S per tile. The price is K_j / V_j read once per tile
// instead of once per two tiles (shared-memory traffic ~160 KB per 128 x 128 block vs MMA 1024 clk).
//   warp 0   TMA: Q once; K_j into a 3-deep ring, V_j into a 2-deep ring;
//   warp 1   MMA: S_{j+1} (into buffer (j+1) & 1 once O += P_{j-1} V_{j-1} has read it), then
//            O += P_j V_j (P_j from buffer j & 1, TS-MMA);
//   warps 2-5 softmax, thread = query row (same one-pass exp2 / lazy-rescale scheme as above).
constexpr int F1_THREADS = 192;
struct Fwd1Smem {
  static constexpr uint32_t Q = 0, K = TILE, V = K + NKS * TILE;
  static constexpr uint32_t BAR = V + NVS * TILE;
  static constexpr uint32_t BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "forward tile set exceeds 227 KB of shared memory");
};

__global__ void __launch_bounds__(F1_THREADS, 1)
    attn_fwd1_sm100_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ o, int64_t ldo,
                           float* __restrict__ lse, int s, int c, int l, float scale_log2, int64_t o_sstride,
                           int64_t lse_sstride, int inorder) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc5::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Fwd1Smem::BAR);
  uint64_t* qfull = bars + 0;
  uint64_t* kfull = bars + 1;    // [3]
  uint64_t* kfree = bars + 4;    // [3]
  uint64_t* vfull = bars + 7;    // [2]
  uint64_t* vfree = bars + 9;    // [2]
  uint64_t* sfull = bars + 11;   // [2] S buffer b holds S_j, j & 1 == b
  uint64_t* pfull = bars + 13;   // [2] P_j written over buffer b (4 warps)
  uint64_t* ofull = bars + 15;   // [2] O += P_j V_j complete (j & 1 == b)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  // warp index through a shuffle: provably warp-uniform, so the role branches below keep the
  // uniform datapath (descriptor arithmetic in uniform registers for tcgen05.mma)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int head = blockIdx.y, sq = blockIdx.z, r0 = (gridDim.x - 1 - blockIdx.x) * AT;
  o += sq * o_sstride;
  lse += sq * lse_sstride;
  const int nkb = (c + min(l, r0 + AT) - 1) / AT + 1;

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int i = 0; i < NKS; ++i) { mbar_init(kfull + i, 1); mbar_init(kfree + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(vfull + i, 1); mbar_init(vfree + i, 1);
      mbar_init(sfull + i, 1); mbar_init(pfull + i, 4); mbar_init(ofull + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
    mbar_expect_tx(qfull, TILE);
    tma_load_4d(sm + Fwd1Smem::Q, &tmQ, 0, c + r0, head, sq, qfull);
    tma_load_4d(sm + Fwd1Smem::Q + HALF, &tmQ, 64, c + r0, head, sq, qfull);
    for (int j = 0; j < nkb; ++j) {
      const int bk = j % NKS, bv = j & 1;
      if (j >= NKS) mbar_wait(kfree + bk, ((j / NKS) - 1) & 1);
      uint8_t* kd = sm + Fwd1Smem::K + bk * TILE;
      mbar_expect_tx(kfull + bk, TILE);
      tma_load_4d(kd, &tmK, 0, j * AT, head, sq, kfull + bk);
      tma_load_4d(kd + HALF, &tmK, 64, j * AT, head, sq, kfull + bk);
      if (j >= NVS) mbar_wait(vfree + bv, ((j >> 1) - 1) & 1);
      uint8_t* vd = sm + Fwd1Smem::V + bv * TILE;
      mbar_expect_tx(vfull + bv, TILE);
      tma_load_4d(vd, &tmV, 0, j * AT, head, sq, vfull + bv);
      tma_load_4d(vd + HALF, &tmV, 64, j * AT, head, sq, vfull + bv);
    }
    }
  } else if (warp == 1) {
    constexpr uint32_t idS = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idO = idesc_bf16(128, 128, false, true);
    const uint32_t q_base = smem_u32(sm + Fwd1Smem::Q);
    auto issue_s = [&](int j) {  // S_j = Q K_j^T into buffer j & 1 (K_j resident)
      const uint32_t k_base = smem_u32(sm + Fwd1Smem::K + (j % NKS) * TILE);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk) {
        const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
        mma_bf16_w(tmem + (j & 1) * 128, make_desc(q_base + off, 16, 1024), make_desc(k_base + off, 16, 1024), idS, kk > 0);
      }
      mma_commit_w(sfull + (j & 1));
      mma_commit_w(kfree + j % NKS);
    };
    mbar_wait(qfull, 0);
    mbar_wait(kfull, 0);
    issue_s(0);
    for (int j = 0; j < nkb; ++j) {
      const int b = j & 1;
      if (j + 1 < nkb) {
        mbar_wait(kfull + (j + 1) % NKS, ((j + 1) / NKS) & 1);
        // buffer (j + 1) & 1 held P_{j-1}: O += P_{j-1} V_{j-1}, issued earlier, reads it first
        // (in-order tcgen05.mma execution; inorder = 0: wait for its completion)
        if (j >= 1 && !inorder) mbar_wait(ofull + ((j - 1) & 1), ((j - 1) >> 1) & 1);
        issue_s(j + 1);
      }
      mbar_wait(vfull + b, (j >> 1) & 1);
      mbar_wait(pfull + b, (j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_base = smem_u32(sm + Fwd1Smem::V + b * TILE);
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk)
        mma_bf16_ts_w(tmem + 256, tmem + b * 128 + kk * 8, make_desc(v_base + kk * 2048, HALF, 1024), idO,
                      (j | kk) != 0);
      mma_commit_w(ofull + b);
      mma_commit_w(vfree + b);
    }
  } else if (warp >= 2) {
    // ---------------- softmax: thread = query row (TMEM lane)
    const int q = warp & 3, row = q * 32 + lane;
    const int qabs = c + r0 + row;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    constexpr uint32_t o_col = 256;
    float m_ref = -INFINITY, lsum = 0.f;
    for (int j = 0; j < nkb; ++j) {
      const int b = j & 1;
      const uint32_t s_col = b * 128;
      mbar_wait(sfull + b, (j >> 1) & 1);
      tc_fence_after();
      const int nvis = qabs - j * AT + 1;
      const bool diag = __any_sync(0xffffffffu, nvis < AT);
      float rs4[4] = {0.f, 0.f, 0.f, 0.f}, m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      uint32_t pk[64];
      const float nm = -m_ref;
      if (j > 0) {
        uint32_t ra[32], rb[32];  // software-pipelined TMEM loads (see the two-tile kernel)
        tmem_ld32_nowait(lane_base + s_col, ra);
        tmem_wait_ld();
#pragma unroll
        for (int ch = 0; ch < AT / 32; ch += 2) {
          tmem_ld32_nowait(lane_base + s_col + (ch + 1) * 32, rb);
          if (diag) exp_max_chunk<true>(ra, ch * 32, nvis, scale_log2, nm, rs4, m4, pk, ch * 16);
          else exp_max_chunk<false>(ra, ch * 32, nvis, scale_log2, nm, rs4, m4, pk, ch * 16);
          tmem_wait_ld();
          if (ch + 2 < AT / 32) tmem_ld32_nowait(lane_base + s_col + (ch + 2) * 32, ra);
          if (diag) exp_max_chunk<true>(rb, (ch + 1) * 32, nvis, scale_log2, nm, rs4, m4, pk, (ch + 1) * 16);
          else exp_max_chunk<false>(rb, (ch + 1) * 32, nvis, scale_log2, nm, rs4, m4, pk, (ch + 1) * 16);
          if (ch + 2 < AT / 32) tmem_wait_ld();
        }
      } else {
#pragma unroll
        for (int ch = 0; ch < AT / 32; ch += 2) {
          uint32_t r[2][32];
          tmem_ld32_nowait(lane_base + s_col + ch * 32, r[0]);
          tmem_ld32_nowait(lane_base + s_col + ch * 32 + 32, r[1]);
          tmem_wait_ld();
          if (diag) row_max_chunk<true>(r, ch * 32, nvis, m4);
          else row_max_chunk<false>(r, ch * 32, nvis, m4);
        }
      }
      const float m_blk = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
      const bool grow = m_blk > m_ref + RESCALE_LOG2;
      if (__any_sync(0xffffffffu, grow)) {
        const float m_new = grow ? m_blk : m_ref;
        const float f = ex2(m_ref - m_new);
        if (j >= 1) {
          mbar_wait(ofull + ((j - 1) & 1), ((j - 1) >> 1) & 1);  // O += P_{j-1} V_{j-1} complete
          tc_fence_after();
#pragma unroll 1
          for (int ch = 0; ch < AT / 32; ++ch) {
            uint32_t r[32];
            tmem_ld32_nowait(lane_base + o_col + ch * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * f);
            tmem_st32(lane_base + o_col + ch * 32, r);
          }
          tmem_wait_st();
        }
        lsum *= f;
        m_ref = m_new;
        const float nm2 = -m_ref;
#pragma unroll
        for (int i = 0; i < 4; ++i) rs4[i] = 0.f;
#pragma unroll
        for (int ch = 0; ch < AT / 32; ++ch) {
          uint32_t r[32];
          tmem_ld32_nowait(lane_base + s_col + ch * 32, r);
          tmem_wait_ld();
          uint32_t pk16[16];
          float mm[4];
          exp_max_chunk16<true>(r, ch * 32, nvis, scale_log2, nm2, rs4, mm, pk16);
#pragma unroll
          for (int u = 0; u < 16; ++u) pk[ch * 16 + u] = pk16[u];
        }
      }
      const float rsum = (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t pk16[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) pk16[u] = pk[ch * 16 + u];
        tmem_st16(lane_base + s_col + ch * 16, pk16);
      }
      lsum += rsum;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(pfull + b);
    }
    mbar_wait(ofull + ((nkb - 1) & 1), ((nkb - 1) >> 1) & 1);
    tc_fence_after();
    const int r = r0 + row;
    const float inv = 1.f / lsum;
    bf16* orow = o + (int64_t)r * ldo + head * AT;
#pragma unroll 1
    for (int ch = 0; ch < AT / 32; ++ch) {
      uint32_t rr[32];
      tmem_ld32_nowait(lane_base + o_col + ch * 32, rr);
      tmem_wait_ld();
      if (r < l) {
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          float v8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v8[e] = __uint_as_float(rr[u + e]) * inv;
          store8<bf16>(orow + ch * 32 + u, v8);
        }
      }
    }
    if (r < l) lse[(int64_t)head * s + c + r] = (m_ref + log2f(lsum)) / LOG2E_F;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ forward, two query tiles, 64-key blocks
// The two-tile kernel above serialises, per tile, softmax(j) -> O += P_j V_j -> S_{j+1} = Q K_{j+1}^T
// (P_j lives in S's TMEM columns, and S is single-buffered because O_0, O_1, S_0, S_1 fill the 512
// columns). Here key blocks are 64 wide, so each tile's S is double-buffered in the same 128
// columns: S_{t,b} = cols t*128 + b*64 (P_{t,b} packed into its first 32), O_t at 256 + t*128.
// S_{j+1} is computed while the softmax works on S_j, and the softmax runs block after block
// without waiting for the tensor pipe. The price: S MMAs at N = 64 (shared-memory bound, 2/3 rate).
//   warp 0     TMA: Q_0, Q_1 once; K_j / V_j (64 x 128) into 4-deep rings;
//   warp 1     MMA: per block j and tile t, once the softmax has written P_t(j): O_t += P_t(j) V_j,
//              then S_t(j+2) into the same buffer (tcgen05.mma executes in issue order, so it cannot
//              overwrite P_t(j) before that MMA has read it): S runs two blocks ahead;
//   warps 2-9  softmax (4 per tile, thread = query row), the one-pass lazy-rescale scheme above.
constexpr int BK3 = 64;                         // keys per block
constexpr uint32_t KT3 = BK3 * AT * 2;          // 16 KiB: [64 keys][128 d]
constexpr uint32_t KHALF3 = KT3 / 2;            // 8 KiB: second 64-column (d) atom
constexpr int NK3 = 4, NV3 = 4;
struct Fwd3Smem {
  static constexpr uint32_t Q = 0, K = 2 * TILE, V = K + NK3 * KT3;
  static constexpr uint32_t BAR = V + NV3 * KT3;
  static constexpr uint32_t BYTES = BAR + 512 + 1024;
  static_assert(BYTES <= 232448, "forward tile set exceeds 227 KB of shared memory");
};
template <bool MASK>
__device__ __forceinline__ void exp_max_chunk32(const uint32_t (&r)[32], int col0, int nvis, float scale_log2,
                                                float nm, float (&rs4)[4], float (&m4)[4], uint32_t (&pk)[32],
                                                int pk0) {
#pragma unroll
  for (int u = 0; u < 32; u += 2) {
    float x0 = __uint_as_float(r[u]), x1 = __uint_as_float(r[u + 1]);
    if (MASK) {
      x0 = col0 + u < nvis ? x0 : -INFINITY;
      x1 = col0 + u + 1 < nvis ? x1 : -INFINITY;
    }
    m4[(u >> 1) & 3] = fmaxf(m4[(u >> 1) & 3], fmaxf(x0, x1));
    const float p0 = ex2(fmaf(x0, scale_log2, nm));
    const float p1 = ex2(fmaf(x1, scale_log2, nm));
    rs4[(u >> 1) & 3] += p0 + p1;
    __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
    pk[pk0 + (u >> 1)] = *reinterpret_cast<uint32_t*>(&h);
  }
}

__global__ void __launch_bounds__(F2_THREADS, 1)
    attn_fwd3_sm100_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ o, int64_t ldo,
                           float* __restrict__ lse, int s, int c, int l, float scale_log2, int64_t o_sstride,
                           int64_t lse_sstride, long long* trace) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc5::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Fwd3Smem::BAR);
  uint64_t* qfull = bars + 0;
  uint64_t* kfull = bars + 1;    // [NK3]
  uint64_t* kfree = bars + 5;    // [NK3]
  uint64_t* vfull = bars + 9;    // [NV3]
  uint64_t* vfree = bars + 13;   // [NV3]
  uint64_t* sfull = bars + 17;   // [tile][buffer]: S_t(j) in buffer j & 1
  uint64_t* pfull = bars + 21;   // [tile][buffer]: P_t(j) written (4 warps)
  uint64_t* ofull = bars + 25;   // [tile][buffer]: O_t += P_t(j) V_j complete, buffer j & 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 29);

  // warp index through a shuffle: provably warp-uniform, so ptxas can use the uniform datapath for
  // the MMA warp's descriptor arithmetic
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int head = blockIdx.y, sq = blockIdx.z, r0 = (gridDim.x - 1 - blockIdx.x) * 2 * AT;
  o += sq * o_sstride;
  lse += sq * lse_sstride;
  const int ntiles = r0 + AT < l ? 2 : 1;
  // key blocks per tile as scalars (a dynamically indexed array lands in local memory, and values
  // loaded from it are not provably warp-uniform: the MMA warp's control flow then loses the uniform
  // datapath and every tcgen05.mma pays an elect + register broadcast)
  const int nkb0 = (c + min(l, r0 + AT) - 1) / BK3 + 1, nkb1 = (c + min(l, r0 + 2 * AT) - 1) / BK3 + 1;
  auto nkb = [&](int t) { return t ? nkb1 : nkb0; };
  const int nkbmax = ntiles > 1 ? nkb1 : nkb0;

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int i = 0; i < NK3; ++i) { mbar_init(kfull + i, 1); mbar_init(kfree + i, 1); }
    for (int i = 0; i < NV3; ++i) { mbar_init(vfull + i, 1); mbar_init(vfree + i, 1); }
    for (int i = 0; i < 4; ++i) { mbar_init(sfull + i, 1); mbar_init(pfull + i, 4); mbar_init(ofull + i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // warp-uniform role branches (lets ptxas use the uniform datapath in the MMA warp)
    if (lane == 0) {
    // ---------------- TMA producer
    mbar_expect_tx(qfull, 2 * TILE);
    for (int t = 0; t < 2; ++t) {
      tma_load_4d(sm + Fwd3Smem::Q + t * TILE, &tmQ, 0, c + r0 + t * AT, head, sq, qfull);
      tma_load_4d(sm + Fwd3Smem::Q + t * TILE + HALF, &tmQ, 64, c + r0 + t * AT, head, sq, qfull);
    }
    for (int j = 0; j < nkbmax; ++j) {
      const int bk = j % NK3, bv = j % NV3;
      if (j >= NK3) mbar_wait(kfree + bk, ((j / NK3) - 1) & 1);
      uint8_t* kd = sm + Fwd3Smem::K + bk * KT3;
      mbar_expect_tx(kfull + bk, KT3);
      tma_load_4d(kd, &tmK, 0, j * BK3, head, sq, kfull + bk);
      tma_load_4d(kd + KHALF3, &tmK, 64, j * BK3, head, sq, kfull + bk);
      if (j >= NV3) mbar_wait(vfree + bv, ((j / NV3) - 1) & 1);
      uint8_t* vd = sm + Fwd3Smem::V + bv * KT3;
      mbar_expect_tx(vfull + bv, KT3);
      tma_load_4d(vd, &tmV, 0, j * BK3, head, sq, vfull + bv);
      tma_load_4d(vd + KHALF3, &tmV, 64, j * BK3, head, sq, vfull + bv);
    }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    constexpr uint32_t idS = idesc_bf16(128, BK3, false, false);
    constexpr uint32_t idO = idesc_bf16(128, 128, false, true);
    // shared-memory addresses as 32-bit arithmetic on the (warp-uniform) window base, so ptxas keeps
    // the descriptors in uniform registers (no per-MMA elect / R2UR broadcast)
    const uint32_t sbase = smem_u32(smem_raw) + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    auto issue_s1 = [&](int t, int j) {  // S_t(j) = Q_t K_j^T into buffer j & 1 (K_j resident)
      const uint32_t k_base = sbase + Fwd3Smem::K + (j % NK3) * KT3;
      const uint32_t q_base = sbase + Fwd3Smem::Q + t * TILE;
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk)
        mma_bf16_w(tmem + t * 128 + (j & 1) * BK3, make_desc(q_base + (kk >> 2) * HALF + (kk & 3) * 32, 16, 1024),
                   make_desc(k_base + (kk >> 2) * KHALF3 + (kk & 3) * 32, 16, 1024), idS, kk > 0);
      mma_commit_w(sfull + t * 2 + (j & 1));
    };
    mbar_wait(qfull, 0);
    for (int j = 0; j < 2 && j < nkbmax; ++j) {  // S(0), S(1): both buffers
      mbar_wait(kfull + j, 0);
      for (int t = 0; t < ntiles; ++t)
        if (j < nkb(t)) issue_s1(t, j);
      mma_commit_w(kfree + j);
    }
    // per block j and tile t, as soon as the softmax has written P_t(j): O_t += P_t(j) V_j, then
    // S_t(j+2) into the same buffer (in issue order after the MMA that reads P_t(j)), so S runs two
    // blocks ahead of the softmax
    for (int j = 0; j < nkbmax; ++j) {
      const int bv = j % NV3, b = j & 1;
      mbar_wait(vfull + bv, (j / NV3) & 1);
      if (lane == 0) TRF(1, 0, j);
      const uint32_t v_base = sbase + Fwd3Smem::V + bv * KT3;
      bool k_waited = false;
      for (int t = 0; t < ntiles; ++t) {
        if (j >= nkb(t)) continue;
        mbar_wait(pfull + t * 2 + b, (j >> 1) & 1);
        if (lane == 0) TRF(1, 1 + t, j);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BK3 / 16; ++kk)
          mma_bf16_ts_w(tmem + 256 + t * 128, tmem + t * 128 + b * BK3 + kk * 8, make_desc(v_base + kk * 2048, KHALF3, 1024),
                        idO, (j | kk) != 0);
        mma_commit_w(ofull + t * 2 + b);
        if (lane == 0) TRF(1, 3 + t, j);
        if (j + 2 < nkb(t)) {
          if (!k_waited) { mbar_wait(kfull + (j + 2) % NK3, ((j + 2) / NK3) & 1); k_waited = true; }
          issue_s1(t, j + 2);
          if (lane == 0) TRF(1, 5 + t, j + 2);
        }
      }
      mma_commit_w(vfree + bv);
      if (k_waited) mma_commit_w(kfree + (j + 2) % NK3);
    }
  } else if (warp >= 2) {
    // ---------------- softmax: tile t = (warp - 2) / 4, thread = query row of the tile
    const int t = (warp - 2) >> 2, q = warp & 3, row = q * 32 + lane;
    if (t < ntiles) {
      const int qabs = c + r0 + t * AT + row;
      const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
      const uint32_t o_col = 256 + t * 128;
      float m_ref = -INFINITY, lsum = 0.f;
      for (int j = 0; j < nkb(t); ++j) {
        const int b = j & 1;
        const uint32_t s_col = t * 128 + b * BK3;
        if (row == 0) TRF(2 + t, 0, j);
        mbar_wait(sfull + t * 2 + b, (j >> 1) & 1);
        if (row == 0) TRF(2 + t, 1, j);
        tc_fence_after();
        const int nvis = qabs - j * BK3 + 1;
        const bool diag = __any_sync(0xffffffffu, nvis < BK3);
        float rs4[4] = {0.f, 0.f, 0.f, 0.f}, m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        uint32_t pk[32];
        const float nm = -m_ref;
        {
          uint32_t r[2][32];
          tmem_ld32_nowait(lane_base + s_col, r[0]);
          tmem_ld32_nowait(lane_base + s_col + 32, r[1]);
          tmem_wait_ld();
          if (j > 0) {
            if (diag) {
              exp_max_chunk32<true>(r[0], 0, nvis, scale_log2, nm, rs4, m4, pk, 0);
              exp_max_chunk32<true>(r[1], 32, nvis, scale_log2, nm, rs4, m4, pk, 16);
            } else {
              exp_max_chunk32<false>(r[0], 0, nvis, scale_log2, nm, rs4, m4, pk, 0);
              exp_max_chunk32<false>(r[1], 32, nvis, scale_log2, nm, rs4, m4, pk, 16);
            }
          } else {
            if (diag) row_max_chunk<true>(r, 0, nvis, m4);
            else row_max_chunk<false>(r, 0, nvis, m4);
          }
        }
        const float m_blk = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
        const bool grow = m_blk > m_ref + RESCALE_LOG2;
        if (__any_sync(0xffffffffu, grow)) {
          const float m_new = grow ? m_blk : m_ref;
          const float f = ex2(m_ref - m_new);
          if (j >= 1) {
            // O_t += P_t(j-1) V_{j-1} complete (its buffer's previous phase, P_t(j-3), completed before
            // S_t(j) was computed: in-order MMAs)
            mbar_wait(ofull + t * 2 + ((j - 1) & 1), ((j - 1) >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int ch = 0; ch < AT / 32; ++ch) {
              uint32_t r[32];
              tmem_ld32_nowait(lane_base + o_col + ch * 32, r);
              tmem_wait_ld();
#pragma unroll
              for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * f);
              tmem_st32(lane_base + o_col + ch * 32, r);
            }
            tmem_wait_st();
          }
          lsum *= f;
          m_ref = m_new;
          const float nm2 = -m_ref;
#pragma unroll
          for (int i = 0; i < 4; ++i) rs4[i] = 0.f;
#pragma unroll
          for (int ch = 0; ch < BK3 / 32; ++ch) {
            uint32_t r[32];
            tmem_ld32_nowait(lane_base + s_col + ch * 32, r);
            tmem_wait_ld();
            uint32_t pk16[16];
            float mm[4];
            exp_max_chunk16<true>(r, ch * 32, nvis, scale_log2, nm2, rs4, mm, pk16);
#pragma unroll
            for (int u = 0; u < 16; ++u) pk[ch * 16 + u] = pk16[u];
          }
        }
        const float rsum = (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t pk16[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) pk16[u] = pk[ch * 16 + u];
          tmem_st16(lane_base + s_col + ch * 16, pk16);
        }
        lsum += rsum;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfull + t * 2 + b);
        if (row == 0) TRF(2 + t, 2, j);
      }
      // epilogue: the last O_t += P V complete (commits track every earlier MMA of the thread)
      const int jl = nkb(t) - 1;
      mbar_wait(ofull + t * 2 + (jl & 1), (jl >> 1) & 1);
      tc_fence_after();
      const int r = r0 + t * AT + row;
      const float inv = 1.f / lsum;
      bf16* orow = o + (int64_t)r * ldo + head * AT;
#pragma unroll 1
      for (int ch = 0; ch < AT / 32; ++ch) {
        uint32_t rr[32];
        tmem_ld32_nowait(lane_base + o_col + ch * 32, rr);
        tmem_wait_ld();
        if (r < l) {
#pragma unroll
          for (int u = 0; u < 32; u += 8) {
            float v8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v8[e] = __uint_as_float(rr[u + e]) * inv;
            store8<bf16>(orow + ch * 32 + u, v8);
          }
        }
      }
      if (r < l) lse[(int64_t)head * s + c + r] = (m_ref + log2f(lsum)) / LOG2E_F;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ======================================================================== backward
// Per (128-key block of the prefix [0, c+l), head, sequence); loop over the slice's 64-query tiles
// that can see the block. The tile loop is software-pipelined so the tensor pipe never waits for
// the softmax-gradient warps: S^T / dP^T of tile i+1 are computed while tile i is in the softmax.
// TMEM (512 columns):
//   buffer b = i & 1 at b*128: S^T [128 keys x 64 q] (cols 0-63) then P^T (bf16, packed over the S
//   columns), dP^T (cols 64-127) then dQ^T [128 d x 64 q] of the same tile;
//   dV at 256, dK at 384 (fp32 [128 keys x 128 d], accumulated over the tiles).
//   S^T = K Q^T, dP^T = V dO^T                                  (M=128 keys, N=64, K=d)
//   softmax warps (thread = key row): P^T = exp2(S^T scale - lse) -> TMEM, dS^T = P^T (dP^T - D) -> smem
//   dV += P^T dO  (A = P^T from TMEM), dK += dS^T Q             (M=128 keys, N=d, K=64; Q/dO MN-major B)
//   dQ^T = K^T dS^T                                             (M=d, N=64 q, K=128 keys; K as MN-major A)
//   dQ^T is drained by the softmax warps into shared memory and added to dq_acc[l][H] by one TMA
//   reduce-add per tile; dK (x scale) / dV are written or added to the fp32 prefix accumulators once.
// Shared memory: K, V (32 KiB each), a 3-deep Q / dO ring (16 KiB tiles), dS^T double-buffered,
// the fp32 dQ staging tile.
constexpr int BQB = 64;                          // query rows per tile (backward)
constexpr uint32_t QT = BQB * AT * 2;            // 16 KiB: [64 q][128 d]
constexpr uint32_t QHALF = QT / 2;               // 8 KiB: second 64-column atom
constexpr uint32_t PT = AT * BQB * 2;            // 16 KiB: [128 keys][64 q] (one atom wide)
constexpr int NQB = 3;                           // Q / dO ring depth
constexpr int BWD_THREADS = 448;                 // TMA, MMA, 8 softmax-gradient warps, 4 dQ drain warps

struct BwdSmem {
  static constexpr uint32_t K = 0, V = TILE, Q = 2 * TILE, O = Q + NQB * QT, DS = O + NQB * QT;
  static constexpr uint32_t DQ = DS + 2 * PT;  // fp32 [64 q][128 d]
  static constexpr uint32_t LD = DQ + 32768;   // fp32 [3 ring slots][lse*log2e[64], D[64]]
  static constexpr uint32_t BAR = LD + NQB * 512;
  static constexpr uint32_t BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "backward tile set exceeds 227 KB of shared memory");
};

// DQ = false: dK / dV only (the split backward: dQ comes from attn_bwd_dq_sm100_kernel) — no dQ^T
// MMA, no dS^T shared-memory copy, no drain warps.
template <bool DQ>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                          const __grid_constant__ CUtensorMap tmdQ, const __grid_constant__ CUtensorMap tmdK,
                          const __grid_constant__ CUtensorMap tmdV, const float* __restrict__ ldg, int s, int c, int l,
                          float scale, float scale_log2, int accumulate, int nheads, volatile int* dbg,
                          long long* trace, int pf_dist, const float* __restrict__ dk_raw,
                          const float* __restrict__ dv_raw, int64_t dkv_sstride, bf16* __restrict__ dkv_out,
                          int64_t ldq, int64_t dq_sstride, int inorder) {
  extern __shared__ uint8_t smem_raw[];
#define DBG(role, v)                                                                    \
  do {                                                                                  \
    if (dbg) { dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + (role)] = (v); __threadfence_system(); } \
  } while (0)
  // TP_ATTN_TRACE: clock64 timeline of CTA (0, 0), slot (role * 8 + event) * 64 + tile
#define TRC(role, ev, i)                                                                  \
  do {                                                                                    \
    if (trace && blockIdx.x == 0 && blockIdx.y == 0 && (i) < 64) trace[((role) * 8 + (ev)) * 64 + (i)] = clock64(); \
  } while (0)
  // 1024-aligned base derived by pointer arithmetic on the __shared__ array (not through an
  // integer cast), so the compiler keeps the shared state space: LDS/STS instead of generic LD/ST
  uint8_t* sm = smem_raw + ((1024u - (tc5::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + BwdSmem::BAR);
  uint64_t* kvfull = bars + 0;
  uint64_t* qfull = bars + 1;    // [3] Q / dO tile landed
  uint64_t* qfree = bars + 4;    // [3] dV / dK MMAs of the tile done (Q, dO, P^T consumed)
  uint64_t* sfull = bars + 7;    // [2] S^T, dP^T in TMEM buffer
  uint64_t* pfull = bars + 9;    // [2] P^T in TMEM, dS^T in smem (8 warps)
  uint64_t* dsfree = bars + 11;  // [2] dK / dQ MMAs done reading dS^T
  uint64_t* dqfull = bars + 13;  // [2] dQ^T in TMEM
  uint64_t* dqfree = bars + 15;  // [2] dQ^T drained (4 warps)
  uint64_t* done = bars + 17;
  uint64_t* dpfull = bars + 18;  // [2] dP^T in TMEM buffer (sfull: S^T)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  // warp index through a shuffle: provably warp-uniform, so the role branches below keep the
  // uniform datapath (descriptor arithmetic in uniform registers for tcgen05.mma)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // raster: the key blocks of one (sequence, head) are consecutive CTAs (heaviest, key block 0,
  // first), so they run concurrently: that head's Q / dO tiles are read from DRAM once and shared
  // through L2, and the fp32 dQ reduce-adds of all its key blocks meet in L2
  const int head = blockIdx.y % nheads, sq = blockIdx.y / nheads, key0 = blockIdx.x * AT;
  ldg += ((int64_t)sq * nheads + head) * ((l + BQB - 1) / BQB) * (2 * BQB);
  const int qt0 = max(0, key0 - c) / BQB, nqt = (l + BQB - 1) / BQB;
  const int ntile = nqt - qt0;  // >= 1 because key0 < c + l

  if (threadIdx.x == 0) {
    mbar_init(kvfull, 1);
    for (int i = 0; i < NQB; ++i) { mbar_init(qfull + i, 1); mbar_init(qfree + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(sfull + i, 1); mbar_init(dpfull + i, 1); mbar_init(pfull + i, 8); mbar_init(dsfree + i, 1);
      mbar_init(dqfull + i, 1); mbar_init(dqfree + i, 4);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) DBG(6, ntile);
  constexpr uint32_t T_DV = 256, T_DK = 384;

  if (warp == 0) {
    if (lane == 0) {
    // ---------------- TMA producer: K, V once; Q_i, dO_i through the 3-deep ring
    mbar_expect_tx(kvfull, 2 * TILE);
    tma_load_4d(sm + BwdSmem::K, &tmK, 0, key0, head, sq, kvfull);
    tma_load_4d(sm + BwdSmem::K + HALF, &tmK, 64, key0, head, sq, kvfull);
    tma_load_4d(sm + BwdSmem::V, &tmV, 0, key0, head, sq, kvfull);
    tma_load_4d(sm + BwdSmem::V + HALF, &tmV, 64, key0, head, sq, kvfull);
    for (int i = 0; i < ntile; ++i) {
      const int b = i % NQB, qt = qt0 + i;
      DBG(0, 100 + i);
      if (i >= NQB) mbar_wait(qfree + b, ((i / NQB) - 1) & 1);
      TRC(0, 0, i);
      uint8_t* qd = sm + BwdSmem::Q + b * QT;
      uint8_t* od = sm + BwdSmem::O + b * QT;
      mbar_expect_tx(qfull + b, 2 * QT + 2 * BQB * 4);
      bulk_load(sm + BwdSmem::LD + b * 512, ldg + qt * (2 * BQB), 2 * BQB * 4, qfull + b);
      tma_load_4d(qd, &tmQ, 0, c + qt * BQB, head, sq, qfull + b);
      tma_load_4d(qd + QHALF, &tmQ, 64, c + qt * BQB, head, sq, qfull + b);
      tma_load_3d(od, &tmdO, head * AT, qt * BQB, sq, qfull + b);
      tma_load_3d(od + QHALF, &tmdO, head * AT + 64, qt * BQB, sq, qfull + b);
      // the ring is only NQB deep and a tile's slot frees late (its dV / dK MMAs): pull the tile
      // pf_dist ahead into L2 now so its TMA load later is an L2 hit, not a DRAM round trip
      if (pf_dist > 0 && i + pf_dist < ntile) {
        const int qp = qt + pf_dist;
        tma_prefetch_4d(&tmQ, 0, c + qp * BQB, head, sq);
        tma_prefetch_4d(&tmQ, 64, c + qp * BQB, head, sq);
        tma_prefetch_3d(&tmdO, head * AT, qp * BQB, sq);
        tma_prefetch_3d(&tmdO, head * AT + 64, qp * BQB, sq);
      }
    }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, warp-uniform control flow; one elected lane issues)
    constexpr uint32_t idS = idesc_bf16(128, BQB, false, false);   // S^T, dP^T
    constexpr uint32_t idKV = idesc_bf16(128, 128, false, true);   // dV (A = P^T in TMEM), dK (B = dO / Q, MN-major)
    constexpr uint32_t idQ = idesc_bf16(128, BQB, true, true);     // dQ^T (A = K MN-major, B = dS^T MN-major)
    // shared-memory addresses as 32-bit arithmetic on the warp-uniform window base (uniform datapath)
    const uint32_t sbase = smem_u32(smem_raw) + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t k_base = sbase + BwdSmem::K, v_base = sbase + BwdSmem::V;
    mbar_wait(kvfull, 0);
    // Per tile j (TMEM buffer j & 1): S^T is issued as early as possible (the softmax warps start the
    // exp2 work on it while dV / dK of the previous tile run), dP^T after dV / dK of j-1 (its
    // columns held dQ^T of j-2, which the drain warps must have read).
    auto issue_s = [&](int j) {
      const int bq = j % NQB, bb = j & 1;
      const uint32_t q_base = sbase + BwdSmem::Q + bq * QT;
      mbar_wait(qfull + bq, (j / NQB) & 1);
      if (lane == 0) TRC(1, 0, j);
      // buffer bb last held tile j-2: its S^T was read by the softmax (pfull(j-2), waited before
      // the MMAs of j-2), its P^T by dV(j-2), issued before this MMA (in-order tcgen05.mma
      // execution; inorder = 0: wait for dV(j-2) to complete, qfree(j-2))
      if (j >= 2 && !inorder) mbar_wait(qfree + (j - 2) % NQB, ((j - 2) / NQB) & 1);
      if (lane == 0) TRC(1, 1, j);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk) {
        const uint32_t ok = (kk >> 2) * HALF + (kk & 3) * 32, oq = (kk >> 2) * QHALF + (kk & 3) * 32;
        mma_bf16_w(tmem + bb * 128, make_desc(k_base + ok, 16, 1024), make_desc(q_base + oq, 16, 1024), idS, kk > 0);
      }
      mma_commit_w(sfull + bb);
      if (lane == 0) TRC(1, 5, j);
    };
    auto issue_dp = [&](int j) {
      const int bq = j % NQB, bb = j & 1;
      const uint32_t o_base = sbase + BwdSmem::O + bq * QT;
      if (DQ && j >= 2) mbar_wait(dqfree + bb, ((j >> 1) - 1) & 1);
      if (lane == 0) TRC(1, 2, j);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk) {
        const uint32_t ok = (kk >> 2) * HALF + (kk & 3) * 32, oq = (kk >> 2) * QHALF + (kk & 3) * 32;
        mma_bf16_w(tmem + bb * 128 + 64, make_desc(v_base + ok, 16, 1024), make_desc(o_base + oq, 16, 1024), idS,
                   kk > 0);
      }
      mma_commit_w(dpfull + bb);
    };
    issue_s(0);
    issue_dp(0);
    for (int i = 0; i < ntile; ++i) {
      const int bq = i % NQB, bb = i & 1;
      const uint32_t q_base = sbase + BwdSmem::Q + bq * QT, o_base = sbase + BwdSmem::O + bq * QT;
      const uint32_t ds_base = sbase + BwdSmem::DS + bb * PT;
      const uint32_t tb = tmem + bb * 128;
      if (lane == 0) DBG(1, 100 + 10 * i);
      if (i + 1 < ntile) issue_s(i + 1);
      // without dQ^T the dP^T columns of buffer (i+1)&1 only held dP^T(i-1), consumed before pfull(i-1):
      // issue dP^T(i+1) right away, so tile i+1's softmax finds both S^T and dP^T ready
      if (!DQ && i + 1 < ntile) issue_dp(i + 1);
      if (lane == 0) DBG(1, 101 + 10 * i);
      mbar_wait(pfull + bb, (i >> 1) & 1);
      if (lane == 0) TRC(1, 3, i);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < BQB / 16; ++kk) {
        // P^T columns: query half h = kk >> 1 was packed at h*32 .. h*32+15 of the S^T columns
        mma_bf16_ts_w(tmem + T_DV, tb + (kk >> 1) * 32 + (kk & 1) * 8, make_desc(o_base + kk * 2048, QHALF, 1024), idKV,
                    (i | kk) != 0);
        // dS^T columns: the softmax warps also wrote it packed into h*32+16 .. h*32+31 (TS-MMA:
        // only Q is read from shared memory)
        mma_bf16_ts_w(tmem + T_DK, tb + (kk >> 1) * 32 + 16 + (kk & 1) * 8, make_desc(q_base + kk * 2048, QHALF, 1024),
                      idKV, (i | kk) != 0);
      }
      mma_commit_w(qfree + bq);
      if (DQ && i + 1 < ntile) issue_dp(i + 1);
      if constexpr (DQ) {
#pragma unroll
        for (int kk = 0; kk < AT / 16; ++kk)
          mma_bf16_w(tb + 64, make_desc(k_base + kk * 2048, HALF, 1024), make_desc(ds_base + kk * 2048, 8192, 1024), idQ,
                   kk > 0);
        mma_commit_w(dqfull + bb);
        mma_commit_w(dsfree + bb);
      }
      if (lane == 0) TRC(1, 4, i);
      if (lane == 0) DBG(1, 105 + 10 * i);
    }
    mma_commit_w(done);
    if (lane == 0) DBG(1, 999);
  } else if (warp >= 10) {
    if constexpr (!DQ) {
      // no dQ^T to drain
    } else {
    // ---------------- dQ drain warps (one per TMEM lane quarter; thread = head-dim index `row`):
    // dQ^T of tile j -> smem [64 q][128 d] -> one TMA reduce-add into dq_acc
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float* dqs = reinterpret_cast<float*>(sm + BwdSmem::DQ);
    const bool leader = threadIdx.x == 320;
    for (int j = 0; j < ntile; ++j) {
      const int bb = j & 1;
      if (leader) tma_wait_reads();  // the previous reduce has finished reading the staging tile
      named_bar(2, 128);
      mbar_wait(dqfull + bb, (j >> 1) & 1);
      if (leader) TRC(2, 4, j);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t r[32];
        tmem_ld32_nowait(lane_base + bb * 128 + 64 + h * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 32; ++t) dqs[(h * 32 + t) * AT + row] = __uint_as_float(r[t]) * scale;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dqfree + bb);
      fence_proxy_async();
      named_bar(2, 128);
      if (leader) { tma_reduce_add_3d(&tmdQ, dqs, head * AT, (qt0 + j) * BQB, sq); TRC(2, 5, j); }
    }
    if (leader) tma_wait_all();
    }
  } else if (warp >= 2) {
    // ---------------- softmax-gradient warps: two per TMEM lane quarter; thread owns key row `row`
    // and query columns [half*32, half*32+32) of the tile (head-dim columns for dK / dV)
    const int q = warp & 3, row = q * 32 + lane, half = (warp - 2) >> 2;
    const int kabs = key0 + row;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    constexpr int HQ = BQB / 2;  // query columns per half
    for (int i = 0; i < ntile; ++i) {
      const int bb = i & 1;
      const int qrow0 = (qt0 + i) * BQB;
      // lse*log2e / D of the tile's queries (rows past the slice: +inf / 0), bulk-loaded with Q / dO
      const float* Ls = reinterpret_cast<const float*>(sm + BwdSmem::LD + (i % NQB) * 512);
      const float* Ds = Ls + BQB;
      if (threadIdx.x == 64) TRC(2, 0, i);
      mbar_wait(qfull + i % NQB, (i / NQB) & 1);
      if (threadIdx.x == 64) TRC(2, 1, i);
      mbar_wait(sfull + bb, (i >> 1) & 1);
      if (threadIdx.x == 64) TRC(2, 2, i);
      tc_fence_after();
      // visible iff c + qr >= kabs (and qr < l, which Ls = +inf enforces)
      const int vis0 = kabs - c - qrow0 - half * HQ;  // first visible column of this key row, in this half
      // phase 1 (needs S^T only): P^T = exp2(S^T scale - lse) -> registers and, packed, into TMEM
      float pv[HQ];
      // this half's 32 S^T columns in one TMEM load (one load latency per tile, not two)
      uint32_t rs32[32];
      tmem_ld32_nowait(lane_base + bb * 128 + half * HQ, rs32);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {  // 16 query columns at a time
        const uint32_t* rs = rs32 + ch * 16;
        const float4* L4 = reinterpret_cast<const float4*>(Ls + half * HQ + ch * 16);
        float Lv[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 a4 = L4[u];
          Lv[4 * u] = a4.x; Lv[4 * u + 1] = a4.y; Lv[4 * u + 2] = a4.z; Lv[4 * u + 3] = a4.w;
        }
        if (ch == 0) tmem_wait_ld();
        uint32_t pk[8];
#pragma unroll
        for (int t = 0; t < 16; t += 2) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = ch * 16 + t + e;
            const float p = ex2(fmaf(__uint_as_float(rs[t + e]), scale_log2, -Lv[t + e]));
            pv[col] = col >= vis0 ? p : 0.f;
          }
          __nv_bfloat162 hp = __floats2bfloat162_rn(pv[ch * 16 + t], pv[ch * 16 + t + 1]);
          pk[t >> 1] = *reinterpret_cast<uint32_t*>(&hp);
        }
        // P^T (this half's 32 queries) packed into the first 16 of this half's own S^T columns;
        // this chunk's S^T columns were consumed above (the second chunk's lie at +16 .. +31)
        tmem_st8(lane_base + bb * 128 + half * HQ + ch * 8, pk);
      }
      // phase 2 (needs dP^T): dS^T = P^T (dP^T - D) -> bf16 -> smem (K-major swizzled)
      mbar_wait(dpfull + bb, (i >> 1) & 1);
      if (DQ && i >= 2) mbar_wait(dsfree + bb, ((i >> 1) - 1) & 1);  // dK / dQ MMAs of tile i-2 read dS^T buffer bb
      tc_fence_after();
      uint8_t* dSt = sm + BwdSmem::DS + bb * PT;
#pragma unroll
      uint32_t rp32[32];  // this half's 32 dP^T columns in one TMEM load
      tmem_ld32_nowait(lane_base + bb * 128 + 64 + half * HQ, rp32);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const uint32_t* rp = rp32 + ch * 16;
        const float4* D4 = reinterpret_cast<const float4*>(Ds + half * HQ + ch * 16);
        float Dv[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 d4 = D4[u];
          Dv[4 * u] = d4.x; Dv[4 * u + 1] = d4.y; Dv[4 * u + 2] = d4.z; Dv[4 * u + 3] = d4.w;
        }
        if (ch == 0) tmem_wait_ld();
        uint32_t dk[8];
#pragma unroll
        for (int t = 0; t < 16; t += 2) {
          const float d0 = pv[ch * 16 + t] * (__uint_as_float(rp[t]) - Dv[t]);
          const float d1 = pv[ch * 16 + t + 1] * (__uint_as_float(rp[t + 1]) - Dv[t + 1]);
          __nv_bfloat162 hd = __floats2bfloat162_rn(d0, d1);
          dk[t >> 1] = *reinterpret_cast<uint32_t*>(&hd);
        }
        if constexpr (DQ) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int cc = half * 4 + ch * 2 + u;
            *reinterpret_cast<uint4*>(dSt + swz(row, cc)) = make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
          }
        }
        // and packed into TMEM (second 16 of this half's S^T columns) as dK's A operand
        tmem_st8(lane_base + bb * 128 + half * HQ + 16 + ch * 8, dk);
      }
      tmem_wait_st();
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) { mbar_arrive(pfull + bb); TRC(3, warp - 2, i); }
      if (threadIdx.x == 64) TRC(2, 3, i);
    }
    if (lane == 0) DBG(2 + q, 900);
    // dK (x scale) and dV of this key block -> 128B-swizzled fp32 staging over the (now idle) Q / dO
    // ring and dS^T buffers: [dK | dV][4 column chunks of 32 d][128 keys][32] -> 8 TMA stores (first
    // slice) or reduce-adds (later slices) into the prefix accumulators; key rows past the prefix
    // are clipped by the tensor map.
    mbar_wait(done, 0);
    if (threadIdx.x == 64) TRC(2, 6, 0);
    tc_fence_after();
    float* stg = reinterpret_cast<float*>(sm + BwdSmem::Q);
#pragma unroll
    for (int cq = 0; cq < 2; ++cq) {
      const int ch = half * 2 + cq;
      uint32_t rk[32], rv[32];
      tmem_ld32_nowait(lane_base + T_DK + ch * 32, rk);
      tmem_ld32_nowait(lane_base + T_DV + ch * 32, rv);
      tmem_wait_ld();
      if (dkv_out && kabs >= c && kabs < c + l) {
        // rows of this slice are final after this launch (later slices were processed before it):
        // dK / dV = this launch's contribution + the earlier launches' accumulator rows, straight to
        // the bf16 dQKV columns [H, 3H) of the job (the separate finalise pass is not needed)
        const int H = nheads * AT;
        bf16* outk = dkv_out + sq * dq_sstride + (int64_t)(kabs - c) * ldq + H + head * AT + ch * 32;
        const int64_t src = sq * dkv_sstride + ((int64_t)head * s + kabs) * AT + ch * 32;
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          float fk[8], fv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) { fk[e] = __uint_as_float(rk[u + e]) * scale; fv[e] = __uint_as_float(rv[u + e]); }
          if (accumulate) {
            float ok[8], ov[8];
            load8<float>(dk_raw + src + u, ok);
            load8<float>(dv_raw + src + u, ov);
#pragma unroll
            for (int e = 0; e < 8; ++e) { fk[e] += ok[e]; fv[e] += ov[e]; }
          }
          store8<bf16>(outk + u, fk);
          store8<bf16>(outk + H + u, fv);
        }
      }
      uint8_t* bk = reinterpret_cast<uint8_t*>(stg + ch * 4096) + row * 128;
      uint8_t* bv = reinterpret_cast<uint8_t*>(stg + 16384 + ch * 4096) + row * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int off = (u ^ (row & 7)) * 16;
        *reinterpret_cast<float4*>(bk + off) =
            make_float4(__uint_as_float(rk[4 * u]) * scale, __uint_as_float(rk[4 * u + 1]) * scale,
                        __uint_as_float(rk[4 * u + 2]) * scale, __uint_as_float(rk[4 * u + 3]) * scale);
        *reinterpret_cast<float4*>(bv + off) = make_float4(__uint_as_float(rv[4 * u]), __uint_as_float(rv[4 * u + 1]),
                                                           __uint_as_float(rv[4 * u + 2]), __uint_as_float(rv[4 * u + 3]));
      }
    }
    fence_proxy_async();
    named_bar(1, 256);
    // a key block entirely inside the slice needs no fp32 accumulator update (its rows were
    // finalised above and no earlier slice reads them)
    if (threadIdx.x == 64 && !(dkv_out && key0 >= c)) {
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        if (accumulate) {
          tma_reduce_add_4d(&tmdK, stg + ch * 4096, ch * 32, key0, head, sq);
          tma_reduce_add_4d(&tmdV, stg + 16384 + ch * 4096, ch * 32, key0, head, sq);
        } else {
          tma_store_4d(&tmdK, stg + ch * 4096, ch * 32, key0, head, sq);
          tma_store_4d(&tmdV, stg + 16384 + ch * 4096, ch * 32, key0, head, sq);
        }
      }
      tma_commit_group();
      tma_wait_all();
      TRC(2, 7, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ backward, dQ (split backward)
// Per (128 query rows of the slice, head, sequence), heaviest first; loop over the key blocks the
// rows see. dQ = scale * sum_j dS_j K_j with dS = P (dP - D), P = exp2(S scale_log2 - lse log2e):
// the same function as the fused kernel's dQ^T, but accumulated in TMEM over the key blocks and
// written once as bf16 (no fp32 partials, no atomics, no conversion pass).
// TMEM: S_0 (cols 0-127), S_1 (128-255), dP (256-383), dQ (384-511).
//   warp 0    TMA: Q and dO once; K_j, V_j through 2-deep rings;
//   warp 1    MMA: S_{j+1} = Q K_{j+1}^T (once dQ has read dS_{j-1} from that buffer), then
//             dP_{j+1} = dO V_{j+1}^T (the softmax has read dP_j), then dQ += dS_j K_j (TS-MMA);
//   warps 2-9 two per query row (TMEM lane), 64 key columns each: P, dS = P (dP - D), packed bf16
//             over S_j's first 64 columns.
constexpr int DQ_THREADS = 320;  // TMA, MMA, 8 softmax warps (two per TMEM lane quarter)
struct DqSmem {
  static constexpr uint32_t Q = 0, O = TILE, K = 2 * TILE, V = K + 2 * TILE;
  static constexpr uint32_t BAR = V + 2 * TILE;
  static constexpr uint32_t BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "dQ tile set exceeds 227 KB of shared memory");
};

__global__ void __launch_bounds__(DQ_THREADS, 1)
    attn_bwd_dq_sm100_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                             const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                             const float* __restrict__ ldg, bf16* __restrict__ dq, int64_t ldq, int64_t dq_sstride,
                             int s, int c, int l, float scale, float scale_log2, int nheads) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc5::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DqSmem::BAR);
  uint64_t* qfull = bars + 0;
  uint64_t* kfull = bars + 1;   // [2]
  uint64_t* kfree = bars + 3;   // [2]
  uint64_t* vfull = bars + 5;   // [2]
  uint64_t* vfree = bars + 7;   // [2]
  uint64_t* sfull = bars + 9;   // [2]
  uint64_t* dpfull = bars + 11;
  uint64_t* pfull = bars + 12;  // [2] dS_j written, dP_j consumed (8 warps)
  uint64_t* dqdone = bars + 14; // [2] dQ += dS_j K_j complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  // warp index through a shuffle: provably warp-uniform, so the role branches below keep the
  // uniform datapath (descriptor arithmetic in uniform registers for tcgen05.mma)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int head = blockIdx.y, sq = blockIdx.z, r0 = (gridDim.x - 1 - blockIdx.x) * AT;
  const int nkb = (c + min(l, r0 + AT) - 1) / AT + 1;

  if (threadIdx.x == 0) {
    mbar_init(qfull, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(kfull + i, 1); mbar_init(kfree + i, 1); mbar_init(vfull + i, 1); mbar_init(vfree + i, 1);
      mbar_init(sfull + i, 1); mbar_init(pfull + i, 8); mbar_init(dqdone + i, 1);
    }
    mbar_init(dpfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t T_DP = 256, T_DQ = 384;

  if (warp == 0) {
    if (lane == 0) {
    mbar_expect_tx(qfull, 2 * TILE);
    tma_load_4d(sm + DqSmem::Q, &tmQ, 0, c + r0, head, sq, qfull);
    tma_load_4d(sm + DqSmem::Q + HALF, &tmQ, 64, c + r0, head, sq, qfull);
    tma_load_3d(sm + DqSmem::O, &tmdO, head * AT, r0, sq, qfull);
    tma_load_3d(sm + DqSmem::O + HALF, &tmdO, head * AT + 64, r0, sq, qfull);
    for (int j = 0; j < nkb; ++j) {
      const int b = j & 1;
      if (j >= 2) mbar_wait(kfree + b, ((j >> 1) - 1) & 1);
      mbar_expect_tx(kfull + b, TILE);
      tma_load_4d(sm + DqSmem::K + b * TILE, &tmK, 0, j * AT, head, sq, kfull + b);
      tma_load_4d(sm + DqSmem::K + b * TILE + HALF, &tmK, 64, j * AT, head, sq, kfull + b);
      if (j >= 2) mbar_wait(vfree + b, ((j >> 1) - 1) & 1);
      mbar_expect_tx(vfull + b, TILE);
      tma_load_4d(sm + DqSmem::V + b * TILE, &tmV, 0, j * AT, head, sq, vfull + b);
      tma_load_4d(sm + DqSmem::V + b * TILE + HALF, &tmV, 64, j * AT, head, sq, vfull + b);
    }
    }
  } else if (warp == 1) {
    constexpr uint32_t idS = idesc_bf16(128, 128, false, false);  // S, dP (both operands K-major)
    constexpr uint32_t idQ = idesc_bf16(128, 128, false, true);   // dQ += dS K (B = K as [keys][d], MN-major)
    const uint32_t q_base = smem_u32(sm + DqSmem::Q), o_base = smem_u32(sm + DqSmem::O);
    auto issue_s = [&](int j) {
      const uint32_t k_base = smem_u32(sm + DqSmem::K + (j & 1) * TILE);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk) {
        const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
        mma_bf16_w(tmem + (j & 1) * 128, make_desc(q_base + off, 16, 1024), make_desc(k_base + off, 16, 1024), idS, kk > 0);
      }
      mma_commit_w(sfull + (j & 1));
    };
    auto issue_dp = [&](int j) {
      const uint32_t v_base = smem_u32(sm + DqSmem::V + (j & 1) * TILE);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk) {
        const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
        mma_bf16_w(tmem + T_DP, make_desc(o_base + off, 16, 1024), make_desc(v_base + off, 16, 1024), idS, kk > 0);
      }
      mma_commit_w(dpfull);
      mma_commit_w(vfree + (j & 1));
    };
    mbar_wait(qfull, 0);
    mbar_wait(kfull, 0);
    issue_s(0);
    mbar_wait(vfull, 0);
    issue_dp(0);
    for (int j = 0; j < nkb; ++j) {
      const int b = j & 1;
      if (j + 1 < nkb) {
        mbar_wait(kfull + (b ^ 1), ((j + 1) >> 1) & 1);
        if (j >= 1) mbar_wait(dqdone + (b ^ 1), ((j - 1) >> 1) & 1);  // dS_{j-1} read from that buffer
        issue_s(j + 1);
      }
      mbar_wait(pfull + b, (j >> 1) & 1);  // dS_j in S buffer b, dP_j consumed
      if (j + 1 < nkb) {  // first, so the next block's softmax is not behind dQ_j
        mbar_wait(vfull + (b ^ 1), ((j + 1) >> 1) & 1);
        issue_dp(j + 1);
      }
      tc_fence_after();
      const uint32_t k_base = smem_u32(sm + DqSmem::K + b * TILE);
#pragma unroll
      for (int kk = 0; kk < AT / 16; ++kk)
        mma_bf16_ts_w(tmem + T_DQ, tmem + b * 128 + kk * 8, make_desc(k_base + kk * 2048, HALF, 1024), idQ,
                      (j | kk) != 0);
      mma_commit_w(dqdone + b);
      mma_commit_w(kfree + b);
    }
  } else if (warp >= 2) {
    const int q = warp & 3, row = q * 32 + lane, half = (warp - 2) >> 2;  // key columns [64 half, +64)
    const int qr = r0 + row;                // row of the slice
    const int qabs = c + qr;
    const bool live = qr < l;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    // lse * log2e and D of this query from the per-64-query-tile staging of bwd_stage_kernel
    const int ntq = (l + BQB - 1) / BQB;
    const float* st = ldg + ((int64_t)sq * nheads + head) * ntq * (2 * BQB) + (qr / BQB) * (2 * BQB) + (qr % BQB);
    const float lse2 = live ? st[0] : 0.f;
    const float Dq = live ? st[BQB] : 0.f;
    for (int j = 0; j < nkb; ++j) {
      const int b = j & 1;
      mbar_wait(sfull + b, (j >> 1) & 1);
      mbar_wait(dpfull, j & 1);
      tc_fence_after();
      const int nvis = live ? qabs - j * AT + 1 : 0;  // keys j*128 .. qabs visible
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int ch = half * 2 + cc;
        uint32_t rs[32], rp[32];
        tmem_ld32_nowait(lane_base + b * 128 + ch * 32, rs);
        tmem_ld32_nowait(lane_base + T_DP + ch * 32, rp);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 32; u += 2) {
          const int col = ch * 32 + u;
          const float p0 = col < nvis ? ex2(fmaf(__uint_as_float(rs[u]), scale_log2, -lse2)) : 0.f;
          const float p1 = col + 1 < nvis ? ex2(fmaf(__uint_as_float(rs[u + 1]), scale_log2, -lse2)) : 0.f;
          const float d0 = p0 * (__uint_as_float(rp[u]) - Dq), d1 = p1 * (__uint_as_float(rp[u + 1]) - Dq);
          __nv_bfloat162 h = __floats2bfloat162_rn(d0, d1);
          pk[u >> 1] = *reinterpret_cast<uint32_t*>(&h);
        }
        // dS packed over S_j's columns [16 ch, 16 ch + 16): for half 0 these are its own already-read
        // columns; for half 1 (ch = 2, 3: columns 32-63) they belong to half 0's second chunk, so half
        // 1 waits until half 0 of the same lane quarter has read them (named barrier per quarter)
        if (cc == (half == 0 ? 1 : 0)) named_bar(3 + q, 64);  // half 0: after reading chunk 1
        tmem_st16(lane_base + b * 128 + ch * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(pfull + b);
    }
    mbar_wait(dqdone + ((nkb - 1) & 1), ((nkb - 1) >> 1) & 1);
    tc_fence_after();
    bf16* out = dq + sq * dq_sstride + (int64_t)qr * ldq + head * AT;
#pragma unroll 1
    for (int ch = half * 2; ch < half * 2 + 2; ++ch) {
      uint32_t rr[32];
      tmem_ld32_nowait(lane_base + T_DQ + ch * 32, rr);
      tmem_wait_ld();
      if (live) {
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          float v8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v8[e] = __uint_as_float(rr[u + e]) * scale;
          store8<bf16>(out + ch * 32 + u, v8);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Per 64-query tile of every (sequence, head): lse*log2e (+inf past the slice) and D = rowsum(dO * O)
// (0 past the slice) as [nseq][a][ntq][lse 64 | D 64] fp32, one 512-byte bulk copy per tile for the
// backward kernel. One warp per query row, lanes over 8-element chunks of all heads.
__global__ void bwd_stage_kernel(const bf16* __restrict__ dO, int64_t ld_do, const bf16* __restrict__ o, int64_t ldo,
                                 const float* __restrict__ lse, int64_t lse_sstride, float* __restrict__ out, int a,
                                 int s, int c, int l, int ntq, int64_t o_sstride) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = blockIdx.x * 4 + w, sq = blockIdx.y;
  if (r >= ntq * BQB) return;
  dO += sq * o_sstride;
  o += sq * o_sstride;
  lse += sq * lse_sstride;
  float* base = out + (int64_t)sq * a * ntq * (2 * BQB) + (r / BQB) * (2 * BQB) + (r % BQB);
  constexpr int CPH = AT / 8;  // 16 chunks per head: two heads per pass of the warp
  for (int hb = 0; hb < a * CPH; hb += 32) {
    const int ch = hb + lane;
    float acc = 0.f;
    if (r < l && ch < a * CPH) {
      float x[8], y[8];
      load8<bf16>(dO + (int64_t)r * ld_do + ch * 8, x);
      load8<bf16>(o + (int64_t)r * ldo + ch * 8, y);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += x[i] * y[i];
    }
#pragma unroll
    for (int off = 1; off < CPH; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (ch < a * CPH && (lane % CPH) == 0) {
      const int head = ch / CPH;
      float* p = base + (int64_t)head * ntq * (2 * BQB);
      p[0] = r < l ? __ldg(lse + (int64_t)head * s + c + r) * LOG2E_F : INFINITY;
      p[BQB] = r < l ? acc : 0.f;
    }
  }
}

__global__ void dq_convert_kernel(const float* __restrict__ dq_acc, int64_t ld_acc, bf16* __restrict__ dq, int64_t ldq,
                                  int H, int l, int64_t dq_sstride) {
  const int r = blockIdx.x, sq = blockIdx.y;
  dq_acc += (int64_t)sq * l * ld_acc;
  dq += sq * dq_sstride;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    float v[8];
    load8<float>(dq_acc + (int64_t)r * ld_acc + i, v);
    store8<bf16>(dq + (int64_t)r * ldq + i, v);
  }
}

}  // namespace

bool attn_sm100_supported(int d) { return d == AT; }

// TP_ATTN_INORDER=0: the MMA warps wait for an MMA's completion before issuing the next MMA that
// overwrites its TMEM operand (A/B knob; default: rely on in-order tcgen05.mma execution)
static int attn_inorder() {
  static const int v = !(getenv("TP_ATTN_INORDER") && atoi(getenv("TP_ATTN_INORDER")) == 0);
  return v;
}

cudaError_t attn_fwd_sm100(const bf16* q, const bf16* k, const bf16* v, bf16* o, int64_t ldo, float* lse, int a, int s,
                           int d, int c, int l, cudaStream_t st, int nseq, int64_t qkv_sstride, int64_t o_sstride,
                           int64_t lse_sstride) {
  if (l == 0 || nseq == 0) return cudaSuccess;
  if (d != AT) return cudaErrorInvalidValue;
  // [seq][a][s][d] viewed as 4-D {d, rows = c + l (prefix), a, seq}: rows past the prefix zero-filled
  const uint64_t dims[4] = {(uint64_t)d, (uint64_t)(c + l), (uint64_t)a, (uint64_t)nseq};
  const uint64_t strides[3] = {(uint64_t)d * 2, (uint64_t)s * d * 2, (uint64_t)(nseq > 1 ? qkv_sstride : (int64_t)a * s * d) * 2};
  const uint32_t box[4] = {64, AT, 1, 1};
  CUtensorMap mq, mk, mv;
  if (!encode_bf16_map(&mq, q, 4, dims, strides, box) || !encode_bf16_map(&mk, k, 4, dims, strides, box) ||
      !encode_bf16_map(&mv, v, 4, dims, strides, box))
    return cudaErrorInvalidValue;
  // TP_ATTN_FWD=1: one query tile per CTA with S double-buffered; =2: two tiles per CTA sharing K/V;
  // =3: two tiles, 64-key blocks, S double-buffered per tile. Default: the two-tile 64-key kernel when
  // its grid fills at least two waves, else the one-tile kernel (wave quantisation of the half-size
  // grid dominates). Measured (scripts/attn_bench.py, one B200; profiles/r02_attn_fwd3.txt):
  // c = 0, l = 2048, 128 heads: 3: 203, 2: 214, 1: 222 us; c = 576, l = 1472: 188 / 200 / 204;
  // c = 0, l = 576: 45.7 / 52.7 / 52.6; c = 1536, l = 512, 80 heads (160 two-tile CTAs): 89 / 86 / 76.
  static const int fwd_env = getenv("TP_ATTN_FWD") ? atoi(getenv("TP_ATTN_FWD")) : 0;
  const long pair_ctas = (long)((l + 2 * AT - 1) / (2 * AT)) * a * nseq;
  const int fwd_impl = fwd_env ? fwd_env : (pair_ctas >= 2L * num_sms() ? 3 : 1);
  if (fwd_impl == 3) {  // two tiles, 64-key blocks, S double-buffered (attn_fwd3_sm100_kernel)
    static bool attr3 = false;
    if (!attr3) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd3_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)Fwd3Smem::BYTES);
      if (e != cudaSuccess) return e;
      attr3 = true;
    }
    const uint32_t box64[4] = {64, BK3, 1, 1};
    CUtensorMap mk64, mv64;
    if (!encode_bf16_map(&mk64, k, 4, dims, strides, box64) || !encode_bf16_map(&mv64, v, 4, dims, strides, box64))
      return cudaErrorInvalidValue;
    dim3 grid3((l + 2 * AT - 1) / (2 * AT), a, nseq);
    static int trace3_left = getenv("TP_ATTN_TRACE") ? atoi(getenv("TP_ATTN_TRACE")) : 0;
    static long long* trace3 = nullptr;
    if (trace3_left > 0 && !trace3) cudaMalloc(&trace3, 4 * 8 * 64 * sizeof(long long));
    if (trace3_left > 0) cudaMemsetAsync(trace3, 0, 4 * 8 * 64 * sizeof(long long), st);
    attn_fwd3_sm100_kernel<<<grid3, F2_THREADS, Fwd3Smem::BYTES, st>>>(mq, mk64, mv64, o, ldo, lse, s, c, l,
                                                                      rsqrtf((float)d) * LOG2E_F, o_sstride,
                                                                      lse_sstride, trace3_left > 0 ? trace3 : nullptr);
    if (trace3_left > 0) {
      --trace3_left;
      long long h[4 * 8 * 64];
      cudaMemcpyAsync(h, trace3, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      long long t0 = 0;
      for (int i = 0; i < 4 * 8 * 64; ++i) if (h[i] && (!t0 || h[i] < t0)) t0 = h[i];
      fprintf(stderr, "attn_fwd3 trace c=%d l=%d: kb | M:vfull M:pfull0 M:pfull1 M:PV0 M:PV1 M:S0 M:S1 | T0:wait T0:sfull T0:pfull | T1:wait T1:sfull T1:pfull\n", c, l);
      for (int i = 0; i < 64; ++i) {
        auto g = [&](int r, int e) { long long v = h[(r * 8 + e) * 64 + i]; return v ? (long long)(v - t0) : -1LL; };
        if (g(1, 0) < 0) break;
        fprintf(stderr, "%3d | %7lld %7lld %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld | %7lld %7lld %7lld\n", i,
                g(1, 0), g(1, 1), g(1, 2), g(1, 3), g(1, 4), g(1, 5), g(1, 6), g(2, 0), g(2, 1), g(2, 2), g(3, 0), g(3, 1), g(3, 2));
      }
    }
    return cudaGetLastError();
  }
  if (fwd_impl == 1) {
    static bool attr1 = false;
    if (!attr1) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd1_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)Fwd1Smem::BYTES);
      if (e != cudaSuccess) return e;
      attr1 = true;
    }
    dim3 grid1((l + AT - 1) / AT, a, nseq);
    attn_fwd1_sm100_kernel<<<grid1, F1_THREADS, Fwd1Smem::BYTES, st>>>(mq, mk, mv, o, ldo, lse, s, c, l,
                                                                      rsqrtf((float)d) * LOG2E_F, o_sstride, lse_sstride,
                                                                      attn_inorder());
    return cudaGetLastError();
  }
  {
    static bool attr2 = false;
    if (!attr2) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd2_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)Fwd2Smem::BYTES);
      if (e != cudaSuccess) return e;
      attr2 = true;
    }
    dim3 grid2((l + 2 * AT - 1) / (2 * AT), a, nseq);
    static int trace2_left = getenv("TP_ATTN_TRACE") ? atoi(getenv("TP_ATTN_TRACE")) : 0;
    static long long* trace2 = nullptr;
    if (trace2_left > 0 && !trace2) cudaMalloc(&trace2, 4 * 8 * 64 * sizeof(long long));
    if (trace2_left > 0) cudaMemsetAsync(trace2, 0, 4 * 8 * 64 * sizeof(long long), st);
    attn_fwd2_sm100_kernel<<<grid2, F2_THREADS, Fwd2Smem::BYTES, st>>>(mq, mk, mv, o, ldo, lse, s, c, l,
                                                                      rsqrtf((float)d) * LOG2E_F, o_sstride, lse_sstride,
                                                                      trace2_left > 0 ? trace2 : nullptr, attn_inorder());
    if (trace2_left > 0) {
      --trace2_left;
      long long h[4 * 8 * 64];
      cudaMemcpyAsync(h, trace2, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      long long t0 = 0;
      for (int i = 0; i < 4 * 8 * 64; ++i) if (h[i] && (!t0 || h[i] < t0)) t0 = h[i];
      fprintf(stderr, "attn_fwd2 trace c=%d l=%d: kb | M:kfull M:S0 M:S1 M:pfull0 M:pfull1 M:PV0 M:PV1 | T0:sfull T0:max T0:pfull | T1:sfull T1:max T1:pfull\n", c, l);
      for (int i = 0; i < 64; ++i) {
        auto g = [&](int r, int e) { long long v = h[(r * 8 + e) * 64 + i]; return v ? (long long)(v - t0) : -1LL; };
        if (g(1, 0) < 0) break;
        fprintf(stderr, "%3d | %7lld %7lld %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld | %7lld %7lld %7lld\n", i,
                g(1, 0), g(1, 1), g(1, 2), g(1, 3), g(1, 4), g(1, 5), g(1, 6), g(2, 0), g(2, 1), g(2, 2), g(3, 0), g(3, 1), g(3, 2));
      }
    }
    return cudaGetLastError();
  }
}

cudaError_t attn_bwd_sm100(const bf16* dO, int64_t ld_do, const bf16* o, int64_t ldo, const bf16* q, const bf16* k,
                           const bf16* v, const float* lse, float* Dvec, float* dq_acc, bf16* dq, int64_t ldq,
                           float* dk_acc, float* dv_acc, int a, int s, int d, int c, int l, int accumulate,
                           cudaStream_t st, int nseq, int64_t qkv_sstride, int64_t o_sstride, int64_t lse_sstride,
                           int64_t dq_sstride, int64_t dkv_sstride, int finalize_dkv) {
  if (l == 0 || nseq == 0) return cudaSuccess;
  if (d != AT) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_sm100_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)BwdSmem::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_sm100_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)BwdSmem::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)DqSmem::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // split backward (TP_ATTN_BWD_SPLIT=1, opt-in): the key-block kernel computes dK / dV only and a
  // query-tile kernel computes dQ in TMEM (no fp32 partials, no atomics, no conversion pass).
  // Measured slower in the N = 1 step (attention backward 25.6-26.3 vs 20.5 ms per step)
  static const bool split = getenv("TP_ATTN_BWD_SPLIT") && atoi(getenv("TP_ATTN_BWD_SPLIT")) != 0;
  const int H = a * d;
  const int ntq = (l + BQB - 1) / BQB;
  cudaError_t e = split ? cudaSuccess : cudaMemsetAsync(dq_acc, 0, sizeof(float) * (size_t)l * H * nseq, st);
  if (e != cudaSuccess) return e;
  bwd_stage_kernel<<<dim3((ntq * BQB + 3) / 4, nseq), 128, 0, st>>>(dO, ld_do, o, ldo, lse, lse_sstride, Dvec, a, s, c,
                                                                     l, ntq, o_sstride);
  const int64_t qs = nseq > 1 ? qkv_sstride : (int64_t)a * s * d;
  const uint64_t kdims[4] = {(uint64_t)d, (uint64_t)(c + l), (uint64_t)a, (uint64_t)nseq};
  const uint64_t kstr[3] = {(uint64_t)d * 2, (uint64_t)s * d * 2, (uint64_t)qs * 2};
  const uint32_t kbox[4] = {64, AT, 1, 1}, qbox[4] = {64, BQB, 1, 1};
  // dO rows of sequence j: dO + j*o_sstride + r*ld_do
  const uint64_t odims[3] = {(uint64_t)H, (uint64_t)l, (uint64_t)nseq};
  const uint64_t ostr[2] = {(uint64_t)ld_do * 2, (uint64_t)(nseq > 1 ? o_sstride : (int64_t)l * ld_do) * 2};
  const uint32_t obox[3] = {64, BQB, 1};
  // dq_acc: [nseq][l][H] fp32
  const uint64_t qdims[3] = {(uint64_t)H, (uint64_t)l, (uint64_t)nseq};
  const uint64_t qstr[2] = {(uint64_t)H * 4, (uint64_t)l * H * 4};
  const uint32_t qrbox[3] = {AT, BQB, 1};
  CUtensorMap mk, mv, mq, mo, mdq;
  if (!encode_bf16_map(&mk, k, 4, kdims, kstr, kbox) || !encode_bf16_map(&mv, v, 4, kdims, kstr, kbox) ||
      !encode_bf16_map(&mq, q, 4, kdims, kstr, qbox) || !encode_bf16_map(&mo, dO, 3, odims, ostr, obox) ||
      !encode_f32_map_noswizzle(&mdq, dq_acc, 3, qdims, qstr, qrbox))
    return cudaErrorInvalidValue;
  // dk_acc / dv_acc: [nseq][a][s][d] fp32, viewed as {d, rows = c + l (prefix), a, seq}
  const uint64_t adims[4] = {(uint64_t)d, (uint64_t)(c + l), (uint64_t)a, (uint64_t)nseq};
  const uint64_t astr[3] = {(uint64_t)d * 4, (uint64_t)s * d * 4,
                            (uint64_t)(nseq > 1 ? dkv_sstride : (int64_t)a * s * d) * 4};
  const uint32_t abox[4] = {32, AT, 1, 1};
  CUtensorMap mdk, mdv;
  if (!encode_f32_map_sw128(&mdk, dk_acc, 4, adims, astr, abox) || !encode_f32_map_sw128(&mdv, dv_acc, 4, adims, astr, abox))
    return cudaErrorInvalidValue;
  const float scale = rsqrtf((float)d);
  dim3 grid((c + l + AT - 1) / AT, a * nseq);
  static int* dbg = nullptr;
  static bool dbg_on = getenv("TP_ATTN_DEBUG") != nullptr;
  if (dbg_on && !dbg) {
    cudaHostAlloc(&dbg, 4096 * sizeof(int), cudaHostAllocMapped);
  }
  int* dbg_dev = nullptr;
  if (dbg_on) { memset(dbg, 0, 4096 * sizeof(int)); cudaHostGetDevicePointer(&dbg_dev, dbg, 0); }
  static int trace_left = getenv("TP_ATTN_TRACE") ? atoi(getenv("TP_ATTN_TRACE")) : 0;
  static long long* trace = nullptr;
  if (trace_left > 0 && !trace) cudaMalloc(&trace, 4 * 8 * 64 * sizeof(long long));
  if (trace_left > 0) cudaMemsetAsync(trace, 0, 4 * 8 * 64 * sizeof(long long), st);
  // L2 prefetch distance of the Q / dO tiles, in tiles ahead of the TMA load (env TP_ATTN_PF; default
  // off: distances 1-4 measured neutral at c = 576, l = 1472, 128 heads, 565-567 us — the kernel is
  // bound by shared-memory bandwidth, ~288 KB per 128 x 64 tile, not by load latency)
  static const int pf_dist = getenv("TP_ATTN_PF") ? atoi(getenv("TP_ATTN_PF")) : 0;
  // dK / dV of the slice's own rows written as bf16 into dQKV by the kernel (TP_ATTN_DKV_FUSED=0: the
  // fp32 accumulators only, finalised by attn_dkv_finalize)
  static const bool dkv_fused_env = !getenv("TP_ATTN_DKV_FUSED") || atoi(getenv("TP_ATTN_DKV_FUSED")) != 0;
  const bool dkv_fused = dkv_fused_env && finalize_dkv;
  auto bwd_kernel = split ? attn_bwd_sm100_kernel<false> : attn_bwd_sm100_kernel<true>;
  bwd_kernel<<<grid, BWD_THREADS, BwdSmem::BYTES, st>>>(mk, mv, mq, mo, mdq, mdk, mdv, Dvec,
                                                           s, c, l, scale, scale * LOG2E_F, accumulate,
                                                           a, dbg_dev, trace_left > 0 ? trace : nullptr, pf_dist,
                                                           dk_acc, dv_acc,
                                                           nseq > 1 ? dkv_sstride : (int64_t)a * s * d, dkv_fused ? dq : nullptr,
                                                           ldq, nseq > 1 ? dq_sstride : 0, attn_inorder());
  e = cudaGetLastError();
  if (trace_left > 0) {
    --trace_left;
    long long h[4 * 8 * 64];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    long long t0 = h[(1 * 8 + 0) * 64];
    for (int i = 0; i < 4 * 8 * 64; ++i) if (h[i] && h[i] < t0) t0 = h[i];
    fprintf(stderr, "attn_bwd trace c=%d l=%d: tile | P:qfree-ok | M:qfull M:bufS M:Sissued M:bufdP M:pfull M:issued | S:stage S:bar S:sfull S:pfull S:dqfull S:dqred\n", c, l);
    for (int i = 0; i < 64; ++i) {
      auto g = [&](int r, int e) { long long v = h[(r * 8 + e) * 64 + i]; return v ? (long long)(v - t0) : -1LL; };
      if (g(1, 0) < 0 && g(2, 0) < 0) break;
      fprintf(stderr, "%3d | %7lld | %7lld %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld %7lld %7lld %7lld | warps", i, g(0, 0), g(1, 0),
              g(1, 1), g(1, 5), g(1, 2), g(1, 3), g(1, 4), g(2, 0), g(2, 1), g(2, 2), g(2, 3), g(2, 4), g(2, 5));
      for (int w = 0; w < 8; ++w) fprintf(stderr, " %lld", g(3, w));
      fprintf(stderr, "\n");
    }
    fprintf(stderr, "done-seen %lld  dkv-stored %lld\n", h[(2 * 8 + 6) * 64] - t0, h[(2 * 8 + 7) * 64] - t0);
  }
  if (dbg_on) {
    for (int it = 0; it < 50 && cudaStreamQuery(st) == cudaErrorNotReady; ++it) usleep(100000);
    if (cudaStreamQuery(st) == cudaErrorNotReady) {
      fprintf(stderr, "attn_bwd_sm100 HUNG: grid %d x %d, c=%d l=%d\n", grid.x, grid.y, c, l);
      for (unsigned b = 0; b < grid.x * grid.y && b < 500; ++b) {
        fprintf(stderr, " cta %u:", b);
        for (int r = 0; r < 8; ++r) fprintf(stderr, " %d", ((volatile int*)dbg)[b * 8 + r]);
        fprintf(stderr, "\n");
      }
      fflush(stderr);
      abort();
    }
  }
  if (e != cudaSuccess) return e;
  if (split) {
    const uint32_t obox128[3] = {64, AT, 1};
    CUtensorMap mq128, mo128;
    if (!encode_bf16_map(&mq128, q, 4, kdims, kstr, kbox) || !encode_bf16_map(&mo128, dO, 3, odims, ostr, obox128))
      return cudaErrorInvalidValue;
    attn_bwd_dq_sm100_kernel<<<dim3((l + AT - 1) / AT, a, nseq), DQ_THREADS, DqSmem::BYTES, st>>>(
        mq128, mo128, mk, mv, Dvec, dq, ldq, nseq > 1 ? dq_sstride : 0, s, c, l, scale, scale * LOG2E_F, a);
  } else {
    dq_convert_kernel<<<dim3(l, nseq), 128, 0, st>>>(dq_acc, H, dq, ldq, H, l, dq_sstride);
  }
  e = cudaGetLastError();
  if (e == cudaSuccess && finalize_dkv && !dkv_fused)  // requested but switched off: the separate pass
    e = attn_dkv_finalize<bf16>(dk_acc, dv_acc, dq, ldq, a, s, d, c, l, st, nseq, nseq > 1 ? dkv_sstride : 0,
                                nseq > 1 ? dq_sstride : 0);
  return e;
}

}  // namespace tp
