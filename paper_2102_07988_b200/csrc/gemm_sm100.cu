// gemm_sm100.cu — the dense contractions of the hot path on 5th-generation tensor cores.
//
//   acc[m][n] = sum_k A(m, k) B(n, k)   (bf16 operands, fp32 accumulation in TMEM)
//
// Every projection of a TeraPipe job is one of these: forward QKV / out-proj /
// FC1 / FC2 / LM head with M = slice tokens, their dX counterparts, and the deferred per-sequence
// weight gradients (K = seq_len, both operands MN-major). The fused epilogues (bias, GeLU,
// residual, Q/K/V scatter into the prefix cache, fp32 accumulate) are in epilogue.cuh.
//
// Design (sm_100a):
//   * persistent CTAs (grid = min(tiles, #SMs)), 128 x BN output tiles (BN = 256 or 128),
//     grouped tile raster (tile_mn: blocks of 2048 rows, m fastest inside a block) so one wave's
//     operand blocks are fetched from DRAM about once and reused from L2;
//   * warp-specialised: warp 0 = TMA producer (one thread), warp 1 = tcgen05.mma issuer (whole
//     warp, one elected lane), warps 2..9 = epilogue (two per TMEM lane quarter, each draining
//     half of the tile's columns: TMEM -> registers -> smem transpose -> fused epilogue -> global);
//   * operands staged by TMA (cp.async.bulk.tensor, 128-byte swizzle) into an NS-deep mbarrier
//     ring; K-major operands are one box per stage, MN-major operands (dW) are 64-wide boxes placed
//     at LBO = 8 KiB steps, described to the tensor core with the canonical SW128 layouts;
//   * the accumulator is double-buffered in TMEM (2 x BN fp32 columns of the 512) so the epilogue
//     of tile t overlaps the MMAs of tile t+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "kernels.h"
#include "tc5.cuh"

namespace tp {

namespace {

using namespace tc5;
constexpr int BM = 128, BK = 64;

// CG = 1: one CTA computes a 128 x BN tile (tcgen05.mma.cta_group::1, M = 128).
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with
//         tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A and half of
//         the BN rows of B, the leader issues the MMAs over both CTAs' shared memory, and each
//         CTA's TMEM receives its 128 rows — halving the per-SM L2->SMEM operand traffic.
// 2 + 8 warps: TMA producer, MMA issuer, and 8 epilogue warps — two per TMEM lane quarter, each
// draining half of the tile's columns (the fused epilogues are instruction-bound, 4 warps cannot
// keep up with a 256-wide tile at K = 2048).
constexpr int GEMM_THREADS = 320;

// WN = 1: tile N = BN with a double-buffered accumulator (epilogue of tile t overlaps the MMAs of
// tile t+1). WN = 2: tile N = 2 * BN as two side-by-side accumulators, single-buffered — 25 % fewer
// operand bytes per FLOP (A is shared by twice the columns) at the price of an un-overlapped
// epilogue; used for long-K GEMMs (dW with K = B*s, FC2 / FC1-dX with K = 4H).
template <int CG, int BN, int WN = 1>
struct Cfg {
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_HALF = (BN / CG) * BK * 2;   // one accumulator's B rows of this CTA
  static constexpr uint32_t B_BYTES = WN * B_HALF;
  static constexpr int TILE_N = WN * BN;
  static constexpr int NACC = WN == 1 ? 2 : 1;             // accumulator buffers in flight
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  static constexpr int NS = (196608 / STAGE) > 8 ? 8 : (196608 / STAGE);  // pipeline depth
  static constexpr uint32_t EPI_SCRATCH = 8 * 32 * 33 * 4;  // per epilogue warp: 32 x 32 fp32 (+1 pad)
  static constexpr uint32_t SMEM = NS * STAGE + EPI_SCRATCH + 1024 /*align slack*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered fp32 accumulator
  static constexpr int TILE_M = BM * CG;
  static_assert(SMEM <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

// Stream-K (data-parallel waves + one stream-K wave): tiles [0, dp_tiles) run whole, round robin
// over the units; the remaining tiles' k-blocks, sk_iters = (tiles - dp_tiles) * kbs in all, are
// cut into one contiguous range per unit (processed last segment first), so every unit ends the
// launch at the same point whatever the tile count. A range that stops inside a tile leaves a fp32 partial in the unit's own
// workspace slot and raises its flag; the unit that processes the tile's LAST k-block (the
// finisher) adds the partials of the earlier units that covered the tile's beginning (waiting on
// their flags; they are lower units, all co-resident: the grid is one CTA per SM) and runs the
// fused epilogue. Each unit leaves at most one partial per launch, so a slot per unit suffices.
struct SplitK {
  int dp_tiles = 0;       // whole tiles; [dp_tiles, tiles) are processed stream-K
  int sk_iters = 0;       // (tiles - dp_tiles) * kbs; the host keeps sk_iters * units < 2^31, so the
                          // device index math stays 32-bit (a 64-bit division is a helper CALL, which
                          // would cost the MMA and TMA warps the uniform datapath)
  float* ws = nullptr;    // [unit * CG + crank][128][TILE_N] fp32 partial slots
  int* flag = nullptr;    // [unit * CG + crank]: 1 = partial ready (reset to 0 by the finisher)
};
__device__ __forceinline__ int sk_r0(int unit, int nunits, int iters) {
  return (int)((unsigned)(iters * unit) / (unsigned)nunits);
}
// Work item `it` of unit `unit`: first its whole tiles (round robin), then the tile segments of its
// stream-K range. kind: 0 = whole tile, 1 = partial (the range ends inside the tile), 2 = finisher
// (the segment ends the tile but does not start it).
__device__ __forceinline__ bool gemm_item(int it, int unit, int nunits, int tiles, int kbs, const SplitK& sk,
                                          int& tile, int& k0, int& k1, int& kind) {
  const int ndp = unit < sk.dp_tiles ? (sk.dp_tiles - unit + nunits - 1) / nunits : 0;
  if (it < ndp) { tile = unit + it * nunits; k0 = 0; k1 = kbs; kind = 0; return true; }
  if (sk.sk_iters <= 0) return false;
  const int r0 = sk_r0(unit, nunits, sk.sk_iters), r1 = sk_r0(unit + 1, nunits, sk.sk_iters);
  if (r1 <= r0) return false;
  // segments in REVERSE order: the range's last segment (a partial other units' finishers wait for)
  // first, its first segment (possibly a finisher, which waits for lower units' partials) last — so
  // no unit waits on a partial that is produced at the end of another unit's range
  const int t0 = r0 / kbs, nseg = (r1 + kbs - 1) / kbs - t0;
  const int n = nseg - 1 - (it - ndp);
  if (n < 0) return false;
  const int pos = n == 0 ? r0 : (t0 + n) * kbs;
  tile = sk.dp_tiles + pos / kbs;
  k0 = pos % kbs;
  k1 = min(kbs, k0 + (r1 - pos));
  kind = (k0 == 0 && k1 == kbs) ? 0 : (k1 < kbs ? 1 : 2);
  return true;
}

// Tile raster: groups of `gm` m-tiles; inside a group m is fastest and n slower, so a wave of
// persistent CTAs covers a compact gm x (units / gm) block of the output — each A row block and
// each B column block is fetched from DRAM about once per group instead of once per n column
// (m-fastest over all of M re-streams A for every column).
__device__ __forceinline__ void tile_mn(int tile, int m_tiles, int n_tiles, int gm, int& mt, int& nt) {
  const int per_group = gm * n_tiles;
  const int g = tile / per_group, w = tile - g * per_group;
  const int first = g * gm;
  const int rows = min(gm, m_tiles - first);
  mt = first + w % rows;
  nt = w / rows;
}
// One output tile's fused epilogue for this warp (TMEM lane quarter q, column chunks [ch0, ch1)),
// specialised on the epilogue kind. mode 0: TMEM -> fused epilogue; 1: TMEM -> raw fp32 partial to
// this CTA's stream-K slot `wsp`; 2 (finisher): TMEM + the partial slots of units [v_lo, v_hi)
// (slot of unit v = ws + (v * CG + crank) * 128 * TILE_N) -> fused epilogue. Per-column work (bias,
// the QKV column -> (part, head, dim) decode) is done once per 32-column chunk and per-row work
// (the QKV row -> (sequence, position) decode) once per tile, so the inner loop is loads, math and
// stores only.
template <int KIND, int CG, int TILE_N, int BN>
__device__ __forceinline__ void epi_tile(const Epi& epi, const SplitK& sk, float* scr, uint32_t tmem_base, int acc, int q,
                                         int lane, int ch0, int ch1, int M, int N, int mode, int m0, int n0, float* wsp,
                                         bool has_dbias, int crank, int v_lo, int v_hi) {
  constexpr bool AUX = KIND == EPI_RESID || KIND == EPI_DGELU;
  constexpr bool BIAS = KIND == EPI_STORE || KIND == EPI_RESID || KIND == EPI_GELU || KIND == EPI_QKV;
  int rows[4];
  int64_t qoff[4];  // QKV: sequence / position offset of each of the thread's 4 rows
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    rows[it] = m0 + q * 32 + it * 8 + (lane >> 2);
    qoff[it] = 0;
    if constexpr (KIND == EPI_QKV) {
      const int sq = rows[it] % epi.bs, pos = epi.row0 + rows[it] / epi.bs;
      qoff[it] = (int64_t)sq * epi.s_len * epi.hidden + (int64_t)pos * epi.head_dim;
    }
  }
  // TMEM loads run one chunk ahead: chunk ch + 1 is loaded while chunk ch's rows are processed
  uint32_t r[32];
  tmem_ld32_async(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + ch0 * 32, r);
#pragma unroll 1
  for (int ch = ch0; ch < ch1; ++ch) {
    const int n = n0 + ch * 32 + (lane & 3) * 8;
    const int nc = n + epi.n_off;  // column in the epilogue's column space
    const bool nok = n < N;
    float aux[4][8];
    if constexpr (AUX) {
      if (mode != 1) {
#pragma unroll
        for (int it = 0; it < 4; ++it)
          if (rows[it] < M && nok) epi_prefetch8<bf16>(epi, rows[it], nc, aux[it]);
      }
    }
    float bias[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if constexpr (BIAS) {
      if (mode != 1 && nok && epi.bias) load8<float>(epi.bias + nc, bias);
    }
    bf16* qkv_col = nullptr;
    if constexpr (KIND == EPI_QKV) {
      const int part = nc / epi.hidden;
      const int within = nc - part * epi.hidden;
      const int head = within / epi.head_dim;
      const int dd = within - head * epi.head_dim;
      qkv_col = reinterpret_cast<bf16*>(part == 0 ? epi.q : (part == 1 ? epi.k : epi.v)) +
                (int64_t)head * epi.s_len * epi.head_dim + dd;
    }
    // the tile's 32 x 32 chunk lands in the warp's padded smem scratch from TMEM; a finisher adds the
    // earlier units' partials of the same rows / columns
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) scr[lane * 33 + i] = __uint_as_float(r[i]);
    if (ch + 1 < ch1) tmem_ld32_async(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + (ch + 1) * 32, r);
    __syncwarp();
    if (mode == 2) {
#pragma unroll 1
      for (int it = 0; it < 4; ++it) {
        const int rr = it * 8 + (lane >> 2);
        const int64_t woff = (int64_t)(q * 32 + rr) * TILE_N + (ch * 32 + (lane & 3) * 8);
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = scr[rr * 33 + (lane & 3) * 8 + i];
        for (int u = v_lo; u < v_hi; ++u) {
          float w[8];
          load8<float>(sk.ws + (int64_t)(u * CG + crank) * 128 * TILE_N + woff, w);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] += w[i];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) scr[rr * 33 + (lane & 3) * 8 + i] = v[i];
      }
      __syncwarp();
    }
    if (mode == 1) {  // raw fp32 partial of this K-part to the workspace
#pragma unroll 1
      for (int it = 0; it < 4; ++it) {
        const int rr = it * 8 + (lane >> 2);
        const int64_t woff = (int64_t)(q * 32 + rr) * TILE_N + (ch * 32 + (lane & 3) * 8);
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = scr[rr * 33 + (lane & 3) * 8 + i];
        if (rows[it] < M && nok) store8<float>(wsp + woff, v);
      }
      __syncwarp();
      continue;
    }
    float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // column sums (Epi::dbias)
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int rr = it * 8 + (lane >> 2);
      const int row = rows[it];
      if (row >= M || !nok) continue;
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = scr[rr * 33 + (lane & 3) * 8 + i] + bias[i];
      if constexpr (KIND == EPI_STORE) {
        if (epi.out_f32) store8<float>(reinterpret_cast<float*>(epi.out) + (int64_t)row * epi.ldo + nc, v);
        else store8<bf16>(reinterpret_cast<bf16*>(epi.out) + (int64_t)row * epi.ldo + nc, v);
      } else if constexpr (KIND == EPI_RESID) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += aux[it][i];
        store8<float>(reinterpret_cast<float*>(epi.out) + (int64_t)row * epi.ldo + nc, v);
      } else if constexpr (KIND == EPI_GELU) {
        float u[8], g[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) u[i] = to_f<bf16>(from_f<bf16>(v[i]));
#pragma unroll
        for (int i = 0; i < 8; ++i) g[i] = gelu_f<bf16>(u[i]);
        store8<bf16>(reinterpret_cast<bf16*>(epi.out) + (int64_t)row * epi.ldo + nc, u);
        store8<bf16>(reinterpret_cast<bf16*>(epi.out2) + (int64_t)row * epi.ldo2 + nc, g);
      } else if constexpr (KIND == EPI_DGELU) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_f<bf16>(aux[it][i]);
        store8<bf16>(reinterpret_cast<bf16*>(epi.out) + (int64_t)row * epi.ldo + nc, v);
        if (has_dbias)
#pragma unroll
          for (int i = 0; i < 8; ++i) cs[i] += v[i];
      } else if constexpr (KIND == EPI_QKV) {
        store8<bf16>(qkv_col + qoff[it], v);
      } else {  // EPI_ACCUM
        float* o = reinterpret_cast<float*>(epi.out) + (int64_t)row * epi.ldo + nc;
        float r0[8];
        load8<float>(o, r0);
#pragma unroll
        for (int i = 0; i < 8; ++i) r0[i] += v[i];
        store8<float>(o, r0);
      }
    }
    if constexpr (KIND == EPI_DGELU) {
      if (has_dbias) {  // the 8 lanes holding the same 8 columns reduce the warp's 32 rows
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], 4);
          cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], 8);
          cs[i] += __shfl_xor_sync(0xffffffffu, cs[i], 16);
        }
        if (lane < 4 && nok) {
          float* d = epi.dbias + nc;
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d), "f"(cs[0]), "f"(cs[1]),
                       "f"(cs[2]), "f"(cs[3]) : "memory");
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d + 4), "f"(cs[4]), "f"(cs[5]),
                       "f"(cs[6]), "f"(cs[7]) : "memory");
        }
      }
    }
    __syncwarp();
  }
}

// KIND: the epilogue (Epi::kind), a template parameter so each kernel compiles only its own
// epilogue (a runtime switch over all kinds in one kernel made ptxas spill the hot epilogue loop)
template <int CG, int BN, bool A_MN, bool B_MN, int WN, int KIND>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                      int K, Epi epi, SplitK sk, int group_m, int epi_pf) {
  using C = Cfg<CG, BN, WN>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned base derived by pointer arithmetic on the __shared__ array (not through an
  // integer cast), so the compiler keeps the shared state space: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (tc5::smem_u32(smem_raw) & 1023u)) & 1023u);
  float* epi_scratch = reinterpret_cast<float*>(smem + C::NS * C::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NS * C::STAGE + C::EPI_SCRATCH);
  uint64_t* empty = full + C::NS;
  uint64_t* tfull = empty + C::NS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  // warp index through a shuffle: provably warp-uniform, so the role branches below keep the
  // uniform datapath (descriptor arithmetic in uniform registers for tcgen05.mma)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? __shfl_sync(0xffffffffu, cluster_rank(), 0) : 0;  // warp-uniform
  const bool leader = crank == 0;
  const int m_tiles = (M + C::TILE_M - 1) / C::TILE_M, n_tiles = (N + C::TILE_N - 1) / C::TILE_N;
  const int tiles = m_tiles * n_tiles, kbs = (K + BK - 1) / BK;
  const int unit = blockIdx.x / CG, nunits = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(tfull + i, 1); mbar_init(tempty + i, 8 * CG); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
    // ---------------- TMA producer (both CTAs of a pair; bytes land on the leader's barrier)
    int stage = 0;
    uint32_t phase = 0;
    int tile, k0, k1, part;
    for (int item = 0; gemm_item(item, unit, nunits, tiles, kbs, sk, tile, k0, k1, part); ++item) {
      int mt, nt;
      tile_mn(tile, m_tiles, n_tiles, group_m, mt, nt);
      const int m0 = mt * C::TILE_M + crank * BM;
      const int nt0 = nt * C::TILE_N + crank * (BN / CG);
      for (int kb = k0; kb < k1; ++kb) {
        mbar_wait(empty + stage, phase ^ 1);
        if (leader) mbar_expect_tx(full + stage, C::STAGE * CG);
        uint8_t* a_dst = smem + stage * C::STAGE;
        if (CG == 1) {
          if (!A_MN) tma_load_2d(a_dst, &tmA, kb * BK, m0, full + stage);
          else
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) tma_load_2d(a_dst + i * 8192, &tmA, m0 + i * 64, kb * BK, full + stage);
#pragma unroll
          for (int h = 0; h < WN; ++h) {
            uint8_t* b_dst = a_dst + C::A_BYTES + h * C::B_HALF;
            const int nb0 = nt0 + h * BN;
            if (!B_MN) tma_load_2d(b_dst, &tmB, kb * BK, nb0, full + stage);
            else
#pragma unroll
              for (int i = 0; i < BN / 64; ++i) tma_load_2d(b_dst + i * 8192, &tmB, nb0 + i * 64, kb * BK, full + stage);
          }
        } else {
          const uint32_t bar = map_to_rank(smem_u32(full + stage), 0);
          if (!A_MN) tma_load_2d_pair(a_dst, &tmA, kb * BK, m0, bar);
          else
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) tma_load_2d_pair(a_dst + i * 8192, &tmA, m0 + i * 64, kb * BK, bar);
#pragma unroll
          for (int h = 0; h < WN; ++h) {
            uint8_t* b_dst = a_dst + C::A_BYTES + h * C::B_HALF;
            const int nb0 = nt0 + h * BN;
            if (!B_MN) tma_load_2d_pair(b_dst, &tmB, kb * BK, nb0, bar);
            else
#pragma unroll
              for (int i = 0; i < BN / CG / 64; ++i) tma_load_2d_pair(b_dst + i * 8192, &tmB, nb0 + i * 64, kb * BK, bar);
          }
        }
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
    }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (whole warp, one elected lane issues for the CTA / CTA pair)
    const uint32_t idesc = (1u << 4)                       // D = fp32
                           | (1u << 7) | (1u << 10)        // A, B = bf16
                           | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16)
                           | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(C::TILE_M >> 4) << 24);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    int tile, k0, k1, part;
    // stage addresses as 32-bit arithmetic on the warp-uniform window base (uniform datapath)
    const uint32_t sbase = smem_u32(smem_raw) + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    for (int item = 0; gemm_item(item, unit, nunits, tiles, kbs, sk, tile, k0, k1, part); ++item) {
      mbar_wait(tempty + acc, acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;  // WN = 2: acc = 0, halves at +0 and +BN
      for (int kb = k0; kb < k1; ++kb) {
        mbar_wait(full + stage, phase);
        tc_fence_after();
        const uint32_t a_base = sbase + stage * C::STAGE;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = A_MN ? make_desc(a_base + k * 2048, 8192, 1024) : make_desc(a_base + k * 32, 16, 1024);
#pragma unroll
          for (int h = 0; h < WN; ++h) {
            const uint32_t b_base = a_base + C::A_BYTES + h * C::B_HALF;
            const uint64_t bd = B_MN ? make_desc(b_base + k * 2048, 8192, 1024) : make_desc(b_base + k * 32, 16, 1024);
            if (CG == 1) mma_bf16_w(d_tmem + h * BN, ad, bd, idesc, (kb != k0) | (k != 0));
            else mma_bf16_pair_w(d_tmem + h * BN, ad, bd, idesc, (kb != k0) | (k != 0));
          }
        }
        if (CG == 1) mma_commit_w(empty + stage); else mma_commit_pair_w(empty + stage);  // frees the smem slot(s)
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
      if (CG == 1) mma_commit_w(tfull + acc); else mma_commit_pair_w(tfull + acc);        // accumulator ready
      if (++acc == C::NACC) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: TMEM lanes (warp % 4) * 32 .. +31 = rows of this CTA's 128
    const int q = warp & 3;
    const uint32_t tempty_leader = CG == 2 ? map_to_rank(smem_u32(tempty), 0) : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    // TMEM (thread = row) -> padded smem transpose -> 4 lanes per row, 8 columns each: every
    // global access of the fused epilogue is a 64/128-byte contiguous row segment.
    float* scr = epi_scratch + (warp - 2) * 32 * 33;
    const bool has_dbias = epi.kind == EPI_DGELU && epi.dbias != nullptr;
    const int ch0 = ((warp - 2) >> 2) * (C::TILE_N / 64), ch1 = ch0 + C::TILE_N / 64;
    auto tile_epilogue = [&](int mode, int m0, int n0, float* wsp, int v_lo, int v_hi) {
      epi_tile<KIND, CG, C::TILE_N, BN>(epi, sk, scr, tmem_base, acc, q, lane, ch0, ch1, M, N, mode, m0, n0, wsp, has_dbias,
                                        crank, v_lo, v_hi);
    };
    int tile, k0, k1, kind;
    for (int item = 0; gemm_item(item, unit, nunits, tiles, kbs, sk, tile, k0, k1, kind); ++item) {
      int mt, nt;
      tile_mn(tile, m_tiles, n_tiles, group_m, mt, nt);
      const int m0 = mt * C::TILE_M + crank * BM, n0 = nt * C::TILE_N;
      // the tile's epilogue operand (RESID: fp32 residual rows, DGELU: U) pulled into L2 while the
      // tile's MMAs run, so the epilogue's loads are L2 hits: one prefetch per 128-byte row segment
      if constexpr (KIND == EPI_RESID || KIND == EPI_DGELU) {
        if (epi_pf && (lane & 3) == 0) {
#pragma unroll 1
          for (int ch = ch0; ch < ch1; ++ch) {
            const int n = n0 + ch * 32;
            if (n >= N) break;
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int row = m0 + q * 32 + it * 8 + (lane >> 2);
              if (row >= M) break;
              const void* a = KIND == EPI_RESID
                                  ? (const void*)(epi.resid + (int64_t)row * epi.ldr + n + epi.n_off)
                                  : (const void*)(reinterpret_cast<const bf16*>(epi.aux) + (int64_t)row * epi.ld_aux + n + epi.n_off);
              asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
            }
          }
        }
      }
      int v_lo = unit, v_hi = unit;
      if (kind == 2) {
        // finisher: the units below whose ranges cover [tile start, this segment's start) left partials
        const int tstart = (tile - sk.dp_tiles) * kbs;
        while (v_lo > 0 && sk_r0(v_lo, nunits, sk.sk_iters) > tstart) --v_lo;
        if (threadIdx.x == 64) {
          for (int u = v_lo; u < v_hi; ++u) {
            const int* f = sk.flag + u * CG + crank;
            int ready = 0;
            do {
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(ready) : "l"(f) : "memory");
            } while (!ready);
          }
        }
        named_bar(1, 256);
      }
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      float* wsp = kind == 1 ? sk.ws + (int64_t)(unit * CG + crank) * 128 * C::TILE_N : nullptr;
      tile_epilogue(kind == 0 ? 0 : (kind == 1 ? 1 : 2), m0, n0, wsp, v_lo, v_hi);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 1) mbar_arrive(tempty + acc);
        else mbar_arrive_cluster(tempty_leader + acc * 8);
      }
      if (++acc == C::NACC) { acc = 0; acc_phase ^= 1; }
      if (kind == 1) {
        // partial written by all 8 epilogue warps: publish it
        named_bar(1, 256);
        if (threadIdx.x == 64) {
          __threadfence();
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sk.flag + unit * CG + crank), "r"(1) : "memory");
        }
      } else if (kind == 2) {
        named_bar(1, 256);  // every warp has read the partials: reset the flags for the next launch
        if (threadIdx.x == 64)
          for (int u = v_lo; u < v_hi; ++u) sk.flag[u * CG + crank] = 0;
      }
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                   : "memory");
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
int g_force_cg = 0;  // test hook: TP_GEMM_CG=1|2 forces the CTA-group size
// Stream-K (TP_GEMM_STREAMK=1 enables, read per launch; off by default, see launch_bn).
int g_stream_k = 0;
int g_num_sms = 0;
std::once_flag g_once;

void init_once() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    if (const char* e = getenv("TP_GEMM_CG")) g_force_cg = atoi(e);

    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  });
}

// 2-D bf16 tensor map: inner dimension `inner` (contiguous), `outer` rows of stride ld elements.
bool make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
              uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int CG, int BN, bool A_MN, bool B_MN, int WN, int KIND>
cudaError_t launch_bn(const GemmDesc& g, const Epi& e, cudaStream_t st) {
  using C = Cfg<CG, BN, WN>;
  auto kern = gemm_sm100_kernel<CG, BN, A_MN, B_MN, WN, KIND>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (r != cudaSuccess) return r;
    attr_set = true;
  }
  CUtensorMap ta, tb;
  bool ok = A_MN ? make_map(&ta, g.A, g.M, g.K, g.lda, 64, 64) : make_map(&ta, g.A, g.K, g.M, g.lda, 64, BM);
  ok = ok && (B_MN ? make_map(&tb, g.B, g.N, g.K, g.ldb, 64, 64) : make_map(&tb, g.B, g.K, g.N, g.ldb, 64, BN / CG));
  if (!ok) return cudaErrorInvalidValue;
  const int tiles = ((g.M + C::TILE_M - 1) / C::TILE_M) * ((g.N + C::TILE_N - 1) / C::TILE_N);
  int units = g.persistent ? std::min(tiles, g_num_sms / CG) : tiles;
  SplitK sk;
  sk.dp_tiles = tiles;
  const int kbs = (g.K + BK - 1) / BK;
  {
    // stream-K is opt-in (TP_GEMM_STREAMK=1): inside the full N = 1 step it measured 3-5 ms slower
    // (144.3-146.5 vs 141.1-141.4 ms, alternating runs on one box) although isolated long-K shapes
    // gain 3-8 % — the partial tiles' fp32 traffic competes with the rest of the step
    const char* e = getenv("TP_GEMM_STREAMK");
    g_stream_k = e ? atoi(e) : 0;
  }
  if (g.persistent && g_stream_k && g.sk_ws && g.sk_cnt) {
    // DP + one stream-K wave when the last wave would leave > 6 % of the units idle and each unit's
    // stream-K range keeps >= 160 k-blocks of MMA work: measured (scripts/bench_kernels.py, one
    // B200) +3-8 % at 173-664 k-blocks per unit (13B FC2 K = 20480, dW K = 16384, FC2 K = 8192 at
    // 3.5 waves) and 12-35 % slower at 51-130 (K <= 5120, or < 1 tile per unit at K = 8192): the
    // partial writes / finisher reads (~128 KB per CTA) and the un-overlapped finisher epilogue
    // need long ranges to amortise
    const int full_units = g_num_sms / CG;
    const int waves = (tiles + full_units - 1) / full_units;
    const double eff = (double)tiles / ((double)waves * full_units);
    const int dp = tiles > full_units ? (tiles / full_units - 1) * full_units : 0;
    const long long iters = (long long)(tiles - dp) * kbs;
    if (eff < 0.94 && iters / full_units >= 160 && iters * (long long)full_units < (1LL << 31)) {
      sk.dp_tiles = dp;
      sk.sk_iters = (int)iters;
      sk.ws = g.sk_ws;
      sk.flag = g.sk_cnt;
      units = full_units;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // raster group: TP_GEMM_GROUP rows of M per group (default 2048; >= M gives the plain m-fastest order)
  const int group_rows = getenv("TP_GEMM_GROUP") ? std::max(1, atoi(getenv("TP_GEMM_GROUP"))) : 2048;
  const int group_m = std::max(1, group_rows / C::TILE_M);
  // L2 prefetch of the epilogue operand ahead of each tile (TP_GEMM_EPI_PF=1; measured neutral in the
  // N = 1 step, off by default)
  static const int epi_pf = getenv("TP_GEMM_EPI_PF") ? atoi(getenv("TP_GEMM_EPI_PF")) : 0;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, g.M, g.N, g.K, e, sk, group_m, epi_pf);
}

template <int CG, int BN, int WN = 1>
cudaError_t launch_major(const GemmDesc& g, const Epi& e, cudaStream_t st) {
  // instantiated (majors x epilogue) pairs: K-major x K-major carries every layer epilogue, the
  // weight-gradient MN-major x MN-major the fp32 store / accumulate, the mixed majors (kernel tests)
  // the store
  if (!g.a_mn && !g.b_mn) {
    switch (e.kind) {
      case EPI_STORE: return launch_bn<CG, BN, false, false, WN, EPI_STORE>(g, e, st);
      case EPI_RESID: return launch_bn<CG, BN, false, false, WN, EPI_RESID>(g, e, st);
      case EPI_GELU: return launch_bn<CG, BN, false, false, WN, EPI_GELU>(g, e, st);
      case EPI_DGELU: return launch_bn<CG, BN, false, false, WN, EPI_DGELU>(g, e, st);
      case EPI_QKV: return launch_bn<CG, BN, false, false, WN, EPI_QKV>(g, e, st);
      case EPI_ACCUM: return launch_bn<CG, BN, false, false, WN, EPI_ACCUM>(g, e, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (g.a_mn && g.b_mn) {
    switch (e.kind) {
      case EPI_STORE: return launch_bn<CG, BN, true, true, WN, EPI_STORE>(g, e, st);
      case EPI_ACCUM: return launch_bn<CG, BN, true, true, WN, EPI_ACCUM>(g, e, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (e.kind != EPI_STORE) return cudaErrorInvalidValue;
  if (g.a_mn) return launch_bn<CG, BN, true, false, WN, EPI_STORE>(g, e, st);
  return launch_bn<CG, BN, false, true, WN, EPI_STORE>(g, e, st);
}

}  // namespace

bool encode_bf16_map(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box) {
  init_once();
  if (!g_encode) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides_bytes[i];
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), d, st, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool encode_f32_map_noswizzle(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims,
                              const uint64_t* strides_bytes, const uint32_t* box) {
  init_once();
  if (!g_encode) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides_bytes[i];
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(ptr), d, st, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool encode_f32_map_sw128(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims,
                          const uint64_t* strides_bytes, const uint32_t* box) {
  init_once();
  if (!g_encode) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides_bytes[i];
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(ptr), d, st, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
void gemm_sm100_workspace(size_t* ws_floats, size_t* cnt_ints) {
  init_once();
  *ws_floats = (size_t)g_num_sms * 128 * 512;  // one 128 x TILE_N (<= 512) fp32 partial slot per CTA
  *cnt_ints = (size_t)g_num_sms;
}
bool tensor_maps_available() {
  init_once();
  return g_encode != nullptr;
}
int num_sms() {
  init_once();
  return g_num_sms;
}

bool gemm_sm100_supported(const GemmDesc& g) {
  init_once();
  if (!g_encode || g_num_sms <= 0) return false;
  if (g.M < 1 || g.N < 1 || g.K < 1) return false;
  if (g.N % 8 || g.lda % 8 || g.ldb % 8) return false;
  if ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) & 15) return false;
  return true;
}

cudaError_t gemm_sm100(const GemmDesc& g, const Epi& e, cudaStream_t st) {
  init_once();
  // Tile shape by a wave-quantisation cost model: every SM gets ceil(tiles / units) tiles of
  // 128 x BN rows-per-SM work, divided by a per-shape efficiency (smaller tiles re-read more
  // operand bytes per FLOP from L2 and issue smaller MMAs). Pair tiles (256 x BN, cta_group::2)
  // need M > 128.
  struct Cand { int cg, bn; double eff; };
  // (efficiencies: per-SM operand bytes per MMA cycle are 64 / 96 / 96 / 128 B for the four shapes
  // against the ~42 B/clk L2 share; calibrated with scripts/bench_kernels.py)
  static const Cand cands[4] = {{2, 256, 1.0}, {2, 128, 0.8}, {1, 256, 0.8}, {1, 128, 0.65}};
  // Wide pair tiles (256 x 512, WN = 2) for long K: 48 instead of 64 B/clk/SM of operands, with the
  // epilogue no longer hidden behind the next tile's MMAs (relative cost ~ 1 + 4 / (K/64) k-blocks).
  // Per-tile efficiency relative to 256 x 256, measured at equal wave quantisation
  // (scripts/bench_kernels.py, profiles/r02_gemm_wide_ab.txt): 1.11 with both operands MN-major (the
  // weight-gradient GEMMs); with K-major A (forward / dX GEMMs, where the 4-stage ring of 48 KB
  // stages hides less latency than the 6-stage ring of the 256 x 256 tiles) ~0.99 at K = 6144-8192
  // and ~1.04 at K = 20480 (13B FC2). TP_GEMM_WIDE=0 disables, =1 forces (when the shape allows).
  const int wide_env = getenv("TP_GEMM_WIDE") ? atoi(getenv("TP_GEMM_WIDE")) : -1;
  if (wide_env != 0 && !g_force_cg && g.persistent && g.M > BM && g.N >= 512 && (g.K >= 4096 || wide_env == 1)) {
    const long units = g_num_sms / 2;
    const long tw = (long)((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + 511) / 512);
    const long t2 = (long)((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + 255) / 256);
    const double kbs = (g.K + BK - 1) / BK;
    const double wide_eff = (g.a_mn && g.b_mn) ? 1.11 : (kbs >= 256 ? 1.05 : 0.99);
    const double cost_wide = (double)((tw + units - 1) / units) * 512 / wide_eff * (1.0 + 4.0 / kbs);
    const double cost_256 = (double)((t2 + units - 1) / units) * 256;
    if (wide_env == 1 || cost_wide < cost_256 * 0.97) return launch_major<2, 256, 2>(g, e, st);
  }
  int best = -1;
  double best_cost = 0;
  for (int i = 0; i < 4; ++i) {
    const Cand& c = cands[i];
    if ((c.cg == 2 && g.M <= BM) || (g_force_cg && c.cg != g_force_cg)) continue;
    const long units = g_num_sms / c.cg;
    const long tiles = (long)((g.M + BM * c.cg - 1) / (BM * c.cg)) * ((g.N + c.bn - 1) / c.bn);
    const double cost = (double)((tiles + units - 1) / units) * c.bn / c.eff;
    if (best < 0 || cost < best_cost * 0.999) { best = i; best_cost = cost; }
  }
  auto launch = [&](int which, const GemmDesc& gg, const Epi& ee) -> cudaError_t {
    switch (which) {
      case 0: return launch_major<2, 256>(gg, ee, st);
      case 1: return launch_major<2, 128>(gg, ee, st);
      case 2: return launch_major<1, 256>(gg, ee, st);
      default: return launch_major<1, 128>(gg, ee, st);
    }
  };
  // Tail split: when the chosen shape leaves a partial last wave, run the n-tile columns that fill
  // whole waves with it and the remaining columns as a second launch with half-width tiles (twice
  // the tiles, half the time each), if the model says that is cheaper: the partial wave then costs
  // half a wave. The second launch sees its columns through Epi::n_off.
  // stream-K (launch_bn) supersedes this split where it can apply: K long enough for >= 2 parts of
  // >= 32 k-blocks each
  const bool sk_on = getenv("TP_GEMM_STREAMK") && atoi(getenv("TP_GEMM_STREAMK")) != 0 && (g.K + BK - 1) / BK >= 64;
  if (!sk_on && g.persistent && !g_force_cg && (best == 0 || best == 2)) {
    const Cand& c = cands[best];
    const Cand& h = cands[best + 1];  // same CTA group, BN / 2
    const long units = g_num_sms / c.cg;
    const long mt = (g.M + BM * c.cg - 1) / (BM * c.cg), nt = (g.N + c.bn - 1) / c.bn;
    const long full = (mt * nt) / units;
    const long n1 = full * units / mt;  // n-tile columns covered by whole waves
    if (full >= 1 && n1 >= 1 && n1 < nt) {
      const long t1 = n1 * mt, t2 = mt * ((g.N - n1 * c.bn + h.bn - 1) / h.bn);
      const double split = (double)((t1 + units - 1) / units) * c.bn / c.eff +
                           (double)((t2 + units - 1) / units) * h.bn / h.eff + 8.0 /* second launch */;
      if (split < best_cost * 0.95) {
        const int N1 = (int)(n1 * c.bn);
        GemmDesc g1 = g, g2 = g;
        g1.N = N1;
        g2.N = g.N - N1;
        const size_t off = g.b_mn ? (size_t)N1 : (size_t)N1 * g.ldb;
        g2.B = reinterpret_cast<const bf16*>(g.B) + off;
        Epi e2 = e;
        e2.n_off = e.n_off + N1;
        cudaError_t r = launch(best, g1, e);
        if (r != cudaSuccess) return r;
        return launch(best + 1, g2, e2);
      }
    }
  }
  return launch(best, g, e);
}

}  // namespace tp
