// runtime.cu — tp_ctx: stage executor, per-stage op lists and the pipeline schedule of tp_step.
//
// Hot path (BASELINE.json:5; §3.2): stage k owns layers [k n/K, (k+1) n/K)
// (uniform cells) and processes one token slice of one sequence at a time.
// For every layer it runs the slice's QKV / out-projection / MLP GEMMs, causal attention of the
// slice's queries against the per-layer prefix K/V cache, and in backward the dK/dV push into
// the earlier slices' rows. Slice activations go to stage k+1 and gradients return to stage k-1
// — as device copies in loopback mode (world == 1) or ncclSend/ncclRecv over
// NVLink (world == K).
//
// Schedule (A-21): each stage runs F(d, i) for d = 0..B-1, i = 1..M, then B(d, i) in
// exact reverse order (GPipe order, store-all); the weight gradients of sequence d
// are accumulated once its last backward slice B(d, 1) is done (deferred dW, K-dim = s).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.h"

namespace tp {

#define CU(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return ::tp::fail(TP_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
  } while (0)
#define NC(x)                                                                              \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess)                                                                 \
      return ::tp::fail(TP_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #x, ncclGetErrorString(r_)); \
  } while (0)
#define TRY(x)                      \
  do {                              \
    tp_status s_ = (x);             \
    if (s_ != TP_OK) return s_;     \
  } while (0)

struct ModelShape {
  int n_layer, H, a, d, V, s, K;
  int partition = 0;  // TP_PARTITION_*
};

// Layers owned by each stage (A-30). Uniform: n/K each. Balanced: the
// last stage also runs the LM head + CE, h = V / (12 H + s) layers' worth of FLOPs per token (head
// 6 H V vs a layer's 72 H^2 + 6 s H); choose the last stage's count nl minimising
// max(ceil((n - nl) / (K - 1)), nl + h) (ties: the larger nl), spread the rest evenly, stages
// 1.. taking the remainder (stage 0 also holds the embedding). synth/__init__.py has the same rule.
static std::vector<int> stage_layer_counts(int n, int K, int H, int V, int s, int partition) {
  std::vector<int> out(K, K > 0 ? n / K : 0);
  if (partition != TP_PARTITION_BALANCED || K == 1) return out;
  const double h = (double)V / (12.0 * H + s);
  int best_nl = n / K;
  double best = 1e300;
  for (int nl = 1; nl <= n - (K - 1); ++nl) {
    const int r = n - nl;
    const double cost = std::max((double)((r + K - 2) / (K - 1)), nl + h);
    if (cost < best || (cost == best && nl > best_nl)) { best = cost; best_nl = nl; }
  }
  const int r = n - best_nl, base = r / (K - 1), extra = r % (K - 1);
  for (int k = 0; k < K - 1; ++k) out[k] = base + ((k >= 1 && k <= extra) ? 1 : 0);
  if (extra == K - 1) out[0] += 1;  // (cannot happen: extra < K - 1)
  out[K - 1] = best_nl;
  return out;
}
static int stage_first_layer(const ModelShape& m, int k) {
  const std::vector<int> c = stage_layer_counts(m.n_layer, m.K, m.H, m.V, m.s, m.partition);
  int f = 0;
  for (int i = 0; i < k; ++i) f += c[i];
  return f;
}
static int stage_nl(const ModelShape& m, int k) {
  return stage_layer_counts(m.n_layer, m.K, m.H, m.V, m.s, m.partition)[k];
}

// Offsets (in floats) of every tensor inside one stage's flat parameter array (include/tp.h).
struct LayerOff {
  size_t ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_1, b_1, w_2, b_2;
};
// Offsets of the fp32 parameters kept on the device as fp32 (LayerNorm, biases, embeddings) inside
// the compact `psmall` array; weight matrices live only as bf16 (or fp32-mode) GEMM operands.
struct SmallOff {
  size_t ln1_g, ln1_b, b_qkv, b_o, ln2_g, ln2_b, b_1, b_2;
};
struct StageLayout {
  size_t wte = 0, wpe = 0, lnf_g = 0, lnf_b = 0, w_out = 0, total = 0;
  std::vector<LayerOff> layers;
  size_t s_wte = 0, s_wpe = 0, s_lnf_g = 0, s_lnf_b = 0, small_total = 0;
  std::vector<SmallOff> small;
};

static StageLayout stage_layout(const ModelShape& m, int k) {
  StageLayout L;
  size_t o = 0;
  const size_t H = m.H;
  if (k == 0) { L.wte = o; o += (size_t)m.V * H; L.wpe = o; o += (size_t)m.s * H; }
  const int nl = stage_nl(m, k);
  for (int j = 0; j < nl; ++j) {
    LayerOff f;
    f.ln1_g = o; o += H; f.ln1_b = o; o += H;
    f.w_qkv = o; o += H * 3 * H; f.b_qkv = o; o += 3 * H;
    f.w_o = o; o += H * H; f.b_o = o; o += H;
    f.ln2_g = o; o += H; f.ln2_b = o; o += H;
    f.w_1 = o; o += H * 4 * H; f.b_1 = o; o += 4 * H;
    f.w_2 = o; o += 4 * H * H; f.b_2 = o; o += H;
    L.layers.push_back(f);
  }
  if (k == m.K - 1) { L.lnf_g = o; o += H; L.lnf_b = o; o += H; L.w_out = o; o += H * (size_t)m.V; }
  L.total = o;
  size_t q = 0;
  if (k == 0) { L.s_wte = q; q += (size_t)m.V * H; L.s_wpe = q; q += (size_t)m.s * H; }
  for (int j = 0; j < nl; ++j) {
    SmallOff f;
    f.ln1_g = q; q += H; f.ln1_b = q; q += H; f.b_qkv = q; q += 3 * H; f.b_o = q; q += H;
    f.ln2_g = q; q += H; f.ln2_b = q; q += H; f.b_1 = q; q += 4 * H; f.b_2 = q; q += H;
    L.small.push_back(f);
  }
  if (k == m.K - 1) { L.s_lnf_g = q; q += H; L.s_lnf_b = q; q += H; }
  L.small_total = q;
  return L;
}

// ---------------------------------------------------------------- kernel statistics
struct KStat {
  const char* name;
  int64_t launches = 0;
  double ms = 0, flops = 0, bytes = 0;
};
enum KClass {
  KC_GEMM_FWD = 0, KC_GEMM_DX, KC_GEMM_DW, KC_ATTN_FWD, KC_ATTN_BWD, KC_LN, KC_EMBED, KC_CE, KC_MISC, KC_COMM, KC_N
};
static const char* kKClassNames[KC_N] = {"gemm_fwd", "gemm_dx", "gemm_dw", "attn_fwd", "attn_bwd",
                                          "layernorm", "embed", "cross_entropy", "misc", "p2p"};

struct Pending {
  int cls;
  double flops, bytes;
  cudaEvent_t a, b;
};

class Instr {
 public:
  bool on = false;
  int64_t launches = 0;
  KStat stats[KC_N];
  std::vector<cudaEvent_t> pool;
  std::vector<Pending> pending;
  size_t next = 0;
  Instr() { for (int i = 0; i < KC_N; ++i) stats[i].name = kKClassNames[i]; }
  ~Instr() { for (auto e : pool) cudaEventDestroy(e); }
  cudaEvent_t ev() {
    if (next == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[next++];
  }
  void begin(cudaStream_t st, int cls, double flops, double bytes, Pending& p) {
    ++launches;
    if (!on) return;
    p.cls = cls; p.flops = flops; p.bytes = bytes;
    p.a = ev(); p.b = ev();
    cudaEventRecord(p.a, st);
  }
  void end(cudaStream_t st, Pending& p) {
    if (!on) return;
    cudaEventRecord(p.b, st);
    pending.push_back(p);
  }
  void resolve() {  // after a device sync
    for (auto& p : pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, p.a, p.b);
      stats[p.cls].launches++;
      stats[p.cls].ms += ms;
      stats[p.cls].flops += p.flops;
      stats[p.cls].bytes += p.bytes;
    }
    pending.clear();
    next = 0;
  }
};

// ---------------------------------------------------------------- schedule
// Per-stage op lists (A-21): GPipe — every F(d, i) in order, then every B in exact
// reverse; 1F1B at group granularity — stage k runs the forwards of its first
// w_k = min(D, K - k) groups, then alternates the backward of its oldest group (slices in reverse)
// with the forward of the next one, then drains. Exported as tp_schedule_oplist and pinned to
// oracle/plan.py (gpipe_oplists / one_f_one_b_oplists).
struct Op {
  bool fwd;
  int d, i;
};
static std::vector<Op> build_oplist(int K, int k, bool one_f_one_b, const std::vector<int>& M) {
  const int D = (int)M.size();
  std::vector<Op> ops;
  auto F = [&](int d) { for (int i = 0; i < M[d]; ++i) ops.push_back({true, d, i}); };
  auto B = [&](int d) { for (int i = M[d] - 1; i >= 0; --i) ops.push_back({false, d, i}); };
  if (!one_f_one_b) {
    for (int d = 0; d < D; ++d) F(d);
    for (int d = D - 1; d >= 0; --d) B(d);
    return ops;
  }
  const int w = std::min(D, K - k);
  for (int d = 0; d < w; ++d) F(d);
  for (int d = 0; d < D; ++d) {
    B(d);
    if (d + w < D) F(d + w);
  }
  return ops;
}

// ---------------------------------------------------------------- engine
struct EngineBase {
  virtual ~EngineBase() = default;
  virtual tp_status load(const float* host, size_t n) = 0;
  virtual tp_status step(const tp_slicing* sl, const int32_t* tokens, bool host_tokens, int batch, float* loss) = 0;
  virtual tp_status step_plan(const tp_batch_plan* pl, const int32_t* tokens, bool host_tokens, int batch,
                              float* loss) = 0;
  virtual tp_status grads(float* host, size_t n) = 0;
  virtual tp_status logits(float* host, size_t n) = 0;
  virtual tp_status profile(int g, int b, int reps, int64_t* ticks, double* fit) = 0;
  virtual tp_status profile_wgrad(int batch, int reps, int64_t* ns_out) = 0;
  virtual tp_status profile_comm(int reps, double* alpha_ns, double* gbs) = 0;
  virtual size_t param_count() const = 0;
  Instr instr;
  cudaStream_t stream = nullptr;
};

template <typename T>
struct Stage {
  int k = 0, nl = 0;
  bool aliased = false;  // loopback: hs[0] / grad_in are the previous stage's hs[nl] / grad_out buffers
  StageLayout L;
  float* psmall = nullptr;  // fp32 LayerNorm / bias / embedding parameters (StageLayout::small offsets)
  float* gflat = nullptr;  // fp32 grads (flat layout)
  // GEMM operands in T: *_t = [out][in] (K-major B for fwd), *_io = [in][out] (K-major B for dX)
  std::vector<T*> wqkv_t, wqkv_io, wo_t, wo_io, w1_t, w1_io, w2_t, w2_io;
  T *wout_t = nullptr, *wout_io = nullptr;
  // activations, store-all over [B][s]
  std::vector<float*> hs;    // nl+1 of [B][s][H] fp32; hs[0] = stage input, hs[nl] = stage output
  std::vector<float*> hmid;  // [B][s][H] fp32
  std::vector<T*> A1, A2, O;      // [B][s][H]
  std::vector<float*> st1, st2;   // [2][B][s] (mean, rstd)
  std::vector<T*> Q, Kc, Vc;      // [B][a][s][d]
  std::vector<float*> LSE;        // [B][a][s]
  std::vector<T*> U, G;           // [B][s][4H]
  T* Af = nullptr; float* stf = nullptr;
  T* Z = nullptr;                 // [B][s][V] logits -> dlogits in place
  float* loss_rows = nullptr;     // [B][s]
  float* logits_keep = nullptr;   // [B][s][V] (TP_FLAG_KEEP_LOGITS)
  float* grad_out = nullptr;      // [B][s][H] dloss/d(stage output)
  float* grad_in = nullptr;       // [B][s][H] dloss/d(stage input)
  // backward stash over [B][s] rows: the operands of the deferred weight-gradient GEMMs
  std::vector<T*> dQKV, dhmid_b, dU, dhout_b;
  std::vector<float*> dk_acc, dv_acc;  // [a][s][d]
  float *gA = nullptr, *gB = nullptr, *gm = nullptr, *dA = nullptr, *Dvec = nullptr, *lnws = nullptr, *dqacc = nullptr;
  T* dO = nullptr;
};

template <typename T>
class Engine final : public EngineBase {
 public:
  ModelShape m;
  int rank, world, k0, k1, precision, flags, max_batch, device;
  bool force_simt;
  bool legacy_attn = false;  // env TP_LEGACY_ATTN=1: mma.sync attention instead of tcgen05 (cross-checks)
  std::vector<Stage<T>> stages;
  std::vector<void*> allocs;
  int32_t* d_tokens = nullptr;
  float* d_loss = nullptr;
  float* sk_ws = nullptr;  // stream-K workspace of the persistent GEMMs on `stream` (fixed size)
  int* sk_cnt = nullptr;
  int* d_bad_tok = nullptr;  // device token check of the *_device steps: count of ids outside [0, V)
  int* h_bad_tok = nullptr;  // pinned
  float* h_loss = nullptr;  // pinned
  int last_batch = 0;
  std::vector<std::pair<size_t, int>> last_groups;  // (seq0, b) of the last step's groups
  int32_t* h_tokens = nullptr;  // pinned staging of the step's tokens
  // CUDA graph of the last (slicing, batch) op list
  bool use_graphs = true;
  std::vector<int64_t> g_key;
  cudaGraphExec_t g_exec = nullptr;
  int64_t g_launches = 0;
  // NCCL (multi-rank, or the single-GPU NCCL loopback of TP_FLAG_NCCL_LOOPBACK)
  bool nccl_lb = false;  // world == 1, K > 1: stage messages through ncclSend/ncclRecv to self
  bool sched_1f1b = false;  // TP_FLAG_SCHEDULE_1F1B: group-granular 1F1B op lists, slot-mapped stash
  // device-initiated p2p (TP_FLAG_DEVICE_P2P, world > 1; p2p.cu): hs[0] / grad_out of the owned stage
  // are NCCL symmetric windows written directly by the neighbours' kernels
  bool dev_p2p = false;
  ncclWindow_t win_in = nullptr, win_gout = nullptr, win_flag = nullptr;
  void *p_in = nullptr, *p_gout = nullptr, *p_flag = nullptr;
  float* peer_in = nullptr;                       // rank + 1's hs[0]
  float* peer_gout = nullptr;                     // rank - 1's grad_out
  unsigned long long* peer_flag_next = nullptr;   // rank + 1's flag slots
  unsigned long long* peer_flag_prev = nullptr;   // rank - 1's flag slots
  unsigned long long* d_epoch = nullptr;
  size_t n_slots = 0;                             // per direction: max jobs per step
  ncclComm_t base = nullptr, commF[2] = {nullptr, nullptr}, commB[2] = {nullptr, nullptr};
  cudaStream_t s_recv_f = nullptr, s_send_f = nullptr, s_recv_b = nullptr, s_send_b = nullptr;
  cudaStream_t s_wgrad = nullptr;  // low priority: deferred weight gradients (multi-rank)
  // second stream of the deferred weight-gradient phase: consecutive dW GEMMs alternate between
  // `stream` and this one, so the partial last wave of one persistent GEMM overlaps the first tiles of
  // the next (TP_DW_STREAMS=1: one stream)
  cudaStream_t s_dw2 = nullptr;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;

  ~Engine() override {
    if (stream) cudaStreamSynchronize(stream);
    if (g_exec) cudaGraphExecDestroy(g_exec);
    if (h_tokens) cudaFreeHost(h_tokens);
    if (d_tokens) cudaFree(d_tokens);
    for (auto& S : stages) if (S.loss_rows) cudaFree(S.loss_rows);
    for (ncclWindow_t w : {win_in, win_gout, win_flag})
      if (w) ncclCommWindowDeregister(base, w);
    for (void* p : {p_in, p_gout, p_flag})
      if (p) ncclMemFree(p);
    for (ncclComm_t c : {commF[0], commF[1], commB[0], commB[1], base})
      if (c) ncclCommDestroy(c);
    for (void* p : allocs) cudaFree(p);
    if (h_loss) cudaFreeHost(h_loss);
    if (h_bad_tok) cudaFreeHost(h_bad_tok);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (cudaStream_t s : {s_recv_f, s_send_f, s_recv_b, s_send_b, s_wgrad, s_dw2, stream})
      if (s) cudaStreamDestroy(s);
  }

  size_t param_count() const override {
    size_t n = 0;
    for (auto& st : stages) n += st.L.total;
    return n;
  }

  template <typename U_>
  tp_status alloc(U_** p, size_t count) {
    if (count == 0) { *p = nullptr; return TP_OK; }
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(U_));
    if (e != cudaSuccess)
      return fail(TP_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", count * sizeof(U_), cudaGetErrorString(e));
    allocs.push_back(q);
    *p = reinterpret_cast<U_*>(q);
    return TP_OK;
  }

  cudaEvent_t event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }

  tp_status init(const tp_model_cfg* cfg, int rank_, int world_, const void* nccl_id, int precision_,
                 int max_batch_, int device_, int flags_) {
    m = {cfg->n_layer, cfg->hidden, cfg->n_head, cfg->hidden / cfg->n_head, cfg->vocab, cfg->seq_len, cfg->n_stages,
         cfg->partition};
    rank = rank_; world = world_; precision = precision_; flags = flags_; max_batch = max_batch_; device = device_;
    force_simt = (flags & TP_FLAG_FORCE_SIMT) != 0 || precision == TP_FP32;
    instr.on = (flags & TP_FLAG_KERNEL_STATS) != 0;
    if (const char* e = std::getenv("TP_LEGACY_ATTN")) legacy_attn = std::atoi(e) != 0;
    if (world == 1) { k0 = 0; k1 = m.K; } else { k0 = rank; k1 = rank + 1; }
    nccl_lb = world == 1 && m.K > 1 && (flags & TP_FLAG_NCCL_LOOPBACK) != 0;
    sched_1f1b = (flags & TP_FLAG_SCHEDULE_1F1B) != 0 ||
                 (std::getenv("TP_SCHEDULE") && std::string(std::getenv("TP_SCHEDULE")) == "1f1b");
    dev_p2p = world > 1 && ((flags & TP_FLAG_DEVICE_P2P) != 0 ||
                            (std::getenv("TP_DEVICE_P2P") && std::atoi(std::getenv("TP_DEVICE_P2P")) != 0));
    CU(cudaSetDevice(device));
    int major = 0;
    CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) return fail(TP_ECUDA, "device %d has compute capability %d.x; this build targets sm_100a", device, major);
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, hi));
    if (!(std::getenv("TP_DW_STREAMS") && std::atoi(std::getenv("TP_DW_STREAMS")) == 1))
      CU(cudaStreamCreateWithPriority(&s_dw2, cudaStreamNonBlocking, hi));
    CU(cudaHostAlloc(&h_loss, sizeof(float), cudaHostAllocDefault));

    use_graphs = std::getenv("TP_NO_GRAPHS") == nullptr && std::getenv("TP_ATTN_DEBUG") == nullptr;
    TRY(alloc(&d_loss, 4));
    CU(cudaHostAlloc(&h_bad_tok, sizeof(int), cudaHostAllocDefault));
    TRY(alloc(&d_bad_tok, 1));
    if (std::is_same<T, bf16>::value && !force_simt) {
      // bf16 mode runs every GEMM on the tcgen05 kernel: no silent SIMT fallback
      if (!tensor_maps_available())
        return fail(TP_ECUDA, "tp_init: cuTensorMapEncodeTiled is unavailable (driver too old?); the bf16 path needs TMA");
      size_t nw = 0, nc = 0;
      gemm_sm100_workspace(&nw, &nc);
      TRY(alloc(&sk_ws, nw));
      TRY(alloc(&sk_cnt, nc));
      CU(cudaMemset(sk_cnt, 0, nc * sizeof(int)));
    }
    stages.resize(k1 - k0);
    for (int k = k0; k < k1; ++k) TRY(alloc_stage(stages[k - k0], k));
    TRY(ensure_batch_capacity(max_batch));
    if (world > 1 || nccl_lb) {
      if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        NC(ncclCommInitRank(&base, world, id, rank));
      } else {
        // one-rank communicator: stage k -> k+1 messages are ncclSend/ncclRecv to self (the same
        // NCCL p2p kernels, streams and events as world == K; runnable on a one-GPU box)
        int dev = device;
        NC(ncclCommInitAll(&base, 1, &dev));
      }
      // one communicator per (direction, edge parity): each rank uses each communicator from
      // exactly one stream, so p2p ops on a communicator are issued in one order on both ends.
      for (int i = 0; i < 2; ++i) {
        NC(ncclCommSplit(base, 0, rank, &commF[i], nullptr));
        NC(ncclCommSplit(base, 0, rank, &commB[i], nullptr));
      }
      if (dev_p2p) TRY(setup_device_p2p());
      CU(cudaStreamCreateWithPriority(&s_recv_f, cudaStreamNonBlocking, hi));
      CU(cudaStreamCreateWithPriority(&s_send_f, cudaStreamNonBlocking, hi));
      CU(cudaStreamCreateWithPriority(&s_recv_b, cudaStreamNonBlocking, hi));
      CU(cudaStreamCreateWithPriority(&s_send_b, cudaStreamNonBlocking, hi));
      // opt-in (TP_SIDE_DW=1): per-group weight gradients on a low-priority stream. Measured on 4 x B200
      // it slows the step (1B 64.2 vs 56.1 ms, 13B 435 vs 418 ms): its one-tile-per-CTA GEMMs hold SMs
      // the critical path needs and the per-group fp32 gradient RMW adds HBM traffic.
      if (std::getenv("TP_SIDE_DW") != nullptr) CU(cudaStreamCreateWithPriority(&s_wgrad, cudaStreamNonBlocking, lo));
    }
    CU(cudaStreamSynchronize(stream));
    return TP_OK;
  }

  tp_status alloc_stage(Stage<T>& S, int k) {
    S.k = k;
    S.nl = stage_nl(m, k);
    S.L = stage_layout(m, k);
    const size_t B = max_batch, s = m.s, H = m.H, a = m.a, nl = S.nl;
    TRY(alloc(&S.psmall, S.L.small_total));
    TRY(alloc(&S.gflat, S.L.total));
    auto vec = [&](auto& v, size_t n, size_t count) -> tp_status {
      v.resize(n);
      for (size_t i = 0; i < n; ++i) TRY(alloc(&v[i], count));
      return TP_OK;
    };
    TRY(vec(S.wqkv_t, nl, 3 * H * H)); TRY(vec(S.wqkv_io, nl, 3 * H * H));
    TRY(vec(S.wo_t, nl, H * H)); TRY(vec(S.wo_io, nl, H * H));
    TRY(vec(S.w1_t, nl, 4 * H * H)); TRY(vec(S.w1_io, nl, 4 * H * H));
    TRY(vec(S.w2_t, nl, 4 * H * H)); TRY(vec(S.w2_io, nl, 4 * H * H));
    const bool first = k == 0, last = k == m.K - 1;
    if (last) { TRY(alloc(&S.wout_t, H * m.V)); TRY(alloc(&S.wout_io, H * m.V)); }
    S.hs.assign(nl + 1, nullptr);
    // loopback: stage k's input buffer IS stage k-1's output buffer (the "send" is free)
    // (1F1B: stages use different slot rows for the same group, so messages are copies)
    const bool alias = world == 1 && k > k0 && !nccl_lb && !sched_1f1b;
    S.aliased = alias;
    if (alias) S.hs[0] = stages[k - 1 - k0].hs[stages[k - 1 - k0].nl];
    // device p2p: hs[0] and grad_out become NCCL symmetric windows (setup_device_p2p, after the comm)
    for (size_t j = (alias || dev_p2p) ? 1 : 0; j <= nl; ++j) TRY(alloc(&S.hs[j], B * s * H));
    TRY(vec(S.hmid, nl, B * s * H));
    TRY(vec(S.A1, nl, B * s * H)); TRY(vec(S.A2, nl, B * s * H)); TRY(vec(S.O, nl, B * s * H));
    TRY(vec(S.st1, nl, 2 * B * s)); TRY(vec(S.st2, nl, 2 * B * s));
    TRY(vec(S.Q, nl, B * s * H)); TRY(vec(S.Kc, nl, B * s * H)); TRY(vec(S.Vc, nl, B * s * H));
    TRY(vec(S.LSE, nl, B * a * s));
    TRY(vec(S.U, nl, B * s * 4 * H)); TRY(vec(S.G, nl, B * s * 4 * H));
    if (last) {
      TRY(alloc(&S.Af, B * s * H)); TRY(alloc(&S.stf, 2 * B * s));
      TRY(alloc(&S.Z, B * s * (size_t)m.V));  // loss_rows: ensure_batch_capacity (batch rows)
      if (flags & TP_FLAG_KEEP_LOGITS) TRY(alloc(&S.logits_keep, B * s * (size_t)m.V));
    }
    if (!dev_p2p) TRY(alloc(&S.grad_out, B * s * H));
    if (alias) {
      // stage k-1's grad_out IS stage k's grad_in
      Stage<T>& P = stages[k - 1 - k0];
      S.grad_in = P.grad_out;
    } else {
      TRY(alloc(&S.grad_in, B * s * H));
    }
    (void)first;
    TRY(vec(S.dQKV, nl, B * s * 3 * H)); TRY(vec(S.dhmid_b, nl, B * s * H));
    TRY(vec(S.dU, nl, B * s * 4 * H)); TRY(vec(S.dhout_b, nl, B * s * H));
    // per job: up to b = max_batch sequences of one slice
    TRY(vec(S.dk_acc, nl, B * s * H)); TRY(vec(S.dv_acc, nl, B * s * H));
    TRY(alloc(&S.gA, B * s * H)); TRY(alloc(&S.gB, B * s * H)); TRY(alloc(&S.gm, B * s * H)); TRY(alloc(&S.dA, B * s * H));
    // Dvec: the sm100 backward's per-tile lse / D staging, [b][a][ceil(l/64)][128]
    TRY(alloc(&S.Dvec, 2 * B * a * (s + 64))); TRY(alloc(&S.dO, B * s * H));
    TRY(alloc(&S.lnws, 2 * H * ((B * s + 3) / 4)));
    TRY(alloc(&S.dqacc, B * s * H));
    return TP_OK;
  }

  // Per-batch (not per-slot) buffers: tokens (device + pinned staging) and the last stage's per-row
  // losses, grown when a 1F1B step's batch exceeds the current capacity (outside any capture; the
  // cached step graph referencing the old buffers is dropped).
  size_t tok_cap = 0;
  tp_status ensure_batch_capacity(int batch) {
    if ((size_t)batch <= tok_cap) return TP_OK;
    if (stream) CU(cudaStreamSynchronize(stream));
    if (g_exec) { cudaGraphExecDestroy(g_exec); g_exec = nullptr; g_key.clear(); }
    if (d_tokens) cudaFree(d_tokens);
    if (h_tokens) cudaFreeHost(h_tokens);
    d_tokens = nullptr; h_tokens = nullptr;
    const size_t n = (size_t)batch * (m.s + 1);
    if (cudaMalloc(&d_tokens, n * sizeof(int32_t)) != cudaSuccess) return fail(TP_ENOMEM, "tokens: cudaMalloc");
    CU(cudaHostAlloc(&h_tokens, n * sizeof(int32_t), cudaHostAllocDefault));
    for (auto& S : stages)
      if (S.k == m.K - 1) {
        if (S.loss_rows) cudaFree(S.loss_rows);
        S.loss_rows = nullptr;
        if (cudaMalloc(&S.loss_rows, (size_t)batch * m.s * sizeof(float)) != cudaSuccess)
          return fail(TP_ENOMEM, "loss rows: cudaMalloc");
      }
    tok_cap = batch;
    return TP_OK;
  }

  // Symmetric windows for the stage's receive buffers and flag slots (collective over the ranks,
  // identical sizes everywhere), and the neighbours' addresses inside them.
  tp_status setup_device_p2p() {
    Stage<T>& S = stages[0];
    const size_t act = (size_t)max_batch * m.s * m.H * sizeof(float);
    const size_t abytes = (act + 4095) / 4096 * 4096;
    n_slots = (size_t)max_batch * m.s;
    const size_t fbytes = (2 * n_slots * sizeof(unsigned long long) + 4095) / 4096 * 4096;
    NC(ncclMemAlloc(&p_in, abytes));
    NC(ncclMemAlloc(&p_gout, abytes));
    NC(ncclMemAlloc(&p_flag, fbytes));
    CU(cudaMemset(p_flag, 0, fbytes));
    NC(ncclCommWindowRegister(base, p_in, abytes, &win_in, NCCL_WIN_COLL_SYMMETRIC));
    NC(ncclCommWindowRegister(base, p_gout, abytes, &win_gout, NCCL_WIN_COLL_SYMMETRIC));
    NC(ncclCommWindowRegister(base, p_flag, fbytes, &win_flag, NCCL_WIN_COLL_SYMMETRIC));
    S.hs[0] = reinterpret_cast<float*>(p_in);
    S.grad_out = reinterpret_cast<float*>(p_gout);
    void* q = nullptr;
    if (rank + 1 < world) {
      CU(p2p_peer_pointer(win_in, rank + 1, &q, stream)); peer_in = reinterpret_cast<float*>(q);
      CU(p2p_peer_pointer(win_flag, rank + 1, &q, stream)); peer_flag_next = reinterpret_cast<unsigned long long*>(q);
    }
    if (rank > 0) {
      CU(p2p_peer_pointer(win_gout, rank - 1, &q, stream)); peer_gout = reinterpret_cast<float*>(q);
      CU(p2p_peer_pointer(win_flag, rank - 1, &q, stream)); peer_flag_prev = reinterpret_cast<unsigned long long*>(q);
    }
    TRY(alloc(&d_epoch, 1));
    CU(cudaMemset(d_epoch, 0, sizeof(unsigned long long)));
    return TP_OK;
  }

  // ------------------------------------------------------------ parameter load
  tp_status load(const float* host, size_t n) override {
    if (n != param_count()) return fail(TP_EINVAL, "tp_load_params: n=%zu, expected %zu", n, param_count());
    // weight matrices go through one fp32 staging buffer into their two GEMM-operand copies
    size_t big = (size_t)4 * m.H * m.H;
    for (auto& S : stages) if (S.k == m.K - 1) big = std::max(big, (size_t)m.H * m.V);
    float* stage_buf = nullptr;
    CU(cudaMalloc(&stage_buf, big * sizeof(float)));
    auto put = [&](float* dst, const float* src, size_t cnt) -> tp_status {
      CU(cudaMemcpyAsync(dst, src, cnt * sizeof(float), cudaMemcpyHostToDevice, stream));
      return TP_OK;
    };
    auto mat = [&](const float* src, int R, int Cc, T* t_copy, T* io_copy) -> tp_status {
      CU(cudaMemcpyAsync(stage_buf, src, (size_t)R * Cc * sizeof(float), cudaMemcpyHostToDevice, stream));
      CU(transpose_convert<T>(stage_buf, t_copy, R, Cc, stream));
      CU(convert_f32<T>(stage_buf, io_copy, (int64_t)R * Cc, stream));
      CU(cudaStreamSynchronize(stream));
      return TP_OK;
    };
    tp_status st = TP_OK;
    size_t off = 0;
    const size_t H = m.H;
    for (auto& S : stages) {
      const float* h = host + off;
      const StageLayout& L = S.L;
      if (S.k == 0) {
        if ((st = put(S.psmall + L.s_wte, h + L.wte, (size_t)m.V * H)) != TP_OK) break;
        if ((st = put(S.psmall + L.s_wpe, h + L.wpe, (size_t)m.s * H)) != TP_OK) break;
      }
      for (int j = 0; j < S.nl && st == TP_OK; ++j) {
        const LayerOff& f = L.layers[j];
        const SmallOff& g = L.small[j];
        const size_t srcs[8] = {f.ln1_g, f.ln1_b, f.b_qkv, f.b_o, f.ln2_g, f.ln2_b, f.b_1, f.b_2};
        const size_t dsts[8] = {g.ln1_g, g.ln1_b, g.b_qkv, g.b_o, g.ln2_g, g.ln2_b, g.b_1, g.b_2};
        const size_t cnts[8] = {H, H, 3 * H, H, H, H, 4 * H, H};
        for (int i = 0; i < 8 && st == TP_OK; ++i) st = put(S.psmall + dsts[i], h + srcs[i], cnts[i]);
        if (st == TP_OK) st = mat(h + f.w_qkv, (int)H, 3 * (int)H, S.wqkv_t[j], S.wqkv_io[j]);
        if (st == TP_OK) st = mat(h + f.w_o, (int)H, (int)H, S.wo_t[j], S.wo_io[j]);
        if (st == TP_OK) st = mat(h + f.w_1, (int)H, 4 * (int)H, S.w1_t[j], S.w1_io[j]);
        if (st == TP_OK) st = mat(h + f.w_2, 4 * (int)H, (int)H, S.w2_t[j], S.w2_io[j]);
      }
      if (st == TP_OK && S.k == m.K - 1) {
        st = put(S.psmall + L.s_lnf_g, h + L.lnf_g, H);
        if (st == TP_OK) st = put(S.psmall + L.s_lnf_b, h + L.lnf_b, H);
        if (st == TP_OK) st = mat(h + L.w_out, (int)H, m.V, S.wout_t, S.wout_io);
      }
      if (st != TP_OK) break;
      off += L.total;
    }
    cudaStreamSynchronize(stream);
    cudaFree(stage_buf);
    return st;
  }

  // ------------------------------------------------------------ launch helpers
  tp_status gemm(int cls, const GemmDesc& g0, const Epi& e, cudaStream_t st = nullptr) {
    if (!st) st = stream;
    GemmDesc g = g0;
    if (st == stream) { g.sk_ws = sk_ws; g.sk_cnt = sk_cnt; }  // one persistent GEMM at a time on `stream`
    Pending p;
    instr.begin(st, cls, 2.0 * g.M * g.N * g.K, 0, p);
    cudaError_t err;
    if (!force_simt && std::is_same<T, bf16>::value) {
      // bf16 mode: the tcgen05 kernel or an error, never a silent ~10x slower SIMT fallback
      if (!gemm_sm100_supported(g))
        return fail(TP_ECUDA, "gemm M=%d N=%d K=%d lda=%lld ldb=%lld: not supported by the sm100 kernel (alignment)",
                    g.M, g.N, g.K, (long long)g.lda, (long long)g.ldb);
      err = gemm_sm100(g, e, st);
    } else {
      Epi e0 = e;
      e0.dbias = nullptr;  // the SIMT epilogue has no fused column sums: a separate pass
      err = gemm_simt<T>(g, e0, st);
      if (err == cudaSuccess && e.dbias)
        err = colsum_accum<T>(reinterpret_cast<const T*>(e.out), e.ldo, e.dbias, g.M, g.N, st);
    }
    instr.end(st, p);
    if (err != cudaSuccess) return fail(TP_ECUDA, "gemm M=%d N=%d K=%d: %s", g.M, g.N, g.K, cudaGetErrorString(err));
    return TP_OK;
  }
  template <typename F>
  tp_status launch(int cls, double flops, double bytes, F&& f) {
    Pending p;
    instr.begin(stream, cls, flops, bytes, p);
    cudaError_t err = f();
    instr.end(stream, p);
    if (err != cudaSuccess) return fail(TP_ECUDA, "launch (%s): %s", kKClassNames[cls], cudaGetErrorString(err));
    return TP_OK;
  }
  static GemmDesc gd(int M, int N, int K, const void* A, int64_t lda, bool amn, const void* B, int64_t ldb, bool bmn) {
    GemmDesc g;
    g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.a_mn = amn; g.B = B; g.ldb = ldb; g.b_mn = bmn;
    return g;
  }

  // ------------------------------------------------------------ forward of one job on one stage
  // Internal row order of every [B][s] activation buffer for a step with batch slice b:
  // A group of b sequences starting at sequence seq0 owns rows [seq0*s, (seq0+b)*s), member j at
  // position p in row seq0*s + p*b + j, so the job (group, slice [c, c+l)) is the contiguous row
  // range [seq0*s + c*b, seq0*s + (c+l)*b) of T = b*l tokens (PAPER.md:362-364 joint batch x token
  // slicing; b = 1 is the plain token slicing of §3.2; groups may differ in b).
  // out_next (device p2p): the stage output rows of this job go straight into the next stage's input
  // buffer (peer memory) from the last layer's FC2 epilogue instead of S.hs[nl]
  // tseq0: the job's first sequence in the batch (tokens, loss rows, kept logits); seq0: its first
  // sequence in this stage's buffers (= tseq0 store-all; the group's slot under 1F1B)
  // in_seq0: its first sequence in the stage INPUT buffer hs[0], which the previous stage fills
  // (1F1B: a slot of the sender's in-flight window, one more than this stage's own)
  tp_status fwd(Stage<T>& S, size_t tseq0, size_t seq0, size_t in_seq0, int c, int l, int b, int batch,
                float* out_next = nullptr) {
    const int H = m.H, s = m.s, a = m.a, dh = m.d, V = m.V;
    const int Tn = b * l;
    const size_t row = seq0 * s + (size_t)c * b;  // first buffer row of this job
    const size_t row_in = in_seq0 * s + (size_t)c * b;  // its first row in hs[0]
    const size_t trow = tseq0 * s + (size_t)c * b;  // first batch row of this job
    const size_t cap = (size_t)max_batch * s;      // rows of the stage buffers (LN stats: mean | rstd)
    const int32_t* tok0 = d_tokens + tseq0 * (s + 1);
    const double ebytes = sizeof(T);
    if (S.k == 0) {
      TRY(launch(KC_EMBED, 0, 8.0 * Tn * H, [&] {
        return embed_fwd(tok0, S.psmall + S.L.s_wte, S.psmall + S.L.s_wpe, S.hs[0] + row_in * H, c, l, b, s, H, V, stream);
      }));
    }
    for (int j = 0; j < S.nl; ++j) {
      const SmallOff& f = S.L.small[j];
      const float* P = S.psmall;
      float* x = S.hs[j] + (j == 0 ? row_in : row) * H;
      float* st1 = S.st1[j];
      TRY(launch(KC_LN, 0, (4.0 + ebytes) * Tn * H, [&] {
        return layernorm_fwd<T>(x, P + f.ln1_g, P + f.ln1_b, S.A1[j] + row * H, st1 + row, st1 + cap + row, Tn, H, stream);
      }));
      Epi eq; eq.kind = EPI_QKV; eq.bias = P + f.b_qkv;
      eq.q = S.Q[j] + seq0 * s * H; eq.k = S.Kc[j] + seq0 * s * H; eq.v = S.Vc[j] + seq0 * s * H;
      eq.s_len = s; eq.head_dim = dh; eq.hidden = H; eq.row0 = c; eq.bs = b;
      TRY(gemm(KC_GEMM_FWD, gd(Tn, 3 * H, H, S.A1[j] + row * H, H, false, S.wqkv_t[j], H, false), eq));
      T* o = S.O[j] + row * H;
      const double attn_flops = 4.0 * H * b * ((double)l * c + 0.5 * l * (l + 1.0));
      TRY(launch(KC_ATTN_FWD, attn_flops, ebytes * b * (2.0 * H * (c + l) + 2.0 * H * l), [&] {
        if constexpr (std::is_same<T, bf16>::value)
          if (!force_simt && attn_sm100_supported(dh) && !legacy_attn)  // all b sequences in one launch
            return attn_fwd_sm100(S.Q[j] + seq0 * s * H, S.Kc[j] + seq0 * s * H, S.Vc[j] + seq0 * s * H, o, (int64_t)b * H,
                                  S.LSE[j] + seq0 * a * s, a, s, dh, c, l, stream, b, (int64_t)s * H, H, (int64_t)a * s);
        for (int jj = 0; jj < b; ++jj) {
          const size_t sq = seq0 + jj;
          const T *q = S.Q[j] + sq * s * H, *kk = S.Kc[j] + sq * s * H, *vv = S.Vc[j] + sq * s * H;
          T* oj = o + (size_t)jj * H;
          float* lse = S.LSE[j] + sq * a * s;
          cudaError_t e;
          if constexpr (std::is_same<T, bf16>::value) {
            if (!force_simt && attn_sm100_supported(dh) && !legacy_attn)
              e = attn_fwd_sm100(q, kk, vv, oj, (int64_t)b * H, lse, a, s, dh, c, l, stream);
            else if (!force_simt)
              e = attn_fwd_tc(q, kk, vv, oj, (int64_t)b * H, lse, a, s, dh, c, l, stream);
            else
              e = attn_fwd_simt<T>(q, kk, vv, oj, (int64_t)b * H, lse, a, s, dh, c, l, stream);
          } else {
            e = attn_fwd_simt<T>(q, kk, vv, oj, (int64_t)b * H, lse, a, s, dh, c, l, stream);
          }
          if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
      }));
      Epi er; er.kind = EPI_RESID; er.bias = P + f.b_o; er.out = S.hmid[j] + row * H; er.ldo = H; er.resid = x; er.ldr = H;
      TRY(gemm(KC_GEMM_FWD, gd(Tn, H, H, o, H, false, S.wo_t[j], H, false), er));
      float* st2 = S.st2[j];
      TRY(launch(KC_LN, 0, (4.0 + ebytes) * Tn * H, [&] {
        return layernorm_fwd<T>(S.hmid[j] + row * H, P + f.ln2_g, P + f.ln2_b, S.A2[j] + row * H, st2 + row, st2 + cap + row, Tn, H, stream);
      }));
      Epi eg; eg.kind = EPI_GELU; eg.bias = P + f.b_1; eg.out = S.U[j] + row * 4 * H; eg.ldo = 4 * H; eg.out2 = S.G[j] + row * 4 * H; eg.ldo2 = 4 * H;
      TRY(gemm(KC_GEMM_FWD, gd(Tn, 4 * H, H, S.A2[j] + row * H, H, false, S.w1_t[j], H, false), eg));
      Epi e2; e2.kind = EPI_RESID; e2.bias = P + f.b_2; e2.ldo = H; e2.resid = S.hmid[j] + row * H; e2.ldr = H;
      e2.out = (out_next && j == S.nl - 1) ? out_next : S.hs[j + 1] + row * H;
      TRY(gemm(KC_GEMM_FWD, gd(Tn, H, 4 * H, S.G[j] + row * 4 * H, 4 * H, false, S.w2_t[j], 4 * H, false), e2));
    }
    if (S.k == m.K - 1) {
      const float* P = S.psmall;
      float* x = S.hs[S.nl] + row * H;
      TRY(launch(KC_LN, 0, (4.0 + ebytes) * Tn * H, [&] {
        return layernorm_fwd<T>(x, P + S.L.s_lnf_g, P + S.L.s_lnf_b, S.Af + row * H, S.stf + row, S.stf + cap + row, Tn, H, stream);
      }));
      Epi ez; ez.kind = EPI_STORE; ez.out = S.Z + row * V; ez.ldo = V;
      TRY(gemm(KC_GEMM_FWD, gd(Tn, V, H, S.Af + row * H, H, false, S.wout_t, H, false), ez));
      const float scale = 1.0f / (float)((double)batch * s);
      float* keep = S.logits_keep ? S.logits_keep + trow * V : nullptr;
      TRY(launch(KC_CE, 0, 2.0 * ebytes * Tn * V, [&] {
        return ce_fwd_bwd<T>(S.Z + row * V, tok0, c, b, s, S.loss_rows + trow, keep, Tn, V, scale, stream);
      }));
    }
    return TP_OK;
  }

  // ------------------------------------------------------------ backward of one job on one stage
  // gin_prev (device p2p): the input-gradient rows of this job go straight into the previous stage's
  // grad_out buffer (peer memory) from the first layer's LayerNorm backward instead of S.grad_in
  tp_status bwd(Stage<T>& S, size_t tseq0, size_t seq0, size_t in_seq0, int c, int l, int b, int batch,
                bool first_bwd_slice, float* gin_prev = nullptr) {
    const int H = m.H, s = m.s, a = m.a, dh = m.d, V = m.V;
    const int Tn = b * l;
    const size_t row = seq0 * s + (size_t)c * b;
    const size_t row_in = in_seq0 * s + (size_t)c * b;
    const size_t cap = (size_t)max_batch * s;
    const int32_t* tok0 = d_tokens + tseq0 * (s + 1);
    const double ebytes = sizeof(T);
    float* gr = S.grad_out + row * H;  // fp32 gradient at the stage output, rows of this job
    if (S.k == m.K - 1) {
      const float* P = S.psmall;
      Epi e; e.kind = EPI_STORE; e.out = S.dA; e.ldo = H; e.out_f32 = std::is_same<T, float>::value;
      TRY(gemm(KC_GEMM_DX, gd(Tn, H, V, S.Z + row * V, V, false, S.wout_io, V, false), e));
      TRY(launch(KC_LN, 0, (12.0 + ebytes) * Tn * H, [&] {
        return layernorm_bwd<T>(reinterpret_cast<const T*>(S.dA), S.hs[S.nl] + row * H, S.stf + row, S.stf + cap + row, P + S.L.s_lnf_g, nullptr, gr,
                                S.dhout_b[S.nl - 1] + row * H, S.gflat + S.L.lnf_g, S.gflat + S.L.lnf_b, S.lnws, Tn, H, stream,
                                S.gflat + S.L.layers[S.nl - 1].b_2);
      }));
    } else {
      TRY(launch(KC_MISC, 0, (4.0 + ebytes) * Tn * H, [&] {
        return convert_f32<T>(gr, S.dhout_b[S.nl - 1] + row * H, (int64_t)Tn * H, stream);
      }));
    }
    for (int j = S.nl - 1; j >= 0; --j) {
      const LayerOff& f = S.L.layers[j];
      const SmallOff& fs = S.L.small[j];
      const float* P = S.psmall;
      float* GR = S.gflat;
      // FFN: dU = (dh W_2^T) * gelu'(U)
      Epi e1; e1.kind = EPI_DGELU; e1.out = S.dU[j] + row * 4 * H; e1.ldo = 4 * H; e1.aux = S.U[j] + row * 4 * H; e1.ld_aux = 4 * H;
      e1.dbias = GR + f.b_1;  // FC1's bias gradient = column sums of dU, fused into this GEMM's epilogue
      TRY(gemm(KC_GEMM_DX, gd(Tn, 4 * H, H, S.dhout_b[j] + row * H, H, false, S.w2_io[j], H, false), e1));
      Epi e2; e2.kind = EPI_STORE; e2.out = S.dA; e2.ldo = H; e2.out_f32 = std::is_same<T, float>::value;
      TRY(gemm(KC_GEMM_DX, gd(Tn, H, 4 * H, S.dU[j] + row * 4 * H, 4 * H, false, S.w1_io[j], 4 * H, false), e2));
      float* st2 = S.st2[j];
      TRY(launch(KC_LN, 0, (16.0 + ebytes) * Tn * H, [&] {
        return layernorm_bwd<T>(reinterpret_cast<const T*>(S.dA), S.hmid[j] + row * H, st2 + row, st2 + cap + row, P + fs.ln2_g, gr, S.gm,
                                S.dhmid_b[j] + row * H, GR + f.ln2_g, GR + f.ln2_b, S.lnws, Tn, H, stream, GR + f.b_o);
      }));
      // attention: dO = dh_mid W_o^T, then slice-vs-prefix attention backward with dK/dV push
      Epi e3; e3.kind = EPI_STORE; e3.out = S.dO; e3.ldo = H;
      TRY(gemm(KC_GEMM_DX, gd(Tn, H, H, S.dhmid_b[j] + row * H, H, false, S.wo_io[j], H, false), e3));
      const double attn_flops = 8.0 * H * b * ((double)l * c + 0.5 * l * (l + 1.0));
      T* dq = S.dQKV[j] + row * 3 * H;
      const int accum = first_bwd_slice ? 0 : 1;
      TRY(launch(KC_ATTN_BWD, attn_flops, b * (ebytes * 4.0 * H * (c + l) + 16.0 * H * (c + l)), [&] {
        if constexpr (std::is_same<T, bf16>::value)
          if (!force_simt && attn_sm100_supported(dh) && !legacy_attn) {  // all b sequences in one launch
            // the kernel also writes the slice rows' final dK / dV into dQKV (no finalise pass)
            return attn_bwd_sm100(S.dO, (int64_t)b * H, S.O[j] + row * H, (int64_t)b * H, S.Q[j] + seq0 * s * H,
                                  S.Kc[j] + seq0 * s * H, S.Vc[j] + seq0 * s * H, S.LSE[j] + seq0 * a * s, S.Dvec,
                                  S.dqacc, dq, (int64_t)b * 3 * H, S.dk_acc[j], S.dv_acc[j], a, s, dh, c, l, accum,
                                  stream, b, (int64_t)s * H, H, (int64_t)a * s, 3 * H, (int64_t)s * H, 1);
          }
        for (int jj = 0; jj < b; ++jj) {
          const size_t sq = seq0 + jj;
          const T *q = S.Q[j] + sq * s * H, *kk = S.Kc[j] + sq * s * H, *vv = S.Vc[j] + sq * s * H;
          const T* dOj = S.dO + (size_t)jj * H;
          const T* Oj = S.O[j] + (row + jj) * H;
          const float* lse = S.LSE[j] + sq * a * s;
          T* dqj = dq + (size_t)jj * 3 * H;
          float* dka = S.dk_acc[j] + (size_t)jj * s * H;
          float* dva = S.dv_acc[j] + (size_t)jj * s * H;
          const int64_t ldb = (int64_t)b * H, ldq = (int64_t)b * 3 * H;
          cudaError_t e;
          if constexpr (std::is_same<T, bf16>::value) {
            if (!force_simt && attn_sm100_supported(dh) && !legacy_attn)
              e = attn_bwd_sm100(dOj, ldb, Oj, ldb, q, kk, vv, lse, S.Dvec, S.dqacc, dqj, ldq, dka, dva, a, s, dh, c, l, accum, stream);
            else if (!force_simt)
              e = attn_bwd_tc(dOj, ldb, Oj, ldb, q, kk, vv, lse, S.Dvec, dqj, ldq, dka, dva, a, s, dh, c, l, accum, stream);
            else
              e = attn_bwd_simt<T>(dOj, ldb, Oj, ldb, q, kk, vv, lse, S.Dvec, dqj, ldq, dka, dva, a, s, dh, c, l, accum, stream);
          } else {
            e = attn_bwd_simt<T>(dOj, ldb, Oj, ldb, q, kk, vv, lse, S.Dvec, dqj, ldq, dka, dva, a, s, dh, c, l, accum, stream);
          }
          if (e == cudaSuccess) e = attn_dkv_finalize<T>(dka, dva, dqj, ldq, a, s, dh, c, l, stream);
          if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
      }));
      Epi e4; e4.kind = EPI_STORE; e4.out = S.dA; e4.ldo = H; e4.out_f32 = std::is_same<T, float>::value;
      TRY(gemm(KC_GEMM_DX, gd(Tn, H, 3 * H, dq, 3 * H, false, S.wqkv_io[j], 3 * H, false), e4));
      float* gnext = j == 0 ? (gin_prev ? gin_prev : S.grad_in + row * H) : (gr == S.gA ? S.gB : S.gA);
      T* copy = j == 0 ? nullptr : S.dhout_b[j - 1] + row * H;
      float* st1 = S.st1[j];
      TRY(launch(KC_LN, 0, (16.0 + ebytes) * Tn * H, [&] {
        return layernorm_bwd<T>(reinterpret_cast<const T*>(S.dA), S.hs[j] + (j == 0 ? row_in : row) * H, st1 + row, st1 + cap + row, P + fs.ln1_g, S.gm, gnext, copy,
                                GR + f.ln1_g, GR + f.ln1_b, S.lnws, Tn, H, stream,
                                j == 0 ? nullptr : GR + S.L.layers[j - 1].b_2);
      }));
      gr = gnext;
    }
    if (S.k == 0) {
      TRY(launch(KC_EMBED, 0, 12.0 * Tn * H, [&] {
        return embed_bwd(tok0, S.grad_in + row * H, S.gflat + S.L.wte, S.gflat + S.L.wpe, c, l, b, s, H, V, stream);
      }));
    }
    return TP_OK;
  }

  // ------------------------------------------------------------ deferred weight gradients
  // One GEMM per weight over all B*s tokens of the step (K = B*s, both operands MN-major), written
  // once (the gradients start at zero), plus the bias column sums: off the per-job critical path and
  // with no fp32 read-modify-write.
  // the instrumented (per-launch CUDA-event) runs keep the dW GEMMs on one stream: overlapping launches
  // would charge each other's time to their event intervals
  tp_status wgrad(Stage<T>& S, int batch) {
    return wgrad_rows(S, 0, batch * m.s, false, stream, true, instr.on ? nullptr : s_dw2);
  }

  // Weight gradients over rows [row0, row0 + K) of the step (K = tokens), written (accum = false) or
  // added; `persistent` = false launches one tile per CTA so a higher-priority stream interleaves.
  tp_status wgrad_rows(Stage<T>& S, size_t row0, int K, bool accum, cudaStream_t st, bool persistent,
                       cudaStream_t st2 = nullptr) {
    const int H = m.H, V = m.V;
    float* GR = S.gflat;
    // dW GEMMs alternate between st and st2 (fork here, join at the end): each writes its own weight's
    // gradient, so they are independent
    int gi = 0;
    if (st2) {
      cudaEvent_t e = event();
      CU(cudaEventRecord(e, st));
      CU(cudaStreamWaitEvent(st2, e, 0));
    }
    auto gemm = [&](int cls, const GemmDesc& g, const Epi& e, cudaStream_t) {
      return this->gemm(cls, g, e, (st2 && (gi++ & 1)) ? st2 : st);
    };
    auto G = [&](int M_, int N_, const void* A_, int64_t lda, const void* B_, int64_t ldb) {
      GemmDesc g = gd(M_, N_, K, A_, lda, true, B_, ldb, true);
      g.persistent = persistent;
      return g;
    };
    for (int j = 0; j < S.nl; ++j) {
      const LayerOff& f = S.L.layers[j];
      Epi e; e.kind = accum ? EPI_ACCUM : EPI_STORE; e.out_f32 = 1;
      e.out = GR + f.w_qkv; e.ldo = 3 * H;
      TRY(gemm(KC_GEMM_DW, G(H, 3 * H, S.A1[j] + row0 * H, H, S.dQKV[j] + row0 * 3 * H, 3 * H), e, st));
      e.out = GR + f.w_o; e.ldo = H;
      TRY(gemm(KC_GEMM_DW, G(H, H, S.O[j] + row0 * H, H, S.dhmid_b[j] + row0 * H, H), e, st));
      e.out = GR + f.w_1; e.ldo = 4 * H;
      TRY(gemm(KC_GEMM_DW, G(H, 4 * H, S.A2[j] + row0 * H, H, S.dU[j] + row0 * 4 * H, 4 * H), e, st));
      e.out = GR + f.w_2; e.ldo = H;
      TRY(gemm(KC_GEMM_DW, G(4 * H, H, S.G[j] + row0 * 4 * H, 4 * H, S.dhout_b[j] + row0 * H, H), e, st));
      Pending p;
      instr.begin(st, KC_MISC, 0, sizeof(T) * 3.0 * K * H, p);
      // b_o and b_2 are summed by the LayerNorm backward that produces their dY, b_1 by the GeLU'
      // epilogue of the FC2 dX GEMM (fused column sums), except b_2 of a non-last stage's last layer,
      // whose dY arrives from the next stage
      cudaError_t r = colsum_accum<T>(S.dQKV[j] + row0 * 3 * H, 3 * H, GR + f.b_qkv, K, 3 * H, st);
      if (r == cudaSuccess && j == S.nl - 1 && S.k != m.K - 1)
        r = colsum_accum<T>(S.dhout_b[j] + row0 * H, H, GR + f.b_2, K, H, st);
      instr.end(st, p);
      if (r != cudaSuccess) return fail(TP_ECUDA, "bias grads: %s", cudaGetErrorString(r));
    }
    if (S.k == m.K - 1) {
      Epi e; e.kind = accum ? EPI_ACCUM : EPI_STORE; e.out_f32 = 1; e.out = GR + S.L.w_out; e.ldo = V;
      TRY(gemm(KC_GEMM_DW, G(H, V, S.Af + row0 * H, H, S.Z + row0 * V, V), e, st));
    }
    if (st2) {
      cudaEvent_t e = event();
      CU(cudaEventRecord(e, st2));
      CU(cudaStreamWaitEvent(st, e, 0));
    }
    return TP_OK;
  }

  // ------------------------------------------------------------ p2p (multi-rank)
  tp_status recv_fwd(Stage<T>& S, size_t row, int l) {  // activation from stage k-1
    cudaEvent_t e = event();
    Pending p;
    instr.begin(s_recv_f, KC_COMM, 0, 4.0 * l * m.H, p);
    NC(ncclRecv(S.hs[0] + row * m.H, (size_t)l * m.H, ncclFloat32, S.k - 1, commF[(S.k - 1) & 1], s_recv_f));
    instr.end(s_recv_f, p);
    CU(cudaEventRecord(e, s_recv_f));
    CU(cudaStreamWaitEvent(stream, e, 0));
    return TP_OK;
  }
  tp_status send_fwd(Stage<T>& S, size_t row, int l) {
    cudaEvent_t e = event();
    CU(cudaEventRecord(e, stream));
    CU(cudaStreamWaitEvent(s_send_f, e, 0));
    NC(ncclSend(S.hs[S.nl] + row * m.H, (size_t)l * m.H, ncclFloat32, S.k + 1, commF[S.k & 1], s_send_f));
    return TP_OK;
  }
  tp_status recv_bwd(Stage<T>& S, size_t row, int l) {  // gradient from stage k+1
    cudaEvent_t e = event();
    NC(ncclRecv(S.grad_out + row * m.H, (size_t)l * m.H, ncclFloat32, S.k + 1, commB[S.k & 1], s_recv_b));
    CU(cudaEventRecord(e, s_recv_b));
    CU(cudaStreamWaitEvent(stream, e, 0));
    return TP_OK;
  }
  tp_status send_bwd(Stage<T>& S, size_t row, int l) {
    cudaEvent_t e = event();
    CU(cudaEventRecord(e, stream));
    CU(cudaStreamWaitEvent(s_send_b, e, 0));
    NC(ncclSend(S.grad_in + row * m.H, (size_t)l * m.H, ncclFloat32, S.k - 1, commB[(S.k - 1) & 1], s_send_b));
    return TP_OK;
  }

  // NCCL loopback (world == 1): the message of one job from stage S to its neighbour T (both owned
  // by this context) as a grouped ncclSend + ncclRecv to self on the direction's comm stream, gated
  // by events exactly like the multi-rank path (sender's compute -> comm stream -> receiver's compute)
  tp_status p2p_self(const float* src, float* dst, size_t count, bool fwd, int edge) {
    cudaStream_t cs = fwd ? s_send_f : s_send_b;
    ncclComm_t comm = fwd ? commF[edge & 1] : commB[edge & 1];
    cudaEvent_t e0 = event(), e1 = event();
    CU(cudaEventRecord(e0, stream));
    CU(cudaStreamWaitEvent(cs, e0, 0));
    Pending p;
    instr.begin(cs, KC_COMM, 0, 4.0 * count, p);
    NC(ncclGroupStart());
    NC(ncclSend(src, count, ncclFloat32, 0, comm, cs));
    NC(ncclRecv(dst, count, ncclFloat32, 0, comm, cs));
    NC(ncclGroupEnd());
    instr.end(cs, p);
    CU(cudaEventRecord(e1, cs));
    CU(cudaStreamWaitEvent(stream, e1, 0));
    return TP_OK;
  }

  // ------------------------------------------------------------ one step
  // Everything one step puts on the device after the tokens are in d_tokens: zero the gradients, the
  // forward and backward op lists of every owned stage, the deferred weight gradients, the loss.
  struct Group {
    size_t seq0;                // first sequence of the group in the batch (tokens, loss, logits)
    int b;
    std::vector<int> off, len;  // slice offsets (M + 1) and lengths (M), tokens
  };
  // Per-stage op lists (A-21): GPipe — every F(d, i) in order, then every B in exact
  // reverse; 1F1B at group granularity (TP_FLAG_SCHEDULE_1F1B) — stage k runs
  // the forwards of its first w_k = min(D, K - k) groups, then alternates the backward of its oldest
  // group (slices in reverse) with the forward of the next one, then drains; oracle/plan.py
  // one_f_one_b_oplists is the same list (tests compare the replayed makespans).
  int inflight(int k, int D) const { return sched_1f1b ? std::min(D, m.K - k) : D; }
  std::vector<Op> oplist(int k, const std::vector<Group>& G) const {
    std::vector<int> M;
    for (const Group& g : G) M.push_back((int)g.len.size());
    return build_oplist(m.K, k, sched_1f1b, M);
  }
  // buffer sequence index of group d on stage k: the group's own sequences (store-all, GPipe) or its
  // slot (d mod w_k) x the largest group size (1F1B: only w_k groups are ever live on stage k)
  size_t bseq0(int k, const std::vector<Group>& G, int d) const {
    if (!sched_1f1b) return G[d].seq0;
    int bmax = 0;
    for (const Group& g : G) bmax = std::max(bmax, g.b);
    return (size_t)(d % inflight(k, (int)G.size())) * bmax;
  }

  // hs[0] of stage k > 0 is written by stage k-1 when IT runs F(d); under 1F1B that can happen before
  // this stage has finished with group d - w_k, so the input buffer cycles through w_{k-1} = w_k + 1
  // slots (stage k-1's window; F(d) on k-1 follows B(d - w_{k-1}) on k-1, hence on k)
  size_t in_bseq0(int k, const std::vector<Group>& G, int d) const {
    if (!sched_1f1b) return G[d].seq0;
    int bmax = 0;
    for (const Group& g : G) bmax = std::max(bmax, g.b);
    return (size_t)(d % inflight(k > 0 ? k - 1 : 0, (int)G.size())) * bmax;
  }

  tp_status enqueue_step(const std::vector<Group>& G, int batch) {
    const int D = (int)G.size();
    const bool multi = world > 1;
    if (multi || nccl_lb) {  // fork: the comm streams join this step's stream order (and any graph capture)
      cudaEvent_t e = event();
      CU(cudaEventRecord(e, stream));
      for (cudaStream_t cs : {s_send_f, s_recv_f, s_send_b, s_recv_b}) CU(cudaStreamWaitEvent(cs, e, 0));
    }
    for (auto& S : stages) CU(cudaMemsetAsync(S.gflat, 0, S.L.total * sizeof(float), stream));
    std::vector<size_t> job0(D + 1, 0);  // global job index of (group d, slice 0): the p2p flag slot
    for (int d = 0; d < D; ++d) job0[d + 1] = job0[d] + G[d].len.size();
    if (dev_p2p) {
      if (job0[D] > n_slots) return fail(TP_EINVAL, "tp_step: %zu jobs exceed the %zu p2p slots", job0[D], n_slots);
      CU(p2p_epoch_inc(d_epoch, stream));
    }
    unsigned long long* flag_local = reinterpret_cast<unsigned long long*>(p_flag);
    // TP_SIDE_DW=1 (GPipe, one stage per GPU, D >= 2): group d's weight gradients go to a low-priority
    // stream as soon as its last backward job is done. 1F1B: group d's weight gradients run in order
    // right after its backward on each stage (its stash slot is reused by a later group).
    const bool side_dw = multi && D >= 2 && s_wgrad && !sched_1f1b;
    std::vector<int> seen_dw(stages.size(), 0);

    auto run_op = [&](size_t si, const Op& op) -> tp_status {
      Stage<T>& S = stages[si];
      const int d = op.d, i = op.i, b = G[d].b;
      const size_t bs0 = bseq0(S.k, G, d), is0 = in_bseq0(S.k, G, d);
      const size_t row = bs0 * m.s + (size_t)G[d].off[i] * b;  // this stage's rows of the job
      const size_t row_in = is0 * m.s + (size_t)G[d].off[i] * b;  // ... in its input buffer hs[0]
      const int Tn = b * G[d].len[i];
      const size_t jb = job0[d] + i;
      if (op.fwd) {
        float* out_next = nullptr;
        if (dev_p2p && S.k < m.K - 1) out_next = peer_in + (in_bseq0(S.k + 1, G, d) * m.s + (size_t)G[d].off[i] * b) * m.H;
        if (dev_p2p && S.k > 0) CU(p2p_wait(flag_local + jb, d_epoch, stream));
        else if (multi && S.k > 0) TRY(recv_fwd(S, row_in, Tn));
        TRY(fwd(S, G[d].seq0, bs0, is0, G[d].off[i], G[d].len[i], b, batch, out_next));
        if (dev_p2p && S.k < m.K - 1) CU(p2p_signal(peer_flag_next + jb, d_epoch, stream));
        else if (multi && S.k < m.K - 1) TRY(send_fwd(S, row, Tn));
        if (world == 1 && si + 1 < stages.size() && !stages[si + 1].aliased) {
          // loopback without aliasing: the message to the next owned stage's input rows
          Stage<T>& R = stages[si + 1];
          float* dst = R.hs[0] + (in_bseq0(R.k, G, d) * m.s + (size_t)G[d].off[i] * b) * m.H;
          if (nccl_lb) TRY(p2p_self(S.hs[S.nl] + row * m.H, dst, (size_t)Tn * m.H, true, S.k));
          else CU(cudaMemcpyAsync(dst, S.hs[S.nl] + row * m.H, sizeof(float) * Tn * m.H, cudaMemcpyDeviceToDevice, stream));
        }
        return TP_OK;
      }
      const bool first_b = i == (int)G[d].len.size() - 1;  // the slice ending at s: first in backward
      float* gin_prev = nullptr;
      if (dev_p2p && S.k > 0) gin_prev = peer_gout + (bseq0(S.k - 1, G, d) * m.s + (size_t)G[d].off[i] * b) * m.H;
      if (dev_p2p && S.k < m.K - 1) CU(p2p_wait(flag_local + n_slots + jb, d_epoch, stream));
      else if (multi && S.k < m.K - 1) TRY(recv_bwd(S, row, Tn));
      TRY(bwd(S, G[d].seq0, bs0, is0, G[d].off[i], G[d].len[i], b, batch, first_b, gin_prev));
      if (dev_p2p && S.k > 0) CU(p2p_signal(peer_flag_prev + n_slots + jb, d_epoch, stream));
      else if (multi && S.k > 0) TRY(send_bwd(S, row, Tn));
      if (world == 1 && si > 0 && !S.aliased) {
        Stage<T>& R = stages[si - 1];
        float* dst = R.grad_out + (bseq0(R.k, G, d) * m.s + (size_t)G[d].off[i] * b) * m.H;
        if (nccl_lb) TRY(p2p_self(S.grad_in + row * m.H, dst, (size_t)Tn * m.H, false, S.k - 1));
        else CU(cudaMemcpyAsync(dst, S.grad_in + row * m.H, sizeof(float) * Tn * m.H, cudaMemcpyDeviceToDevice, stream));
      }
      if (i == 0 && sched_1f1b) {  // group d's backward done on this stage: its weight gradients, in order
        TRY(wgrad_rows(S, bs0 * m.s, b * m.s, seen_dw[si] > 0, stream, true));
        ++seen_dw[si];
      }
      if (i == 0 && side_dw) {
        cudaEvent_t e = event();
        CU(cudaEventRecord(e, stream));
        CU(cudaStreamWaitEvent(s_wgrad, e, 0));
        TRY(wgrad_rows(S, bs0 * m.s, b * m.s, d != D - 1, s_wgrad, false));
      }
      return TP_OK;
    };

    std::vector<std::vector<Op>> lists;
    for (auto& S : stages) lists.push_back(oplist(S.k, G));
    if (stages.size() == 1) {
      for (const Op& op : lists[0]) TRY(run_op(0, op));
    } else {
      // all stages on one stream (loopback): a topological merge of the per-stage lists — an op runs
      // once its producer (F on the stage before, B on the stage after, or F on the last stage) ran
      const size_t NS = stages.size();
      std::vector<size_t> pos(NS, 0);
      std::vector<std::vector<char>> fdone(NS, std::vector<char>(job0[D], 0)), bdone = fdone;
      size_t left = 0;
      for (auto& l : lists) left += l.size();
      while (left) {
        bool progressed = false;
        for (size_t si = 0; si < NS; ++si) {
          while (pos[si] < lists[si].size()) {
            const Op& op = lists[si][pos[si]];
            const size_t jb = job0[op.d] + op.i;
            const bool ready = op.fwd ? (si == 0 || fdone[si - 1][jb]) : (si + 1 == NS ? fdone[si][jb] : bdone[si + 1][jb]);
            if (!ready) break;
            TRY(run_op(si, op));
            (op.fwd ? fdone : bdone)[si][jb] = 1;
            ++pos[si];
            --left;
            progressed = true;
          }
        }
        if (!progressed) return fail(TP_EINVAL, "tp_step: schedule deadlock (internal)");
      }
    }
    if (side_dw) {
      cudaEvent_t e = event();
      CU(cudaEventRecord(e, s_wgrad));
      CU(cudaStreamWaitEvent(stream, e, 0));
    } else if (!sched_1f1b) {
      for (auto& S : stages) TRY(wgrad(S, batch));
    }
    // loss: sum of per-token NLL on the last stage, mean over batch*seq_len (A-9)
    Stage<T>* last = nullptr;
    for (auto& S : stages) if (S.k == m.K - 1) last = &S;
    if (last) {
      TRY(launch(KC_MISC, 0, 4.0 * batch * m.s, [&] { return sum_rows(last->loss_rows, batch * m.s, d_loss, stream); }));
    } else {
      CU(cudaMemsetAsync(d_loss, 0, sizeof(float), stream));
    }
    if (multi || nccl_lb) {
      // the comm streams must have drained before the step ends
      for (cudaStream_t cs : {s_send_f, s_recv_f, s_send_b, s_recv_b}) {
        cudaEvent_t e = event();
        CU(cudaEventRecord(e, cs));
        CU(cudaStreamWaitEvent(stream, e, 0));
      }
      if (multi) NC(ncclAllReduce(d_loss, d_loss, 1, ncclFloat32, ncclSum, base, stream));
    }
    CU(cudaMemcpyAsync(h_loss, d_loss, sizeof(float), cudaMemcpyDeviceToHost, stream));
    return TP_OK;
  }

  tp_status step(const tp_slicing* sl, const int32_t* tokens, bool host_tokens, int batch, float* loss_out) override {
    if (!sl || !sl->lengths) return fail(TP_EINVAL, "tp_step: null slicing");
    if (batch < 1) return fail(TP_EINVAL, "tp_step: batch %d < 1", batch);
    const int b = sl->batch_slice;
    if (b < 1 || batch % b != 0)
      return fail(TP_EINVAL, "tp_step: batch_slice %d must be >= 1 and divide batch %d", b, batch);
    const int M = sl->n_slices;
    if (M < 1 || M > m.s) return fail(TP_EINVAL, "tp_step: n_slices %d", M);
    Group g0;
    g0.b = b;
    g0.off.assign(M + 1, 0);
    for (int i = 0; i < M; ++i) {
      if (sl->lengths[i] <= 0) return fail(TP_EINVAL, "tp_step: slice %d has length %d", i, sl->lengths[i]);
      g0.off[i + 1] = g0.off[i] + sl->lengths[i];
      g0.len.push_back(sl->lengths[i]);
    }
    if (g0.off[M] != m.s) return fail(TP_EINVAL, "tp_step: slice lengths sum to %d, seq_len is %d", g0.off[M], m.s);
    std::vector<Group> G(batch / b, g0);
    for (int d = 0; d < batch / b; ++d) G[d].seq0 = (size_t)d * b;
    return run_step(G, tokens, host_tokens, batch, loss_out);
  }

  tp_status step_plan(const tp_batch_plan* pl, const int32_t* tokens, bool host_tokens, int batch,
                      float* loss_out) override {
    if (!pl || !pl->batch_slice || !pl->n_slices || !pl->lengths) return fail(TP_EINVAL, "tp_step_plan: null plan");
    if (batch < 1) return fail(TP_EINVAL, "tp_step_plan: batch %d < 1", batch);
    if (pl->n_groups < 1 || pl->n_groups > batch) return fail(TP_EINVAL, "tp_step_plan: n_groups %d", pl->n_groups);
    if (pl->n_groups > pl->capacity_groups)
      return fail(TP_EINVAL, "tp_step_plan: n_groups %d exceeds capacity_groups %d", pl->n_groups, pl->capacity_groups);
    std::vector<Group> G(pl->n_groups);
    size_t seq0 = 0, pos = 0;
    for (int d = 0; d < pl->n_groups; ++d) {
      const int b = pl->batch_slice[d], M = pl->n_slices[d];
      if (b < 1) return fail(TP_EINVAL, "tp_step_plan: group %d has batch_slice %d", d, b);
      if (M < 1 || M > m.s) return fail(TP_EINVAL, "tp_step_plan: group %d has n_slices %d", d, M);
      if (pos + M > (size_t)pl->capacity_lengths) return fail(TP_EINVAL, "tp_step_plan: lengths[] overrun at group %d", d);
      G[d].seq0 = seq0;
      G[d].b = b;
      G[d].off.assign(M + 1, 0);
      for (int i = 0; i < M; ++i) {
        const int l = pl->lengths[pos + i];
        if (l <= 0) return fail(TP_EINVAL, "tp_step_plan: group %d slice %d has length %d", d, i, l);
        G[d].off[i + 1] = G[d].off[i] + l;
        G[d].len.push_back(l);
      }
      if (G[d].off[M] != m.s)
        return fail(TP_EINVAL, "tp_step_plan: group %d slice lengths sum to %d, seq_len is %d", d, G[d].off[M], m.s);
      seq0 += b;
      pos += M;
    }
    if ((int)seq0 != batch) return fail(TP_EINVAL, "tp_step_plan: batch slices sum to %zu, batch is %d", seq0, batch);
    return run_step(G, tokens, host_tokens, batch, loss_out);
  }

  tp_status run_step(const std::vector<Group>& G, const int32_t* tokens, bool host_tokens, int batch,
                     float* loss_out) {
    if (!tokens) return fail(TP_EINVAL, "tp_step: null tokens");
    CU(cudaSetDevice(device));
    // capacity: store-all (GPipe) holds the whole batch in the stage buffers (batch <= max_batch);
    // 1F1B holds at most w_k = min(D, K - k) groups per stage, so the batch may exceed max_batch as
    // long as w_k * (largest group) <= max_batch on every owned stage (the memory bound of 1F1B)
    int bmax = 0;
    for (const Group& g : G) bmax = std::max(bmax, g.b);
    if (!sched_1f1b) {
      if (batch > max_batch) return fail(TP_EINVAL, "tp_step: batch %d > max_batch %d", batch, max_batch);
    } else {
      for (auto& S : stages) {
        const int w = std::max(inflight(S.k, (int)G.size()), S.k > 0 ? inflight(S.k - 1, (int)G.size()) : 0);
        if ((size_t)w * bmax > (size_t)max_batch)
          return fail(TP_EINVAL, "tp_step (1F1B): stage %d holds %d groups of up to %d sequences > max_batch %d", S.k, w,
                      bmax, max_batch);
      }
      if ((flags & TP_FLAG_KEEP_LOGITS) && batch > max_batch)
        return fail(TP_EINVAL, "tp_step: TP_FLAG_KEEP_LOGITS keeps at most max_batch = %d sequences", max_batch);
    }
    TRY(ensure_batch_capacity(batch));
    last_batch = batch;
    last_groups.clear();
    for (const Group& g : G) last_groups.push_back({g.seq0, g.b});
    // tokens -> d_tokens, outside any graph (the caller's pointer may change between calls)
    const size_t ntok = (size_t)batch * (m.s + 1);
    // token ids outside [0, V) are rejected (TP_EINVAL), never clamped: host tokens before anything
    // runs, device tokens by a device count read back with the loss
    if (host_tokens) {
      for (size_t i = 0; i < ntok; ++i)
        if (tokens[i] < 0 || tokens[i] >= m.V)
          return fail(TP_EINVAL, "tp_step: token id %d at [%zu][%zu] outside [0, %d)", tokens[i], i / (m.s + 1),
                      i % (m.s + 1), m.V);
      std::memcpy(h_tokens, tokens, ntok * sizeof(int32_t));
      CU(cudaMemcpyAsync(d_tokens, h_tokens, ntok * sizeof(int32_t), cudaMemcpyHostToDevice, stream));
      *h_bad_tok = 0;
    } else {
      CU(cudaMemcpyAsync(d_tokens, tokens, ntok * sizeof(int32_t), cudaMemcpyDeviceToDevice, stream));
      CU(count_bad_tokens(d_tokens, (int64_t)ntok, m.V, d_bad_tok, stream));
      CU(cudaMemcpyAsync(h_bad_tok, d_bad_tok, sizeof(int), cudaMemcpyDeviceToHost, stream));
    }
    // The op list of a plan is static: the first step with a new key runs eagerly, the second is
    // captured into a CUDA graph, later ones replay it (no per-kernel host launch cost).
    std::vector<int64_t> key = {batch, (int64_t)G.size()};
    for (const Group& g : G) {
      key.push_back(g.b);
      key.push_back((int64_t)g.len.size());
      for (int l : g.len) key.push_back(l);
    }
    const bool graphs = use_graphs && !instr.on;
    if (graphs && g_exec && key == g_key) {
      CU(cudaGraphLaunch(g_exec, stream));
      instr.launches = g_launches;
    } else if (graphs && key == g_key) {
      instr.launches = 0;
      ev_next = 0;
      CU(cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed));
      tp_status st = enqueue_step(G, batch);
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(stream, &graph);
      if (st != TP_OK) { if (graph) cudaGraphDestroy(graph); return st; }
      if (ce != cudaSuccess) return fail(TP_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
      // launch count of a replayed step = the kernel nodes of the captured graph (includes the
      // launches made inside helpers that bypass the instrumentation, e.g. colsum / dkv_finalize)
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      int64_t kn = 0;
      if (nn && cudaGraphGetNodes(graph, nodes.data(), &nn) == cudaSuccess)
        for (auto nd : nodes) {
          cudaGraphNodeType t;
          if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++kn;
        }
      ce = cudaGraphInstantiate(&g_exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) { g_exec = nullptr; return fail(TP_ECUDA, "graph instantiate: %s", cudaGetErrorString(ce)); }
      g_launches = kn;
      instr.launches = kn;
      CU(cudaGraphLaunch(g_exec, stream));
    } else {
      if (g_exec) { cudaGraphExecDestroy(g_exec); g_exec = nullptr; }
      g_key = key;
      instr.launches = 0;
      ev_next = 0;
      TRY(enqueue_step(G, batch));
    }
    CU(cudaStreamSynchronize(stream));
    CU(cudaGetLastError());
    instr.resolve();
    if (*h_bad_tok)
      return fail(TP_EINVAL, "tp_step_device: %d token ids outside [0, %d); the step's results are invalid", *h_bad_tok, m.V);
    if (loss_out) *loss_out = (float)(*h_loss / ((double)batch * m.s));
    return TP_OK;
  }

  tp_status grads(float* host, size_t n) override {
    if (n != param_count()) return fail(TP_EINVAL, "tp_get_grads: n=%zu, expected %zu", n, param_count());
    size_t off = 0;
    for (auto& S : stages) {
      CU(cudaMemcpy(host + off, S.gflat, S.L.total * sizeof(float), cudaMemcpyDeviceToHost));
      off += S.L.total;
    }
    return TP_OK;
  }
  tp_status logits(float* host, size_t n) override {
    Stage<T>* last = nullptr;
    for (auto& S : stages) if (S.k == m.K - 1) last = &S;
    if (!last || !last->logits_keep) return fail(TP_ESTATE, "tp_get_logits: needs TP_FLAG_KEEP_LOGITS and the last stage");
    const size_t need = (size_t)last_batch * m.s * m.V;
    if (n != need) return fail(TP_EINVAL, "tp_get_logits: n=%zu, expected %zu", n, need);
    std::vector<float> tmp(need);
    CU(cudaMemcpy(tmp.data(), last->logits_keep, need * sizeof(float), cudaMemcpyDeviceToHost));
    // internal row seq0*s + p*b + j of a group (seq0, b)  ->  [sequence seq0 + j][position p]
    const size_t s = m.s, V = m.V;
    for (const auto& gr : last_groups) {
      const size_t seq0 = gr.first, b = (size_t)gr.second;
      for (size_t p = 0; p < s; ++p)
        for (size_t j = 0; j < b; ++j)
          std::memcpy(host + ((seq0 + j) * s + p) * V, tmp.data() + (seq0 * s + p * b + j) * V, V * sizeof(float));
    }
    return TP_OK;
  }
  tp_status profile(int g, int b, int reps, int64_t* ticks, double* fit) override;
  tp_status profile_wgrad(int batch, int reps, int64_t* ns_out) override;
  tp_status profile_comm(int reps, double* alpha_ns, double* gbs) override;
  tp_status profile_stage(Stage<T>& S, int g, int bsl, int reps, std::vector<int64_t>& ticks, double* fit);
  std::vector<int> stage_types() const;
  double comm_alpha_ns = 0.0, comm_gbs = 0.0;  // tp_profile_comm (0: no transmission term)
};

// ---------------------------------------------------------------- tp_profile
// measure t(l, 0) for every l, fit t_ctx(l, c) = a0 + a1 l + a2 c + a3 l c on a
// subset of (l, c) by least squares, fill the table with t(l, 0) + t_ctx(l, c). Done for every
// owned stage TYPE (first: embedding + layers, middle: layers, last: layers + head + CE; DESIGN.md
// A-16) and reduced by element-wise max — over the owned types here, over the ranks with an NCCL
// max when world > 1 — plus the data-transmission term of PAPER.md:243 when stages talk.
template <typename T>
tp_status Engine<T>::profile_stage(Stage<T>& S, int g, int bsl, int reps, std::vector<int64_t>& ticks,
                                   double* fit) {
  const int n = m.s / g;
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  // tokens for sequence 0 (values do not affect dense cost); finite dK/dV accumulators for the
  // reduce-add path of non-final slices
  CU(cudaMemsetAsync(d_tokens, 0, sizeof(int32_t) * (m.s + 1) * bsl, stream));
  for (int j = 0; j < S.nl; ++j) {
    CU(cudaMemsetAsync(S.dk_acc[j], 0, sizeof(float) * (size_t)bsl * m.s * m.H, stream));
    CU(cudaMemsetAsync(S.dv_acc[j], 0, sizeof(float) * (size_t)bsl * m.s * m.H, stream));
  }
  auto time_job = [&](int l, int c, double* out_ns) -> tp_status {
    std::vector<float> v;
    for (int r = 0; r < reps + 2; ++r) {
      CU(cudaEventRecord(e0, stream));
      TRY(fwd(S, 0, 0, 0, c, l, bsl, bsl));
      // as the step runs it: the slice ending at s (the first in backward) stores dK/dV, every other
      // slice reduce-adds into the c + l prefix rows
      TRY(bwd(S, 0, 0, 0, c, l, bsl, bsl, c + l == m.s));
      CU(cudaEventRecord(e1, stream));
      CU(cudaEventSynchronize(e1));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) v.push_back(ms);
    }
    std::sort(v.begin(), v.end());
    *out_ns = 1e6 * v[v.size() / 2];
    return TP_OK;
  };
  std::vector<double> base(n + 1, 0.0);
  for (int u = 1; u <= n; ++u) TRY(time_job(u * g, 0, &base[u]));
  // context samples on a grid: l in {g * 2^k} U {s}, c in {0, s/8, 2s/8, ...} U {s - l}
  std::vector<int> lgrid;
  for (int lu = 1; lu < n; lu *= 2) lgrid.push_back(lu);
  lgrid.push_back(n);
  const int cstep = std::max(1, n / 8);
  std::vector<std::array<double, 3>> samp;                  // (l, c, t_ctx) in tokens / ns
  std::vector<std::vector<std::pair<int, double>>> cs_of(lgrid.size());  // per grid l: (cu, t_ctx)
  for (size_t li = 0; li < lgrid.size(); ++li) {
    const int lu = lgrid[li];
    std::vector<int> cus;
    for (int cu = 0; cu + lu <= n; cu += cstep) cus.push_back(cu);
    if (cus.back() != n - lu) cus.push_back(n - lu);
    for (int cu : cus) {
      double t = base[lu];
      if (cu > 0) TRY(time_job(lu * g, cu * g, &t));
      cs_of[li].push_back({cu, t - base[lu]});
      samp.push_back({(double)lu * g, (double)cu * g, t - base[lu]});
    }
  }
  // least squares for a0..a3 via normal equations (4x4, Gaussian elimination with pivoting)
  double A[4][5] = {};
  for (auto& sp : samp) {
    const double x[4] = {1.0, sp[0], sp[1], sp[0] * sp[1]};
    for (int i = 0; i < 4; ++i) {
      for (int j = 0; j < 4; ++j) A[i][j] += x[i] * x[j];
      A[i][4] += x[i] * sp[2];
    }
  }
  double coef[4] = {0, 0, 0, 0};
  {
    bool ok = true;
    for (int col = 0; col < 4 && ok; ++col) {
      int best = col;
      for (int r = col + 1; r < 4; ++r) if (std::fabs(A[r][col]) > std::fabs(A[best][col])) best = r;
      if (std::fabs(A[best][col]) < 1e-30) { ok = false; break; }
      for (int j = 0; j < 5; ++j) std::swap(A[col][j], A[best][j]);
      for (int r = 0; r < 4; ++r) {
        if (r == col) continue;
        const double f = A[r][col] / A[col][col];
        for (int j = 0; j < 5; ++j) A[r][j] -= f * A[col][j];
      }
    }
    if (ok) for (int i = 0; i < 4; ++i) coef[i] = A[i][4] / A[i][i];
  }
  double maxrel = 0.0;
  for (auto& sp : samp) {
    const double pred = coef[0] + coef[1] * sp[0] + coef[2] * sp[1] + coef[3] * sp[0] * sp[1];
    const int lu = (int)sp[0] / g;
    const double full = base[lu] + sp[2];
    if (full > 0) maxrel = std::max(maxrel, std::fabs(base[lu] + pred - full) / full);
  }
  // Table fill. Default: t(l, c) = t(l, 0) + t_ctx(l, c) with t_ctx interpolated from the measured
  // grid (piecewise-linear in c at each grid l, then linear in l) — on B200 small-slice attention is
  // latency-bound, so t_ctx is not the bilinear a0 + a1 l + a2 c + a3 l c of PAPER.md:294 (the fit
  // above is still reported). TP_CTX_FIT=linear fills the table from the paper's linear fit.
  const bool linear = std::getenv("TP_CTX_FIT") && std::string(std::getenv("TP_CTX_FIT")) == "linear";
  // TP_PROFILE_DENSE=1 (cost-model study, NEXT(3)): every (l, c) entry measured directly
  const bool dense = std::getenv("TP_PROFILE_DENSE") && std::atoi(std::getenv("TP_PROFILE_DENSE")) != 0;
  auto ctx_at = [&](size_t li, int cu) -> double {  // t_ctx at grid l index li, any cu >= 0
    const auto& v = cs_of[li];
    if (v.size() == 1) return v[0].second;
    size_t k = 1;
    while (k + 1 < v.size() && v[k].first < cu) ++k;
    const double x0 = v[k - 1].first, x1 = v[k].first, y0 = v[k - 1].second, y1 = v[k].second;
    return y0 + (y1 - y0) * (cu - x0) / (x1 - x0);  // extrapolates past the last point
  };
  ticks.assign((size_t)n * (n + 1), 0);
  for (int lu = 1; lu <= n; ++lu)
    for (int cu = 0; cu + lu <= n; ++cu) {
      const double l = lu * g, c = cu * g;
      double tc;
      if (cu == 0) {
        tc = 0.0;
      } else if (dense) {
        double t = 0.0;
        TRY(time_job(lu * g, cu * g, &t));
        tc = t - base[lu];
      } else if (linear) {
        tc = coef[0] + coef[1] * l + coef[2] * c + coef[3] * l * c;
      } else {
        size_t hi = 0;
        while (lgrid[hi] < lu) ++hi;
        if (lgrid[hi] == lu || hi == 0) {
          tc = ctx_at(hi, cu);
        } else {
          const double w = (double)(lu - lgrid[hi - 1]) / (lgrid[hi] - lgrid[hi - 1]);
          tc = (1.0 - w) * ctx_at(hi - 1, cu) + w * ctx_at(hi, cu);
        }
        tc = std::max(0.0, tc);  // more context never costs less
      }
      ticks[(size_t)(lu - 1) * (n + 1) + cu] = std::max<int64_t>(1, (int64_t)std::llround(base[lu] + tc));
    }
  CU(cudaEventDestroy(e0));
  CU(cudaEventDestroy(e1));
  if (fit) { for (int i = 0; i < 4; ++i) fit[i] = coef[i]; fit[4] = maxrel; }
  return TP_OK;
}

// indices (into `stages`) of the first owned stage of each type: first / middle / last (A-16)
template <typename T>
std::vector<int> Engine<T>::stage_types() const {
  std::vector<int> out;
  int seen = 0;
  for (size_t i = 0; i < stages.size(); ++i) {
    const int k = stages[i].k;
    const int type = (k == 0 ? 1 : 0) | (k == m.K - 1 ? 2 : 0);  // 0 middle, 1 first, 2 last, 3 both
    if (!(seen & (1 << type))) { seen |= 1 << type; out.push_back((int)i); }
  }
  // a middle stage does a subset of the first stage's work (no embedding): skip it when a first
  // stage is measured too
  if ((seen & 2) && (seen & 1)) {
    std::vector<int> kept;
    for (int i : out) if (stages[i].k == 0 || stages[i].k == m.K - 1) kept.push_back(i);
    out = kept;
  }
  return out;
}

template <typename T>
tp_status Engine<T>::profile(int g, int bsl, int reps, int64_t* ticks, double* fit) {
  if (g < 1 || m.s % g != 0) return fail(TP_EINVAL, "tp_profile: granularity %d must divide seq_len %d", g, m.s);
  if (reps < 1) return fail(TP_EINVAL, "tp_profile: reps must be >= 1");
  if (bsl < 1 || bsl > max_batch) return fail(TP_EINVAL, "tp_profile: batch_slice %d not in [1, max_batch]", bsl);
  if (!ticks) return fail(TP_EINVAL, "tp_profile: null ticks_out");
  CU(cudaSetDevice(device));
  const int n = m.s / g;
  const size_t N = (size_t)n * (n + 1);
  bool saved = instr.on;
  instr.on = false;
  std::vector<int64_t> best(N, 0), t;
  double best_base = -1.0;
  for (int si : stage_types()) {
    double f[5];
    tp_status st = profile_stage(stages[si], g, bsl, reps, t, f);
    if (st != TP_OK) { instr.on = saved; return st; }
    for (size_t i = 0; i < N; ++i) best[i] = std::max(best[i], t[i]);
    const double tb = (double)t[(size_t)(n - 1) * (n + 1)];  // t(s, 0): the heaviest stage's fit is reported
    if (tb > best_base) { best_base = tb; if (fit) std::memcpy(fit, f, sizeof f); }
  }
  instr.on = saved;
  // data transmission (t = computation latency + data transmission latency): one fp32
  // T x H activation forward and one gradient backward per job, t_comm(T) = alpha + 4 H T / beta,
  // with alpha / beta measured by tp_profile_comm (world > 1) or set by the caller (TP_COMM_ALPHA_NS,
  // TP_COMM_GBS; e.g. to plan K > 1 stages from one GPU). Loopback without NCCL has no messages.
  double alpha = comm_alpha_ns, gbs = comm_gbs;
  if (const char* e = std::getenv("TP_COMM_ALPHA_NS")) alpha = std::atof(e);
  if (const char* e = std::getenv("TP_COMM_GBS")) gbs = std::atof(e);
  if (m.K > 1 && gbs > 0) {
    for (int lu = 1; lu <= n; ++lu) {
      const double bytes = 4.0 * m.H * (double)bsl * lu * g;
      const int64_t tc = (int64_t)std::llround(2.0 * (alpha + bytes / gbs));  // GB/s == bytes/ns
      for (int cu = 0; cu + lu <= n; ++cu) best[(size_t)(lu - 1) * (n + 1) + cu] += tc;
    }
  }
  if (world > 1) {  // bottleneck over the ranks' stages (collective: every rank calls tp_profile)
    int64_t* d = nullptr;
    CU(cudaMalloc(&d, N * sizeof(int64_t)));
    cudaError_t ce = cudaMemcpy(d, best.data(), N * sizeof(int64_t), cudaMemcpyHostToDevice);
    ncclResult_t nr = ncclSuccess;
    if (ce == cudaSuccess) nr = ncclAllReduce(d, d, N, ncclInt64, ncclMax, base, stream);
    if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaStreamSynchronize(stream);
    if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaMemcpy(best.data(), d, N * sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (nr != ncclSuccess) return fail(TP_ENCCL, "tp_profile: max over ranks: %s", ncclGetErrorString(nr));
    if (ce != cudaSuccess) return fail(TP_ECUDA, "tp_profile: max over ranks: %s", cudaGetErrorString(ce));
  }
  std::memcpy(ticks, best.data(), N * sizeof(int64_t));
  return TP_OK;
}

// Deferred weight-gradient GEMMs of one step (slicing-independent, excluded from the table): the
// time of the slowest owned stage type for `batch` sequences, max over ranks when world > 1.
template <typename T>
tp_status Engine<T>::profile_wgrad(int batch, int reps, int64_t* ns_out) {
  if (batch < 1 || batch > max_batch) return fail(TP_EINVAL, "tp_profile_wgrad: batch %d not in [1, max_batch]", batch);
  if (reps < 1 || !ns_out) return fail(TP_EINVAL, "tp_profile_wgrad: bad arguments");
  CU(cudaSetDevice(device));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  bool saved = instr.on;
  instr.on = false;
  double worst = 0.0;
  for (int si : stage_types()) {
    std::vector<float> v;
    for (int r = 0; r < reps + 1; ++r) {
      CU(cudaEventRecord(e0, stream));
      tp_status st = wgrad(stages[si], batch);
      if (st != TP_OK) { instr.on = saved; return st; }
      CU(cudaEventRecord(e1, stream));
      CU(cudaEventSynchronize(e1));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 1) v.push_back(ms);
    }
    std::sort(v.begin(), v.end());
    worst = std::max(worst, 1e6 * v[v.size() / 2]);
  }
  instr.on = saved;
  CU(cudaEventDestroy(e0));
  CU(cudaEventDestroy(e1));
  int64_t t = (int64_t)std::llround(worst);
  if (world > 1) {
    int64_t* d = nullptr;
    CU(cudaMalloc(&d, sizeof(int64_t)));
    CU(cudaMemcpy(d, &t, sizeof t, cudaMemcpyHostToDevice));
    NC(ncclAllReduce(d, d, 1, ncclInt64, ncclMax, base, stream));
    CU(cudaStreamSynchronize(stream));
    CU(cudaMemcpy(&t, d, sizeof t, cudaMemcpyDeviceToHost));
    cudaFree(d);
  }
  *ns_out = t;
  return TP_OK;
}

// alpha / beta of one stage-to-stage message, measured with ncclSend / ncclRecv
// ping-pongs between neighbouring ranks (edges (0,1), (2,3), .. then (1,2), (3,4), ..): the median
// one-way time of a small (4 KiB) and a large (the largest job's T x H fp32) message; alpha = t_small,
// beta = (bytes_large - bytes_small) / (t_large - t_small). Worst (max alpha, min beta) over the
// edges, identical on every rank; stored in the context and folded into later tp_profile tables.
template <typename T>
tp_status Engine<T>::profile_comm(int reps, double* alpha_ns, double* gbs) {
  if (world < 2) return fail(TP_ESTATE, "tp_profile_comm: needs world > 1 (one stage per GPU)");
  if (reps < 1) return fail(TP_EINVAL, "tp_profile_comm: reps must be >= 1");
  CU(cudaSetDevice(device));
  Stage<T>& S = stages[0];
  const size_t big = std::min((size_t)max_batch * m.s * m.H, (size_t)64 << 20);  // floats
  const size_t sizes[2] = {1024, big};
  double t1[2] = {0.0, 0.0};
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  double my_alpha = 0.0, my_gbs = 1e30;
  for (int phase = 0; phase < 2; ++phase) {
    // this rank's partner in the phase, initiator = the lower rank of the edge
    int peer = -1;
    if ((rank & 1) == phase) peer = rank + 1 < world ? rank + 1 : -1;
    else peer = rank - 1 >= 0 ? rank - 1 : -1;
    if (phase == 1 && rank == 0) peer = -1;
    const bool init = peer > rank;
    for (int z = 0; z < 2; ++z) {
      std::vector<float> v;
      for (int r = 0; r < reps + 2 && peer >= 0; ++r) {
        CU(cudaEventRecord(e0, stream));
        if (init) {
          NC(ncclSend(S.grad_out, sizes[z], ncclFloat32, peer, base, stream));
          NC(ncclRecv(S.grad_out, sizes[z], ncclFloat32, peer, base, stream));
        } else {
          NC(ncclRecv(S.grad_out, sizes[z], ncclFloat32, peer, base, stream));
          NC(ncclSend(S.grad_out, sizes[z], ncclFloat32, peer, base, stream));
        }
        CU(cudaEventRecord(e1, stream));
        CU(cudaEventSynchronize(e1));
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        if (r >= 2) v.push_back(ms);
      }
      if (!v.empty()) { std::sort(v.begin(), v.end()); t1[z] = 0.5e6 * v[v.size() / 2]; }
    }
    if (peer >= 0 && init) {
      const double a = t1[0];
      const double b = (double)(sizes[1] - sizes[0]) * 4.0 / std::max(1.0, t1[1] - t1[0]);
      my_alpha = std::max(my_alpha, a);
      my_gbs = std::min(my_gbs, b);
    }
    // all ranks finish the phase before the next one (a 1-float all-reduce as the barrier)
    NC(ncclAllReduce(d_loss, d_loss, 1, ncclFloat32, ncclSum, base, stream));
    CU(cudaStreamSynchronize(stream));
  }
  CU(cudaEventDestroy(e0));
  CU(cudaEventDestroy(e1));
  double* d = nullptr;
  double h[2] = {my_alpha, -my_gbs};
  CU(cudaMalloc(&d, 2 * sizeof(double)));
  CU(cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice));
  NC(ncclAllReduce(d, d, 2, ncclFloat64, ncclMax, base, stream));
  CU(cudaStreamSynchronize(stream));
  CU(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
  cudaFree(d);
  comm_alpha_ns = h[0];
  comm_gbs = -h[1];
  if (alpha_ns) *alpha_ns = comm_alpha_ns;
  if (gbs) *gbs = comm_gbs;
  return TP_OK;
}

}  // namespace tp

// ==================================================================== C ABI
struct tp_ctx {
  std::unique_ptr<tp::EngineBase> eng;
};

using namespace tp;

extern "C" tp_status tp_stage_param_count(const tp_model_cfg* cfg, int32_t stage, size_t* out) {
  TP_CHECK_ARG(cfg && out, "tp_stage_param_count: null argument");
  TP_CHECK_ARG(cfg->n_stages >= 1 && stage >= 0 && stage < cfg->n_stages, "tp_stage_param_count: bad stage");
  TP_CHECK_ARG(cfg->partition == TP_PARTITION_UNIFORM || cfg->partition == TP_PARTITION_BALANCED, "bad partition");
  TP_CHECK_ARG(cfg->partition == TP_PARTITION_BALANCED ? cfg->n_layer >= cfg->n_stages : cfg->n_layer % cfg->n_stages == 0,
               "n_layer %d does not split over %d stages", cfg->n_layer, cfg->n_stages);
  ModelShape m{cfg->n_layer, cfg->hidden, cfg->n_head, cfg->n_head ? cfg->hidden / cfg->n_head : 0,
               cfg->vocab, cfg->seq_len, cfg->n_stages, cfg->partition};
  *out = stage_layout(m, stage).total;
  return TP_OK;
}

extern "C" tp_status tp_schedule_oplist(int32_t n_stages, int32_t stage, int32_t schedule, int32_t n_groups,
                                        const int32_t* n_slices, int32_t capacity, int32_t* ops_out, int32_t* n_ops) {
  TP_CHECK_ARG(n_stages >= 1 && stage >= 0 && stage < n_stages, "tp_schedule_oplist: bad stage %d of %d", stage, n_stages);
  TP_CHECK_ARG(schedule == 0 || schedule == 1, "tp_schedule_oplist: schedule %d", schedule);
  TP_CHECK_ARG(n_groups >= 1 && n_slices && ops_out && n_ops, "tp_schedule_oplist: null / empty argument");
  std::vector<int> M(n_slices, n_slices + n_groups);
  std::vector<int> first(n_groups + 1, 0);
  for (int d = 0; d < n_groups; ++d) {
    TP_CHECK_ARG(M[d] >= 1, "tp_schedule_oplist: group %d has %d slices", d, M[d]);
    first[d + 1] = first[d] + M[d];
  }
  TP_CHECK_ARG(capacity >= 2 * first[n_groups], "tp_schedule_oplist: capacity %d < %d", capacity, 2 * first[n_groups]);
  const std::vector<Op> ops = build_oplist(n_stages, stage, schedule == 1, M);
  for (size_t t = 0; t < ops.size(); ++t) {
    const int j = first[ops[t].d] + ops[t].i;
    ops_out[t] = ops[t].fwd ? j + 1 : -(j + 1);
  }
  *n_ops = (int32_t)ops.size();
  return TP_OK;
}

extern "C" tp_status tp_stage_layers(const tp_model_cfg* cfg, int32_t* counts_out) {
  TP_CHECK_ARG(cfg && counts_out && cfg->n_stages >= 1 && cfg->n_layer >= cfg->n_stages, "tp_stage_layers: bad argument");
  TP_CHECK_ARG(cfg->partition == TP_PARTITION_BALANCED || cfg->n_layer % cfg->n_stages == 0,
               "tp_stage_layers: n_layer %% n_stages != 0");
  const std::vector<int> c = stage_layer_counts(cfg->n_layer, cfg->n_stages, cfg->hidden, cfg->vocab, cfg->seq_len,
                                                cfg->partition);
  for (int k = 0; k < cfg->n_stages; ++k) counts_out[k] = c[k];
  return TP_OK;
}

extern "C" tp_status tp_nccl_unique_id(void* out128) {
  TP_CHECK_ARG(out128, "tp_nccl_unique_id: null");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(TP_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof id);
  return TP_OK;
}

extern "C" tp_status tp_init(const tp_model_cfg* cfg, int32_t rank, int32_t world, const void* nccl_id,
                             int32_t precision, int32_t max_batch, int32_t device, int32_t flags, tp_ctx** out) {
  TP_CHECK_ARG(cfg && out, "tp_init: null argument");
  *out = nullptr;
  TP_CHECK_ARG(cfg->partition == TP_PARTITION_UNIFORM || cfg->partition == TP_PARTITION_BALANCED,
               "tp_init: bad partition %d", cfg->partition);
  TP_CHECK_ARG(cfg->n_layer >= 1 && cfg->n_stages >= 1 &&
               (cfg->partition == TP_PARTITION_BALANCED ? cfg->n_layer >= cfg->n_stages : cfg->n_layer % cfg->n_stages == 0),
               "tp_init: n_layer (%d) must be a positive multiple of n_stages (%d) (balanced: >= n_stages)", cfg->n_layer,
               cfg->n_stages);
  TP_CHECK_ARG(cfg->n_head >= 1 && cfg->hidden % cfg->n_head == 0, "tp_init: hidden %% n_head != 0");
  const int d = cfg->hidden / cfg->n_head;
  TP_CHECK_ARG(d % 16 == 0 && d <= 128, "tp_init: head_dim %d must be a multiple of 16 and <= 128", d);
  TP_CHECK_ARG(cfg->hidden % 64 == 0, "tp_init: hidden %d must be a multiple of 64", cfg->hidden);
  TP_CHECK_ARG(cfg->vocab >= 1 && cfg->vocab % 8 == 0, "tp_init: vocab %d must be a positive multiple of 8", cfg->vocab);
  TP_CHECK_ARG(cfg->seq_len >= 1, "tp_init: seq_len must be >= 1");
  TP_CHECK_ARG(world == 1 || world == cfg->n_stages, "tp_init: world (%d) must be 1 (loopback) or n_stages (%d)", world, cfg->n_stages);
  TP_CHECK_ARG(rank >= 0 && rank < world, "tp_init: rank %d not in [0, %d)", rank, world);
  TP_CHECK_ARG(world == 1 || nccl_id, "tp_init: nccl_id required for world > 1");
  TP_CHECK_ARG(precision == TP_BF16 || precision == TP_FP32, "tp_init: bad precision %d", precision);
  TP_CHECK_ARG(max_batch >= 1, "tp_init: max_batch must be >= 1");
  auto ctx = std::make_unique<tp_ctx>();
  tp_status st;
  if (precision == TP_BF16) {
    auto e = std::make_unique<Engine<bf16>>();
    st = e->init(cfg, rank, world, nccl_id, precision, max_batch, device, flags);
    ctx->eng = std::move(e);
  } else {
    auto e = std::make_unique<Engine<float>>();
    st = e->init(cfg, rank, world, nccl_id, precision, max_batch, device, flags);
    ctx->eng = std::move(e);
  }
  if (st != TP_OK) return st;
  *out = ctx.release();
  return TP_OK;
}

extern "C" tp_status tp_param_count(const tp_ctx* ctx, size_t* out) {
  TP_CHECK_ARG(ctx && out, "tp_param_count: null argument");
  *out = ctx->eng->param_count();
  return TP_OK;
}
extern "C" tp_status tp_load_params(tp_ctx* ctx, const float* host, size_t n) {
  TP_CHECK_ARG(ctx && host, "tp_load_params: null argument");
  return ctx->eng->load(host, n);
}
extern "C" tp_status tp_step(tp_ctx* ctx, const tp_slicing* sl, const int32_t* tokens, int32_t batch, float* loss) {
  TP_CHECK_ARG(ctx, "tp_step: null ctx");
  return ctx->eng->step(sl, tokens, true, batch, loss);
}
extern "C" tp_status tp_step_device(tp_ctx* ctx, const tp_slicing* sl, const int32_t* tokens, int32_t batch, float* loss) {
  TP_CHECK_ARG(ctx, "tp_step_device: null ctx");
  return ctx->eng->step(sl, tokens, false, batch, loss);
}
extern "C" tp_status tp_step_plan(tp_ctx* ctx, const tp_batch_plan* pl, const int32_t* tokens, int32_t batch,
                                  float* loss) {
  TP_CHECK_ARG(ctx, "tp_step_plan: null ctx");
  return ctx->eng->step_plan(pl, tokens, true, batch, loss);
}
extern "C" tp_status tp_step_plan_device(tp_ctx* ctx, const tp_batch_plan* pl, const int32_t* tokens, int32_t batch,
                                         float* loss) {
  TP_CHECK_ARG(ctx, "tp_step_plan_device: null ctx");
  return ctx->eng->step_plan(pl, tokens, false, batch, loss);
}
extern "C" tp_status tp_get_grads(tp_ctx* ctx, float* host, size_t n) {
  TP_CHECK_ARG(ctx && host, "tp_get_grads: null argument");
  return ctx->eng->grads(host, n);
}
extern "C" tp_status tp_get_logits(tp_ctx* ctx, float* host, size_t n) {
  TP_CHECK_ARG(ctx && host, "tp_get_logits: null argument");
  return ctx->eng->logits(host, n);
}
extern "C" tp_status tp_profile(tp_ctx* ctx, int32_t g, int32_t batch_slice, int32_t reps, int64_t* ticks,
                                double* fit) {
  TP_CHECK_ARG(ctx, "tp_profile: null ctx");
  return ctx->eng->profile(g, batch_slice, reps, ticks, fit);
}
extern "C" tp_status tp_profile_wgrad(tp_ctx* ctx, int32_t batch, int32_t reps, int64_t* ns_out) {
  TP_CHECK_ARG(ctx, "tp_profile_wgrad: null ctx");
  return ctx->eng->profile_wgrad(batch, reps, ns_out);
}
extern "C" tp_status tp_profile_comm(tp_ctx* ctx, int32_t reps, double* alpha_ns, double* gbs) {
  TP_CHECK_ARG(ctx, "tp_profile_comm: null ctx");
  return ctx->eng->profile_comm(reps, alpha_ns, gbs);
}
extern "C" tp_status tp_get_stream(tp_ctx* ctx, void** out) {
  TP_CHECK_ARG(ctx && out, "tp_get_stream: null argument");
  *out = (void*)ctx->eng->stream;
  return TP_OK;
}
extern "C" tp_status tp_kernel_stats(tp_ctx* ctx, int32_t i, char* name32, int64_t* launches, double* ms,
                                     double* flops, double* bytes, int32_t* n_classes) {
  TP_CHECK_ARG(ctx, "tp_kernel_stats: null ctx");
  if (n_classes) *n_classes = KC_N;
  if (i < 0 || i >= KC_N) return i == -1 ? TP_OK : fail(TP_EINVAL, "tp_kernel_stats: class %d", i);
  const KStat& s = ctx->eng->instr.stats[i];
  if (name32) { std::strncpy(name32, s.name, 31); name32[31] = 0; }
  if (launches) *launches = s.launches;
  if (ms) *ms = s.ms;
  if (flops) *flops = s.flops;
  if (bytes) *bytes = s.bytes;
  return TP_OK;
}
extern "C" tp_status tp_kernel_stats_reset(tp_ctx* ctx) {
  TP_CHECK_ARG(ctx, "tp_kernel_stats_reset: null ctx");
  for (auto& s : ctx->eng->instr.stats) { s.launches = 0; s.ms = s.flops = s.bytes = 0; }
  return TP_OK;
}
extern "C" tp_status tp_kernel_stats_enable(tp_ctx* ctx, int32_t on) {
  TP_CHECK_ARG(ctx, "tp_kernel_stats_enable: null ctx");
  ctx->eng->instr.on = on != 0;
  return TP_OK;
}
extern "C" tp_status tp_last_step_launches(tp_ctx* ctx, int64_t* out) {
  TP_CHECK_ARG(ctx && out, "tp_last_step_launches: null argument");
  *out = ctx->eng->instr.launches;
  return TP_OK;
}
extern "C" void tp_destroy(tp_ctx* ctx) { delete ctx; }
