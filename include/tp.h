/*
 * tp.h — C ABI of the B200-native TeraPipe hot path (arXiv 2102.07988).
 *
 * Two calls follow the paper's problem statement (§3.3): "given a partitioned
 * Transformer-based LM F = c_K o ... o c_1 and a training input sequence of length L, find the
 * slicing scheme l_1..l_M to minimize the total forward and backward propagation latency":
 *   tp_plan  — the dynamic program of §3.3 (Eq. 5-8, Algorithm 1) over a
 *              t_fwd+bwd(slice_len, context_len) cost table;
 *   tp_step  — one synchronous forward+backward of a causal GPT stack,
 *              token-sliced and pipelined over K stages.
 * The rest (tp_init, tp_load_params, tp_profile, getters) is the plumbing those two need.
 *
 * Conventions
 *   - Every call returns tp_status (0 = TP_OK, < 0 = error). On error, tp_last_error() returns a
 *     thread-local, NUL-terminated message valid until the next failing call on that thread.
 *   - Bad arguments are rejected, never clamped (TP_EINVAL). No call falls back to a CPU path:
 *     without a usable sm_100a GPU, tp_init fails with TP_ECUDA.
 *   - The caller owns every host buffer passed in; the library copies what it keeps and never
 *     retains a caller pointer past the call. The library owns all device memory, CUDA streams and
 *     the NCCL communicator inside a tp_ctx.
 *   - Host integers are little-endian; all sizes are element counts unless named *_bytes.
 *
 * Parameter layout (shared DATA, not code, with oracle/ and synth/): for stage k of K, one flat
 * float32 array, in this order —
 *     stage 0 only:   wte[V][H], wpe[s][H]
 *     each owned layer l (stage k's contiguous block: k*n/K .. (k+1)*n/K - 1 for uniform cells,
 *       PAPER.md:193-194; tp_stage_layers for TP_PARTITION_BALANCED):
 *         ln1_g[H], ln1_b[H], w_qkv[H][3H], b_qkv[3H], w_o[H][H], b_o[H],
 *         ln2_g[H], ln2_b[H], w_1[H][4H], b_1[4H], w_2[4H][H], b_2[H]
 *       (matrices row-major [in][out]; w_qkv columns are [q | k | v], head j at j*d..(j+1)*d)
 *     stage K-1 only: lnf_g[H], lnf_b[H], w_out[H][V]
 *   A context that owns several stages (loopback, world == 1) uses the concatenation in stage
 *   order. Gradients (tp_get_grads) use exactly the same layout.
 */
#ifndef TP_H_
#define TP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TP_OK = 0,
  TP_EINVAL = -1,       /* bad argument / shape (SPEC.md exit code 2)                        */
  TP_EINFEASIBLE = -2,  /* no slicing satisfies the constraints (SPEC.md exit code 3)       */
  TP_ETOOBIG = -3,      /* instance too large for the requested operation                  */
  TP_ECUDA = -4,        /* CUDA runtime/driver error, or no sm_100 device                   */
  TP_ENCCL = -5,        /* NCCL error                                                      */
  TP_ENOMEM = -6,       /* device or host allocation failed                                */
  TP_ESTATE = -7        /* call not valid in the context's current state                   */
} tp_status;

enum { TP_BF16 = 0, /* bf16 GEMM/attention operands, fp32 accumulation, fp32 residual stream,
                       softmax, LayerNorm statistics and stage messages (A-23)      */
       TP_FP32 = 1  /* true fp32 arithmetic everywhere (SIMT FFMA; A-18)           */ };

enum { TP_FLAG_KEEP_LOGITS = 1,   /* keep fp32 logits of the last step for tp_get_logits     */
       TP_FLAG_KERNEL_STATS = 2,  /* bracket launches with CUDA events (tp_kernel_stats)      */
       TP_FLAG_FORCE_SIMT = 4,    /* bf16 mode: use SIMT GEMM/attention (kernel cross-checks)  */
       TP_FLAG_NCCL_LOOPBACK = 8, /* world == 1, n_stages > 1: send every stage message through
                                     ncclSend/ncclRecv to self on a one-rank communicator (grouped
                                     per message, on the same per-direction comm streams, NCCL
                                     communicators and events as world == n_stages) instead of
                                     aliasing the buffers; lets the p2p path run on one GPU        */
       TP_FLAG_DEVICE_P2P = 16,   /* world == n_stages > 1: device-initiated messages instead of
                                     ncclSend/ncclRecv — each stage's receive buffers are NCCL
                                     symmetric windows (ncclMemAlloc + ncclCommWindowRegister); the
                                     last layer's FC2 epilogue and the first layer's LayerNorm
                                     backward write straight into the neighbour's buffer over
                                     NVLink, a release-store flag per job signals it, the consumer
                                     spins on its flag before the job; env
                                     TP_DEVICE_P2P=1 sets it too                                   */
       TP_FLAG_SCHEDULE_1F1B = 32 /* 1F1B at sequence-group granularity instead of GPipe order
                                     (A-21): stage k runs the forwards
                                     of w_k = min(D, K - k) groups, then alternates the backward of
                                     its oldest group with the forward of the next; each group's
                                     weight gradients run right after its backward; the stage
                                     buffers hold only w_k groups (slots), so a step's batch may
                                     exceed max_batch as long as w_k x (largest group) <= max_batch;
                                     env TP_SCHEDULE=1f1b sets it too                              */ };

enum { TP_PARTITION_UNIFORM = 0,  /* stage k owns n_layer / n_stages layers   */
       TP_PARTITION_BALANCED = 1  /* the last stage, which also runs the LM head + CE, owns fewer
                                     layers so the per-stage FLOPs balance (A-30;
                                     counts: tp_stage_layers)                                      */ };

/* Model shape. hidden % n_head == 0; head_dim = hidden / n_head must be a multiple of 16 and <= 128;
 * hidden % 64 == 0; seq_len >= 1; partition TP_PARTITION_UNIFORM (n_layer % n_stages == 0) or
 * TP_PARTITION_BALANCED (n_layer >= n_stages). Stage k owns a contiguous block of layers. */
typedef struct {
  int32_t n_layer, hidden, n_head, vocab, seq_len, n_stages;
  int32_t partition;
} tp_model_cfg;

/* Layers owned by each stage (counts_out[n_stages], in stage order) under cfg->partition. */
tp_status tp_stage_layers(const tp_model_cfg* cfg, int32_t* counts_out);

/* Cost table t_{fwd+bwd}(l, c) of ONE pipeline stage (the bottleneck stage; A-16), in
 * integer ticks (A-15). l and c are in units of `granularity` tokens (g | seq_len, n_units =
 * seq_len / g). ticks[(l-1)*(n_units+1) + c] = t(l*g tokens, c*g tokens of context), for
 * 1 <= l, 0 <= c, l + c <= n_units; other entries are ignored. Used entries must be > 0.
 * ticks_per_ms is informational (e.g. 1000000 for ns). Caller-owned, read-only during the call. */
typedef struct {
  int32_t granularity;
  int32_t n_units;
  const int64_t* ticks;
  int64_t ticks_per_ms;
} tp_cost_table;

/* A slicing scheme [(b, [l_1..l_M])] * (B/b) in the paper's notation.
 * lengths: caller-owned array of `capacity` int32 (tokens; multiples of g, sum = seq_len).
 * batch_slice b: sequences per job (b | batch): every job is b sequences x one token slice, so
 * D = batch / b jobs share each slice index (joint batch x token slicing). */
typedef struct {
  int32_t batch_slice;
  int32_t n_slices;          /* M                                          */
  int32_t capacity;          /* size of `lengths` (>= n_units for tp_plan) */
  int32_t* lengths;          /* l_1..l_M in tokens                         */
  int64_t t_max_ticks;       /* max_i t_i of the scheme (tp_plan output)   */
  int64_t predicted_ticks;   /* n_micro * sum t_i + (K-1) * max t_i        */
} tp_slicing;

/* ---------------------------------------------------------------- planner (host only) */
/* The paper's DP: candidates = the distinct table values, ascending, thinned
 * so each evaluated t_max is >= the previous evaluated one + eps_ticks (the largest
 * value is always evaluated); for each, Algorithm 1 with smallest-k
 * backpointers; keep the scheme minimising T = n_micro * sum t_i + (K-1) * max t_i (Eq. 5 with
 * D = n_micro jobs per slice index, A-20; n_micro = 1 is Eq. 5 exactly), replacing only
 * on strict improvement; stop once (n_micro + K - 1) * t_max >= best (A-14).
 * eps_ticks = 0 gives the exact optimum, identical (T and boundaries) to brute force over all
 * compositions with the tie-break (T, max t, reversed lengths). n_layer and hidden are validated
 * (n_layer >= n_stages, hidden > 0) and otherwise informational. Pure, deterministic,
 * thread-safe. Threads: env TP_PLAN_THREADS (default: hardware concurrency, max 64).
 * Errors: TP_EINVAL (shape, table, capacity), TP_EINFEASIBLE (cannot happen for valid tables). */
tp_status tp_plan(int32_t n_layer, int32_t hidden, int32_t seq_len, int32_t n_stages,
                  const tp_cost_table* cost, int32_t n_micro, int64_t eps_ticks, tp_slicing* out);

/* A batch plan [(b_1, l^1), (b_2, l^2), ..]: group d is b_d consecutive
 * sequences x its own token slicing l^d (multiples of g, sum = seq_len); sum_d b_d = batch. Groups
 * run in order d = 1..D, each group's jobs in slice order (GPipe order, A-21). All arrays
 * caller-owned: batch_slice[] / n_slices[] hold `capacity_groups` entries, lengths[] (the groups'
 * slicings concatenated) holds `capacity_lengths`. A uniform tp_slicing is the plan with D = batch/b
 * identical groups. */
typedef struct {
  int32_t n_groups;          /* D                                                      */
  int32_t capacity_groups;   /* size of batch_slice[] and n_slices[]                   */
  int32_t* batch_slice;      /* b_1..b_D                                               */
  int32_t* n_slices;         /* M_1..M_D                                               */
  int32_t capacity_lengths;  /* size of lengths[]                                      */
  int32_t* lengths;          /* l^1_1..l^1_{M_1}, l^2_1.., in tokens                    */
  int64_t t_max_ticks;       /* max over all jobs of the plan (tp_plan_joint output)   */
  int64_t predicted_ticks;   /* sum over all jobs + (K-1) * max (A-20b)      */
} tp_batch_plan;

/* Joint batch x token planning: cost tables costs[i] of jobs of b_values[i]
 * sequences (tp_profile with batch_slice = b_values[i], all with the same granularity); chooses
 * b_1 + .. + b_D = batch and a slicing per group minimising the exact pipelined makespan
 * sum_jobs t + (K-1) * max_jobs t (A-20b: the bubble is paid once for the whole batch).
 * For each t_max candidate (the union of the tables' distinct values, ascending, eps-thinned, the
 * largest always kept): Algorithm 1 per table, then the 1-D knapsack C(m) = min_b C(m-b) + S*_b
 * (smallest b wins ties), then the exact objective of the plan; strict improvements only; stop
 * once K * t_max >= best. eps_ticks = 0 is the exact optimum (pinned to brute force over all
 * partitions x slicings). Groups are returned in knapsack backtrack order from m = batch. Output:
 * out->capacity_groups >= batch, out->capacity_lengths >= batch * seq_len / g.
 * Errors: TP_EINVAL (shapes, tables, capacities, duplicate b), TP_EINFEASIBLE (batch not a sum of
 * the available b). Pure, deterministic, thread-safe. */
tp_status tp_plan_joint(int32_t n_layer, int32_t hidden, int32_t seq_len, int32_t n_stages, int32_t n_b,
                        const int32_t* b_values, const tp_cost_table* const* costs, int32_t batch,
                        int64_t eps_ticks, tp_batch_plan* out);

/* The op list tp_step runs on stage `stage` of n_stages (A-21) for groups with
 * n_slices[d] token slices each (jobs numbered group-major: job j = slice i of group d, j = first(d) +
 * i): ops_out[t] = j + 1 for the forward of job j, -(j + 1) for its backward. schedule 0 = GPipe
 * (all forwards in order, then all backwards in exact reverse), 1 = 1F1B at group granularity
 * (TP_FLAG_SCHEDULE_1F1B). capacity >= 2 * total jobs; *n_ops = 2 * total jobs. Pure host function
 * (pinned to oracle/plan.py gpipe_oplists / one_f_one_b_oplists). */
tp_status tp_schedule_oplist(int32_t n_stages, int32_t stage, int32_t schedule, int32_t n_groups,
                             const int32_t* n_slices, int32_t capacity, int32_t* ops_out, int32_t* n_ops);

/* Number of float32 parameters of stage `stage` (see "Parameter layout"). */
tp_status tp_stage_param_count(const tp_model_cfg* cfg, int32_t stage, size_t* out);

/* ---------------------------------------------------------------- runtime (one process per GPU) */
typedef struct tp_ctx tp_ctx;

/* Writes a fresh 128-byte ncclUniqueId into out128 (rank 0 calls it; the harness broadcasts it). */
tp_status tp_nccl_unique_id(void* out128);

/* Creates a context on CUDA device `device`.
 *  world == 1: this context owns ALL cfg->n_stages stages on one GPU ("loopback": stage k's input
 *              buffer is stage k-1's output buffer, no copy and no NCCL; with TP_FLAG_NCCL_LOOPBACK
 *              every message is an NCCL send/recv to self instead; nccl_id may be NULL).
 *  world == cfg->n_stages > 1: this context owns stage `rank`; neighbours exchange slice
 *              activations / gradients with ncclSend/ncclRecv over NVLink.
 * precision: TP_BF16 or TP_FP32. max_batch: largest `batch` tp_step will be called with (sizes the
 * store-all activation buffers). flags: TP_FLAG_*. */
tp_status tp_init(const tp_model_cfg* cfg, int32_t rank, int32_t world, const void* nccl_id,
                  int32_t precision, int32_t max_batch, int32_t device, int32_t flags,
                  tp_ctx** out);

/* Total float32 parameter count of the stages this context owns. */
tp_status tp_param_count(const tp_ctx* ctx, size_t* out);

/* Copies host parameters (stage-local flat layout, n == tp_param_count) to the device. In bf16
 * mode matrices are rounded to bf16 (round-to-nearest-even) on the device. */
tp_status tp_load_params(tp_ctx* ctx, const float* host_params, size_t n);

/* One synchronous forward+backward of one batch with the given slicing: gradients are zeroed on
 * entry, every stage runs F(d,i) for d = 0..B-1, i = 1..M, then B(d,i) in exact reverse order
 * (GPipe order, store-all, A-21); weight gradients are accumulated per sequence.
 * tokens: HOST int32 [batch][seq_len+1] (input = [:, :s], target = [:, 1:], A-8); read by the
 * first and last stage; every id must lie in [0, vocab): an id outside it is rejected with
 * TP_EINVAL before any device work (never clamped). loss_out (may be NULL): mean cross-entropy over
 * batch*seq_len targets, identical on every rank. Returns after all local device work has completed. */
tp_status tp_step(tp_ctx* ctx, const tp_slicing* slicing, const int32_t* tokens, int32_t batch,
                  float* loss_out);

/* Same as tp_step with DEVICE tokens (already resident in HBM on this context's device). Ids outside
 * [0, vocab) are counted on the device (the kernels never read or scatter out of range with them)
 * and the call returns TP_EINVAL after the step; its loss, logits and gradients are then invalid. */
tp_status tp_step_device(tp_ctx* ctx, const tp_slicing* slicing, const int32_t* dev_tokens,
                         int32_t batch, float* loss_out);

/* tp_step with a heterogeneous batch plan (tp_plan_joint's output): group d is
 * sequences [b_1+..+b_{d-1}, +b_d) with its own token slicing; forward jobs run group by group,
 * each in slice order, backward in exact reverse. sum b_d must equal batch <= max_batch; every
 * group's lengths must be positive and sum to seq_len (TP_EINVAL otherwise). Same tokens / loss /
 * gradient contract as tp_step (a uniform tp_slicing is the plan of batch/b identical groups). */
tp_status tp_step_plan(tp_ctx* ctx, const tp_batch_plan* plan, const int32_t* tokens, int32_t batch,
                       float* loss_out);
/* Same with DEVICE tokens. */
tp_status tp_step_plan_device(tp_ctx* ctx, const tp_batch_plan* plan, const int32_t* dev_tokens, int32_t batch,
                              float* loss_out);

/* Copies the last step's gradients (same layout as tp_load_params) to host_out[n]. */
tp_status tp_get_grads(tp_ctx* ctx, float* host_out, size_t n);

/* Copies the last step's logits, float32 [batch][seq_len][vocab], to host_out[n]. Requires
 * TP_FLAG_KEEP_LOGITS and a context owning the last stage (else TP_ESTATE). */
tp_status tp_get_logits(tp_ctx* ctx, float* host_out, size_t n);

/* The cost table t_{fwd+bwd}(l, c) of PAPER.md:292-298 for jobs of batch_slice sequences x l tokens
 * with c tokens of context, in ns (median of `reps` after 2 warm-ups), measured the way tp_step runs
 * each job (the slice ending at seq_len stores dK/dV, every other one reduce-adds them into its
 * prefix rows). The base curve t(l, 0) is measured for every l = g, 2g, .., s; the
 * context term t_ctx(l, c) on a grid (l in {g 2^k} U {s}, c in multiples of s/8 U {s - l}), and
 * ticks_out[(l/g-1)*(n+1) + c/g] = t(l,0) + t_ctx(l,c) with t_ctx interpolated from the grid (env
 * TP_CTX_FIT=linear: the paper's least-squares t_ctx = a0 + a1 l + a2 c + a3 l c instead,
 * PAPER.md:292-296). Every owned stage TYPE is measured (first: embedding + layers; middle: layers;
 * last: layers + LM head + CE) and the table is their element-wise max (the bottleneck stage,
 * DESIGN.md A-16); with world > 1 the max is also taken over all ranks (COLLECTIVE: every rank must
 * call tp_profile with the same arguments). With n_stages > 1 the data-transmission term of
 * PAPER.md:243 is added to every entry: 2 * (alpha + 4 * hidden * batch_slice * l / beta) (one
 * fp32 activation forward, one gradient backward), alpha / beta from tp_profile_comm (world > 1) or
 * the env TP_COMM_ALPHA_NS / TP_COMM_GBS (e.g. to plan a K-GPU pipeline from one GPU); none if
 * neither is set. n = s/g; caller-owned, n*(n+1) int64. fit_out (may be NULL): the linear fit's
 * a0..a3 (ns, ns/token, ns/token, ns/token^2) and its max relative error on the grid samples (the
 * paper reports < 2%), for the stage type with the largest t(s, 0). Parameters must be loaded. */
tp_status tp_profile(tp_ctx* ctx, int32_t granularity, int32_t batch_slice, int32_t reps,
                     int64_t* ticks_out, double* fit_out /* [5] */);

/* Time of the deferred weight-gradient GEMMs of one step of `batch` sequences (K = batch * seq_len,
 * slicing-independent, so not part of the cost table): median of `reps`, ns, for the slowest owned
 * stage type, max over ranks when world > 1 (COLLECTIVE then). The step latency model is
 * predicted_ticks of the plan + this constant (the last stage's dW overlaps, the first stage's does
 * not). */
tp_status tp_profile_wgrad(tp_ctx* ctx, int32_t batch, int32_t reps, int64_t* ns_out);

/* alpha (ns) and beta (GB/s = bytes/ns) of one stage-to-stage message, measured with
 * NCCL ping-pongs between neighbouring ranks (median one-way time of a 4 KiB and a large message),
 * worst over the edges, identical on every rank. COLLECTIVE; requires world > 1 (TP_ESTATE
 * otherwise). Stored in the context and added by later tp_profile calls. Either output may be
 * NULL. */
tp_status tp_profile_comm(tp_ctx* ctx, int32_t reps, double* alpha_ns, double* gbs);

/* The CUDA stream (cudaStream_t) all compute of this context is issued on. */
tp_status tp_get_stream(tp_ctx* ctx, void** stream_out);

/* Kernel statistics collected while TP_FLAG_KERNEL_STATS is set: for class index i (0 <= i <
 * *n_classes), name (<= 31 chars), launches, summed device ms (CUDA events on the launching
 * stream), summed algorithmic FLOPs and bytes. tp_kernel_stats_reset clears them. */
tp_status tp_kernel_stats(tp_ctx* ctx, int32_t i, char* name32, int64_t* launches, double* ms,
                          double* flops, double* bytes, int32_t* n_classes);
tp_status tp_kernel_stats_reset(tp_ctx* ctx);
/* Turns the per-launch CUDA-event bracketing of TP_FLAG_KERNEL_STATS on (1) or off (0). */
tp_status tp_kernel_stats_enable(tp_ctx* ctx, int32_t on);

/* Number of kernel launches issued by the last tp_step on this context. For a step replayed from
 * the CUDA graph this is the number of kernel nodes in the captured graph (every launch, NCCL p2p
 * kernels included); for an eager step it counts the instrumented launches only. */
tp_status tp_last_step_launches(tp_ctx* ctx, int64_t* out);

void tp_destroy(tp_ctx* ctx);
const char* tp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TP_H_ */
