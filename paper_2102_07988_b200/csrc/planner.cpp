// planner.cpp — tp_plan: the slicing dynamic program of TeraPipe §3.3.
//
// Costs are int64 ticks (A-15), so sums are exact and the result is bit-identical to
// brute force over all compositions (proof sketch: SURVEY.md §8(c) "Why DP == brute force").
//
// Structure:
//   candidates = distinct t(k, j), k >= 1, k + j <= n, ascending, thinned by eps
//   (A-13/A-13b); for each candidate t_max in ascending order:
//     prune: stop once (D + K - 1) * t_max >= best T      (A-14, A-20)
//     Algorithm 1: S(0) = 0,
//         S(i) = min_{k: t(k, i-k) <= t_max} S(i-k) + t(k, i-k), q_i = smallest argmin (A-11, A-12)
//     backtrack q, recompute T = D * sum t_i + (K-1) * max t_i, keep on strict improvement.
//
// B200-host design: the table is re-laid out by END position (tt[i][k] = t(k, i-k)) so the
// inner min-plus loop over k is contiguous, and candidates are evaluated in parallel batches by
// a thread pool; the batch results are merged in ascending candidate order with the same pruning
// and strict-improvement rule, which makes the parallel result identical to the sequential one
// (SPEC.md:174 merge rule).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <thread>
#include <vector>

#include "common.h"

namespace {

constexpr int64_t kInf = INT64_MAX / 4;

struct DpResult {
  bool feasible = false;
  int64_t T = 0, mx = 0;
  std::vector<int32_t> lengths;  // in units
};

// Algorithm 1 for one t_max. tt: [(n+1)][(n+1)], tt[i*(n+1)+k] = t(k, i-k).
static void dp_fixed_tmax(const int64_t* tt, int n, int64_t t_max, int64_t D, int64_t K,
                          std::vector<int64_t>& S, std::vector<int32_t>& q, DpResult& out) {
  const int ld = n + 1;
  S[0] = 0;
  for (int i = 1; i <= n; ++i) {
    const int64_t* row = tt + (int64_t)i * ld;
    int64_t best = kInf;
    int32_t arg = 0;
    for (int k = 1; k <= i; ++k) {
      const int64_t t = row[k];
      const int64_t prev = S[i - k];
      const int64_t v = (t <= t_max) ? prev + t : kInf;
      if (v < best) { best = v; arg = k; }   // strict: the smallest k wins ties (A-12)
    }
    S[i] = best;
    q[i] = arg;
  }
  if (S[n] >= kInf) { out.feasible = false; return; }
  out.feasible = true;
  out.lengths.clear();
  for (int i = n; i > 0; i -= q[i]) out.lengths.push_back(q[i]);
  std::reverse(out.lengths.begin(), out.lengths.end());
  int64_t sum = 0, mx = 0;
  int c = 0;
  for (int32_t l : out.lengths) {
    const int64_t t = tt[(int64_t)(c + l) * ld + l];
    sum += t;
    mx = std::max(mx, t);
    c += l;
  }
  out.T = D * sum + (K - 1) * mx;
  out.mx = mx;
}

}  // namespace

extern "C" tp_status tp_plan(int32_t n_layer, int32_t hidden, int32_t seq_len, int32_t n_stages,
                             const tp_cost_table* cost, int32_t n_micro, int64_t eps_ticks,
                             tp_slicing* out) {
  TP_CHECK_ARG(cost && out, "tp_plan: null cost table or output");
  TP_CHECK_ARG(n_stages >= 1, "tp_plan: n_stages must be >= 1 (got %d)", n_stages);
  TP_CHECK_ARG(n_layer >= 1 && n_layer >= n_stages,
               "tp_plan: n_layer (%d) must be a positive multiple of n_stages (%d)", n_layer, n_stages);
  TP_CHECK_ARG(hidden > 0, "tp_plan: hidden must be > 0");
  TP_CHECK_ARG(n_micro >= 1, "tp_plan: n_micro must be >= 1");
  TP_CHECK_ARG(eps_ticks >= 0, "tp_plan: eps_ticks must be >= 0");
  const int g = cost->granularity;
  TP_CHECK_ARG(g >= 1 && seq_len >= g && seq_len % g == 0,
               "tp_plan: seq_len (%d) must be a positive multiple of granularity (%d)", seq_len, g);
  const int n = seq_len / g;
  TP_CHECK_ARG(cost->n_units == n, "tp_plan: cost->n_units (%d) != seq_len/g (%d)", cost->n_units, n);
  TP_CHECK_ARG(n <= 65536, "tp_plan: n_units %d too large", n);
  TP_CHECK_ARG(cost->ticks != nullptr, "tp_plan: null ticks");
  TP_CHECK_ARG(out->lengths != nullptr && out->capacity >= n,
               "tp_plan: out->lengths capacity %d < n_units %d", out->capacity, n);

  const int ld = n + 1;
  std::vector<int64_t> tt((size_t)ld * ld, kInf);
  std::vector<int64_t> vals;
  vals.reserve((size_t)n * (n + 1) / 2);
  for (int l = 1; l <= n; ++l)
    for (int c = 0; c + l <= n; ++c) {
      const int64_t v = cost->ticks[(int64_t)(l - 1) * ld + c];
      if (v <= 0)
        return tp::fail(TP_EINVAL, "tp_plan: non-positive tick %lld at l=%d c=%d", (long long)v, l, c);
      tt[(int64_t)(l + c) * ld + l] = v;
      vals.push_back(v);
    }
  std::sort(vals.begin(), vals.end());
  vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
  std::vector<int64_t> cand;
  for (int64_t v : vals)
    if (cand.empty() || eps_ticks == 0 || v >= cand.back() + eps_ticks) cand.push_back(v);
  if (cand.back() != vals.back()) cand.push_back(vals.back());  // A-13b

  int nthreads = (int)std::thread::hardware_concurrency();
  if (const char* e = std::getenv("TP_PLAN_THREADS")) nthreads = std::atoi(e);
  nthreads = std::max(1, std::min(nthreads, 64));
  // Small problems: threads cost more than they save.
  if ((int64_t)n * n < 4096) nthreads = 1;

  const int64_t D = n_micro, K = n_stages;
  bool have = false;
  DpResult best;
  std::vector<DpResult> res(nthreads);
  std::vector<std::vector<int64_t>> Ss(nthreads, std::vector<int64_t>(n + 1));
  std::vector<std::vector<int32_t>> qs(nthreads, std::vector<int32_t>(n + 1));

  size_t pos = 0;
  bool stop = false;
  while (pos < cand.size() && !stop) {
    if (have && (D + K - 1) * cand[pos] >= best.T) break;
    const int batch = (int)std::min<size_t>(nthreads, cand.size() - pos);
    if (batch == 1) {
      dp_fixed_tmax(tt.data(), n, cand[pos], D, K, Ss[0], qs[0], res[0]);
    } else {
      std::vector<std::thread> pool;
      for (int w = 1; w < batch; ++w)
        pool.emplace_back([&, w] { dp_fixed_tmax(tt.data(), n, cand[pos + w], D, K, Ss[w], qs[w], res[w]); });
      dp_fixed_tmax(tt.data(), n, cand[pos], D, K, Ss[0], qs[0], res[0]);
      for (auto& th : pool) th.join();
    }
    // merge in ascending candidate order: identical to the sequential loop
    for (int w = 0; w < batch; ++w) {
      if (have && (D + K - 1) * cand[pos + w] >= best.T) { stop = true; break; }
      if (!res[w].feasible) continue;
      if (!have || res[w].T < best.T) { best = res[w]; have = true; }
    }
    pos += batch;
  }
  if (!have) return tp::fail(TP_EINFEASIBLE, "tp_plan: no feasible slicing scheme");

  out->n_slices = (int32_t)best.lengths.size();
  for (size_t i = 0; i < best.lengths.size(); ++i) out->lengths[i] = best.lengths[i] * g;
  out->t_max_ticks = best.mx;
  out->predicted_ticks = best.T;
  if (out->batch_slice <= 0) out->batch_slice = 1;
  return TP_OK;
}

// ---------------------------------------------------------------- tp_plan_joint
// PAPER.md:362-364 with reading A-20b: per t_max candidate, Algorithm 1 for every
// batch-slice size, a 1-D knapsack over the batch, the exact plan objective; see tp.h.
extern "C" tp_status tp_plan_joint(int32_t n_layer, int32_t hidden, int32_t seq_len, int32_t n_stages, int32_t n_b,
                                   const int32_t* b_values, const tp_cost_table* const* costs, int32_t batch,
                                   int64_t eps_ticks, tp_batch_plan* out) {
  TP_CHECK_ARG(out && b_values && costs, "tp_plan_joint: null argument");
  TP_CHECK_ARG(n_b >= 1, "tp_plan_joint: n_b must be >= 1");
  TP_CHECK_ARG(batch >= 1, "tp_plan_joint: batch must be >= 1");
  TP_CHECK_ARG(n_stages >= 1 && n_layer >= 1 && n_layer >= n_stages && hidden > 0,
               "tp_plan_joint: bad model shape (n_layer %d, n_stages %d, hidden %d)", n_layer, n_stages, hidden);
  TP_CHECK_ARG(eps_ticks >= 0, "tp_plan_joint: eps_ticks must be >= 0");
  TP_CHECK_ARG(costs[0] != nullptr, "tp_plan_joint: null cost table 0");
  const int g = costs[0]->granularity;
  TP_CHECK_ARG(g >= 1 && seq_len >= g && seq_len % g == 0,
               "tp_plan_joint: seq_len (%d) must be a positive multiple of granularity (%d)", seq_len, g);
  const int n = seq_len / g, ld = n + 1;
  TP_CHECK_ARG(n <= 65536, "tp_plan_joint: n_units %d too large", n);
  TP_CHECK_ARG(out->batch_slice && out->n_slices && out->lengths && out->capacity_groups >= batch &&
                   (int64_t)out->capacity_lengths >= (int64_t)batch * n,
               "tp_plan_joint: output capacities too small (need %d groups, %lld lengths)", batch,
               (long long)batch * n);
  // per-b end-indexed tables (tt[i][k] = t(k, i-k)) and the union of their values
  std::vector<std::vector<int64_t>> tts(n_b);
  std::vector<int64_t> vals;
  for (int ib = 0; ib < n_b; ++ib) {
    const tp_cost_table* cost = costs[ib];
    TP_CHECK_ARG(cost && cost->ticks, "tp_plan_joint: null cost table %d", ib);
    TP_CHECK_ARG(cost->granularity == g && cost->n_units == n, "tp_plan_joint: table %d shape mismatch", ib);
    TP_CHECK_ARG(b_values[ib] >= 1, "tp_plan_joint: b_values[%d] = %d", ib, b_values[ib]);
    for (int jb = 0; jb < ib; ++jb)
      TP_CHECK_ARG(b_values[jb] != b_values[ib], "tp_plan_joint: duplicate batch-slice size %d", b_values[ib]);
    tts[ib].assign((size_t)ld * ld, kInf);
    for (int l = 1; l <= n; ++l)
      for (int c = 0; c + l <= n; ++c) {
        const int64_t v = cost->ticks[(int64_t)(l - 1) * ld + c];
        if (v <= 0)
          return tp::fail(TP_EINVAL, "tp_plan_joint: non-positive tick in table %d at l=%d c=%d", ib, l, c);
        tts[ib][(int64_t)(l + c) * ld + l] = v;
        vals.push_back(v);
      }
  }
  std::sort(vals.begin(), vals.end());
  vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
  std::vector<int64_t> cand;
  for (int64_t v : vals)
    if (cand.empty() || eps_ticks == 0 || v >= cand.back() + eps_ticks) cand.push_back(v);
  if (cand.back() != vals.back()) cand.push_back(vals.back());  // A-13b
  // b values in ascending order (knapsack tie-break: the smallest b wins)
  std::vector<int> order(n_b);
  for (int i = 0; i < n_b; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int x, int y) { return b_values[x] < b_values[y]; });

  const int64_t K = n_stages;
  std::vector<int64_t> S(n + 1);
  std::vector<int32_t> q(n + 1);
  std::vector<DpResult> res(n_b);
  std::vector<int64_t> C(batch + 1);
  std::vector<int32_t> choice(batch + 1);
  bool have = false;
  int64_t best_T = 0, best_mx = 0;
  std::vector<int32_t> best_b;
  std::vector<std::vector<int32_t>> best_len;
  for (int64_t tau : cand) {
    if (have && K * tau >= best_T) break;
    for (int ib = 0; ib < n_b; ++ib) dp_fixed_tmax(tts[ib].data(), n, tau, 1, K, S, q, res[ib]);
    C[0] = 0;
    for (int m = 1; m <= batch; ++m) {
      C[m] = kInf;
      choice[m] = -1;
      for (int ib : order) {
        const int b = b_values[ib];
        if (b > m || !res[ib].feasible || C[m - b] >= kInf) continue;
        const int64_t sum = res[ib].T - (K - 1) * res[ib].mx;  // Algorithm 1's S*: sum of the slice costs
        const int64_t v = C[m - b] + sum;
        if (v < C[m]) { C[m] = v; choice[m] = ib; }
      }
    }
    if (C[batch] >= kInf) continue;
    int64_t mx = 0;
    std::vector<int32_t> bs;
    std::vector<std::vector<int32_t>> lens;
    for (int m = batch; m > 0; m -= b_values[choice[m]]) {
      const int ib = choice[m];
      bs.push_back(b_values[ib]);
      lens.push_back(res[ib].lengths);
      mx = std::max(mx, res[ib].mx);
    }
    const int64_t T = C[batch] + (K - 1) * mx;
    if (!have || T < best_T) {
      have = true;
      best_T = T;
      best_mx = mx;
      best_b = bs;
      best_len = lens;
    }
  }
  if (!have) return tp::fail(TP_EINFEASIBLE, "tp_plan_joint: batch %d is not a sum of the given batch-slice sizes", batch);
  out->n_groups = (int32_t)best_b.size();
  int32_t pos = 0;
  for (size_t d = 0; d < best_b.size(); ++d) {
    out->batch_slice[d] = best_b[d];
    out->n_slices[d] = (int32_t)best_len[d].size();
    for (int32_t l : best_len[d]) out->lengths[pos++] = l * g;
  }
  out->t_max_ticks = best_mx;
  out->predicted_ticks = best_T;
  return TP_OK;
}
