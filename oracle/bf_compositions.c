/* TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Brute force over ALL 2^(n-1) compositions of n units — the definition of the optimal slicing
 * scheme of TeraPipe §3.3 (Eq. 5), generalised to D jobs per slice index
 * (reading A-20):  T = D * sum_i t_i + (K-1) * max_i t_i,  t_i = t(l_i, c_i).
 * Tie-break: lexicographic minimum of (T, max t_i, reversed lengths) — identical to
 * oracle/plan.py:brute_force. Written for n = 32 (the tiny config, BASELINE.json:7, at g = 1),
 * where Python is too slow. No pruning: every composition is scored.
 *
 * Input  (stdin, text):  n K D   then n*(n+1) int64 ticks, row-major t[l-1][c].
 * Output (stdout, text): T m M l_1 ... l_M
 * Build: gcc -O2 -fopenmp -o oracle/bf_compositions oracle/bf_compositions.c   (done by build()).
 *
 * Parity status: pinned — agrees with oracle/plan.py:brute_force on random instances with
 * n <= 14 (tests/test_oracle_plan.py::test_c_brute_force_matches_python).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXN 40

static int n, K, D;
static int64_t *tab; /* [n][n+1] */

typedef struct {
  int64_t T, m;
  int M;
  int len[MAXN];
} best_t;

/* is reversed(a) lexicographically smaller than reversed(b)? */
static int rev_less(const int *a, int Ma, const int *b, int Mb) {
  int i = Ma - 1, j = Mb - 1;
  while (i >= 0 && j >= 0) {
    if (a[i] != b[j]) return a[i] < b[j];
    --i; --j;
  }
  return i < 0 && j >= 0; /* a is a proper prefix (cannot happen for compositions of n) */
}

static void consider(best_t *b, int64_t sum, int64_t mx, const int *len, int M) {
  int64_t T = (int64_t)D * sum + (int64_t)(K - 1) * mx;
  if (b->M == 0 || T < b->T || (T == b->T && (mx < b->m || (mx == b->m && rev_less(len, M, b->len, b->M))))) {
    b->T = T; b->m = mx; b->M = M;
    memcpy(b->len, len, sizeof(int) * M);
  }
}

/* positions p = start+1 .. n: decide whether slice [start, p) closes at p. */
static void dfs(best_t *b, int start, int p, int64_t sum, int64_t mx, int *len, int M) {
  if (p == n) {
    int l = n - start;
    int64_t t = tab[(int64_t)(l - 1) * (n + 1) + start];
    len[M] = l;
    consider(b, sum + t, t > mx ? t : mx, len, M + 1);
    return;
  }
  /* cut at p */
  {
    int l = p - start;
    int64_t t = tab[(int64_t)(l - 1) * (n + 1) + start];
    len[M] = l;
    dfs(b, p, p + 1, sum + t, t > mx ? t : mx, len, M + 1);
  }
  /* no cut at p */
  dfs(b, start, p + 1, sum, mx, len, M);
}

int main(void) {
  if (scanf("%d %d %d", &n, &K, &D) != 3 || n < 1 || n > MAXN || K < 1 || D < 1) {
    fprintf(stderr, "bad header\n");
    return 2;
  }
  tab = (int64_t *)malloc(sizeof(int64_t) * n * (n + 1));
  for (int i = 0; i < n * (n + 1); ++i) {
    long long v;
    if (scanf("%lld", &v) != 1) { fprintf(stderr, "short table\n"); return 2; }
    tab[i] = v;
  }
  /* split the first P cut decisions into 2^P independent tasks */
  int P = n - 1 < 8 ? n - 1 : 8;
  int ntask = 1 << P;
  best_t *res = (best_t *)calloc(ntask, sizeof(best_t));
#pragma omp parallel for schedule(dynamic, 1)
  for (int task = 0; task < ntask; ++task) {
    int len[MAXN];
    int M = 0, start = 0;
    int64_t sum = 0, mx = 0;
    for (int p = 1; p <= P; ++p) {
      if ((task >> (p - 1)) & 1) { /* cut at p */
        int l = p - start;
        int64_t t = tab[(int64_t)(l - 1) * (n + 1) + start];
        len[M++] = l; sum += t; if (t > mx) mx = t; start = p;
      }
    }
    dfs(&res[task], start, P + 1, sum, mx, len, M);
  }
  /* merge with the same tie-break */
  best_t b;
  memset(&b, 0, sizeof b);
  for (int task = 0; task < ntask; ++task) {
    best_t *r = &res[task];
    if (!r->M) continue;
    if (b.M == 0 || r->T < b.T || (r->T == b.T && (r->m < b.m || (r->m == b.m && rev_less(r->len, r->M, b.len, b.M)))))
      b = *r;
  }
  printf("%lld %lld %d", (long long)b.T, (long long)b.m, b.M);
  for (int i = 0; i < b.M; ++i) printf(" %d", b.len[i]);
  printf("\n");
  free(res); free(tab);
  return 0;
}
