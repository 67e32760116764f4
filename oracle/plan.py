"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The slicing planner of TeraPipe §3.3, written out step by step, plus the
brute force that defines its optimum and the schedule simulators behind Eq. 5.

Costs are int64 ticks (reading A-15): t(l, c) is the fwd+bwd time of a slice of l units with
c units of context, given as a table `t[l-1][c]` of shape [n][n+1]
(units of the granularity g; only l + c <= n is used; used entries must be > 0).
With integer costs every sum is exact, so "DP == brute force" holds exactly, not within a
tolerance.

Objective (Eq. 5, generalised by reading A-20 to D jobs per slice index):
    T(l_1..l_M) = D * sum_i t_i + (K - 1) * max_i t_i,   t_i = t(l_i, sum_{j<i} l_j).
D = 1 is exactly the paper's Eq. 5.

Joint batch x token plan (reading A-20b): joint_optimize == joint_brute_force on
random integer instances (tests/test_oracle_plan.py).

Parity status: pinned (tests/test_oracle_plan.py) — optimize() == brute_force() exactly on
random integer instances; SPEC.md:146-147 worked examples (T = 4, T = 10); closed form ==
flow-shop simulation (SPEC.md:253-264 examples and random vectors); epsilon gap <= K*eps
(PAPER.md:290); pruning soundness.

Schedules (A-21, A-27): gpipe_oplists / one_f_one_b_oplists are the per-stage op lists
(GPipe order of PAPER.md:373; 1F1B at group granularity) and oplist_replay replays any lists with
the pipeline's data dependencies. Pinned: replay of the GPipe lists == oplist_makespan (the
two-wave replay, itself == the A-19 closed form); 1F1B with one-job groups and uniform durations
== the textbook (D + K - 1)(t_f + t_b); in-flight groups == min(D, K - k); deadlock detection.
"""
from __future__ import annotations

import itertools
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

INF = None  # marker for "no feasible scheme"


def slice_costs(t: np.ndarray, lengths: Sequence[int]) -> List[int]:
    """t_i = t_fwd(l_i, sum_{j<i} l_j)."""
    out, c = [], 0
    for l in lengths:
        out.append(int(t[l - 1, c]))
        c += l
    return out


def objective(t: np.ndarray, lengths: Sequence[int], K: int, D: int = 1) -> int:
    """Eq. 5 with D jobs per slice index (A-20)."""
    ts = slice_costs(t, lengths)
    return D * sum(ts) + (K - 1) * max(ts)


def dp_fixed_tmax(t: np.ndarray, n: int, t_max: int) -> Optional[Tuple[int, List[int]]]:
    """Algorithm 1: S*(0) = 0; for i = 1..n,
    S*(i) = min_{1<=k<=i} { S*(i-k) + t(k, i-k) | t(k, i-k) <= t_max } (Eq. 8),
    q_i = argmin (reading A-11: r_{i-k} is S*(i-k); A-12: the smallest k wins ties),
    then backtrack l.prepend(q_i), i -= q_i. Returns (S*(n), [l_1..l_M]) or None if infeasible."""
    S: List[Optional[int]] = [None] * (n + 1)
    q = [0] * (n + 1)
    S[0] = 0
    for i in range(1, n + 1):
        best, arg = None, 0
        for k in range(1, i + 1):
            if S[i - k] is None:
                continue
            tk = int(t[k - 1, i - k])
            if tk > t_max:
                continue
            v = S[i - k] + tk
            if best is None or v < best:
                best, arg = v, k
        S[i], q[i] = best, arg
    if S[n] is None:
        return None
    lengths: List[int] = []
    i = n
    while i > 0:
        lengths.insert(0, q[i])
        i -= q[i]
    return S[n], lengths


def candidates(t: np.ndarray, n: int, eps: int = 0) -> List[int]:
    """All distinct t(k, j), k >= 1, k + j <= n, ascending, thinned so each kept
    value is >= the last kept one + eps (reading A-13: keep the first of a cluster)."""
    vals = sorted({int(t[k - 1, j]) for k in range(1, n + 1) for j in range(0, n - k + 1)})
    if eps <= 0:
        return vals
    out: List[int] = []
    for v in vals:
        if not out or v >= out[-1] + eps:
            out.append(v)
    # reading A-13b: the largest value is always evaluated, so thinning can never make every
    # evaluated t_max infeasible (at t_max = max t, the all-ones scheme is feasible).
    if out[-1] != vals[-1]:
        out.append(vals[-1])
    return out


def optimize(t: np.ndarray, n: int, K: int, D: int = 1, eps: int = 0,
             prune: bool = True) -> Tuple[int, int, List[int]]:
    """Enumerate t_max ascending (Eq. 6-7), run Algorithm 1 for each, keep the
    scheme with the smallest T (replace only on strict improvement, A-12); stop when
    (D + K - 1) * t_max >= best T (PAPER.md:290 'K * t_max greater than the current best',
    generalised to D jobs and to >=, reading A-14). Returns (T, t_max_of_scheme, lengths)."""
    best: Optional[Tuple[int, int, List[int]]] = None
    for c in candidates(t, n, eps):
        if prune and best is not None and (D + K - 1) * c >= best[0]:
            break
        r = dp_fixed_tmax(t, n, c)
        if r is None:
            continue
        _, lengths = r
        ts = slice_costs(t, lengths)
        T = D * sum(ts) + (K - 1) * max(ts)
        if best is None or T < best[0]:
            best = (T, max(ts), lengths)
    if best is None:
        raise ValueError("infeasible: no slicing scheme")
    return best


def compositions(n: int) -> Iterable[Tuple[int, ...]]:
    """All 2^(n-1) compositions of n (ordered positive parts)."""
    for cuts in itertools.product((0, 1), repeat=n - 1):
        parts, last = [], 0
        for i, cut in enumerate(cuts, start=1):
            if cut:
                parts.append(i - last)
                last = i
        parts.append(n - last)
        yield tuple(parts)


def brute_force(t: np.ndarray, n: int, K: int, D: int = 1) -> Tuple[int, int, List[int]]:
    """The definition of the optimum: score every composition of n with Eq. 5 and take the
    lexicographic minimum of (T, max t_i, reversed lengths) — the same deterministic tie-break
    Algorithm 1 with smallest-k backpointers produces (reading A-12)."""
    if n > 22:
        raise ValueError("too big for the Python brute force (use oracle/bf_compositions.c)")
    best = None
    for comp in compositions(n):
        ts = slice_costs(t, comp)
        key = (D * sum(ts) + (K - 1) * max(ts), max(ts), tuple(reversed(comp)))
        if best is None or key < best:
            best = key
    T, m, rev = best
    return T, m, list(reversed(rev))


# ---------------------------------------------------------------- joint batch x token plan
# PAPER.md:362-364 (§3.4): run the DP for every batch-slice size b, then choose b_1 + .. + b_D = B
# (a 1-D knapsack). Reading A-20b: all D groups' jobs are pipelined back to back, so the objective
# of a batch plan {(b_d, l^d)} is  sum_d sum_i t_{b_d}(l^d_i, c^d_i) + (K - 1) * max over all jobs,
# i.e. the fill/drain bubble is paid once for the whole batch (A-20 with heterogeneous groups; a
# uniform plan [(b, l)] * D is exactly tp_plan's D * sum + (K - 1) * max).

def joint_objective(tables, plan: Sequence[Tuple[int, Sequence[int]]], K: int) -> int:
    ts = [x for b, lengths in plan for x in slice_costs(tables[b], lengths)]
    return sum(ts) + (K - 1) * max(ts)


def joint_candidates(tables, n: int, eps: int = 0) -> List[int]:
    """Union over b of the per-table candidates, thinned as in candidates()."""
    vals = sorted({v for t in tables.values() for v in candidates(t, n, 0)})
    if eps <= 0:
        return vals
    out: List[int] = []
    for v in vals:
        if not out or v >= out[-1] + eps:
            out.append(v)
    if out[-1] != vals[-1]:
        out.append(vals[-1])
    return out


def knapsack(costs, B: int):
    """C(0) = 0, C(m) = min_{b <= m, costs[b] finite} C(m - b) + costs[b] (PAPER.md:364 '1D
    knapsack'); ties keep the smallest b. Returns (C(B), [b_1, b_2, ..]) by backtracking from B, or
    None if B cannot be composed."""
    C: List[Optional[int]] = [None] * (B + 1)
    choice = [0] * (B + 1)
    C[0] = 0
    for m in range(1, B + 1):
        for b in sorted(costs):
            if b > m or costs[b] is None or C[m - b] is None:
                continue
            v = C[m - b] + costs[b]
            if C[m] is None or v < C[m]:
                C[m], choice[m] = v, b
    if C[B] is None:
        return None
    parts, m = [], B
    while m > 0:
        parts.append(choice[m])
        m -= choice[m]
    return C[B], parts


def joint_optimize(tables, n: int, B: int, K: int, eps: int = 0):
    """For each t_max candidate (ascending): Algorithm 1 per batch-slice size b (the smallest sum
    S*_b with every slice <= t_max), the knapsack over b, and the exact objective of the resulting
    plan; keep strict improvements; stop once K * t_max >= best (any plan whose largest job is
    >= t_max costs at least max + (K - 1) * max). Returns (T, [(b_d, lengths_d), ..])."""
    best = None
    for tau in joint_candidates(tables, n, eps):
        if best is not None and K * tau >= best[0]:
            break
        per_b, schemes = {}, {}
        for b, t in tables.items():
            r = dp_fixed_tmax(t, n, tau)
            per_b[b] = None if r is None else r[0]
            if r is not None:
                schemes[b] = r[1]
        ks = knapsack(per_b, B)
        if ks is None:
            continue
        plan = [(b, schemes[b]) for b in ks[1]]
        T = joint_objective(tables, plan, K)
        if best is None or T < best[0]:
            best = (T, plan)
    if best is None:
        raise ValueError("infeasible: no batch plan")
    return best


def partitions(B: int, parts: Sequence[int], max_part: Optional[int] = None) -> Iterable[Tuple[int, ...]]:
    """Non-increasing partitions of B into the allowed part sizes."""
    if B == 0:
        yield ()
        return
    for p in sorted(parts, reverse=True):
        if p <= B and (max_part is None or p <= max_part):
            for rest in partitions(B - p, parts, p):
                yield (p,) + rest


def joint_brute_force(tables, n: int, B: int, K: int) -> int:
    """The definition of the joint optimum: every partition of B into the available batch-slice
    sizes, every slicing of every group, scored with the A-20b objective. Returns the minimum T."""
    comps = list(compositions(n))
    best = None
    for parts in partitions(B, list(tables)):
        for choice in itertools.product(comps, repeat=len(parts)):
            T = joint_objective(tables, list(zip(parts, choice)), K)
            if best is None or T < best:
                best = T
    return best


def uniform_schemes(n: int) -> List[List[int]]:
    """[n/d] * d for every divisor d of n (SPEC.md:165 'DP dominates uniform')."""
    return [[n // d] * d for d in range(1, n + 1) if n % d == 0]


# ---------------------------------------------------------------- schedule models
def closed_form(ts: Sequence[float], K: int, D: int = 1):
    """Eq. 5: sum_i t_i + (K-1) max_j t_j, for D repetitions of the slice list."""
    return D * sum(ts) + (K - 1) * max(ts)


def flowshop_makespan(durations: Sequence[float], K: int):
    """Pipeline semantics of Fig. 2(c)/Fig. 5: job i on stage k starts when job i-1 left stage k
    and job i left stage k-1: start(i,k) = max(end(i-1,k), end(i,k-1)), end = start + t_i."""
    M = len(durations)
    end = [[0.0] * (K + 1) for _ in range(M + 1)]
    for i in range(1, M + 1):
        for k in range(1, K + 1):
            end[i][k] = max(end[i - 1][k], end[i][k - 1]) + durations[i - 1]
    return end[M][K]


def oplist_makespan(tf: Sequence[Sequence[float]], tb: Sequence[Sequence[float]],
                    comm: float = 0.0) -> float:
    """Replays the runtime's per-stage op lists (GPipe order, reading A-21): stage k runs
    F(j) for j = 0..J-1 then B(j) for j = J-1..0, each op waiting for its cross-stage input
    (F(j) on k-1, resp. B(j) on k+1; B(j) on the last stage waits for its own F(j)) plus `comm`.
    tf[k][j], tb[k][j]: per-stage, per-job durations. Returns the makespan."""
    K, J = len(tf), len(tf[0])
    fend = [[0.0] * J for _ in range(K)]
    bend = [[0.0] * J for _ in range(K)]
    free = [0.0] * K
    # forward wave: stage-major is a valid topological order for a DAG with edges k-1 -> k
    for k in range(K):
        for j in range(J):
            dep = fend[k - 1][j] + comm if k > 0 else 0.0
            st = max(free[k], dep)
            fend[k][j] = st + tf[k][j]
            free[k] = fend[k][j]
    for k in reversed(range(K)):
        for j in reversed(range(J)):
            dep = bend[k + 1][j] + comm if k < K - 1 else fend[k][j]
            st = max(free[k], dep)
            bend[k][j] = st + tb[k][j]
            free[k] = bend[k][j]
    return max(free)


def gpipe_oplists(groups: Sequence[int], K: int) -> List[List[Tuple[str, int]]]:
    """GPipe order (reading A-21): every stage runs F of all jobs in order, then B in exact reverse.
    groups[d] = number of token-slice jobs of group d; jobs are numbered group-major."""
    J = sum(groups)
    ops = [("F", j) for j in range(J)] + [("B", j) for j in reversed(range(J))]
    return [list(ops) for _ in range(K)]


def one_f_one_b_oplists(groups: Sequence[int], K: int) -> List[List[Tuple[str, int]]]:
    """1F1B at sequence (group) granularity (north star "1F1B-style", DESIGN.md
    A-21: inside one group the backward of its last slice needs every forward, so the unit that
    interleaves is the group): stage k first runs the forwards of w_k = min(D, K - k) groups (the
    warm-up), then alternates the backward of its oldest in-flight group (slices in reverse) with
    the forward of the next group, then drains the remaining backwards. Each stage holds at most
    w_k groups' activations (the memory bound the schedule exists for)."""
    D = len(groups)
    first = [sum(groups[:d]) for d in range(D)]
    F = lambda d: [("F", first[d] + i) for i in range(groups[d])]
    Bk = lambda d: [("B", first[d] + i) for i in reversed(range(groups[d]))]
    out = []
    for k in range(K):
        w = min(D, K - k)
        ops: List[Tuple[str, int]] = []
        for d in range(w):
            ops += F(d)
        for d in range(D):
            ops += Bk(d)
            if d + w < D:
                ops += F(d + w)
        out.append(ops)
    return out


def oplist_replay(oplists: Sequence[Sequence[Tuple[str, int]]], tf: Sequence[Sequence[float]],
                  tb: Sequence[Sequence[float]], comm: float = 0.0) -> float:
    """Replays arbitrary per-stage op lists with the pipeline's data dependencies: F(j) on stage k
    starts after F(j) on k-1 (+ comm), B(j) on stage k after B(j) on k+1 (+ comm), B(j) on the last
    stage after its own F(j); each stage executes its list in order, one op at a time. Returns the
    makespan; raises ValueError on a deadlocking order. tf[k][j], tb[k][j]: per-stage durations."""
    K = len(oplists)
    end: Dict[Tuple[str, int, int], float] = {}
    pos = [0] * K
    free = [0.0] * K
    remaining = sum(len(o) for o in oplists)
    while remaining:
        progressed = False
        for k in range(K):
            while pos[k] < len(oplists[k]):
                kind, j = oplists[k][pos[k]]
                if kind == "F":
                    dep = ("F", k - 1, j) if k > 0 else None
                    extra = comm if k > 0 else 0.0
                else:
                    dep = ("B", k + 1, j) if k < K - 1 else ("F", k, j)
                    extra = comm if k < K - 1 else 0.0
                if dep is not None and dep not in end:
                    break
                ready = end[dep] + extra if dep is not None else 0.0
                st = max(free[k], ready)
                free[k] = st + (tf[k][j] if kind == "F" else tb[k][j])
                end[(kind, k, j)] = free[k]
                pos[k] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            raise ValueError("op lists deadlock")
    return max(free)


def max_inflight_groups(oplists: Sequence[Sequence[Tuple[str, int]]], groups: Sequence[int]) -> List[int]:
    """Per stage: the largest number of groups whose forward has started and whose backward has not
    finished (the activation-memory footprint of the schedule, in groups)."""
    gid = [d for d, m in enumerate(groups) for _ in range(m)]
    out = []
    for ops in oplists:
        started, done_b = set(), {}
        live = peak = 0
        for kind, j in ops:
            d = gid[j]
            if kind == "F" and d not in started:
                started.add(d)
                live += 1
            if kind == "B":
                done_b[d] = done_b.get(d, 0) + 1
                if done_b[d] == groups[d]:
                    live -= 1
            peak = max(peak, live)
        out.append(peak)
    return out
