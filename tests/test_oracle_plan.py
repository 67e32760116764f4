"""Pins for oracle/plan.py (CPU only).

  * SPEC.md:135-147 worked examples (T = 4 and T = 10, dp_fixed_tmax examples);
  * SPEC.md:253-264 schedule examples ([1,3],K=2 -> 7; [1,3,1],K=3 -> 11);
  * Algorithm 1 + enumeration == brute force over all compositions (the definition), exactly,
    on random integer instances including heavy ties (BASELINE.json:5 invariant (b));
  * closed form (Eq. 5) == flow-shop simulation (invariant (c)) and the fwd+bwd GPipe-order
    op-list replay == D*sum(tf+tb) + (K-1)(max tf + max tb) (reading A-19);
  * pruning soundness and the epsilon gap <= K*eps of PAPER.md:290.
"""
import subprocess
import os

import numpy as np
import pytest

from oracle import plan as op
from synth import random_int_table, gpu_like_table

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BF = os.path.join(ROOT, "oracle", "bf_compositions")


def table_from(fn, n):
    t = np.zeros((n, n + 1), dtype=np.int64)
    for l in range(1, n + 1):
        for c in range(0, n - l + 1):
            t[l - 1, c] = fn(l, c)
    return t


def test_spec_examples():
    t = table_from(lambda l, c: l, 3)
    assert op.dp_fixed_tmax(t, 3, 1) == (3, [1, 1, 1])
    T, m, lens = op.optimize(t, 3, K=2)
    assert (T, lens) == (4, [1, 1, 1])
    t = table_from(lambda l, c: 1 + l, 3)
    T, m, lens = op.optimize(t, 3, K=3)
    assert (T, lens) == (10, [1, 1, 1])
    const = table_from(lambda l, c: 5, 6)
    assert op.dp_fixed_tmax(const, 6, 5) == (5, [6])
    assert op.dp_fixed_tmax(const, 6, 4) is None
    assert op.optimize(const, 6, K=1) == (5, 5, [6])


def test_schedule_examples_and_closed_form():
    assert op.flowshop_makespan([1, 3], 2) == 7
    assert op.closed_form([1, 3], 2) == 7
    assert op.closed_form([1, 3, 1], 3) == 11 == op.flowshop_makespan([1, 3, 1], 3)
    assert op.flowshop_makespan([4.5], 5) == 5 * 4.5
    rng = np.random.default_rng(0)
    for _ in range(1000):
        M, K, D = rng.integers(1, 12), rng.integers(1, 9), rng.integers(1, 4)
        ts = list(rng.integers(1, 100, size=M))
        assert op.flowshop_makespan(ts * D, K) == op.closed_form(ts, K, D)


def test_oplist_replay_matches_two_wave_closed_form():
    rng = np.random.default_rng(1)
    for _ in range(300):
        M, K, D = rng.integers(1, 7), rng.integers(1, 6), rng.integers(1, 4)
        tf = list(rng.integers(1, 50, size=M)) * D
        tb = list(rng.integers(1, 90, size=M)) * D
        ms = op.oplist_makespan([tf] * K, [tb] * K)
        assert ms == sum(tf) + sum(tb) + (K - 1) * (max(tf) + max(tb))
        # with t_b proportional to t_f it reduces to Eq. 5 on t_f + t_b
        tb2 = [2 * x for x in tf]
        assert op.oplist_makespan([tf] * K, [tb2] * K) == op.closed_form(
            [a + b for a, b in zip(tf, tb2)], K)


@pytest.mark.parametrize("seed", range(8))
def test_dp_equals_brute_force_random(seed):
    rng = np.random.default_rng(100 + seed)
    for trial in range(30):
        n = int(rng.integers(1, 12))
        K = int(rng.integers(1, 5))
        D = int(rng.choice([1, 2, 8]))
        hi = int(rng.choice([3, 10, 1000]))
        t = random_int_table(n, rng, 1, hi)
        bf = op.brute_force(t, n, K, D)
        dp = op.optimize(t, n, K, D)
        assert dp == bf, (n, K, D, t, dp, bf)
        assert op.optimize(t, n, K, D, prune=False)[0] == bf[0]              # pruning soundness


def test_dp_dominates_uniform_and_eps_gap():
    rng = np.random.default_rng(7)
    for _ in range(20):
        n = int(rng.integers(8, 33))
        K = int(rng.integers(1, 9))
        t = gpu_like_table(n, rng)
        T0, _, lens = op.optimize(t, n, K)
        assert sum(lens) == n and min(lens) >= 1
        for u in op.uniform_schemes(n):
            assert T0 <= op.objective(t, u, K)
        for eps in (5_000, 10_000, 50_000):                                   # ticks (ns)
            Te, _, _ = op.optimize(t, n, K, eps=eps)
            assert T0 <= Te <= T0 + K * eps


def _c_brute(t, n, K, D):
    inp = f"{n} {K} {D}\n" + " ".join(str(int(v)) for v in t.reshape(-1)) + "\n"
    r = subprocess.run([BF], input=inp, capture_output=True, text=True, check=True, timeout=600)
    v = [int(x) for x in r.stdout.split()]
    return v[0], v[1], v[3:3 + v[2]]


@pytest.fixture(scope="module")
def c_brute():
    if not os.path.exists(BF):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-o", BF, BF + ".c"], check=True)
    return _c_brute


def test_c_brute_force_matches_python(c_brute):
    rng = np.random.default_rng(5)
    for _ in range(40):
        n = int(rng.integers(1, 14))
        K, D = int(rng.integers(1, 5)), int(rng.choice([1, 2, 8]))
        t = random_int_table(n, rng, 1, int(rng.choice([3, 50])))
        assert c_brute(t, n, K, D) == op.brute_force(t, n, K, D)


@pytest.mark.slow
def test_tiny_config_dp_equals_c_brute_force_2pow31(c_brute):
    """Tiny config (BASELINE.json:7): s = 32, g = 1, K = 2, D = 1 — all 2^31 compositions."""
    rng = np.random.default_rng(32)
    t = gpu_like_table(32, rng, knee=4, base_ns=10_000, per_unit_ns=900, ctx_ns=300)
    assert c_brute(t, 32, 2, 1) == op.optimize(t, 32, 2, 1)


# ---------------------------------------------------------------- joint batch x token plan
from oracle.plan import (joint_brute_force, joint_objective, joint_optimize, knapsack,  # noqa: E402
                         partitions)


def test_knapsack_spec_example():
    # T_1 = 5, T_2 = 8 -> C(2) = min(T_2, 2 T_1) = 8, partition [2]
    assert knapsack({1: 5, 2: 8}, 2) == (8, [2])
    # ties keep the smallest b: T_2 = 2 T_1 exactly -> all ones
    assert knapsack({1: 4, 2: 8}, 2) == (8, [1, 1])
    assert knapsack({2: 3}, 3) is None


def test_partitions_count():
    # p(6) over parts {1..6} = 11; parts {1, 2} of 6: 4 (2+2+2, 2+2+1+1, 2+1*4, 1*6)
    assert len(list(partitions(6, [1, 2, 3, 4, 5, 6]))) == 11
    assert len(list(partitions(6, [1, 2]))) == 4


def _monotone_tables(rng, n, bs):
    # per-b tables: larger b costs more per job (b sequences), context makes later slices dearer
    base = rng.integers(1, 20, size=(n, n + 1)).astype(np.int64)
    return {b: base * b + rng.integers(0, 5 * b, size=(n, n + 1)) for b in bs}


@pytest.mark.parametrize("seed", range(40))
def test_joint_optimize_equals_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 5))
    B = int(rng.integers(1, 5))
    K = int(rng.integers(1, 5))
    bs = sorted(set(int(x) for x in rng.integers(1, B + 1, size=rng.integers(1, 3)))) or [1]
    if 1 not in bs:
        bs = [1] + bs  # every B is composable
    tables = _monotone_tables(rng, n, bs)
    T, plan = joint_optimize(tables, n, B, K)
    assert sum(b for b, _ in plan) == B and all(sum(l) == n for _, l in plan)
    assert T == joint_objective(tables, plan, K)
    assert T == joint_brute_force(tables, n, B, K)


def test_joint_reduces_to_uniform_objective():
    # a single allowed batch-slice size b: the joint plan is [(b, l)] * (B / b) with the tp_plan
    # objective D * sum + (K - 1) * max (reading A-20)
    rng = np.random.default_rng(7)
    n, K, B, b = 5, 3, 4, 2
    t = rng.integers(1, 30, size=(n, n + 1)).astype(np.int64)
    T, plan = joint_optimize({b: t}, n, B, K)
    T_u, _, lengths = op.optimize(t, n, K, D=B // b)
    assert T == T_u and [x for x, _ in plan] == [b, b]


# ---------------------------------------------------------------- op-list schedules (GPipe, 1F1B)
def test_generic_replay_equals_gpipe_replay():
    rng = np.random.default_rng(17)
    for _ in range(100):
        K, J = int(rng.integers(1, 6)), int(rng.integers(1, 9))
        tf = rng.uniform(0.5, 3.0, size=(K, J)).tolist()
        tb = rng.uniform(0.5, 3.0, size=(K, J)).tolist()
        comm = float(rng.uniform(0, 0.5))
        assert abs(op.oplist_replay(op.gpipe_oplists([J], K), tf, tb, comm) -
                   op.oplist_makespan(tf, tb, comm)) < 1e-9


def test_1f1b_textbook_closed_form():
    """One job per group (microbatch) and uniform durations: 1F1B's makespan is the textbook
    (D + K - 1)(t_f + t_b) (the same bubble as GPipe), and stage k holds min(D, K - k) groups."""
    for K in range(1, 6):
        for D in range(1, 9):
            tf, tb = 1.0, 2.0
            ops = op.one_f_one_b_oplists([1] * D, K)
            ms = op.oplist_replay(ops, [[tf] * D] * K, [[tb] * D] * K)
            assert abs(ms - (D + K - 1) * (tf + tb)) < 1e-9, (K, D, ms)
            assert op.max_inflight_groups(ops, [1] * D) == [min(D, K - k) for k in range(K)]
            assert op.max_inflight_groups(op.gpipe_oplists([1] * D, K), [1] * D) == [D] * K


def test_1f1b_single_group_is_gpipe_and_lists_are_permutations():
    rng = np.random.default_rng(5)
    for _ in range(50):
        K = int(rng.integers(1, 6))
        groups = [int(x) for x in rng.integers(1, 5, size=int(rng.integers(1, 6)))]
        a, b = op.one_f_one_b_oplists(groups, K), op.gpipe_oplists(groups, K)
        for x, y in zip(a, b):
            assert sorted(x) == sorted(y)
        if len(groups) == 1:
            assert a == b
        J = sum(groups)
        tf = rng.uniform(0.5, 2.0, size=(K, J)).tolist()
        tb = rng.uniform(0.5, 2.0, size=(K, J)).tolist()
        ms = op.oplist_replay(a, tf, tb)           # never deadlocks
        lower = max(sum(tf[k]) + sum(tb[k]) for k in range(K))
        assert ms >= lower - 1e-9


def test_replay_detects_deadlock():
    with pytest.raises(ValueError):
        op.oplist_replay([[("B", 0), ("F", 0)], [("F", 0), ("B", 0)]], [[1.0], [1.0]], [[1.0], [1.0]])
