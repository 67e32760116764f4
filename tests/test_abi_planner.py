"""C ABI on the CPU host: libtp.so loads, exports every symbol include/tp.h declares, validates
arguments, and tp_plan (host-only) equals the oracle's brute force bit-exactly (BASELINE.json:5
invariant (b)). No GPU compute is called here."""
import os
import re
import subprocess
import time

import numpy as np
import pytest

import paper_2102_07988_b200 as tp
from oracle import plan as op
from synth import CONFIGS, ModelCfg, gpu_like_table, random_int_table, stage_param_count

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="tp.h"):
    src = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:tp_status|void|const char\*)\s+(tpk?_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", tp.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (tpk?_\w+)$", out, re.M))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(tp.EXPORTED) == syms
    ksyms = declared_symbols("tp_kernels.h")
    assert sorted(tp.KEXPORTED) == ksyms and all(s in exported for s in ksyms)
    for s in syms + ksyms:
        getattr(tp.lib(), s)


def test_stage_param_count_matches_layout():
    for name in ("tiny", "gpt3-1b", "gpt3-13b", "small"):
        cfg, _ = CONFIGS[name]
        for k in range(cfg.n_stages):
            assert tp.stage_param_count(cfg, k) == stage_param_count(cfg, k)


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg, _ = CONFIGS["tiny"]
    with pytest.raises(tp.TpError) as e:
        tp.Context(cfg)
    assert e.value.status == tp.TP_ECUDA


def test_init_rejects_bad_shapes():
    with pytest.raises(tp.TpError) as e:
        tp.Context(ModelCfg(3, 64, 4, 128, 32, 2))       # n_layer % n_stages
    assert e.value.status == tp.TP_EINVAL
    with pytest.raises(tp.TpError) as e:
        tp.Context(ModelCfg(2, 96, 4, 128, 32, 1))       # head_dim 24 not a multiple of 16
    assert e.value.status == tp.TP_EINVAL


def _plan(t, n, K, D=1, eps=0, g=1):
    return tp.plan(t, g, n_layer=K, hidden=64, seq_len=n * g, n_stages=K, n_micro=D, eps_ticks=eps)


def test_plan_spec_examples():
    t = np.zeros((3, 4), np.int64)
    for l in range(1, 4):
        for c in range(0, 4 - l):
            t[l - 1, c] = l
    s = _plan(t, 3, 2)
    assert s.lengths == [1, 1, 1] and s.predicted == 4
    t2 = t + (t > 0)
    s = _plan(t2, 3, 3)
    assert s.lengths == [1, 1, 1] and s.predicted == 10


@pytest.mark.parametrize("seed", range(6))
def test_plan_bit_exact_vs_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(40):
        n = int(rng.integers(1, 13))
        K = int(rng.integers(1, 5))
        D = int(rng.choice([1, 2, 8]))
        t = random_int_table(n, rng, 1, int(rng.choice([3, 12, 10 ** 6])))
        T, m, lens = op.brute_force(t, n, K, D)
        s = _plan(t, n, K, D)
        assert (s.predicted, s.t_max, s.lengths) == (T, m, lens)


def test_plan_matches_oracle_dp_with_eps_and_threads(monkeypatch):
    rng = np.random.default_rng(9)
    for n in (16, 40):
        t = gpu_like_table(n, rng)
        for K in (2, 8):
            for eps in (0, 20_000):
                T, m, lens = op.optimize(t, n, K, 1, eps)
                s = tp.plan(t, 8, n_layer=K, hidden=64, seq_len=8 * n, n_stages=K, eps_ticks=eps)
                assert s.lengths == [8 * x for x in lens] and s.predicted == T and s.t_max == m


def test_plan_rejects_bad_tables():
    t = np.ones((4, 5), np.int64)
    t[1, 2] = 0
    with pytest.raises(tp.TpError) as e:
        _plan(t, 4, 2)
    assert e.value.status == tp.TP_EINVAL
    with pytest.raises(tp.TpError):
        tp.plan(np.ones((4, 5), np.int64), 4, n_layer=2, hidden=64, seq_len=12, n_stages=2)  # n_units mismatch


def test_plan_s2048_g8_within_a_minute():
    """PAPER.md:290 'the dynamic programming can finish within a minute' — s = 2048, g = 8, exact."""
    rng = np.random.default_rng(2048)
    t = gpu_like_table(256, rng, knee=32, base_ns=1_500_000, per_unit_ns=45_000, ctx_ns=2_000)
    t0 = time.time()
    s = tp.plan(t, 8, n_layer=40, hidden=5120, seq_len=2048, n_stages=8, n_micro=8)
    assert time.time() - t0 < 60
    assert sum(s.lengths) == 2048


@pytest.mark.slow
def test_plan_tiny_config_vs_2pow31_brute_force():
    """Tiny config (BASELINE.json:7): s = 32, g = 1, K = 2, D = 1 against all 2^31 compositions."""
    bf = os.path.join(ROOT, "oracle", "bf_compositions")
    if not os.path.exists(bf):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-o", bf, bf + ".c"], check=True)
    rng = np.random.default_rng(31)
    for trial in range(2):
        t = gpu_like_table(32, rng, knee=4, base_ns=10_000, per_unit_ns=900, ctx_ns=300) if trial == 0 \
            else random_int_table(32, rng, 1, 40)
        inp = "32 2 1\n" + " ".join(str(int(v)) for v in t.reshape(-1))
        out = [int(x) for x in subprocess.run([bf], input=inp, capture_output=True, text=True, check=True).stdout.split()]
        s = _plan(t, 32, 2)
        assert (s.predicted, s.t_max, s.lengths) == (out[0], out[1], out[3:3 + out[2]])


# ---------------------------------------------------------------- tp_plan_joint
def _joint_tables(rng, n, bs):
    base = rng.integers(1, 20, size=(n, n + 1)).astype(np.int64)
    return {b: base * b + rng.integers(0, 5 * b, size=(n, n + 1)).astype(np.int64) for b in bs}


@pytest.mark.parametrize("seed", range(60))
def test_plan_joint_bit_exact_vs_oracle(seed):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(1, 9))
    B = int(rng.integers(1, 9))
    K = int(rng.integers(1, 6))
    bs = sorted({1} | {int(x) for x in rng.integers(1, B + 1, size=int(rng.integers(0, 3)))})
    tables = _joint_tables(rng, n, bs)
    g = 8
    T, plan = op.joint_optimize(tables, n, B, K)
    got = tp.plan_joint(tables, g, K, 64, n * g, K, B)
    assert got.predicted == T
    assert got.groups == [(b, [x * g for x in ls]) for b, ls in plan]
    assert got.t_max == max(x for b, ls in plan for x in op.slice_costs(tables[b], ls))


@pytest.mark.parametrize("seed", range(20))
def test_plan_joint_vs_brute_force(seed):
    rng = np.random.default_rng(7000 + seed)
    n, B, K = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 5))
    bs = sorted({1} | {int(rng.integers(1, B + 1))})
    tables = _joint_tables(rng, n, bs)
    got = tp.plan_joint(tables, 1, K, 64, n, K, B)
    assert got.predicted == op.joint_brute_force(tables, n, B, K)
    assert sum(b for b, _ in got.groups) == B


def test_plan_joint_single_b_equals_plan():
    # one batch-slice size: the joint plan is tp_plan with n_micro = B / b (reading A-20)
    rng = np.random.default_rng(11)
    n, K, B, b, g = 16, 4, 8, 2, 64
    t = random_int_table(n, rng, 1, 1000)
    j = tp.plan_joint({b: t}, g, K, 64, n * g, K, B)
    u = tp.plan(t, g, K, 64, n * g, K, n_micro=B // b)
    assert j.predicted == u.predicted and j.groups == [(b, u.lengths)] * (B // b)


def test_plan_joint_rejects_bad_input():
    t = np.ones((2, 3), dtype=np.int64)
    with pytest.raises(tp.TpError) as e:
        tp.plan_joint({2: t}, 1, 1, 64, 2, 1, 3)  # 3 is not a sum of 2s
    assert e.value.status == tp.TP_EINFEASIBLE
    with pytest.raises(tp.TpError) as e:
        tp.plan_joint({1: t, 2: np.ones((3, 4), dtype=np.int64)}, 1, 1, 64, 2, 1, 2)
    assert e.value.status == tp.TP_EINVAL
    bad = t.copy()
    bad[0, 0] = 0
    with pytest.raises(tp.TpError):
        tp.plan_joint({1: bad}, 1, 1, 64, 2, 1, 1)


def test_batch_plan_notation():
    p = tp.BatchPlan([(2, [384, 384]), (2, [384, 384]), (1, [768])])
    assert p.notation() == "[(2, [384, 384])] * 2 + [(1, [768])] * 1" and p.batch() == 5


# ---------------------------------------------------------------- schedules (A-21)
@pytest.mark.parametrize("seed", range(30))
def test_schedule_oplist_equals_oracle(seed):
    """tp_schedule_oplist (the op lists tp_step executes) equals oracle/plan.py's GPipe and 1F1B lists
    on every stage, and the 1F1B lists never deadlock and keep at most min(D, K - k) groups live."""
    rng = np.random.default_rng(300 + seed)
    K = int(rng.integers(1, 7))
    groups = [int(x) for x in rng.integers(1, 5, size=int(rng.integers(1, 7)))]
    ref_g, ref_1 = op.gpipe_oplists(groups, K), op.one_f_one_b_oplists(groups, K)
    for k in range(K):
        assert tp.schedule_oplist(K, k, groups, False) == ref_g[k]
        assert tp.schedule_oplist(K, k, groups, True) == ref_1[k]
    lists = [tp.schedule_oplist(K, k, groups, True) for k in range(K)]
    J = sum(groups)
    ms = op.oplist_replay(lists, [[1.0] * J] * K, [[2.0] * J] * K)
    assert ms > 0
    assert op.max_inflight_groups(lists, groups) == [min(len(groups), K - k) for k in range(K)]


def test_schedule_oplist_rejects_bad_input():
    with pytest.raises(tp.TpError):
        tp.schedule_oplist(2, 2, [1], True)
    with pytest.raises(tp.TpError):
        tp.schedule_oplist(2, 0, [0, 1], True)


# ---------------------------------------------------------------- stage partition (A-30)
def test_stage_layers_uniform_and_balanced_match_synth():
    """tp_stage_layers (the library's layout) equals synth's stage_layer_counts for both partitions
    over many shapes, every stage owns >= 1 layer, the counts sum to n_layer, and the balanced split
    never has a larger max per-stage FLOP cost (layers + h on the last stage) than the uniform one."""
    from synth import ModelCfg, stage_layer_counts
    rng = np.random.default_rng(42)
    shapes = [(24, 2048, 2048, 50304, K) for K in (1, 2, 3, 4, 6, 8)] + \
             [(40, 5120, 2048, 50304, K) for K in (1, 2, 4, 5, 8)] + [(24, 12288, 2048, 50304, 8)]
    for _ in range(60):
        K = int(rng.integers(1, 9))
        shapes.append((int(rng.integers(K, 5 * K + 1)), int(rng.choice([256, 1024, 2048, 5120])),
                       int(rng.choice([128, 2048, 8192])), int(rng.choice([512, 50304])), K))
    for n, H, s, V, K in shapes:
        for part in (0, 1):
            if part == 0 and n % K:
                continue
            cfg = ModelCfg(n, H, 16, V, s, K, part)
            got = tp.stage_layers(cfg)
            assert got == stage_layer_counts(cfg), (n, H, s, V, K, part)
            assert sum(got) == n and min(got) >= 1
        if n % K == 0:
            h = V / (12.0 * H + s)
            bal = stage_layer_counts(ModelCfg(n, H, 16, V, s, K, 1))
            cost = lambda c: max(max(c[:-1], default=0), c[-1] + h)
            assert cost(bal) <= cost([n // K] * K) + 1e-12


def test_balanced_partition_1b_examples():
    from synth import ModelCfg
    assert tp.stage_layers(ModelCfg(24, 2048, 16, 50304, 2048, 4, 1)) == [6, 7, 6, 5]
    assert tp.stage_layers(ModelCfg(24, 2048, 16, 50304, 2048, 8, 1)) == [3, 4, 3, 3, 3, 3, 3, 2]
    assert tp.stage_layers(ModelCfg(40, 5120, 40, 50304, 2048, 4, 1)) == [10] * 4   # 13B: uniform is optimal
    with pytest.raises(tp.TpError):
        tp.stage_layers(ModelCfg(3, 64, 4, 128, 32, 2, 0))
