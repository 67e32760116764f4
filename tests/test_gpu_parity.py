"""GPU parity: tp_step (token-sliced, pipelined over K stages) against the fp64 oracle's unsliced
forward/backward — invariant (a) of BASELINE.json:5 — within 2e-2 (bf16) / 1e-4 (fp32) per-tensor
relative L2 (A-23), on seeded random weights and tokens, for many slicings including
[s], [1]*s, ragged and paper-shaped (non-monotone) ones. All calls go through the C ABI."""
import numpy as np
import pytest

import paper_2102_07988_b200 as tp
from synth import CONFIGS, ModelCfg
from tests.gpu_util import gpu_run, gpu_run_plan, oracle_run, rel, worst_errors

pytestmark = pytest.mark.gpu

TINY, _ = CONFIGS["tiny"]
SMALL, SMALL_B = CONFIGS["small"]
TINY_SLICINGS = [[32], [1] * 32, [5, 9, 2, 16], [16, 8, 8], [3, 29], [8, 8, 8, 8]]


def check(errs, tol):
    bad = {k: v for k, v in errs.items() if not v < tol}
    assert not bad, (bad, max(errs.values()))


@pytest.mark.parametrize("lengths", TINY_SLICINGS)
def test_tiny_fp32(lengths):
    params, tokens, ref = oracle_run(TINY, 1, 0, False)
    loss, logits, grads, _ = gpu_run(TINY, 1, params, tokens, lengths, tp.TP_FP32)
    check(worst_errors(loss, logits, grads, ref), 1e-4)


@pytest.mark.parametrize("lengths", TINY_SLICINGS)
def test_tiny_bf16(lengths):
    params, tokens, ref = oracle_run(TINY, 1, 0, True)
    loss, logits, grads, launches = gpu_run(TINY, 1, params, tokens, lengths, tp.TP_BF16)
    assert launches > 0
    check(worst_errors(loss, logits, grads, ref), 2e-2)


@pytest.mark.parametrize("K", [1, 2, 4])
def test_small_bf16_stages(K):
    cfg = SMALL.with_(n_stages=K)
    params, tokens, ref = oracle_run(cfg, SMALL_B, 3, True)
    loss, logits, grads, _ = gpu_run(cfg, SMALL_B, params, tokens, [40, 24, 64], tp.TP_BF16)
    check(worst_errors(loss, logits, grads, ref), 2e-2)


def test_small_fp32_batch2():
    params, tokens, ref = oracle_run(SMALL, SMALL_B, 4, False)
    loss, logits, grads, _ = gpu_run(SMALL, SMALL_B, params, tokens, [8, 56, 8, 56], tp.TP_FP32)
    check(worst_errors(loss, logits, grads, ref), 1e-4)


def test_fp32_sliced_equals_unsliced_on_gpu():
    params, tokens, _ = oracle_run(SMALL, SMALL_B, 5, False)
    a = gpu_run(SMALL, SMALL_B, params, tokens, [128], tp.TP_FP32)
    b = gpu_run(SMALL, SMALL_B, params, tokens, [8] * 16, tp.TP_FP32)
    assert abs(a[0] - b[0]) < 1e-6 * abs(a[0])
    assert rel(b[1], a[1]) < 1e-5
    for k in a[2]:
        assert rel(b[2][k], a[2][k]) < 1e-5, k


def test_bf16_default_vs_force_simt():
    """The tensor-core kernels against the independent SIMT kernels on identical inputs."""
    params, tokens, ref = oracle_run(SMALL, SMALL_B, 6, True)
    a = gpu_run(SMALL, SMALL_B, params, tokens, [72, 56], tp.TP_BF16)
    b = gpu_run(SMALL, SMALL_B, params, tokens, [72, 56], tp.TP_BF16, tp.TP_FLAG_KEEP_LOGITS | tp.TP_FLAG_FORCE_SIMT)
    check(worst_errors(*a[:3], ref), 2e-2)
    check(worst_errors(*b[:3], ref), 2e-2)


def test_parity_mid_13b_width():
    """SURVEY.md §8(c) parity-mid: 2 layers at the real 13B width (H=5120, a=40, d=128), s=512,
    unaligned slice offsets."""
    cfg, B = CONFIGS["parity-mid"]
    params, tokens, ref = oracle_run(cfg, B, 7, True)
    loss, logits, grads, _ = gpu_run(cfg, B, params, tokens, [200, 136, 104, 72], tp.TP_BF16)
    check(worst_errors(loss, logits, grads, ref), 2e-2)


def test_wide_hidden_175b_width():
    """GPT-3 175B width (H = 12288, 96 heads of 128) on one layer: the wide-row LayerNorm backward
    (768 threads x 2 chunks, shared-memory gradient partials) and the GEMMs at that width."""
    cfg = ModelCfg(1, 12288, 96, 256, 64, 1)
    params, tokens, ref = oracle_run(cfg, 1, 17, True)
    loss, logits, grads, _ = gpu_run(cfg, 1, params, tokens, [40, 24], tp.TP_BF16)
    check(worst_errors(loss, logits, grads, ref), 2e-2)


def test_parity_mid_batch2_tail_split():
    """13B width, b = 2 unsliced: 1024-row GEMMs whose partial last wave is split into a second
    half-width-tile launch (QKV scatter, GeLU, residual and dX epilogues through Epi::n_off)."""
    cfg, _ = CONFIGS["parity-mid"]
    B = 2
    params, tokens, ref = oracle_run(cfg, B, 13, True)
    loss, logits, grads, _ = gpu_run(cfg, B, params, tokens, [512], tp.TP_BF16, batch_slice=2)
    check(worst_errors(loss, logits, grads, ref), 2e-2)


@pytest.mark.parametrize("precision,tol", [(tp.TP_BF16, 2e-2), (tp.TP_FP32, 1e-4)])
@pytest.mark.parametrize("K,b,lengths", [(2, 2, [40, 24, 64]), (1, 4, [128]), (2, 2, [8] * 16), (4, 4, [56, 72])])
def test_joint_batch_token_slicing(K, b, lengths, precision, tol):
    """Jobs of b sequences x one token slice: same result as the unsliced oracle."""
    cfg = SMALL.with_(n_stages=K)
    B = 4
    params, tokens, ref = oracle_run(cfg, B, 8, precision == tp.TP_BF16)
    loss, logits, grads, _ = gpu_run(cfg, B, params, tokens, lengths, precision, batch_slice=b)
    check(worst_errors(loss, logits, grads, ref), tol)


@pytest.mark.parametrize("precision,tol", [(tp.TP_BF16, 2e-2), (tp.TP_FP32, 1e-4)])
@pytest.mark.parametrize("K,groups", [
    (2, [(2, [40, 24, 64]), (1, [128]), (1, [8] * 16)]),      # three groups, three slicings
    (1, [(1, [64, 64]), (3, [16, 112])]),
    (4, [(3, [128]), (1, [32, 32, 32, 32])]),
])
def test_heterogeneous_batch_plan(K, groups, precision, tol):
    """Groups of different batch-slice sizes, each with its own token slicing (PAPER.md:362-364,
    tp_plan_joint's output): the same function as the unsliced oracle."""
    cfg = SMALL.with_(n_stages=K)
    B = 4
    params, tokens, ref = oracle_run(cfg, B, 9, precision == tp.TP_BF16)
    loss, logits, grads = gpu_run_plan(cfg, B, params, tokens, groups, precision)
    check(worst_errors(loss, logits, grads, ref), tol)


def test_heterogeneous_plan_rejects_bad_plans():
    params, tokens, _ = oracle_run(TINY, 2, 0, True)
    for groups in ([(1, [32])], [(1, [32]), (2, [32])], [(1, [16, 8]), (1, [32])], [(0, [32]), (2, [32])]):
        with pytest.raises(tp.TpError) as e:
            gpu_run_plan(TINY, 2, params, tokens, groups, tp.TP_BF16)
        assert e.value.status == tp.TP_EINVAL


def test_rejects_bad_slicing():
    params, tokens, _ = oracle_run(TINY, 1, 0, True)
    with pytest.raises(tp.TpError) as e:
        gpu_run(TINY, 1, params, tokens, [16, 8], tp.TP_BF16)
    assert e.value.status == tp.TP_EINVAL
    with pytest.raises(tp.TpError) as e:                        # batch_slice must divide batch
        gpu_run(TINY, 1, params, tokens, [32], tp.TP_BF16, batch_slice=2)
    assert e.value.status == tp.TP_EINVAL


def test_profile_plan_step_end_to_end():
    """a1 -> a2 -> tp_step: the measured cost table feeds the DP
    and the chosen slicing runs with parity against the oracle; the DP result equals the oracle's
    Algorithm 1 on the same table."""
    from oracle import plan as op
    cfg = SMALL.with_(n_stages=2)
    B = 2
    params, tokens, ref = oracle_run(cfg, B, 9, True)
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=B, device=0, flags=tp.TP_FLAG_KEEP_LOGITS)
    try:
        from synth import pack_all_stages, unpack_all_stages
        ctx.load_params(pack_all_stages(params, cfg))
        g = 16
        for b in (1, 2):
            ticks, fit = ctx.profile(g, reps=3, batch_slice=b)
            n = cfg.seq_len // g
            assert ticks.shape == (n, n + 1)
            assert all(ticks[l - 1, c] > 0 for l in range(1, n + 1) for c in range(0, n - l + 1))
            assert fit.shape == (5,) and np.isfinite(fit).all()
            sl = tp.plan(ticks, g, cfg.n_layer, cfg.hidden, cfg.seq_len, 2, n_micro=B // b)
            T, m, lens = op.optimize(ticks, n, 2, B // b)
            assert sl.lengths == [g * x for x in lens] and sl.predicted == T
            loss = ctx.step(tp.Slicing(sl.lengths, b), tokens)
            grads = unpack_all_stages(ctx.grads(), cfg)
            check(worst_errors(loss, ctx.logits(B), grads, ref), 2e-2)
    finally:
        ctx.close()


def test_graph_replay_identical():
    """tp_step runs a new (slicing, batch) eagerly, captures it into a CUDA graph on the second call
    and replays the graph afterwards: all three give identical results, and a different slicing in
    between invalidates the graph."""
    cfg = SMALL.with_(n_stages=2)
    B = 2
    params, tokens, ref = oracle_run(cfg, B, 10, True)
    from synth import pack_all_stages
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=B, device=0)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        sl = tp.Slicing([40, 24, 64])
        outs = []
        for _ in range(3):
            loss = ctx.step(sl, tokens)
            outs.append((loss, ctx.grads(), ctx.last_step_launches()))
        ctx.step(tp.Slicing([64, 64], 2), tokens)
        outs.append((ctx.step(sl, tokens), ctx.grads(), ctx.last_step_launches()))
        for loss, g, n in outs[1:]:
            assert abs(loss - outs[0][0]) <= 1e-6 * abs(outs[0][0])
            assert rel(g, outs[0][1]) < 1e-6
        # eager steps count the instrumented launches, captured / replayed steps the graph's kernel
        # nodes (every launch): the replays agree, and the eager count is a lower bound
        assert outs[1][2] == outs[2][2] and 0 < outs[0][2] <= outs[1][2]
        assert abs(outs[0][0] - ref["loss"]) < 2e-2 * abs(ref["loss"])
    finally:
        ctx.close()


def test_rejects_token_ids_outside_vocab():
    """Token ids outside [0, V) are rejected (TP_EINVAL), never clamped: host tokens before the step
    runs, device tokens by the device-side count read back with the loss (include/tp.h)."""
    import torch
    params, tokens, _ = oracle_run(TINY, 1, 0, True)
    from synth import pack_all_stages
    ctx = tp.Context(TINY, precision=tp.TP_BF16, max_batch=1, device=0)
    try:
        ctx.load_params(pack_all_stages(params, TINY))
        sl = tp.Slicing([16, 16])
        for bad in (-1, TINY.vocab):
            t = tokens.copy()
            t[0, 7] = bad
            with pytest.raises(tp.TpError) as e:
                ctx.step(sl, t)
            assert e.value.status == tp.TP_EINVAL
            dt = torch.from_numpy(t.astype(np.int32)).cuda()
            with pytest.raises(tp.TpError) as e:
                ctx.step_device(sl, dt.data_ptr(), 1)
            assert e.value.status == tp.TP_EINVAL
        # valid tokens still work afterwards (device and host)
        dt = torch.from_numpy(tokens.astype(np.int32)).cuda()
        a = ctx.step_device(sl, dt.data_ptr(), 1)
        b = ctx.step(sl, tokens)
        assert np.isfinite(a) and abs(a - b) <= 1e-6 * abs(b)
        with pytest.raises(tp.TpError):
            ctx.step(sl, tokens[:, :-1])  # wrong token row length
    finally:
        ctx.close()


def test_tiny_measured_table_vs_2pow31_brute_force():
    """SURVEY.md §8 acceptance (i) with a MEASURED table: tp_profile of the tiny config (s = 32,
    g = 1, BASELINE.json:7) feeds tp_plan (K = 2, D = 1), and the result equals the oracle's brute
    force over all 2^31 compositions (oracle/bf_compositions.c) on the same table, bit-exactly in T,
    t_max and the slice boundaries."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    bf = os.path.join(root, "oracle", "bf_compositions")
    if not os.path.exists(bf):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-o", bf, bf + ".c"], check=True)
    params, tokens, _ = oracle_run(TINY, 1, 0, True)
    from synth import pack_all_stages
    ctx = tp.Context(TINY, precision=tp.TP_BF16, max_batch=1, device=0)
    try:
        ctx.load_params(pack_all_stages(params, TINY))
        ticks, _ = ctx.profile(1, reps=3)
    finally:
        ctx.close()
    n = TINY.seq_len
    inp = f"{n} 2 1\n" + " ".join(str(int(v)) for v in ticks.reshape(-1))
    out = [int(x) for x in subprocess.run([bf], input=inp, capture_output=True, text=True, check=True,
                                          timeout=600).stdout.split()]
    s = tp.plan(ticks, 1, TINY.n_layer, TINY.hidden, n, 2)
    assert (s.predicted, s.t_max, s.lengths) == (out[0], out[1], out[3:3 + out[2]])


def test_profile_stage_types_comm_term_and_wgrad(monkeypatch):
    """tp_profile over a K = 2 loopback context measures both stage types (first: embedding, last:
    LM head + CE) and returns their element-wise max (A-16); TP_COMM_ALPHA_NS / TP_COMM_GBS add the
    transmission term 2 (alpha + 4 H b l / beta) of PAPER.md:243 to every entry; tp_profile_wgrad
    times the slicing-independent dW GEMMs; tp_profile_comm needs world > 1."""
    cfg = SMALL.with_(n_stages=2)
    params, tokens, _ = oracle_run(cfg, 2, 9, True)
    from synth import pack_all_stages
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=2, device=0)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        g, b = 32, 2
        t0, _ = ctx.profile(g, reps=5, batch_slice=b)
        alpha, gbs = 2.0e6, 0.5  # 2 ms + 0.5 GB/s: far above the measurement noise
        monkeypatch.setenv("TP_COMM_ALPHA_NS", str(alpha))
        monkeypatch.setenv("TP_COMM_GBS", str(gbs))
        t1, _ = ctx.profile(g, reps=5, batch_slice=b)
        n = cfg.seq_len // g
        for lu in range(1, n + 1):
            want = 2.0 * (alpha + 4.0 * cfg.hidden * b * lu * g / gbs)
            got = t1[lu - 1, 0] - t0[lu - 1, 0]
            assert abs(got - want) < 0.05 * want, (lu, got, want)
        w = ctx.profile_wgrad(2, reps=3)
        assert 0 < w < 1e9
        with pytest.raises(tp.TpError) as e:
            ctx.profile_comm()
        assert e.value.status == tp.TP_ESTATE
    finally:
        ctx.close()


# ---------------------------------------------------------------- 1F1B schedule
@pytest.mark.parametrize("K,groups,flags", [
    (2, [(1, [40, 24, 64])] * 4, 0),
    (4, [(1, [40, 24, 64])] * 4, 0),
    (4, [(2, [40, 24, 64]), (1, [128]), (1, [8] * 16)], 0),
    (2, [(1, [64, 64])] * 4, tp.TP_FLAG_NCCL_LOOPBACK),
])
@pytest.mark.parametrize("precision,tol", [(tp.TP_BF16, 2e-2), (tp.TP_FP32, 1e-4)])
def test_1f1b_schedule_parity(K, groups, flags, precision, tol):
    """TP_FLAG_SCHEDULE_1F1B: the group-granular 1F1B op lists (tp_schedule_oplist), slot-mapped stage
    buffers and per-group weight gradients compute the same function as the unsliced oracle."""
    cfg = SMALL.with_(n_stages=K)
    B = sum(b for b, _ in groups)
    params, tokens, ref = oracle_run(cfg, B, 9, precision == tp.TP_BF16)
    # 1F1B slots hold the largest group: w_k x max b sequences per stage (here <= 2 x B)
    loss, logits, grads = gpu_run_plan(cfg, B, params, tokens, groups, precision,
                                       flags=tp.TP_FLAG_KEEP_LOGITS | tp.TP_FLAG_SCHEDULE_1F1B | flags,
                                       max_batch=2 * B)
    check(worst_errors(loss, logits, grads, ref), tol)


def test_1f1b_batch_exceeds_max_batch():
    """1F1B bounds the stage memory: stage k holds w_k = min(D, K - k) groups, so with K = 2 a batch of
    6 single-sequence groups runs in buffers sized for max_batch = 2 (GPipe would need 6), with the
    same loss and gradients as the oracle; GPipe rejects it."""
    from synth import pack_all_stages, unpack_all_stages
    cfg = SMALL.with_(n_stages=2)
    B = 6
    params, tokens, ref = oracle_run(cfg, B, 14, True)
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=2, device=0, flags=tp.TP_FLAG_SCHEDULE_1F1B)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        losses = [ctx.step(tp.Slicing([40, 24, 64]), tokens) for _ in range(3)]  # eager, capture, replay
        grads = unpack_all_stages(ctx.grads(), cfg)
    finally:
        ctx.close()
    errs = {"loss": abs(losses[-1] - ref["loss"]) / abs(ref["loss"])}
    errs.update({k: rel(grads[k], g) for k, g in ref["grads"].items()})
    check(errs, 2e-2)
    assert abs(losses[0] - losses[2]) <= 1e-5 * abs(losses[0])
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=2, device=0)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        with pytest.raises(tp.TpError) as e:
            ctx.step(tp.Slicing([40, 24, 64]), tokens)
        assert e.value.status == tp.TP_EINVAL
    finally:
        ctx.close()


@pytest.mark.parametrize("K,flags", [(2, 0), (3, 0), (4, 0), (4, tp.TP_FLAG_NCCL_LOOPBACK), (4, tp.TP_FLAG_SCHEDULE_1F1B)])
def test_balanced_partition_parity(K, flags):
    """TP_PARTITION_BALANCED (A-30): non-uniform contiguous layer blocks per stage (the last
    stage, which runs the LM head, owns fewer layers); same function as the unsliced oracle."""
    base, B = CONFIGS["small-deep"]
    cfg = base.with_(n_stages=K)
    assert K == 2 or len(set(tp.stage_layers(cfg))) > 1
    params, tokens, ref = oracle_run(cfg, B, 15, True)
    loss, logits, grads = gpu_run_plan(cfg, B, params, tokens, [(1, [40, 24, 64])] * B, tp.TP_BF16,
                                       flags=tp.TP_FLAG_KEEP_LOGITS | flags)
    check(worst_errors(loss, logits, grads, ref), 2e-2)


@pytest.mark.parametrize("flags", [0, tp.TP_FLAG_NCCL_LOOPBACK, tp.TP_FLAG_SCHEDULE_1F1B])
def test_eight_stage_pipeline_parity(flags):
    """K = 8 stages (one layer each, the depth of an 8-GPU run) executed on one GPU: GPipe and 1F1B op
    lists, in-process and NCCL-loopback transports, heterogeneous slicing; same function as the
    unsliced fp64 oracle."""
    base, B = CONFIGS["small-deep"]
    cfg = base.with_(n_stages=8)
    assert tp.stage_layers(cfg) == [1] * 8
    params, tokens, ref = oracle_run(cfg, B, 17, True)
    loss, logits, grads = gpu_run_plan(cfg, B, params, tokens, [(1, [40, 24, 64]), (1, [64, 64])], tp.TP_BF16,
                                       flags=tp.TP_FLAG_KEEP_LOGITS | flags)
    check(worst_errors(loss, logits, grads, ref), 2e-2)
