"""Parity on the kernel paths bench.py's full-size step takes, against the fp64 oracle.

At BASELINE.json's 1B width (H = 2048, 16 heads of 128) and full sequence length (s = 2048), with
B = 4 sequences, the deferred weight-gradient GEMMs have K = B*s = 8192 (both operands MN-major):
the 256 x 512 pair tiles (`gemm_sm100_kernel<2,256,1,1,2>`) and the stream-K tail are taken
exactly as in the bench (gemm_sm100.cu tile rules, K >= 4096), and the attention backward sees
long prefixes with b > 1 sequences per job. Two layers (one per stage, K = 2 loopback) and a
reduced vocabulary (1024) keep the fp64 oracle (oracle/model.py, the unsliced definition,
PAPER.md:164-180) at ~1 min on the GPU box's host.

Checks (A-23, plus per-slice / per-row maxima so a wrong slice cannot hide in a
per-tensor norm): loss, logits and EVERY gradient within 2e-2 relative L2; every slice's logits
within 2e-2; every logits row and every wpe-gradient row (the position-specific gradient, rows
[c, c+l) of each slice) within 0.1 relative — a row computed from the wrong slice, offset or
prefix is O(1) off."""
import numpy as np
import pytest

import paper_2102_07988_b200 as tp
from synth import ModelCfg, make_params, make_tokens, pack_all_stages, unpack_all_stages
from oracle.model import gpt_forward_backward
from tests.gpu_util import rel

pytestmark = pytest.mark.gpu

CFG = ModelCfg(2, 2048, 16, 1024, 2048, 2)
B = 4
PLANS = [([576, 1472], 2), ([328, 712, 1008], 1)]  # [(2, [576, 1472])] * 2 and [(1, [328, 712, 1008])] * 4
TOL = 2e-2
ROW_TOL = 0.1


@pytest.fixture(scope="module")
def oracle():
    params = make_params(CFG, seed=21, bf16=True)
    tokens = make_tokens(CFG, B, seed=22)
    ref = gpt_forward_backward(params, tokens, CFG.n_layer, CFG.n_head)
    return params, tokens, ref


def row_rel(a, b):
    """Per-row relative L2 over the last axis."""
    a = a.reshape(-1, a.shape[-1]).astype(np.float64)
    b = b.reshape(-1, b.shape[-1]).astype(np.float64)
    return np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-30)


@pytest.mark.parametrize("lengths,b", PLANS)
def test_benchsize_every_gradient_vs_oracle(oracle, lengths, b):
    params, tokens, ref = oracle
    ctx = tp.Context(CFG, precision=tp.TP_BF16, max_batch=B, device=0, flags=tp.TP_FLAG_KEEP_LOGITS)
    try:
        ctx.load_params(pack_all_stages(params, CFG))
        sl = tp.Slicing(lengths, b)
        losses = [ctx.step(sl, tokens) for _ in range(3)]  # eager, capture, replay (bench configuration)
        grads = unpack_all_stages(ctx.grads(), CFG)
        logits = ctx.logits(B)
    finally:
        ctx.close()
    errs = {"loss": abs(losses[-1] - ref["loss"]) / abs(ref["loss"]), "logits": rel(logits, ref["logits"])}
    for k, g in ref["grads"].items():
        errs[k] = rel(grads[k], g)
    bad = {k: v for k, v in errs.items() if not v < TOL}
    assert not bad, (bad, errs)
    assert abs(losses[0] - losses[2]) <= 1e-5 * abs(losses[0])
    # per slice: logits rows [c, c+l) of every sequence, and the wpe gradient rows [c, c+l)
    c = 0
    for l in lengths:
        e = rel(logits[:, c:c + l], ref["logits"][:, c:c + l])
        assert e < TOL, (c, l, e)
        e = rel(grads["wpe"][c:c + l], ref["grads"]["wpe"][c:c + l])
        assert e < TOL, ("wpe", c, l, e)
        c += l
    # per row: no single position of any sequence may be off
    rl = row_rel(logits, ref["logits"])
    assert rl.max() < ROW_TOL, (int(rl.argmax()), float(rl.max()))
    rw = row_rel(grads["wpe"][:CFG.seq_len], ref["grads"]["wpe"][:CFG.seq_len])
    assert rw.max() < ROW_TOL, (int(rw.argmax()), float(rw.max()))


def test_one_layer_1b_width_random_slicing():
    """SURVEY.md §8(c) third parity config: one 1B-width layer at s = 2048 with a random
    non-uniform slicing (unaligned offsets at length), B = 1."""
    cfg = ModelCfg(1, 2048, 16, 512, 2048, 1)
    params = make_params(cfg, seed=31, bf16=True)
    tokens = make_tokens(cfg, 1, seed=32)
    ref = gpt_forward_backward(params, tokens, cfg.n_layer, cfg.n_head)
    rng = np.random.default_rng(33)
    cuts = np.sort(rng.choice(np.arange(1, 2048), size=6, replace=False))
    lengths = np.diff(np.concatenate([[0], cuts, [2048]])).tolist()
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=1, device=0, flags=tp.TP_FLAG_KEEP_LOGITS)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        loss = ctx.step(tp.Slicing(lengths), tokens)
        grads = unpack_all_stages(ctx.grads(), cfg)
        logits = ctx.logits(1)
    finally:
        ctx.close()
    assert abs(loss - ref["loss"]) < TOL * abs(ref["loss"])
    assert rel(logits, ref["logits"]) < TOL
    for k, g in ref["grads"].items():
        assert rel(grads[k], g) < TOL, (k, rel(grads[k], g), lengths)
    assert row_rel(logits, ref["logits"]).max() < ROW_TOL
    assert row_rel(grads["wpe"], ref["grads"]["wpe"]).max() < ROW_TOL
