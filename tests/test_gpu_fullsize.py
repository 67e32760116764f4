"""Parity at BASELINE.json's full size, in the launch configuration bench.py times (GPT-3 1B,
B = 8, s = 2048, bf16, joint batch x token slicing [(8, [576, 1472])], CUDA-graph replay).

The oracle cannot run the whole step in a test's time, so it checks sampled outputs it can compute
on its own: causality (Eq. 2) makes the logits of positions < P depend only on tokens
< P, so the fp64 oracle runs the full-width, full-depth model on a P-token prefix of two sequences
and their logits are compared with the GPU's full-size step. The rest is checked through properties
that hold at any size: the sliced step equals the unsliced one (slicing changes
the schedule, not the function) in loss and logits, and graph replays repeat the eager step.
Tolerance: the north-star bf16 bound, 2e-2 per-tensor relative L2 (A-23)."""
import numpy as np
import pytest

import paper_2102_07988_b200 as tp
from tests.gpu_util import rel
from oracle.model import gpt_forward_backward
from synth import CONFIGS, make_stage_flat, make_tokens, round_bf16, unpack_all_stages

pytestmark = pytest.mark.gpu

P = 128                # oracle prefix length
SEQS = [0, 5]          # sampled sequences of the batch
SLICED = ([576, 1472], 8)
UNSLICED = ([2048], 8)


@pytest.fixture(scope="module")
def full():
    cfg, B = CONFIGS["gpt3-1b"]
    flat = round_bf16(make_stage_flat(cfg, 0, seed=0))  # the bench's weights, bf16-representable
    tokens = make_tokens(cfg, B, seed=1)
    return cfg, B, flat, tokens


def run(cfg, B, flat, tokens, lengths, b):
    ctx = tp.Context(cfg, precision=tp.TP_BF16, max_batch=B, device=0, flags=tp.TP_FLAG_KEEP_LOGITS)
    try:
        ctx.load_params(flat)
        sl = tp.Slicing(lengths, b)
        losses = [ctx.step(sl, tokens) for _ in range(3)]  # eager, capture + launch, replay
        logits = ctx.logits(B)[SEQS].copy()
    finally:
        ctx.close()
    return losses, logits


@pytest.fixture(scope="module")
def sliced(full):
    cfg, B, flat, tokens = full
    return run(cfg, B, flat, tokens, *SLICED)


def test_fullsize_prefix_logits_vs_oracle(full, sliced):
    cfg, B, flat, tokens = full
    params = unpack_all_stages(flat, cfg)
    ref = gpt_forward_backward(params, tokens[SEQS, :P + 1], cfg.n_layer, cfg.n_head, need_grads=False)
    _, logits = sliced
    err = rel(logits[:, :P], ref["logits"])
    assert err < 2e-2, err


def test_fullsize_sliced_equals_unsliced(full, sliced):
    cfg, B, flat, tokens = full
    losses_s, logits_s = sliced
    losses_u, logits_u = run(cfg, B, flat, tokens, *UNSLICED)
    assert abs(losses_s[-1] - losses_u[-1]) <= 2e-3 * abs(losses_u[-1])
    assert rel(logits_s, logits_u) < 2e-2
    # graph replays repeat the eager step (same kernels, same inputs)
    assert abs(losses_s[2] - losses_s[0]) <= 1e-5 * abs(losses_s[0])
    assert np.isfinite(losses_s[-1]) and 10.0 < losses_s[-1] < 11.5  # ~ln V for a random-init model
