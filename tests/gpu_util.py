"""Shared helpers for the GPU parity tests (test-only)."""
import functools

import numpy as np

import paper_2102_07988_b200 as tp
from oracle.model import gpt_forward_backward
from synth import make_params, make_tokens, pack_all_stages, unpack_all_stages


def rel(a, b):
    """Per-tensor relative L2 error ||a - b|| / ||b|| (reading A-23)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@functools.lru_cache(maxsize=16)
def oracle_run(cfg, B, seed, bf16):
    params = make_params(cfg, seed=seed, bf16=bf16)
    tokens = make_tokens(cfg, B, seed=seed + 1)
    ref = gpt_forward_backward(params, tokens, cfg.n_layer, cfg.n_head)
    return params, tokens, ref


def gpu_run(cfg, B, params, tokens, lengths, precision, flags=tp.TP_FLAG_KEEP_LOGITS, batch_slice=1):
    ctx = tp.Context(cfg, precision=precision, max_batch=B, device=0, flags=flags)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        loss = ctx.step(tp.Slicing(lengths, batch_slice), tokens)
        grads = unpack_all_stages(ctx.grads(), cfg)
        logits = ctx.logits(B) if flags & tp.TP_FLAG_KEEP_LOGITS else None
        launches = ctx.last_step_launches()
    finally:
        ctx.close()
    return loss, logits, grads, launches


def worst_errors(loss, logits, grads, ref):
    errs = {"loss": abs(loss - ref["loss"]) / abs(ref["loss"])}
    if logits is not None:
        errs["logits"] = rel(logits, ref["logits"])
    for k, g in ref["grads"].items():
        errs[k] = rel(grads[k], g)
    return errs


def gpu_run_plan(cfg, B, params, tokens, groups, precision, flags=tp.TP_FLAG_KEEP_LOGITS, max_batch=None):
    """One step with a heterogeneous batch plan [(b_d, lengths_d), ..] (tp_step_plan)."""
    ctx = tp.Context(cfg, precision=precision, max_batch=max_batch or B, device=0, flags=flags)
    try:
        ctx.load_params(pack_all_stages(params, cfg))
        loss = ctx.step_plan(tp.BatchPlan(groups), tokens)
        grads = unpack_all_stages(ctx.grads(), cfg)
        logits = ctx.logits(B) if flags & tp.TP_FLAG_KEEP_LOGITS else None
    finally:
        ctx.close()
    return loss, logits, grads
