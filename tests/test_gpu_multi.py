"""Multi-GPU (NCCL send/recv over NVLink) parity: K = world stages, one process per GPU, against
the fp64 oracle. Skipped when fewer GPUs are visible."""
import json
import numpy as np
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(world, cfg, precision, lengths, tmp_path, env=None, batch=None):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "tests", "mp_parity_worker.py"),
           cfg, precision, lengths, str(tmp_path)] + ([str(batch)] if batch else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [json.load(open(tmp_path / f"rank{k}.json")) for k in range(world)]


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
def test_tiny_two_stages_nccl(precision, tol, tmp_path):
    for errs in run(2, "tiny", precision, "5,9,2,16", tmp_path):
        assert max(errs.values()) < tol, errs


def test_small_two_stages_nccl_side_stream_dw(tmp_path):
    """D = B/b = 2 groups with TP_SIDE_DW=1: the weight gradients of the first group run on the
    low-priority stream (opt-in; measured slower than the end-of-step dW)."""
    for errs in run(2, "small", "bf16", "40,24,64", tmp_path, env={"TP_SIDE_DW": "1"}):
        assert max(errs.values()) < 2e-2, errs


def test_profile_collectives_two_ranks(tmp_path):
    """tp_profile_comm (NCCL ping-pong alpha / beta), tp_profile (bottleneck table: max
    over the ranks' stages inside the library, A-16, plus the transmission term) and
    tp_profile_wgrad give identical results on every rank."""
    import json as _json
    run(2, "small", "bf16", "40,24,64", tmp_path, env={"TP_TEST_PROFILE": "1"})
    p = [_json.load(open(tmp_path / f"rank{k}_prof.json")) for k in range(2)]
    assert p[0] == p[1]
    assert 0 < p[0]["alpha_ns"] < 1e6 and 1.0 < p[0]["gbs"] < 5000.0
    t = np.array(p[0]["table"])
    assert (t[:, 0] > 0).all()


@pytest.mark.parametrize("world,cfg,lengths,batch", [(2, "tiny", "5,9,2,16", None), (2, "small", "40,24,64", None),
                                                     (2, "small", "2:40,24,64;1:128", 3), (4, "small", "40,24,64", None)])
def test_device_initiated_p2p(world, cfg, lengths, batch, tmp_path):
    """TP_DEVICE_P2P=1: stage messages written by the producing kernels straight
    into the neighbour's NCCL symmetric window, signalled by per-job release flags, no ncclSend/Recv
    on the data path; same parity bar, repeated steps (epoch-based flags) and graph replay."""
    for errs in run(world, cfg, "bf16", lengths, tmp_path, env={"TP_DEVICE_P2P": "1"}, batch=batch):
        assert max(errs.values()) < 2e-2, errs


@pytest.mark.parametrize("world,env", [(2, {"TP_SCHEDULE": "1f1b"}), (4, {"TP_SCHEDULE": "1f1b"}),
                                       (4, {"TP_SCHEDULE": "1f1b", "TP_DEVICE_P2P": "1"})])
def test_1f1b_nccl(world, env, tmp_path):
    """1F1B over NCCL (and over device-initiated p2p): four groups of b = 1, one stage per GPU."""
    for errs in run(world, "small", "bf16", "1:40,24,64;1:40,24,64;1:40,24,64;1:40,24,64", tmp_path, env=env, batch=4):
        assert max(errs.values()) < 2e-2, errs


@pytest.mark.parametrize("world,env", [(2, {}), (4, {}), (4, {"TP_DEVICE_P2P": "1"})])
def test_balanced_partition_multi(world, env, tmp_path):
    """TP_PARTITION_BALANCED over NCCL / device p2p: stages of different layer counts."""
    for errs in run(world, "small-deep", "bf16", "40,24,64", tmp_path, env=env):
        assert max(errs.values()) < 2e-2, errs


def test_small_four_stages_nccl(tmp_path):
    for errs in run(4, "small", "bf16", "40,24,64", tmp_path):
        assert max(errs.values()) < 2e-2, errs


def test_small_two_stages_heterogeneous_batch_plan(tmp_path):
    """tp_step_plan over NCCL: groups of different batch-slice sizes with their own slicings (jobs
    of different row counts and message sizes on the p2p edges)."""
    for errs in run(2, "small", "bf16", "2:40,24,64;1:128", tmp_path, batch=3):
        assert max(errs.values()) < 2e-2, errs


# ---------------------------------------------------------------- NCCL p2p on one GPU
# TP_FLAG_NCCL_LOOPBACK: all K stages in one context, every stage message (rows a11 / a16: the
# slice's fp32 activation to stage k+1, its gradient back to stage k-1) goes through
# ncclSend / ncclRecv to self on a one-rank communicator, on the same per-direction comm streams,
# split communicators and events as the one-process-per-GPU path. Runs on a one-GPU box.
from synth import CONFIGS as _CONFIGS  # noqa: E402
import paper_2102_07988_b200 as tp  # noqa: E402
from tests.gpu_util import gpu_run, gpu_run_plan, oracle_run, worst_errors  # noqa: E402

NL = tp.TP_FLAG_KEEP_LOGITS | tp.TP_FLAG_NCCL_LOOPBACK


@pytest.mark.parametrize("precision,tol", [(tp.TP_BF16, 2e-2), (tp.TP_FP32, 1e-4)])
@pytest.mark.parametrize("lengths", [[5, 9, 2, 16], [32], [1] * 32])
def test_tiny_nccl_loopback(precision, tol, lengths):
    cfg, B = _CONFIGS["tiny"]
    params, tokens, ref = oracle_run(cfg, B, 0, precision == tp.TP_BF16)
    loss, logits, grads, launches = gpu_run(cfg, B, params, tokens, lengths, precision, flags=NL)
    errs = worst_errors(loss, logits, grads, ref)
    assert max(errs.values()) < tol, errs


@pytest.mark.parametrize("K", [2, 4])
def test_small_nccl_loopback(K):
    base, B = _CONFIGS["small"]
    cfg = base.with_(n_stages=K)
    params, tokens, ref = oracle_run(cfg, B, 3, True)
    loss, logits, grads, _ = gpu_run(cfg, B, params, tokens, [40, 24, 64], tp.TP_BF16, flags=NL)
    errs = worst_errors(loss, logits, grads, ref)
    assert max(errs.values()) < 2e-2, errs


@pytest.mark.parametrize("K,groups", [(2, [(2, [40, 24, 64]), (1, [128]), (1, [8] * 16)]),
                                      (4, [(3, [128]), (1, [32, 32, 32, 32])])])
def test_heterogeneous_plan_nccl_loopback(K, groups):
    base, _ = _CONFIGS["small"]
    cfg = base.with_(n_stages=K)
    params, tokens, ref = oracle_run(cfg, 4, 9, True)
    loss, logits, grads = gpu_run_plan(cfg, 4, params, tokens, groups, tp.TP_BF16, flags=NL)
    errs = worst_errors(loss, logits, grads, ref)
    assert max(errs.values()) < 2e-2, errs


def test_nccl_loopback_equals_aliasing_loopback():
    """The same step with messages through NCCL and with aliased buffers gives identical results
    up to the order of float atomics in the gradient reductions (the messages are exact fp32 copies),
    and the captured NCCL graph replays the eager step."""
    base, B = _CONFIGS["small"]
    cfg = base.with_(n_stages=4)
    params, tokens, _ = oracle_run(cfg, B, 5, False)
    from synth import pack_all_stages, unpack_all_stages
    outs = []
    for fl in (0, tp.TP_FLAG_NCCL_LOOPBACK):
        ctx = tp.Context(cfg, precision=tp.TP_FP32, max_batch=B, device=0, flags=fl)
        try:
            ctx.load_params(pack_all_stages(params, cfg))
            ls = [ctx.step(tp.Slicing([40, 24, 64]), tokens) for _ in range(3)]
            outs.append((ls, ctx.grads()))
        finally:
            ctx.close()
    (la, ga), (lb, gb) = outs
    assert abs(la[0] - lb[0]) <= 1e-6 * abs(la[0]) and abs(lb[0] - lb[2]) <= 1e-6 * abs(lb[0])
    assert float(np.linalg.norm(ga - gb) / np.linalg.norm(ga)) < 1e-6
