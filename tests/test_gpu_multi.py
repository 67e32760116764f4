"""Multi-GPU (NCCL send/recv over NVLink) parity: K = world stages, one process per GPU, against
the fp64 oracle. Skipped when fewer GPUs are visible."""
import json
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


@pytest.mark.parametrize("g", ["1", "2"])
def test_small_two_stages_group_dw(g, tmp_path):
    """TP_GROUP_DW=g: the first stage computes the weight gradients of every run of g finished groups
    in order (three groups of different b: flushes of one or two groups, then the rest at the end)."""
    for errs in run(2, "small", "bf16", "1:40,24,64;1:128;2:64,64", tmp_path, batch=4, env={"TP_GROUP_DW": g}):
        assert max(errs.values()) < 2e-2, errs


def test_small_four_stages_nccl(tmp_path):
    for errs in run(4, "small", "bf16", "40,24,64", tmp_path):
        assert max(errs.values()) < 2e-2, errs


def test_small_two_stages_heterogeneous_batch_plan(tmp_path):
    """tp_step_plan over NCCL: groups of different batch-slice sizes with their own slicings (jobs
    of different row counts and message sizes on the p2p edges)."""
    for errs in run(2, "small", "bf16", "2:40,24,64;1:128", tmp_path, batch=3):
        assert max(errs.values()) < 2e-2, errs
