"""World-size-2 gloo tests (CPU) of the multi-process host logic used by bench.py at N > 1:
NCCL-id sharing, the bottleneck (max over stages) cost table, and that all ranks plan the same
slicing with tp_plan (host-only)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2102_07988_b200 as tp
    from paper_2102_07988_b200 import dist as tdist
    from synth import gpu_like_table
    try:
        nid = tdist.share_nccl_id(rank, make_id=lambda: bytes(range(128)))
        n = 32
        t = gpu_like_table(n, np.random.default_rng(rank), knee=4, base_ns=50_000 * (1 + rank))
        tb = tdist.bottleneck_table(t)
        sl = tp.plan(tb, 8, n_layer=4, hidden=64, seq_len=8 * n, n_stages=world, n_micro=4)
        q.put((rank, nid, tb, sl.lengths, tdist.agreed(sl.lengths), tdist.max_over_ranks(float(rank))))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from synth import gpu_like_table
    t0 = gpu_like_table(32, np.random.default_rng(0), knee=4, base_ns=50_000)
    t1 = gpu_like_table(32, np.random.default_rng(1), knee=4, base_ns=100_000)
    for rank, nid, tb, lens, ok, mx in res:
        assert nid == bytes(range(128))
        assert np.array_equal(tb, np.maximum(t0, t1))
        assert ok and mx == 1.0
    assert res[0][3] == res[1][3] and sum(res[0][3]) == 256
