"""Host-side plumbing for one-process-per-GPU runs (torch.distributed is used only here and only
for plumbing): share the library's NCCL unique id, build the bottleneck cost table (element-wise
max over stages, A-16) and check that every rank plans the same slicing."""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _tp


def _dev():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def share_nccl_id(rank: int, make_id=None) -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId (tp_nccl_unique_id) and broadcasts it."""
    buf = torch.zeros(128, dtype=torch.uint8, device=_dev())
    if rank == 0:
        raw = (make_id or _tp.nccl_unique_id)()
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def bottleneck_table(ticks: np.ndarray) -> np.ndarray:
    """Element-wise max of every stage's measured t(l, c) table (A-16)."""
    t = torch.from_numpy(np.ascontiguousarray(ticks, dtype=np.int64)).to(_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def agreed(values) -> bool:
    """True iff every rank passed identical integer values (e.g. the planned slice lengths)."""
    v = torch.tensor(list(values), dtype=torch.int64, device=_dev())
    lo, hi = v.clone(), v.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    return bool(torch.equal(lo, hi))


def max_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=_dev())
    dist.all_reduce(t)
    return float(t.item())
