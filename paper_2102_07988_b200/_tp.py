"""ctypes binding of include/tp.h — argument marshalling only; every step runs in libtp.so.

Loading fails loudly (ImportError) when libtp.so is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TP_LIB: an alternative build of the same library (A/B of kernel variants across two builds)
LIB_PATH = os.environ.get("TP_LIB") or os.path.join(_HERE, "libtp.so")

TP_OK, TP_EINVAL, TP_EINFEASIBLE, TP_ETOOBIG, TP_ECUDA, TP_ENCCL, TP_ENOMEM, TP_ESTATE = 0, -1, -2, -3, -4, -5, -6, -7
TP_BF16, TP_FP32 = 0, 1
TP_FLAG_KEEP_LOGITS, TP_FLAG_KERNEL_STATS, TP_FLAG_FORCE_SIMT, TP_FLAG_NCCL_LOOPBACK, TP_FLAG_DEVICE_P2P = 1, 2, 4, 8, 16
TP_FLAG_SCHEDULE_1F1B = 32
TP_PARTITION_UNIFORM, TP_PARTITION_BALANCED = 0, 1

EXPORTED = ["tp_plan", "tp_plan_joint", "tp_schedule_oplist", "tp_stage_layers", "tp_step_plan", "tp_step_plan_device", "tp_stage_param_count", "tp_nccl_unique_id", "tp_init", "tp_param_count",
            "tp_load_params", "tp_step", "tp_step_device", "tp_get_grads", "tp_get_logits",
            "tp_profile", "tp_profile_wgrad", "tp_profile_comm", "tp_get_stream", "tp_kernel_stats", "tp_kernel_stats_reset", "tp_kernel_stats_enable",
            "tp_last_step_launches", "tp_destroy", "tp_last_error"]
KEXPORTED = ["tpk_gemm", "tpk_attention_fwd", "tpk_attention_bwd", "tpk_layernorm_fwd", "tpk_layernorm_bwd"]


class TpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"tp status {status}: {msg}")
        self.status = status


class ModelCfgC(C.Structure):
    _fields_ = [("n_layer", C.c_int32), ("hidden", C.c_int32), ("n_head", C.c_int32),
                ("vocab", C.c_int32), ("seq_len", C.c_int32), ("n_stages", C.c_int32), ("partition", C.c_int32)]


class CostTableC(C.Structure):
    _fields_ = [("granularity", C.c_int32), ("n_units", C.c_int32),
                ("ticks", C.POINTER(C.c_int64)), ("ticks_per_ms", C.c_int64)]


class SlicingC(C.Structure):
    _fields_ = [("batch_slice", C.c_int32), ("n_slices", C.c_int32), ("capacity", C.c_int32),
                ("lengths", C.POINTER(C.c_int32)), ("t_max_ticks", C.c_int64),
                ("predicted_ticks", C.c_int64)]


class BatchPlanC(C.Structure):
    _fields_ = [("n_groups", C.c_int32), ("capacity_groups", C.c_int32), ("batch_slice", C.POINTER(C.c_int32)),
                ("n_slices", C.POINTER(C.c_int32)), ("capacity_lengths", C.c_int32),
                ("lengths", C.POINTER(C.c_int32)), ("t_max_ticks", C.c_int64), ("predicted_ticks", C.c_int64)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built — run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sigs = {
        "tp_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(CostTableC), C.c_int32,
                              C.c_int64, C.POINTER(SlicingC)]),
        "tp_plan_joint": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                    C.POINTER(C.POINTER(CostTableC)), C.c_int32, C.c_int64, C.POINTER(BatchPlanC)]),
        "tp_step_plan": (C.c_int, [P, C.POINTER(BatchPlanC), P, C.c_int32, C.POINTER(C.c_float)]),
        "tp_step_plan_device": (C.c_int, [P, C.POINTER(BatchPlanC), P, C.c_int32, C.POINTER(C.c_float)]),
        "tp_stage_param_count": (C.c_int, [C.POINTER(ModelCfgC), C.c_int32, C.POINTER(C.c_size_t)]),
        "tp_stage_layers": (C.c_int, [C.POINTER(ModelCfgC), C.POINTER(C.c_int32)]),
        "tp_schedule_oplist": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "tp_nccl_unique_id": (C.c_int, [P]),
        "tp_init": (C.c_int, [C.POINTER(ModelCfgC), C.c_int32, C.c_int32, P, C.c_int32, C.c_int32, C.c_int32,
                              C.c_int32, C.POINTER(P)]),
        "tp_param_count": (C.c_int, [P, C.POINTER(C.c_size_t)]),
        "tp_load_params": (C.c_int, [P, P, C.c_size_t]),
        "tp_step": (C.c_int, [P, C.POINTER(SlicingC), P, C.c_int32, C.POINTER(C.c_float)]),
        "tp_step_device": (C.c_int, [P, C.POINTER(SlicingC), P, C.c_int32, C.POINTER(C.c_float)]),
        "tp_get_grads": (C.c_int, [P, P, C.c_size_t]),
        "tp_get_logits": (C.c_int, [P, P, C.c_size_t]),
        "tp_profile": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, P, P]),
        "tp_profile_wgrad": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
        "tp_profile_comm": (C.c_int, [P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "tp_get_stream": (C.c_int, [P, C.POINTER(P)]),
        "tp_kernel_stats": (C.c_int, [P, C.c_int32, C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
        "tp_kernel_stats_reset": (C.c_int, [P]),
        "tp_kernel_stats_enable": (C.c_int, [P, C.c_int32]),
        "tp_last_step_launches": (C.c_int, [P, C.POINTER(C.c_int64)]),
        "tp_destroy": (None, [P]),
        "tpk_gemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, P, C.c_int64, C.c_int32, P, C.c_int64, C.c_int32,
                               P, C.c_int64, C.c_int32, P]),
        "tpk_attention_fwd": (C.c_int, [P, P, P, P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, P]),
        "tpk_attention_bwd": (C.c_int, [P, P, P, P, P, P, P, C.c_int64, P, P, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.c_int32, C.c_int32, P]),
        "tpk_layernorm_fwd": (C.c_int, [P, P, P, P, P, P, C.c_int32, C.c_int32, P]),
        "tpk_layernorm_bwd": (C.c_int, [P, P, P, P, P, P, P, P, P, P, P, C.c_int32, C.c_int32, P]),
        "tp_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()


def lib() -> C.CDLL:
    return _lib


def _check(st: int) -> None:
    if st != TP_OK:
        raise TpError(st, (_lib.tp_last_error() or b"").decode())


def _cfg(cfg) -> ModelCfgC:
    return ModelCfgC(cfg.n_layer, cfg.hidden, cfg.n_head, cfg.vocab, cfg.seq_len, cfg.n_stages,
                     int(getattr(cfg, "partition", 0)))


class Slicing:
    """A slicing scheme [(b, [l_1..l_M])] * (B/b) (PAPER.md:494-641 notation)."""

    def __init__(self, lengths: Sequence[int], batch_slice: int = 1, t_max: int = 0, predicted: int = 0):
        self.lengths = [int(x) for x in lengths]
        self.batch_slice = int(batch_slice)
        self.t_max = int(t_max)
        self.predicted = int(predicted)
        self._arr = (C.c_int32 * max(1, len(self.lengths)))(*self.lengths)
        self._c = SlicingC(self.batch_slice, len(self.lengths), len(self.lengths), self._arr,
                           self.t_max, self.predicted)

    @property
    def c(self) -> SlicingC:
        return self._c

    def notation(self, batch: int) -> str:
        return f"[({self.batch_slice}, {self.lengths})] * {batch // self.batch_slice}"

    def __repr__(self):
        return f"Slicing({self.lengths})"


def plan(ticks: np.ndarray, granularity: int, n_layer: int, hidden: int, seq_len: int, n_stages: int,
         n_micro: int = 1, eps_ticks: int = 0, ticks_per_ms: int = 1_000_000) -> Slicing:
    """tp_plan (include/tp.h): the DP of PAPER.md:254-290 over t[l-1][c] (int64 ticks, [n][n+1])."""
    n = seq_len // granularity if granularity > 0 else 0
    t = np.ascontiguousarray(ticks, dtype=np.int64)
    if t.shape != (n, n + 1):
        raise TpError(TP_EINVAL, f"ticks shape {t.shape} != ({n}, {n + 1})")
    table = CostTableC(granularity, n, t.ctypes.data_as(C.POINTER(C.c_int64)), ticks_per_ms)
    buf = (C.c_int32 * max(1, n))()
    out = SlicingC(1, 0, n, buf, 0, 0)
    _check(_lib.tp_plan(n_layer, hidden, seq_len, n_stages, C.byref(table), n_micro, eps_ticks, C.byref(out)))
    return Slicing([buf[i] for i in range(out.n_slices)], out.batch_slice, out.t_max_ticks, out.predicted_ticks)


class BatchPlan:
    """A batch plan [(b_1, l^1), (b_2, l^2), ..]: group d = b_d consecutive
    sequences with its own token slicing. Uniform slicings are the special case of identical groups."""

    def __init__(self, groups: Sequence[Tuple[int, Sequence[int]]], t_max: int = 0, predicted: int = 0):
        self.groups = [(int(b), [int(x) for x in ls]) for b, ls in groups]
        self.t_max = int(t_max)
        self.predicted = int(predicted)
        D = len(self.groups)
        flat = [x for _, ls in self.groups for x in ls]
        self._b = (C.c_int32 * max(1, D))(*[b for b, _ in self.groups])
        self._m = (C.c_int32 * max(1, D))(*[len(ls) for _, ls in self.groups])
        self._l = (C.c_int32 * max(1, len(flat)))(*flat)
        self._c = BatchPlanC(D, D, self._b, self._m, len(flat), self._l, self.t_max, self.predicted)

    @classmethod
    def uniform(cls, slicing: "Slicing", batch: int) -> "BatchPlan":
        return cls([(slicing.batch_slice, slicing.lengths)] * (batch // slicing.batch_slice), slicing.t_max,
                   slicing.predicted)

    @property
    def c(self) -> BatchPlanC:
        return self._c

    def batch(self) -> int:
        return sum(b for b, _ in self.groups)

    def notation(self) -> str:
        """The paper's notation, runs of identical groups collapsed: [(b, [l..])] * k + ..."""
        runs: List[List] = []
        for g in self.groups:
            if runs and runs[-1][0] == g:
                runs[-1][1] += 1
            else:
                runs.append([g, 1])
        return " + ".join(f"[({b}, {ls})] * {k}" for (b, ls), k in runs)

    def __repr__(self):
        return f"BatchPlan({self.groups})"


def plan_joint(tables: Dict[int, np.ndarray], granularity: int, n_layer: int, hidden: int, seq_len: int,
               n_stages: int, batch: int, eps_ticks: int = 0, ticks_per_ms: int = 1_000_000) -> BatchPlan:
    """tp_plan_joint (include/tp.h): per-b tables t_b[l-1][c] -> the batch plan minimising the
    pipelined makespan (A-20b)."""
    n = seq_len // granularity if granularity > 0 else 0
    bs = sorted(int(b) for b in tables)
    arrs = [np.ascontiguousarray(tables[b], dtype=np.int64) for b in bs]
    for b, t in zip(bs, arrs):
        if t.shape != (n, n + 1):
            raise TpError(TP_EINVAL, f"table for b={b}: shape {t.shape} != ({n}, {n + 1})")
    cts = [CostTableC(granularity, n, t.ctypes.data_as(C.POINTER(C.c_int64)), ticks_per_ms) for t in arrs]
    ptrs = (C.POINTER(CostTableC) * len(cts))(*[C.pointer(ct) for ct in cts])
    bvals = (C.c_int32 * len(bs))(*bs)
    gb, gm = (C.c_int32 * batch)(), (C.c_int32 * batch)()
    lens = (C.c_int32 * max(1, batch * n))()
    out = BatchPlanC(0, batch, gb, gm, batch * n, lens, 0, 0)
    _check(_lib.tp_plan_joint(n_layer, hidden, seq_len, n_stages, len(bs), bvals, ptrs, batch, eps_ticks,
                              C.byref(out)))
    groups, pos = [], 0
    for d in range(out.n_groups):
        groups.append((gb[d], [lens[pos + i] for i in range(gm[d])]))
        pos += gm[d]
    return BatchPlan(groups, out.t_max_ticks, out.predicted_ticks)


def schedule_oplist(n_stages: int, stage: int, groups: Sequence[int], one_f_one_b: bool = False) -> List[Tuple[str, int]]:
    """tp_schedule_oplist: the op list tp_step runs on `stage` for groups of groups[d] slices, as
    ("F" | "B", job) pairs (oracle/plan.py's format)."""
    g = (C.c_int32 * max(1, len(groups)))(*groups)
    cap = 2 * sum(groups)
    out = (C.c_int32 * max(1, cap))()
    n = C.c_int32()
    _check(_lib.tp_schedule_oplist(n_stages, stage, 1 if one_f_one_b else 0, len(groups), g, cap, out, C.byref(n)))
    return [("F", v - 1) if v > 0 else ("B", -v - 1) for v in out[:n.value]]


def stage_layers(cfg) -> List[int]:
    """tp_stage_layers: layers per stage under cfg.partition."""
    out = (C.c_int32 * cfg.n_stages)()
    _check(_lib.tp_stage_layers(C.byref(_cfg(cfg)), out))
    return list(out)


def stage_param_count(cfg, stage: int) -> int:
    n = C.c_size_t()
    _check(_lib.tp_stage_param_count(C.byref(_cfg(cfg)), stage, C.byref(n)))
    return n.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.tp_nccl_unique_id(buf))
    return buf.raw


class Context:
    """tp_ctx: one process per GPU (or all stages on one GPU when world == 1)."""

    def __init__(self, cfg, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 precision: int = TP_BF16, max_batch: int = 1, device: int = 0, flags: int = 0):
        self.cfg = cfg
        self.max_batch = max_batch
        self._h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(_lib.tp_init(C.byref(_cfg(cfg)), rank, world, idbuf, precision, max_batch, device, flags,
                            C.byref(self._h)))

    def close(self):
        if self._h:
            _lib.tp_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def param_count(self) -> int:
        n = C.c_size_t()
        _check(_lib.tp_param_count(self._h, C.byref(n)))
        return n.value

    def load_params(self, flat: np.ndarray) -> None:
        a = np.ascontiguousarray(flat, dtype=np.float32)
        _check(_lib.tp_load_params(self._h, a.ctypes.data, a.size))

    def _tokens(self, tokens: np.ndarray) -> np.ndarray:
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.ndim != 2 or tok.shape[1] != self.cfg.seq_len + 1:
            raise TpError(TP_EINVAL, f"tokens shape {tok.shape} != (batch, seq_len + 1 = {self.cfg.seq_len + 1})")
        return tok

    def step(self, slicing: Slicing, tokens: np.ndarray) -> float:
        tok = self._tokens(tokens)
        loss = C.c_float()
        _check(_lib.tp_step(self._h, C.byref(slicing.c), tok.ctypes.data, tok.shape[0], C.byref(loss)))
        return loss.value

    def step_device(self, slicing: Slicing, dev_tokens_ptr: int, batch: int) -> float:
        loss = C.c_float()
        _check(_lib.tp_step_device(self._h, C.byref(slicing.c), C.c_void_p(dev_tokens_ptr), batch, C.byref(loss)))
        return loss.value

    def step_plan(self, plan: BatchPlan, tokens: np.ndarray) -> float:
        tok = self._tokens(tokens)
        loss = C.c_float()
        _check(_lib.tp_step_plan(self._h, C.byref(plan.c), tok.ctypes.data, tok.shape[0], C.byref(loss)))
        return loss.value

    def step_plan_device(self, plan: BatchPlan, dev_tokens_ptr: int, batch: int) -> float:
        loss = C.c_float()
        _check(_lib.tp_step_plan_device(self._h, C.byref(plan.c), C.c_void_p(dev_tokens_ptr), batch,
                                        C.byref(loss)))
        return loss.value

    def grads(self) -> np.ndarray:
        out = np.empty(self.param_count(), dtype=np.float32)
        _check(_lib.tp_get_grads(self._h, out.ctypes.data, out.size))
        return out

    def logits(self, batch: int) -> np.ndarray:
        c = self.cfg
        out = np.empty((batch, c.seq_len, c.vocab), dtype=np.float32)
        _check(_lib.tp_get_logits(self._h, out.ctypes.data, out.size))
        return out

    def profile(self, granularity: int, reps: int = 5, batch_slice: int = 1) -> Tuple[np.ndarray, np.ndarray]:
        n = self.cfg.seq_len // granularity
        ticks = np.zeros((n, n + 1), dtype=np.int64)
        fit = np.zeros(5, dtype=np.float64)
        _check(_lib.tp_profile(self._h, granularity, batch_slice, reps, ticks.ctypes.data, fit.ctypes.data))
        return ticks, fit

    def profile_wgrad(self, batch: int, reps: int = 3) -> int:
        """ns of one step's deferred weight-gradient GEMMs (slowest stage type / rank)."""
        ns = C.c_int64()
        _check(_lib.tp_profile_wgrad(self._h, batch, reps, C.byref(ns)))
        return ns.value

    def profile_comm(self, reps: int = 5) -> Tuple[float, float]:
        """(alpha_ns, GB/s) of one stage message, measured by NCCL ping-pong (collective, world > 1)."""
        a, b = C.c_double(), C.c_double()
        _check(_lib.tp_profile_comm(self._h, reps, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stream(self) -> int:
        p = C.c_void_p()
        _check(_lib.tp_get_stream(self._h, C.byref(p)))
        return p.value or 0

    def kernel_stats(self) -> Dict[str, Dict[str, float]]:
        n = C.c_int32()
        _check(_lib.tp_kernel_stats(self._h, -1, None, None, None, None, None, C.byref(n)))
        out = {}
        for i in range(n.value):
            name = C.create_string_buffer(32)
            la, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            _check(_lib.tp_kernel_stats(self._h, i, name, C.byref(la), C.byref(ms), C.byref(fl), C.byref(by), None))
            out[name.value.decode()] = {"launches": la.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
        return out

    def kernel_stats_reset(self) -> None:
        _check(_lib.tp_kernel_stats_reset(self._h))

    def kernel_stats_enable(self, on: bool) -> None:
        _check(_lib.tp_kernel_stats_enable(self._h, 1 if on else 0))

    def last_step_launches(self) -> int:
        n = C.c_int64()
        _check(_lib.tp_last_step_launches(self._h, C.byref(n)))
        return n.value


# ---------------------------------------------------------------- kernel-level entry points (tp_kernels.h)
def k_gemm(M, N, K, A_ptr, lda, a_mn, B_ptr, ldb, b_mn, out_ptr, ldo, impl=0, stream=0):
    _check(_lib.tpk_gemm(M, N, K, A_ptr, lda, int(a_mn), B_ptr, ldb, int(b_mn), out_ptr, ldo, impl, stream))


def k_attention_fwd(q, k, v, o, lse, a, s, d, c, l, impl=0, stream=0):
    _check(_lib.tpk_attention_fwd(q, k, v, o, lse, a, s, d, c, l, impl, stream))


def k_attention_bwd(dO, o, q, k, v, lse, dq, ldq, dk_acc, dv_acc, a, s, d, c, l, accumulate, impl=0, stream=0):
    _check(_lib.tpk_attention_bwd(dO, o, q, k, v, lse, dq, ldq, dk_acc, dv_acc, a, s, d, c, l, accumulate, impl,
                                  stream))


def k_layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, H, stream=0):
    _check(_lib.tpk_layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, H, stream))


def k_layernorm_bwd(dy, x, mean, rstd, gamma, resid, dx_out, dx_copy, dgamma, dbeta, dbias, rows, H, stream=0):
    _check(_lib.tpk_layernorm_bwd(dy, x, mean, rstd, gamma, resid, dx_out, dx_copy, dgamma, dbeta, dbias, rows, H,
                                  stream))
