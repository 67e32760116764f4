"""Seeded synthetic inputs shared by the oracle (oracle/) and the CUDA path's tests/bench.

This module holds NO arithmetic of the method (no layer maths, no DP, no cost formula):
only configurations, random number draws, bf16 rounding of inputs, and the flat
parameter layout that `tp_load_params` / `tp_get_grads` use (include/tp.h).

Input recipe:
  * configs follow BASELINE.json:7-11 (tiny, GPT-3 1B, 13B, 13B-long, 175B-24L) plus the
    parity configs of SURVEY.md §8(c) ("parity-mid");
  * vocab: 128 for tiny, 50304 (50257 padded to x64) for GPT-3 shapes (reading A-6);
  * tokens uniform in [0, V), shape [B][s+1], numpy PCG64 seed 1 (A-8, A-25);
  * weights: 'test' init makes every parameter random so every gradient path is non-trivial
    (W, b ~ N(0, 0.02); gamma = 1 + N(0, 0.1); beta ~ N(0, 0.02)); 'gpt2' init is the GPT-2
    recipe (N(0, 0.02), W_o / W_2 scaled by 1/sqrt(2n), zero biases, unit gamma) used by bench.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Tuple

import numpy as np

__all__ = [
    "ModelCfg", "CONFIGS", "param_specs", "stage_param_specs", "stage_layers",
    "make_params", "make_tokens", "round_bf16", "pack_stage", "unpack_stage",
    "pack_all_stages", "stage_param_count", "random_int_table", "gpu_like_table",
]


@dataclasses.dataclass(frozen=True)
class ModelCfg:
    n_layer: int
    hidden: int
    n_head: int
    vocab: int
    seq_len: int
    n_stages: int = 1
    partition: int = 0          # 0 uniform n/K layers per stage; 1 balanced for the LM head (A-30)

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_head

    def with_(self, **kw) -> "ModelCfg":
        return dataclasses.replace(self, **kw)


# BASELINE.json:7-11 and SURVEY.md §8(c) parity configs. Batch sizes live with the callers.
CONFIGS: Dict[str, Tuple[ModelCfg, int]] = {
    "tiny": (ModelCfg(2, 64, 4, 128, 32, 2), 1),              # BASELINE.json:7
    "gpt3-1b": (ModelCfg(24, 2048, 16, 50304, 2048, 1), 8),   # BASELINE.json:8
    "gpt3-13b": (ModelCfg(40, 5120, 40, 50304, 2048, 8), 8),  # BASELINE.json:9
    "gpt3-13b-8k": (ModelCfg(40, 5120, 40, 50304, 8192, 8), 2),  # BASELINE.json:10
    "gpt3-175b-24l": (ModelCfg(24, 12288, 96, 50304, 2048, 8), 2),  # BASELINE.json:11
    "parity-mid": (ModelCfg(2, 5120, 40, 1024, 512, 2), 1),   # SURVEY.md §8(c) parity-mid (vocab reduced)
    "small": (ModelCfg(4, 256, 2, 512, 128, 2), 2),           # several tiles, d=128
    # a head worth ~1.3 layers: the balanced partition (A-30) gives non-uniform stages
    "small-deep": (ModelCfg(8, 256, 2, 4096, 128, 2, 1), 2),
}

LAYER_PARAMS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")


def _layer_shapes(H: int) -> List[Tuple[str, Tuple[int, ...]]]:
    return [("ln1_g", (H,)), ("ln1_b", (H,)), ("w_qkv", (H, 3 * H)), ("b_qkv", (3 * H,)),
            ("w_o", (H, H)), ("b_o", (H,)), ("ln2_g", (H,)), ("ln2_b", (H,)),
            ("w_1", (H, 4 * H)), ("b_1", (4 * H,)), ("w_2", (4 * H, H)), ("b_2", (H,))]


def stage_layer_counts(cfg: ModelCfg) -> List[int]:
    """Layers per stage (the parameter LAYOUT shared with the library, tp_stage_layers; no method
    arithmetic). partition 0: n/K each (uniform cells). partition 1 (DESIGN.md
    A-30): the last stage, which also holds the LM head worth h = V / (12 H + s) layers, gets the nl
    minimising max(ceil((n - nl) / (K - 1)), nl + h) (ties: larger nl); stages 1..r%(K-1) get one
    more of the remaining layers."""
    n, K = cfg.n_layer, cfg.n_stages
    if cfg.partition == 0 or K == 1:
        return [n // K] * K
    h = cfg.vocab / (12.0 * cfg.hidden + cfg.seq_len)
    best_nl, best = n // K, float("inf")
    for nl in range(1, n - (K - 1) + 1):
        r = n - nl
        cost = max(float((r + K - 2) // (K - 1)), nl + h)
        if cost < best or (cost == best and nl > best_nl):
            best, best_nl = cost, nl
    r = n - best_nl
    base, extra = divmod(r, K - 1)
    return [base + (1 if 1 <= k <= extra else 0) for k in range(K - 1)] + [best_nl]


def stage_layers(cfg: ModelCfg, k: int) -> range:
    """Stage k owns a contiguous block of layers (stage_layer_counts)."""
    c = stage_layer_counts(cfg)
    first = sum(c[:k])
    return range(first, first + c[k])


def stage_param_specs(cfg: ModelCfg, k: int) -> List[Tuple[str, Tuple[int, ...]]]:
    """Flat per-stage layout (include/tp.h, 'Parameter layout'):
    stage 0: wte[V][H], wpe[s][H]; each owned layer: LAYER_PARAMS in order (weights stored
    [in][out] row-major); stage K-1: lnf_g[H], lnf_b[H], w_out[H][V]."""
    H, V, s = cfg.hidden, cfg.vocab, cfg.seq_len
    out: List[Tuple[str, Tuple[int, ...]]] = []
    if k == 0:
        out += [("wte", (V, H)), ("wpe", (s, H))]
    for li in stage_layers(cfg, k):
        out += [(f"l{li}.{n}", shp) for n, shp in _layer_shapes(H)]
    if k == cfg.n_stages - 1:
        out += [("lnf_g", (H,)), ("lnf_b", (H,)), ("w_out", (H, V))]
    return out


def param_specs(cfg: ModelCfg) -> List[Tuple[str, Tuple[int, ...]]]:
    out = []
    for k in range(cfg.n_stages):
        out += stage_param_specs(cfg, k)
    return out


def stage_param_count(cfg: ModelCfg, k: int) -> int:
    return sum(int(np.prod(s)) for _, s in stage_param_specs(cfg, k))


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (round-to-nearest-even), returned as float32.
    Precision policy A-23: both sides consume the same bf16-rounded parameters."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = (rounded & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    # keep NaN/Inf untouched (never produced by our generators)
    return out.reshape(x.shape)


def make_params(cfg: ModelCfg, seed: int = 0, init: str = "test",
                bf16: bool = False) -> Dict[str, np.ndarray]:
    """All parameters of the model as float32 arrays keyed by name (see stage_param_specs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = cfg.n_layer
    params: Dict[str, np.ndarray] = {}
    for name, shape in param_specs(cfg):
        base = name.split(".")[-1]
        if init == "test":
            if base.endswith("_g"):
                v = 1.0 + 0.1 * rng.standard_normal(shape)
            else:
                v = 0.02 * rng.standard_normal(shape)
        elif init == "gpt2":
            if base.endswith("_g"):
                v = np.ones(shape)
            elif base.startswith("b_") or base.endswith("_b"):
                v = np.zeros(shape)
            else:
                v = 0.02 * rng.standard_normal(shape, dtype=np.float32)
                if base in ("w_o", "w_2"):
                    v = v / math.sqrt(2.0 * n)
        else:
            raise ValueError(init)
        v = np.asarray(v, dtype=np.float32)
        params[name] = round_bf16(v) if bf16 else v
    return params


def make_tokens(cfg: ModelCfg, batch: int, seed: int = 1) -> np.ndarray:
    """tokens[B][s+1] int32 uniform in [0, V); input = [:, :s], target = [:, 1:] (A-8)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, cfg.vocab, size=(batch, cfg.seq_len + 1), dtype=np.int64).astype(np.int32)


def pack_stage(params: Dict[str, np.ndarray], cfg: ModelCfg, k: int) -> np.ndarray:
    parts = [np.asarray(params[name], dtype=np.float32).reshape(-1) for name, _ in stage_param_specs(cfg, k)]
    return np.concatenate(parts) if parts else np.zeros(0, np.float32)


def pack_all_stages(params: Dict[str, np.ndarray], cfg: ModelCfg) -> np.ndarray:
    return np.concatenate([pack_stage(params, cfg, k) for k in range(cfg.n_stages)])


def unpack_stage(flat: np.ndarray, cfg: ModelCfg, k: int) -> Dict[str, np.ndarray]:
    out, off = {}, 0
    for name, shape in stage_param_specs(cfg, k):
        cnt = int(np.prod(shape))
        out[name] = flat[off:off + cnt].reshape(shape)
        off += cnt
    if off != flat.size:
        raise ValueError(f"flat size {flat.size} != layout size {off}")
    return out


def unpack_all_stages(flat: np.ndarray, cfg: ModelCfg) -> Dict[str, np.ndarray]:
    out, off = {}, 0
    for k in range(cfg.n_stages):
        cnt = stage_param_count(cfg, k)
        out.update(unpack_stage(flat[off:off + cnt], cfg, k))
        off += cnt
    return out


# ---------------------------------------------------------------- planner inputs
def random_int_table(n: int, rng: np.random.Generator, lo: int = 1, hi: int = 20) -> np.ndarray:
    """Random positive integer cost table t[l-1][c] (units of g) with l+c <= n; other entries 0.
    Shape [n][n+1], the layout of tp_cost_table.ticks (include/tp.h)."""
    t = np.zeros((n, n + 1), dtype=np.int64)
    for l in range(1, n + 1):
        for c in range(0, n - l + 1):
            t[l - 1, c] = rng.integers(lo, hi + 1)
    return t


def gpu_like_table(n: int, rng: np.random.Generator, knee: int = 32, base_ns: int = 200_000,
                   per_unit_ns: int = 6_000, ctx_ns: int = 900, noise: float = 0.01) -> np.ndarray:
    """A synthetic table shaped like a measured GPU stage: flat until `knee` units, then linear
    in the slice length, plus a context term growing with l*c (PAPER.md:218-223 qualitative shape),
    with multiplicative noise. Integer ns ticks, layout [n][n+1]. Generator only: the planner does
    not assume any of this structure."""
    t = np.zeros((n, n + 1), dtype=np.int64)
    for l in range(1, n + 1):
        base = base_ns + per_unit_ns * max(0, l - knee)
        for c in range(0, n - l + 1):
            v = (base + ctx_ns * l * c / 8.0) * (1.0 + noise * rng.standard_normal())
            t[l - 1, c] = max(1, int(round(v)))
    return t


def _tensor_seed(seed: int, name: str) -> int:
    h = 1469598103934665603
    for ch in name.encode():
        h = ((h ^ ch) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return (h ^ (seed * 0x9E3779B97F4A7C15)) & 0xFFFFFFFFFFFFFFFF


def make_stage_flat(cfg: ModelCfg, k: int, seed: int = 0, init: str = "gpt2") -> np.ndarray:
    """Flat float32 parameters of stage k only (bench at GPT-3 sizes: a rank builds just its stage).
    Same recipes as make_params, but every tensor is a window, at a per-(seed, name) random offset,
    of one 2^24-entry N(0, 1) pool, tiled — so multi-GB stages are built at memcpy speed. Values do
    not affect the dense cost being measured."""
    pool_rng = np.random.Generator(np.random.PCG64(seed))
    pool = pool_rng.standard_normal(1 << 24, dtype=np.float32)
    out = np.empty(stage_param_count(cfg, k), dtype=np.float32)
    off = 0
    for name, shape in stage_param_specs(cfg, k):
        cnt = int(np.prod(shape))
        base = name.split(".")[-1]
        dst = out[off:off + cnt]
        if base.endswith("_g"):
            dst[:] = 1.0
        elif init == "gpt2" and (base.startswith("b_") or base.endswith("_b")):
            dst[:] = 0.0
        else:
            start = _tensor_seed(seed, name) % pool.size
            scale = 0.02 / (math.sqrt(2.0 * cfg.n_layer) if base in ("w_o", "w_2") else 1.0)
            done = 0
            while done < cnt:
                take = min(cnt - done, pool.size - start)
                np.multiply(pool[start:start + take], scale, out=dst[done:done + take])
                done += take
                start = 0
        off += cnt
    return out
