"""Cost-model study (Fig. 4 and :292-298).

On one GPU, one pipeline stage of a GPT-3 shaped model (default: 13B width, 10 of its 40 layers =
one of K = 4 stages): measures the cost table with tp_profile twice -- once with the paper's
least-squares linear context term t_ctx = a0 + a1 l + a2 c + a3 l c (TP_CTX_FIT=linear) and once
with the measured (l, c) grid interpolation used by default -- and reports
  * the base curve t(l, 0) and the stage's tokens/s vs l (the B200 analogue of Fig. 4: throughput
    is flat below the GEMM ridge and saturates above it),
  * the linear fit's coefficients and its max relative error on its own samples (the paper: < 2%),
  * the relative difference between the two tables over all l + c <= s.
Prints one JSON object (rank 0) and writes it to --out.

  python scripts/cost_model_study.py --config gpt3-13b --layers 10 --out profiles/r01_cost_model_13b.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2102_07988_b200 as tp  # noqa: E402
from synth import CONFIGS, make_stage_flat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt3-13b")
    ap.add_argument("--layers", type=int, default=10)
    ap.add_argument("--granularity", type=int, default=64)
    ap.add_argument("--batch-slice", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    base, _ = CONFIGS[args.config]
    cfg = base.with_(n_layer=args.layers, n_stages=1)
    g, b = args.granularity, args.batch_slice
    ctx = tp.Context(cfg, max_batch=b, device=0)
    ctx.load_params(make_stage_flat(cfg, 0, seed=0))
    tables = {}
    for mode in ("linear", "grid"):
        if mode == "linear":
            os.environ["TP_CTX_FIT"] = "linear"
        else:
            os.environ.pop("TP_CTX_FIT", None)
        ticks, fit = ctx.profile(g, reps=args.reps, batch_slice=b)
        tables[mode] = (ticks.astype(np.float64), fit)
    ctx.close()
    n = cfg.seq_len // g
    lin, grid = tables["linear"][0], tables["grid"][0]
    valid = np.zeros_like(lin, dtype=bool)
    for li in range(n):
        valid[li, : n - li] = True  # l + c <= s
    diff = np.abs(lin - grid)[valid] / np.maximum(grid[valid], 1.0)
    ls = np.arange(1, n + 1) * g
    base_ms = grid[:, 0] / 1e6
    out = {
        "config": args.config, "layers": args.layers, "hidden": cfg.hidden, "seq_len": cfg.seq_len,
        "granularity": g, "batch_slice": b,
        "base_curve": [{"l": int(l), "ms": float(t), "tokens_per_s": float(b * l / (t / 1e3))} for l, t in zip(ls, base_ms)],
        "linear_fit": {"a": [float(x) for x in tables["linear"][1][:4]], "max_rel_err_on_samples": float(tables["linear"][1][4])},
        "linear_vs_grid_table": {"max_rel_diff": float(diff.max()), "mean_rel_diff": float(diff.mean()),
                                 "p95_rel_diff": float(np.percentile(diff, 95))},
    }
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
