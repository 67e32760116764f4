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

  python scripts/cost_model_study.py --config gpt3-13b --layers 10 --out profiles/r02_cost_model_13b.json

Also measures the table DENSELY (every (l, c), TP_PROFILE_DENSE=1) and reports both models' error
against it (NEXT(3): the paper's "< 2 %"), and one layer's base curve at --fine-granularity (the
per-layer Fig. 4 curve).
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
    ap.add_argument("--fine-granularity", type=int, default=8)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    base, _ = CONFIGS[args.config]
    cfg = base.with_(n_layer=args.layers, n_stages=1)
    g, b = args.granularity, args.batch_slice
    ctx = tp.Context(cfg, max_batch=b, device=0)
    ctx.load_params(make_stage_flat(cfg, 0, seed=0))
    tables = {}
    for mode in ("linear", "grid", "dense"):
        os.environ.pop("TP_CTX_FIT", None)
        os.environ.pop("TP_PROFILE_DENSE", None)
        if mode == "linear":
            os.environ["TP_CTX_FIT"] = "linear"
        if mode == "dense":
            os.environ["TP_PROFILE_DENSE"] = "1"  # every (l, c) measured
        ticks, fit = ctx.profile(g, reps=args.reps, batch_slice=b)
        tables[mode] = (ticks.astype(np.float64), fit)
    os.environ.pop("TP_PROFILE_DENSE", None)
    ctx.close()
    # Fig. 4 analogue: ONE layer's fwd+bwd latency and throughput vs slice length
    # at a fine granularity
    cfg1 = base.with_(n_layer=1, n_stages=1)
    ctx = tp.Context(cfg1, max_batch=b, device=0)
    ctx.load_params(make_stage_flat(cfg1, 0, seed=0))
    t1, _ = ctx.profile(args.fine_granularity, reps=args.reps, batch_slice=b)
    ctx.close()
    n = cfg.seq_len // g
    lin, grid, dense = tables["linear"][0], tables["grid"][0], tables["dense"][0]
    valid = np.zeros_like(lin, dtype=bool)
    for li in range(n):
        valid[li, : n - li] = True  # l + c <= s
    diff = np.abs(lin - grid)[valid] / np.maximum(grid[valid], 1.0)

    def err(x):
        e = np.abs(x - dense)[valid] / np.maximum(dense[valid], 1.0)
        return {"max_rel_err": float(e.max()), "mean_rel_err": float(e.mean()), "p95_rel_err": float(np.percentile(e, 95)),
                "frac_within_2pct": float((e < 0.02).mean())}
    gf = args.fine_granularity
    fine = [{"l": int((i + 1) * gf), "ms": float(t1[i, 0] / 1e6), "tokens_per_s": float(b * (i + 1) * gf / (t1[i, 0] / 1e9))}
            for i in range(cfg1.seq_len // gf)]
    ls = np.arange(1, n + 1) * g
    base_ms = grid[:, 0] / 1e6
    out = {
        "config": args.config, "layers": args.layers, "hidden": cfg.hidden, "seq_len": cfg.seq_len,
        "granularity": g, "batch_slice": b,
        "base_curve": [{"l": int(l), "ms": float(t), "tokens_per_s": float(b * l / (t / 1e3))} for l, t in zip(ls, base_ms)],
        "linear_fit": {"a": [float(x) for x in tables["linear"][1][:4]], "max_rel_err_on_samples": float(tables["linear"][1][4])},
        "linear_vs_grid_table": {"max_rel_diff": float(diff.max()), "mean_rel_diff": float(diff.mean()),
                                 "p95_rel_diff": float(np.percentile(diff, 95))},
        # the paper's claim: the fitted table is within 2 % of dense profiling
        "linear_fit_vs_dense": err(lin), "grid_interp_vs_dense": err(grid),
        "fig4_one_layer": {"granularity": gf, "curve": fine},
    }
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
