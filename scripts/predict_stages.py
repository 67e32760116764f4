"""Model-based estimate for pipeline depths that cannot be measured here (8 GPUs were not
available): for K stages of n_layer / K layers, the bottleneck cost table of PAPER.md:292-298 is
measured on ONE GPU as the element-wise max over the stage types (A-16): a loopback
context holding a first stage (embedding + n/K layers) and a last stage (n/K layers + LM head + CE)
— a middle stage does a subset of the first stage's work — for every batch-slice size b, plus the
data-transmission term alpha + 4 H T / beta measured on 2 GPUs (TP_COMM_ALPHA_NS / TP_COMM_GBS,
PAPER.md:243) and the deferred weight-gradient constant (tp_profile_wgrad). For each K it asks the
planner for the joint plan (tp_plan_joint, A-20b) and computes the unsliced GPipe makespan
(B/b + K - 1) * t(s, 0) on the same table; predicted step = makespan + dW.

  TP_COMM_ALPHA_NS=... TP_COMM_GBS=... python scripts/predict_stages.py --config gpt3-13b --stages 4,8
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
    ap.add_argument("--stages", default="4,8")
    ap.add_argument("--granularity", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    base, B = CONFIGS[args.config]
    g = args.granularity
    n = base.seq_len // g
    lines = []
    for K in [int(x) for x in args.stages.split(",")]:
        L = base.n_layer // K
        types = min(K, 2)
        cfg = base.with_(n_layer=L * types, n_stages=types, partition=0)  # uniform cells
        ctx = tp.Context(cfg, max_batch=B, device=0)
        ctx.load_params(np.concatenate([make_stage_flat(cfg, k, seed=0) for k in range(types)]))
        bsl = [b for b in (1, 2, 4, 8, 16) if B % b == 0 and b <= B]
        tables = {b: ctx.profile(g, reps=args.reps, batch_slice=b)[0] for b in bsl}
        wgrad = ctx.profile_wgrad(B)
        ctx.close()
        plan = tp.plan_joint(tables, g, base.n_layer, base.hidden, base.seq_len, K, B)
        gpipe = min(((B // b + K - 1) * int(t[n - 1, 0]), b) for b, t in tables.items())
        line = {"config": args.config, "stages": K, "layers_per_stage": L, "batch": B,
                "dp_plan": plan.notation(), "dp_predicted_ms": plan.predicted / 1e6,
                "gpipe_plan": f"[({gpipe[1]}, [{base.seq_len}])] * {B // gpipe[1]}", "gpipe_predicted_ms": gpipe[0] / 1e6,
                "wgrad_ms": wgrad / 1e6,
                "dp_predicted_step_ms": (plan.predicted + wgrad) / 1e6,
                "gpipe_predicted_step_ms": (gpipe[0] + wgrad) / 1e6,
                "predicted_speedup": (gpipe[0] + wgrad) / (plan.predicted + wgrad),
                "comm": {"alpha_ns": os.environ.get("TP_COMM_ALPHA_NS"), "gbs": os.environ.get("TP_COMM_GBS")},
                "note": "bottleneck table = max over the first / last stage types measured on one GPU "
                        "(A-16), + p2p term when TP_COMM_* are set, + the dW constant"}
        print(json.dumps(line), flush=True)
        lines.append(line)
    if args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
