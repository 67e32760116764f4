"""Model-based estimate for pipeline depths that cannot be measured here (8 GPUs were not
available): profiles ONE pipeline stage of a GPT-3 shaped model on one GPU (n_layer / K layers,
the cost tables of PAPER.md:292-298 for every batch-slice size b), then for each K asks the planner
for the joint plan (tp_plan_joint, A-20b) and computes the unsliced GPipe makespan
(B/b + K - 1) * t(s, 0) with the same table. Prints one JSON object per K: the predicted DP and GPipe
step times (one stage's fwd+bwd only: no weight-gradient GEMMs, no communication) and their ratio.
The K = 4 line can be compared with the measured 4 x B200 runs (profiles/r01_pipe_*_n4.json).

  python scripts/predict_stages.py --config gpt3-13b --stages 4,8 --out profiles/r01_predict_13b.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2102_07988_b200 as tp  # noqa: E402
from synth import CONFIGS, make_stage_flat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt3-13b")
    ap.add_argument("--stages", default="4,8")
    ap.add_argument("--granularity", type=int, default=64)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    base, B = CONFIGS[args.config]
    g = args.granularity
    n = base.seq_len // g
    lines = []
    for K in [int(x) for x in args.stages.split(",")]:
        cfg = base.with_(n_layer=base.n_layer // K, n_stages=1)
        ctx = tp.Context(cfg, max_batch=B, device=0)
        ctx.load_params(make_stage_flat(cfg, 0, seed=0))
        bsl = [b for b in (1, 2, 4, 8, 16) if B % b == 0 and b <= B]
        tables = {b: ctx.profile(g, reps=5, batch_slice=b)[0] for b in bsl}
        ctx.close()
        plan = tp.plan_joint(tables, g, base.n_layer, base.hidden, base.seq_len, K, B)
        gpipe = min(((B // b + K - 1) * int(t[n - 1, 0]), b) for b, t in tables.items())
        line = {"config": args.config, "stages": K, "layers_per_stage": cfg.n_layer, "batch": B,
                "dp_plan": plan.notation(), "dp_predicted_ms": plan.predicted / 1e6,
                "gpipe_plan": f"[({gpipe[1]}, [{base.seq_len}])] * {B // gpipe[1]}", "gpipe_predicted_ms": gpipe[0] / 1e6,
                "predicted_speedup": gpipe[0] / plan.predicted,
                "note": "one stage's fwd+bwd cost model only (no dW GEMMs, no p2p), K stages assumed identical"}
        print(json.dumps(line), flush=True)
        lines.append(line)
    if args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
