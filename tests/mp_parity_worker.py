"""torchrun worker for tests/test_gpu_multi.py: one stage per GPU, NCCL send/recv between stages,
compared with the fp64 oracle on its own stage's gradients (and logits on the last stage)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import paper_2102_07988_b200 as tp
from paper_2102_07988_b200 import dist as tdist
from oracle.model import gpt_forward_backward
from synth import CONFIGS, make_params, make_tokens, pack_stage, unpack_stage
from tests.gpu_util import rel


def main():
    # lengths: "l1,l2,.." (uniform slicing, b = 1) or a batch plan "b:l1,l2;b:l1,.." (tp_step_plan);
    # optional argv[5]: batch size override
    cfg_name, precision, lengths, out_dir = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base, B = CONFIGS[cfg_name]
    if len(sys.argv) > 5:
        B = int(sys.argv[5])
    cfg = base.with_(n_stages=world)
    prec = tp.TP_BF16 if precision == "bf16" else tp.TP_FP32
    params = make_params(cfg, seed=11, bf16=(prec == tp.TP_BF16))
    tokens = make_tokens(cfg, B, seed=12)
    nid = tdist.share_nccl_id(rank)
    ctx = tp.Context(cfg, rank=rank, world=world, nccl_id=nid, precision=prec, max_batch=B, device=local,
                     flags=tp.TP_FLAG_KEEP_LOGITS if rank == world - 1 else 0)
    ctx.load_params(pack_stage(params, cfg, rank))
    if ":" in lengths:
        plan = tp.BatchPlan([(int(g.split(":")[0]), [int(x) for x in g.split(":")[1].split(",")])
                             for g in lengths.split(";")])
        losses = [ctx.step_plan(plan, tokens) for _ in range(2)]  # twice: grads are re-zeroed per step
    else:
        sl = tp.Slicing([int(x) for x in lengths.split(",")])
        losses = [ctx.step(sl, tokens) for _ in range(2)]          # twice: grads are re-zeroed per step
    grads = unpack_stage(ctx.grads(), cfg, rank)
    ref = gpt_forward_backward(params, tokens, cfg.n_layer, cfg.n_head)
    errs = {k: rel(v, ref["grads"][k]) for k, v in grads.items()}
    errs["loss"] = abs(losses[-1] - ref["loss"]) / abs(ref["loss"])
    errs["loss_repeat"] = abs(losses[0] - losses[1]) / abs(losses[0])
    if rank == world - 1:
        errs["logits"] = rel(ctx.logits(B), ref["logits"])
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(errs, f)
    if os.environ.get("TP_TEST_PROFILE") == "1":
        # collective profiling calls: alpha / beta by NCCL ping-pong, the bottleneck table (max over
        # ranks inside the library), the dW constant — identical on every rank
        a, gbs = ctx.profile_comm(reps=3)
        t, _ = ctx.profile(16, reps=3)
        w = ctx.profile_wgrad(B, reps=2)
        with open(os.path.join(out_dir, f"rank{rank}_prof.json"), "w") as f:
            json.dump({"alpha_ns": a, "gbs": gbs, "table": t.tolist(), "wgrad": w}, f)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
