#!/usr/bin/env python
"""bench.py — one JSON line for the driver.

A step = one synchronous tp_step_plan: token-sliced, pipelined forward+backward of one batch of a
GPT-3 shaped model (BASELINE.json:5, metric BASELINE.json:2) with the batch x token plan chosen by
tp_plan_joint from the cost tables tp_profile measured on this box for every batch-slice size b
(the max over stages, A-16, A-20b). The unsliced GPipe schedule [(b, [s])] * B/b
(best predicted b) on the same kernels is timed beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt3-1b] [--impl reference]

N = 1: the GPT-3 1B config (BASELINE.json:8) on one GPU (K = 1 stage). N > 1 (torchrun): K = N
pipeline stages, one process per GPU, NCCL send/recv between neighbours; total work is fixed
(strong scaling). `value` = tokens of the batch / max-over-ranks device time per step.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd iteration latency & tokens/s, 1/2/4/8 B200, MFU vs unsliced pipeline"


def model_flops(cfg, B):
    """Algorithmic FLOPs of one iteration: B*[n*(72 s H^2 + 6 H s (s+1)) + 6 s H V]."""
    n, H, s, V = cfg.n_layer, cfg.hidden, cfg.seq_len, cfg.vocab
    return B * (n * (72.0 * s * H * H + 6.0 * H * s * (s + 1)) + 6.0 * s * H * V)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region. nvidia-smi
    takes up to a second to start reporting, so start() waits for its first line and stop() keeps
    only the lines that arrived after that (a short timed region, e.g. 5 x 50 ms at N = 4, would
    otherwise see no sample at all)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = str(gpu_index)
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.n0 = len(self.lines)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "n0", 0):]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8 or parts[0] != self.idx:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_sample(cfg, B, reps=1, warmup=0):
    """The fp64 oracle (oracle/model.py) as it stands, on a bounded sample of the workload: one
    sequence through embedding + ONE layer + LM head at the config's full width, seq_len and vocab,
    fwd+bwd (median of `reps` timed runs after `warmup`). Extrapolated to the whole model with the
    algorithmic FLOP model (n layers + head), reported as tokens/s."""
    from oracle.model import gpt_forward_backward
    from synth import make_params, make_tokens
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    one = cfg.with_(n_layer=1, n_stages=1)
    params = make_params(one, seed=0, init="gpt2")
    tokens = make_tokens(one, 1, seed=1)
    times = []
    for i in range(warmup + reps):
        t0 = time.time()
        gpt_forward_backward(params, tokens, 1, one.n_head)
        if i >= warmup:
            times.append(time.time() - t0)
    dt = statistics.median(times)
    H, s, V, n = cfg.hidden, cfg.seq_len, cfg.vocab, cfg.n_layer
    layer = 72.0 * s * H * H + 6.0 * H * s * (s + 1)
    head = 6.0 * s * H * V
    t_seq = dt * (n * layer + head) / (layer + head)
    tokps = s / t_seq
    return {"value": tokps, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"fp64 numpy oracle, 1 sequence x (embed + 1 of {n} layers + LM head) at H={H}, s={s}, "
                      f"V={V}, fwd+bwd, median {dt:.1f} s of {reps}; extrapolated by algorithmic FLOPs to {n} layers "
                      f"(t_seq = {t_seq:.0f} s)"}


# The JSON result line is the only thing on stdout: keep a private handle on the original stdout and
# point fd 1 at stderr, so banners printed by native libraries (e.g. NCCL's version line at
# communicator init) cannot interleave with it.
_RESULT_OUT = None


def emit(line):
    global _RESULT_OUT
    out = _RESULT_OUT if _RESULT_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _isolate_stdout():
    global _RESULT_OUT
    sys.stdout.flush()
    _RESULT_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    _isolate_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="gpt3-1b")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--max-batch", type=int, default=0,
                    help="sequences the stage buffers hold (default: the batch; 1F1B may use fewer, DESIGN.md A-27)")
    ap.add_argument("--granularity", type=int, default=64)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-gpipe", action="store_true")
    ap.add_argument("--profile-reps", type=int, default=7, help="tp_profile repetitions per (l, c) point (median)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slicing", default="dp", help="dp | gpipe | comma-separated lengths")
    ap.add_argument("--batch-slices", default="auto", help="auto | comma-separated batch-slice sizes b to plan over")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from synth import CONFIGS, make_stage_flat, make_tokens
    base_cfg, B0 = CONFIGS[args.config]
    B = args.batch or B0
    K = max(world, 1)
    # stage partition: balanced for the LM head by default (A-30; identical to uniform cells
    # when the head is lighter than a layer, e.g. 13B); TP_PARTITION=uniform for n/K layers per stage
    part = 0 if os.environ.get("TP_PARTITION", "balanced") == "uniform" else 1
    cfg = base_cfg.with_(n_stages=K, partition=part)

    if args.impl == "reference":
        # The reference arm is the CPU oracle (tier framing): rank 0 only, on the host cores.
        if rank != 0:
            return 0
        cpu = cpu_oracle_sample(cfg, B, reps=max(1, args.steps), warmup=min(args.warmup, 1))
        per_step_s = B * cfg.seq_len / cpu["value"]
        line = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_s * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": args.config, "batch": B, "stages": K},
                "cpu_baseline": cpu, "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                                             "d2h_bytes_per_step": 0}}
        emit(line)
        return 0

    import torch
    import torch.distributed as dist
    import paper_2102_07988_b200 as tp

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2102_07988_b200 import dist as tdist
    nid = tdist.share_nccl_id(rank) if world > 1 else None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        return tdist.max_over_ranks(x) if world > 1 else x

    def allsum(x):
        return tdist.sum_over_ranks(x) if world > 1 else x

    stage = rank if world > 1 else 0
    # stage messages (world > 1): device-initiated p2p over NCCL symmetric windows by default (the
    # producing kernels store into the neighbour's buffer; measured faster than
    # ncclSend/ncclRecv on 4 x B200); TP_DEVICE_P2P=0 selects ncclSend/ncclRecv
    p2p_device = world > 1 and os.environ.get("TP_DEVICE_P2P", "1") != "0"
    p2p_note = None
    mb = args.max_batch or B
    free0 = torch.cuda.mem_get_info()[0]
    try:
        ctx = tp.Context(cfg, rank=rank, world=world, nccl_id=nid, precision=tp.TP_BF16, max_batch=mb,
                         device=local_rank, flags=tp.TP_FLAG_DEVICE_P2P if p2p_device else 0)
    except tp.TpError as e:
        if not p2p_device:
            raise
        # symmetric-memory windows unavailable on this box: the ncclSend/ncclRecv transport (every
        # rank fails the collective registration alike, so all retry with a fresh communicator)
        p2p_device, p2p_note = False, f"device p2p unavailable ({e}); ncclSend/ncclRecv used"
        print(p2p_note, file=sys.stderr)
        nid = tdist.share_nccl_id(rank)
        ctx = tp.Context(cfg, rank=rank, world=world, nccl_id=nid, precision=tp.TP_BF16, max_batch=mb,
                         device=local_rank, flags=0)
    ctx_mem_gb = (free0 - torch.cuda.mem_get_info()[0]) / 1e9  # the library's device allocations
    flat = make_stage_flat(cfg, stage, seed=0) if world > 1 else np.concatenate(
        [make_stage_flat(cfg, k, seed=0) for k in range(K)])
    ctx.load_params(flat)
    del flat
    tokens = make_tokens(cfg, B, seed=1)
    tok_dev = torch.from_numpy(tokens).cuda()
    tok_pin = torch.from_numpy(tokens).pin_memory()
    stream = torch.cuda.ExternalStream(ctx.stream())

    # --- cost tables (this stage; max over stages = bottleneck table, A-16) and the DP plan.
    # Joint batch x token slicing: one table per batch-slice size b, then
    # tp_plan_joint (per-b Algorithm 1 + 1-D knapsack over the batch under a shared t_max, A-20b);
    # the per-b uniform plans (tp_plan with D = B/b, A-20) are reported as candidates.
    g = args.granularity
    bsl = [int(x) for x in args.batch_slices.split(",")] if args.batch_slices != "auto" else \
        [x for x in (1, 2, 4, 8, 16) if B % x == 0 and x <= min(B, mb)]
    dp, fit, t_prof, t_plan, plans = None, None, 0.0, 0.0, []
    gpipe = tp.BatchPlan.uniform(tp.Slicing([cfg.seq_len]), B)
    comm, t_wgrad = None, None
    if args.slicing in ("dp", "gpipe") and (args.slicing == "dp" or len(bsl) > 1):
        t0 = time.time()
        tables = {}
        if world > 1:  # alpha / beta of a stage message, folded into every table entry
            comm = ctx.profile_comm(reps=5)
        for b in bsl:
            # the library measures every stage type this rank owns and (world > 1) takes the max over
            # all ranks: the bottleneck table of DESIGN.md A-16
            ticks, f = ctx.profile(g, reps=args.profile_reps, batch_slice=b)
            tables[b] = ticks
            t1 = time.time()
            sl = tp.plan(ticks, g, cfg.n_layer, cfg.hidden, cfg.seq_len, K, n_micro=B // b, eps_ticks=0)
            t_plan += time.time() - t1
            sl = tp.Slicing(sl.lengths, b, sl.t_max, sl.predicted)
            n = cfg.seq_len // g
            gp_pred = (B // b + K - 1) * int(ticks[n - 1, 0])   # unsliced [(b, [s])] * (B/b)
            plans.append({"b": b, "slicing": sl, "fit": f, "gpipe_pred": gp_pred})
        # slicing-independent constant of the step model (the stage buffers hold at most max_batch
        # sequences; a 1F1B batch beyond that is modelled as proportionally more dW)
        wb = min(B, mb)
        t_wgrad = ctx.profile_wgrad(wb, reps=3) * B // wb
        t1 = time.time()
        dp = tp.plan_joint(tables, g, cfg.n_layer, cfg.hidden, cfg.seq_len, K, B, eps_ticks=0)
        t_plan += time.time() - t1
        t_prof = time.time() - t0 - t_plan
        fit = min(plans, key=lambda p: (p["slicing"].predicted, -p["b"]))["fit"]
        gbest = min(plans, key=lambda p: (p["gpipe_pred"], -p["b"]))
        gpipe = tp.BatchPlan.uniform(tp.Slicing([cfg.seq_len], gbest["b"]), B)
        flat_plan = [x for bb, ls in dp.groups for x in [bb] + ls] + [gbest["b"]]
        if world > 1 and not tdist.agreed(flat_plan):
            raise RuntimeError("ranks planned different slicings")
    # tie-break (A-31): a DP plan predicted to beat the unsliced GPipe plan by less than
    # TIE_MARGIN of the step is within the cost table's per-job timing noise (the step model's error
    # is a few %), and the plan with fewer slices is taken — at K = 1 slicing cannot remove a bubble
    TIE_MARGIN = 0.02
    tie_break = False
    if args.slicing == "dp":
        main_sl = dp
        if dp.groups != gpipe.groups and dp.predicted + t_wgrad > (1 - TIE_MARGIN) * (gbest["gpipe_pred"] + t_wgrad):
            main_sl, tie_break = gpipe, True
    elif args.slicing == "gpipe":
        main_sl = gpipe
    else:
        main_sl = tp.BatchPlan.uniform(tp.Slicing([int(x) for x in args.slicing.split(",")],
                                                  int(args.batch_slices.split(",")[0])
                                                  if args.batch_slices != "auto" else 1), B)

    def timed(sl, steps, device_tokens=True):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        loss = None
        for _ in range(steps):
            if device_tokens:
                loss = ctx.step_plan_device(sl, tok_dev.data_ptr(), B)
            else:
                loss = ctx.step_plan(sl, tok_pin.numpy())
        e1.record(stream)
        e1.synchronize()
        barrier()
        return allmax(e0.elapsed_time(e1) / steps), loss

    for _ in range(args.warmup):
        ctx.step_plan_device(main_sl, tok_dev.data_ptr(), B)
    clocks = ClockSampler(local_rank)
    clocks.start()
    # TP_PROFILE_RANGE=1 limits an `ncu --profile-from-start off` capture to the timed device region
    prof_range = os.environ.get("TP_PROFILE_RANGE") == "1"
    if prof_range:
        torch.cuda.profiler.start()
    ms, loss = timed(main_sl, args.steps)
    if prof_range:
        torch.cuda.profiler.stop()
    clk = clocks.stop()
    launches = allsum(ctx.last_step_launches()) * args.steps
    # e2e through the public API with host tokens (pinned) and the loss read back every step
    ms_e2e, _ = timed(main_sl, args.steps, device_tokens=False)
    # unsliced GPipe on the same kernels
    ms_gpipe = None
    same = main_sl.groups == gpipe.groups
    if not args.no_gpipe and not same:
        for _ in range(1):
            ctx.step_plan_device(gpipe, tok_dev.data_ptr(), B)
        ms_gpipe, _ = timed(gpipe, args.steps)
    elif same:
        ms_gpipe = ms
    # kernel statistics: a second timed region with CUDA events around every launch (on the
    # library's stream, which every kernel is launched on)
    ctx.kernel_stats_reset()
    ctx.kernel_stats_enable(True)
    ms_instr, _ = timed(main_sl, args.steps)
    ctx.kernel_stats_enable(False)
    kstats = ctx.kernel_stats()
    peak_burst, peak_sust, hbm, peak_kind = load_peaks()
    tokens_per_step = B * cfg.seq_len
    flops = model_flops(cfg, B)
    value = tokens_per_step / (ms / 1e3)
    mfu = flops / (ms / 1e3) / (args.gpus * peak_burst * 1e12)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": args.config, "n_layer": cfg.n_layer, "hidden": cfg.hidden, "heads": cfg.n_head,
                   "seq_len": cfg.seq_len, "batch": B, "vocab": cfg.vocab, "stages": K,
                   "parallelism": f"pipeline{K}", "slicing": main_sl.notation(), "granularity": g,
                   "p2p": (("device" if p2p_device else "nccl") if world > 1 else None) if not p2p_note else p2p_note,
                   "stage_layers": tp.stage_layers(cfg), "max_batch": mb,
                   "device_mem_gb": allmax(ctx_mem_gb),
                   "schedule": "1f1b" if os.environ.get("TP_SCHEDULE") == "1f1b" else "gpipe",
                   "l2": "working set > L2 (bf16 weights alone exceed 126 MB); no flush"},
        "mfu": mfu, "mfu_sustained_peak": flops / (ms / 1e3) / (args.gpus * peak_sust * 1e12),
        "gpipe": None if ms_gpipe is None else {
            "slicing": gpipe.notation(), "ms_per_step": ms_gpipe, "tokens_per_s": tokens_per_step / (ms_gpipe / 1e3),
            "mfu": flops / (ms_gpipe / 1e3) / (args.gpus * peak_burst * 1e12),
            "speedup_of_dp": ms_gpipe / ms},
        "plan": None if dp is None else {
            "predicted_ms": dp.predicted / 1e6, "t_max_ms": dp.t_max / 1e6, "profile_s": t_prof, "plan_s": t_plan,
            "wgrad_ms": t_wgrad / 1e6,
            "predicted_step_ms": (dp.predicted + t_wgrad) / 1e6,
            "predicted_step_err": ((dp.predicted + t_wgrad) / 1e6 - ms) / ms if main_sl is dp else
                                  (((gbest["gpipe_pred"] + t_wgrad) / 1e6 - ms) / ms if tie_break else None),
            "dp_slicing": dp.notation(),
            "tie_break": ("DP plan predicted within %d %% of the unsliced GPipe plan: GPipe timed" % round(100 * TIE_MARGIN))
                         if tie_break else None,
            "comm": None if comm is None else {"alpha_us": comm[0] / 1e3, "gbs": comm[1]},
            "fit": {"a": [float(x) for x in fit[:4]], "max_rel_err": float(fit[4])},
            "joint": "tp_plan_joint over b in " + str(bsl),
            "candidates": [{"b": p["b"], "slicing": p["slicing"].notation(B), "predicted_ms": p["slicing"].predicted / 1e6,
                            "gpipe_predicted_ms": p["gpipe_pred"] / 1e6} for p in plans],
            "gpipe_predicted_step_ms": (gbest["gpipe_pred"] + t_wgrad) / 1e6},
        "loss": loss,
        "clocks": clk,
        "e2e": {"value": tokens_per_step / (ms_e2e / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(tokens.nbytes), "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches),
    }
    # roofline + cpu baseline are filled by the rank-0 tail below
    if rank == 0:
        line["roofline"] = roofline(kstats, ms_instr, args.steps, peak_sust, hbm, peak_kind)
        line["kernel_classes"] = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                                      "tflops": (v["flops"] / (v["ms"] * 1e9)) if v["ms"] > 0 and v["flops"] > 0 else None,
                                      "gbs": (v["bytes"] / (v["ms"] * 1e6)) if v["ms"] > 0 and v["bytes"] > 0 else None}
                                  for k, v in kstats.items() if v["launches"]}
        line["roofline_hbm"] = roofline_hbm(kstats, ms_instr, args.steps, hbm, peak_kind)
        line["ms_per_step_instrumented"] = ms_instr
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_oracle_sample(cfg, B)
        emit(line)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def roofline(kstats, ms_step, steps, peak_tflops, hbm_gbs, peak_kind):
    """Dominant kernel class of the step (largest summed device time): its ALGORITHMIC FLOPs (or
    bytes) per launch / its mean CUDA-event launch duration, against the measured sustained bf16
    peak (a kernel timed inside a long step) or the measured HBM copy bandwidth."""
    live = {k: v for k, v in kstats.items() if v["launches"] and v["ms"] > 0}
    if not live:
        return None
    name, v = max(live.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = v["ms"] / v["launches"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(name)
    except Exception:
        pass
    if v["flops"] > 0:
        ach = v["flops"] / v["launches"] / (per_launch_ms * 1e-3) / 1e12
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": ach / peak_tflops, "traffic": traffic, "peak_kind": f"{peak_kind} sustained bf16",
                "share_of_step": v["ms"] / steps / ms_step, "launches_per_step": v["launches"] / steps,
                "flops_per_launch": v["flops"] / v["launches"]}
    ach = v["bytes"] / v["launches"] / (per_launch_ms * 1e-3) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm_gbs, "unit": "GB/s", "frac": ach / hbm_gbs,
            "traffic": traffic, "peak_kind": peak_kind, "share_of_step": v["ms"] / steps / ms_step}


def roofline_hbm(kstats, ms_step, steps, hbm_gbs, peak_kind):
    """The HBM-bound kernel classes (no FLOPs counted: LayerNorm fwd/bwd, embedding, cross-entropy,
    the dK/dV finalise / dQ convert / column-sum passes in "misc"): ALGORITHMIC bytes per launch (the
    per-unit figures of DESIGN.md §6 x the tokens of one job) / mean CUDA-event launch duration,
    against the measured HBM copy bandwidth. The dominant one (largest summed time) leads."""
    live = {k: v for k, v in kstats.items() if v["launches"] and v["ms"] > 0 and v["bytes"] > 0 and v["flops"] == 0}
    if not live:
        return None
    out = []
    for name, v in sorted(live.items(), key=lambda kv: -kv[1]["ms"]):
        ach = v["bytes"] / (v["ms"] * 1e-3) / 1e9
        out.append({"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm_gbs, "unit": "GB/s",
                    "frac": ach / hbm_gbs, "peak_kind": peak_kind, "share_of_step": v["ms"] / steps / ms_step,
                    "launches_per_step": v["launches"] / steps, "bytes_per_launch": v["bytes"] / v["launches"]})
    return out


if __name__ == "__main__":
    sys.exit(main())
