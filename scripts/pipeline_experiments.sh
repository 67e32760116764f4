#!/bin/bash
# North-star experiment (BASELINE.json:5): on N GPUs of one box, the DP-chosen
# token slicing vs the unsliced GPipe schedule on the same kernels, for the GPT-3 shaped configs.
# Usage (under gpurun --gpus N): bash scripts/pipeline_experiments.sh N "gpt3-13b gpt3-13b-8k ..."
N=${1:-4}
CONFIGS=${2:-"gpt3-13b gpt3-13b-8k gpt3-175b-24l"}
mkdir -p gpurun_out
for cfg in $CONFIGS; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29541 bench.py --gpus $N --config $cfg --steps 3 --warmup 2 --no-cpu-baseline \
    > gpurun_out/pipe_${cfg}_n${N}.json 2> gpurun_out/pipe_${cfg}_n${N}.err
  echo "$cfg rc=$?"
  tail -2 gpurun_out/pipe_${cfg}_n${N}.err
  python - "$cfg" "$N" <<'PY'
import json, sys
cfg, n = sys.argv[1], sys.argv[2]
try:
    d = json.loads([l for l in open(f"gpurun_out/pipe_{cfg}_n{n}.json") if l.startswith("{")][-1])
    g = d.get("gpipe") or {}
    print(cfg, "DP", d["config"]["slicing"], f'{d["ms_per_step"]:.1f} ms', f'mfu {d["mfu"]:.3f}',
          "| GPipe", f'{g.get("ms_per_step", float("nan")):.1f} ms', f'mfu {g.get("mfu", float("nan")):.3f}',
          f'speedup {g.get("speedup_of_dp", float("nan")):.3f}', "| predicted", d["plan"] and d["plan"]["predicted_ms"])
except Exception as e:
    print(cfg, "no result", e)
PY
done
