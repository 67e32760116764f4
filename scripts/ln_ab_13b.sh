#!/bin/bash
# 4 x B200 A/B of the LayerNorm-backward grid at the 13B width (H = 5120, the wide kernel):
# TP_LNB_CTAS = CTAs per SM the row groups are sized for (default 4 for H > 2048), on the K = 4
# pipeline with the DP plan [(4, [128, 192*10])] * 2 fixed. Prints step ms and the LayerNorm class.
mkdir -p gpurun_out
SL=128,192,192,192,192,192,192,192,192,192,192
for rep in 1 2; do
  for c in 4 2; do
    TP_LNB_CTAS=$c timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29541 bench.py --gpus 4 --config gpt3-13b --steps 3 --warmup 3 --slicing $SL --batch-slices 4 \
      --no-gpipe --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json, sys
d = json.loads(sys.stdin.read())
ln = d['kernel_classes']['layernorm']
print('lnb_ctas=$c rep=$rep step_ms %.2f ln_ms(rank0) %.3f ln_gbs %.0f sm_mhz %s' % (d['ms_per_step'], ln['ms_per_step'], ln['gbs'], d['clocks']['sm_mhz']))"
  done
done
