#!/bin/bash
# A/B of the LayerNorm-backward launch configuration (TP_LNB_CTAS = CTAs per SM the row groups are
# sized for; a TP_LNB_MINB=3 80-register variant was measured too and removed: it spilled and was slower) on the default
# N = 1 bench workload with a fixed plan; prints step ms and the LayerNorm class ms / GB/s.
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in "4 1" "2 1" "1 1"; do
    set -- $cfg
    TP_LNB_CTAS=$1 TP_LNB_MINB=$2 timeout 300 python bench.py --steps 10 --warmup 3 --slicing 576,1472 \
      --batch-slices 8 --no-gpipe --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json, sys
d = json.loads(sys.stdin.read())
ln = d['kernel_classes']['layernorm']
print('ctas=$1 minb=$2 rep=$rep step_ms %.2f instr_ms %.2f ln_ms %.3f ln_gbs %.0f sm_mhz %s' % (d['ms_per_step'],
      d['ms_per_step_instrumented'], ln['ms_per_step'], ln['gbs'], d['clocks']['sm_mhz']))"
  done
done
