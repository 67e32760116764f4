#!/bin/bash
# A/B of environment settings on the default N = 1 bench workload with a fixed plan:
#   VARS="TP_GEMM_GROUP=2048 TP_GEMM_GROUP=100000" scripts/env_ab.sh [reps] [extra bench args]
# Prints step ms and the per-class kernel times for every setting, alternating over reps.
mkdir -p gpurun_out
REPS=${1:-2}; shift
for rep in $(seq 1 $REPS); do
  for kv in $VARS; do
    env $kv timeout 300 python bench.py --steps 10 --warmup 3 --slicing ${SLICING:-576,1472} \
      --batch-slices ${BSL:-8} --no-gpipe --no-cpu-baseline "$@" 2>/dev/null | grep '^{' | python -c "
import json, sys
d = json.loads(sys.stdin.read())
kc = d['kernel_classes']
cls = ' '.join('%s=%.2f' % (k, v['ms_per_step']) for k, v in sorted(kc.items()))
print('$kv rep=$rep step_ms %.2f instr_ms %.2f sm_mhz %s | %s' % (d['ms_per_step'], d['ms_per_step_instrumented'],
      d['clocks']['sm_mhz'], cls))"
  done
done
