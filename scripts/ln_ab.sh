#!/bin/bash
# A/B of the LayerNorm launch configurations on the default N = 1 bench workload with a fixed plan:
# TP_LNB_CTAS = CTAs per SM the backward row groups are sized for. Measured and removed (neutral or
# slower): an 80-register 3-CTA/SM backward variant (spills) and 4-row forward CTAs (TP_LNF_RPC=4);
# profiles/r01_lnb_ab_n1.txt, profiles/r01_ln_ab_n1.txt. Prints step ms and the LayerNorm class.
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in ${CONFIGS:-"8 4" "8 2" "8 1"}; do
    set -- $cfg
    TP_LNF_RPC=$1 TP_LNB_CTAS=$2 timeout 300 python bench.py --steps 10 --warmup 3 --slicing 576,1472 \
      --batch-slices 8 --no-gpipe --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json, sys
d = json.loads(sys.stdin.read())
ln = d['kernel_classes']['layernorm']
print('lnf_rpc=$1 lnb_ctas=$2 rep=$rep step_ms %.2f instr_ms %.2f ln_ms %.3f ln_gbs %.0f sm_mhz %s' % (d['ms_per_step'],
      d['ms_per_step_instrumented'], ln['ms_per_step'], ln['gbs'], d['clocks']['sm_mhz']))"
  done
done
