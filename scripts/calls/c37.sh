# GEMM wide-tile rule check on the bench's T = 16384 shapes: default vs TP_GEMM_WIDE=0 / =1
mkdir -p gpurun_out/c37
for w in d 0 1 d 0 1; do
  if [ $w = d ]; then timeout 600 python scripts/bench_kernels.py --which gemm --filter "T=16384" > gpurun_out/c37/gemm_default.$RANDOM.jsonl 2>&1
  else TP_GEMM_WIDE=$w timeout 600 python scripts/bench_kernels.py --which gemm --filter "T=16384" > gpurun_out/c37/gemm_wide$w.$RANDOM.jsonl 2>&1; fi
done
