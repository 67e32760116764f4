# softmax instruction-mix micro, ncu --set full of the two-tile attention forward, LN bulk-forward A/B
mkdir -p gpurun_out/c24
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/ex2_rate.cu -o /tmp/ex2_rate && /tmp/ex2_rate > gpurun_out/c24/ex2_rate.txt 2>&1
TP_ATTN_FWD=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd2 -c 1 -o gpurun_out/c24/fwd2 \
  python scripts/attn_bench.py 128 2048 0 2048 1 > gpurun_out/c24/ncu_fwd2.log 2>&1
TP_ATTN_FWD=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd1 -c 1 -o gpurun_out/c24/fwd1 \
  python scripts/attn_bench.py 128 2048 0 2048 1 > gpurun_out/c24/ncu_fwd1.log 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k layernorm > gpurun_out/c24/pytest_ln.log 2>&1
echo rc=$? >> gpurun_out/c24/pytest_ln.log
for b in 1 0 1 0; do TP_LN_BULK=$b timeout 300 python scripts/bench_kernels.py --which ln >> gpurun_out/c24/ln_kernels.jsonl 2>&1; done
VARS="TP_LN_BULK=1 TP_LN_BULK=0" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c24/ab.txt 2>&1
