# single-warp softmax-mix rate; wide (H = 5120) bulk LayerNorm: tests + isolated GB/s
mkdir -p gpurun_out/c26
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/ex2_rate.cu -o /tmp/ex2_rate && /tmp/ex2_rate > gpurun_out/c26/ex2_rate.txt 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k layernorm > gpurun_out/c26/pytest_ln.log 2>&1
echo rc=$? >> gpurun_out/c26/pytest_ln.log
for b in 1 0 1 0; do TP_LN_BULK=$b timeout 300 python scripts/bench_kernels.py --which ln >> gpurun_out/c26/ln_kernels.jsonl 2>&1; done
