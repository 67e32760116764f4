# bulk-staged LayerNorm kernels: unit tests, isolated GB/s (bulk vs register-prefetch), step A/B
mkdir -p gpurun_out/c23
timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k layernorm > gpurun_out/c23/pytest_ln.log 2>&1
echo rc=$? >> gpurun_out/c23/pytest_ln.log
for b in 1 0 1 0; do TP_LN_BULK=$b timeout 300 python scripts/bench_kernels.py --which ln >> gpurun_out/c23/ln_kernels.jsonl 2>&1; done
VARS="TP_LN_BULK=1 TP_LN_BULK=0" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c23/ab.txt 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c23/pytest.log 2>&1
echo rc=$? >> gpurun_out/c23/pytest.log
# attention forward timeline (CTA 0 = the heaviest tile pair, 16 key blocks), both forward kernels
for f in 2 1; do
  TP_ATTN_TRACE=1 TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py 128 2048 0 2048 2 > gpurun_out/c23/fwd_trace_$f.txt 2>&1
done
