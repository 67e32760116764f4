# in-order tcgen05.mma issue (no completion waits before TMEM-operand reuse): parity, kernel A/B, step A/B
mkdir -p gpurun_out/c25
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "attention or layernorm" > gpurun_out/c25/pytest_k.log 2>&1
echo rc=$? >> gpurun_out/c25/pytest_k.log
for io in 1 0; do
  for f in 2 1; do
    echo "TP_ATTN_INORDER=$io TP_ATTN_FWD=$f" >> gpurun_out/c25/attn.txt
    for shp in "128 2048 0 2048" "128 2048 576 1472" "128 2048 0 576" "80 2048 1536 512"; do
      TP_ATTN_INORDER=$io TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py $shp 20 >> gpurun_out/c25/attn.txt 2>&1
    done
  done
done
TP_ATTN_TRACE=1 TP_ATTN_FWD=2 timeout 120 python scripts/attn_bench.py 128 2048 0 2048 2 > gpurun_out/c25/fwd_trace_2.txt 2>&1
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c25/pytest.log 2>&1
echo rc=$? >> gpurun_out/c25/pytest.log
VARS="TP_ATTN_INORDER=1 TP_ATTN_INORDER=0" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c25/ab.txt 2>&1
