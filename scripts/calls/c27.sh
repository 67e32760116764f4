# attention backward: dQ^T over the S^T columns with dP^T(i+1) / S^T(i+1) issued before the softmax
# of tile i is waited (TP_ATTN_DQS=1, default) vs the round-1 TMEM layout (TP_ATTN_DQS=0)
mkdir -p gpurun_out/c27
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "attention" > gpurun_out/c27/pytest_k.log 2>&1
echo rc=$? >> gpurun_out/c27/pytest_k.log
for d in 1 0 1 0; do
  echo "TP_ATTN_DQS=$d" >> gpurun_out/c27/attn.txt
  for shp in "128 2048 0 2048" "128 2048 576 1472" "128 2048 0 576" "80 2048 1536 512"; do
    TP_ATTN_DQS=$d timeout 120 python scripts/attn_bench.py $shp 20 >> gpurun_out/c27/attn.txt 2>&1
  done
done
TP_ATTN_TRACE=1 timeout 120 python scripts/attn_bench.py 128 2048 0 2048 2 > gpurun_out/c27/bwd_trace.txt 2>&1
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c27/pytest.log 2>&1
echo rc=$? >> gpurun_out/c27/pytest.log
VARS="TP_ATTN_DQS=1 TP_ATTN_DQS=0" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c27/ab.txt 2>&1
