# 64-key double-buffered two-tile attention forward (TP_ATTN_FWD=3): parity + kernel timing vs 1 / 2
mkdir -p gpurun_out/c29
TP_ATTN_FWD=3 timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "attention" -x > gpurun_out/c29/pytest_k.log 2>&1
echo rc=$? >> gpurun_out/c29/pytest_k.log
for f in 3 2 1 3 2 1; do
  echo "TP_ATTN_FWD=$f" >> gpurun_out/c29/attn.txt
  for shp in "128 2048 0 2048" "128 2048 576 1472" "128 2048 0 576" "80 2048 1536 512"; do
    TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py $shp 20 >> gpurun_out/c29/attn.txt 2>&1
  done
done
TP_ATTN_FWD=3 timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py -x > gpurun_out/c29/pytest.log 2>&1
echo rc=$? >> gpurun_out/c29/pytest.log
