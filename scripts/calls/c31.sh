# fwd3 with per-tile PV -> S(j+2) issue order: tests (forced and default dispatch), timing; K = 8 loopback parity
mkdir -p gpurun_out/c31
TP_ATTN_FWD=3 timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "attention" -x > gpurun_out/c31/pytest_k3.log 2>&1
echo rc=$? >> gpurun_out/c31/pytest_k3.log
for f in 3 2 3 2; do
  echo "TP_ATTN_FWD=$f" >> gpurun_out/c31/attn.txt
  for shp in "128 2048 0 2048" "128 2048 576 1472" "128 2048 0 576"; do
    TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py $shp 20 >> gpurun_out/c31/attn.txt 2>&1
  done
done
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py -k "eight_stage or balanced" > gpurun_out/c31/pytest_k8.log 2>&1
echo rc=$? >> gpurun_out/c31/pytest_k8.log
TP_ATTN_FWD=3 timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py -x > gpurun_out/c31/pytest.log 2>&1
echo rc=$? >> gpurun_out/c31/pytest.log
