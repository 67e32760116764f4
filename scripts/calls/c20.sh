mkdir -p gpurun_out/c20
for v in new; do
  timeout 120 python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c20/attn.txt 2>&1
  timeout 120 python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c20/attn.txt 2>&1
  timeout 120 python scripts/attn_bench.py 80 2048 1536 512 20 >> gpurun_out/c20/attn.txt 2>&1
done
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k attention tests/test_gpu_parity.py > gpurun_out/c20/pytest.log 2>&1
echo rc=$? >> gpurun_out/c20/pytest.log
VARS="X=1" scripts/env_ab.sh 2 > gpurun_out/c20/ab.txt 2>&1
