mkdir -p gpurun_out/c14
for sp in 1 0; do
  echo "TP_ATTN_BWD_SPLIT=$sp" >> gpurun_out/c14/attn.txt
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c14/attn.txt 2>&1
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c14/attn.txt 2>&1
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 80 2048 1536 512 20 >> gpurun_out/c14/attn.txt 2>&1
done
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c14/pytest.log 2>&1
echo rc=$? >> gpurun_out/c14/pytest.log
VARS="TP_ATTN_BWD_SPLIT=1 TP_ATTN_BWD_SPLIT=0 TP_GEMM_EPI_PF=0" scripts/env_ab.sh 2 > gpurun_out/c14/ab.txt 2>&1
