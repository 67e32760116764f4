mkdir -p gpurun_out/c5
for pf in 0 1 2 3 4; do
  echo "TP_ATTN_PF=$pf" >> gpurun_out/c5/attn.txt
  TP_ATTN_PF=$pf python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c5/attn.txt 2>&1
  TP_ATTN_PF=$pf python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c5/attn.txt 2>&1
done
TP_ATTN_TRACE=1 TP_ATTN_PF=2 python scripts/attn_bench.py 128 2048 576 1472 1 > gpurun_out/c5/trace.txt 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_kernels.py -k attention > gpurun_out/c5/pytest.log 2>&1
echo rc=$? >> gpurun_out/c5/pytest.log
