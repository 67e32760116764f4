mkdir -p gpurun_out/c4
for m in 0 1 2; do
  echo "TP_ATTN_DQ=$m" >> gpurun_out/c4/attn.txt
  TP_ATTN_DQ=$m python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c4/attn.txt 2>&1
  TP_ATTN_DQ=$m python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c4/attn.txt 2>&1
done
for m in 1 2; do
  TP_ATTN_DQ=$m timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_kernels.py -k attention \
    tests/test_gpu_parity.py::test_parity_mid_13b_width > gpurun_out/c4/pytest_$m.log 2>&1
  echo rc=$? >> gpurun_out/c4/pytest_$m.log
done
TP_ATTN_TRACE=1 python scripts/attn_bench.py 128 2048 576 1472 1 > gpurun_out/c4/trace.txt 2>&1
