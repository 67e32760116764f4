mkdir -p gpurun_out/c16
for sp in 1 0; do
  echo "TP_ATTN_BWD_SPLIT=$sp" >> gpurun_out/c16/attn.txt
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c16/attn.txt 2>&1
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c16/attn.txt 2>&1
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 80 2048 1536 512 20 >> gpurun_out/c16/attn.txt 2>&1
done
TP_ATTN_BWD_SPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c16/split_launches.csv python scripts/attn_bench.py 128 2048 576 1472 3 > gpurun_out/c16/split.log 2>&1
TP_ATTN_BWD_SPLIT=1 timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k attention tests/test_gpu_parity.py::test_parity_mid_13b_width tests/test_gpu_parity.py::test_small_bf16_stages > gpurun_out/c16/pytest.log 2>&1
echo rc=$? >> gpurun_out/c16/pytest.log
