mkdir -p gpurun_out/c2
timeout 1500 python -m pytest -q --timeout 900 -p no:cacheprovider tests/test_gpu_kernels.py::test_gemm_weight_grad_shapes \
  tests/test_gpu_parity.py tests/test_gpu_multi.py > gpurun_out/c2/pytest.log 2>&1
echo pytest rc=$? >> gpurun_out/c2/pytest.log
B="python bench.py --steps 1 --warmup 3 --slicing 576,1472 --batch-slices 8 --no-gpipe --no-cpu-baseline"
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"attn_bwd_sm100" -c 1 -o gpurun_out/c2/attn_bwd $B > gpurun_out/c2/ncu_bwd.log 2>&1
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"attn_fwd2_sm100" --launch-skip 24 -c 1 -o gpurun_out/c2/attn_fwd $B > gpurun_out/c2/ncu_fwd.log 2>&1
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/c2/metrics.csv $B > gpurun_out/c2/ncu_metrics.log 2>&1
