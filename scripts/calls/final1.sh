# final 1-GPU validation of the tree: the full GPU suite, smoke, the default bench line (plain, then
# under ncu: the per-launch device-time list and the per-kernel DRAM / tensor-pipe metrics pass)
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/final/pytest_gpu.log 2>&1
echo rc=$? >> gpurun_out/final/pytest_gpu.log
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/final/smoke.log 2>&1
echo rc=$? >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err
B="python bench.py --steps 1 --warmup 3 --slicing 576,1472 --batch-slices 8 --no-gpipe --no-cpu-baseline"
$B > gpurun_out/final/plain.log 2>&1 && \
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/final/launches.csv $B > gpurun_out/final/ncu_launches.log 2>&1
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/final/metrics.csv $B > gpurun_out/final/ncu_metrics.log 2>&1
