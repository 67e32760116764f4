# LayerNorm forward: one-pass shifted statistics (one block barrier per row): tests, isolated GB/s, step A/B
mkdir -p gpurun_out/c41
timeout 600 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k layernorm > gpurun_out/c41/pytest_ln.log 2>&1
echo rc=$? >> gpurun_out/c41/pytest_ln.log
for lib in libtp.so libtp_base.so libtp.so libtp_base.so; do
  echo "TP_LIB=$lib" >> gpurun_out/c41/ln.txt
  TP_LIB=paper_2102_07988_b200/$lib timeout 300 python scripts/bench_kernels.py --which ln >> gpurun_out/c41/ln.txt 2>&1
done
VARS="TP_LIB=paper_2102_07988_b200/libtp.so TP_LIB=paper_2102_07988_b200/libtp_base.so" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c41/ab.txt 2>&1
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c41/pytest.log 2>&1
echo rc=$? >> gpurun_out/c41/pytest.log
