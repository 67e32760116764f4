mkdir -p gpurun_out/c8
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_benchsize.py > gpurun_out/c8/pytest.log 2>&1
echo rc=$? >> gpurun_out/c8/pytest.log
scripts/micro/ex2_rate > gpurun_out/c8/ex2.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/c8/smoke.log 2>&1
