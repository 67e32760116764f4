mkdir -p gpurun_out/c21
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k gemm tests/test_gpu_parity.py::test_parity_mid_13b_width tests/test_gpu_benchsize.py > gpurun_out/c21/pytest.log 2>&1
echo rc=$? >> gpurun_out/c21/pytest.log
VARS="X=1 TP_LIB=/root/repo/paper_2102_07988_b200/libtp_base.so" scripts/env_ab.sh 3 > gpurun_out/c21/ab.txt 2>&1
