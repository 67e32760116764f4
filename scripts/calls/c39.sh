# deferred dW GEMMs on two alternating streams (tail overlap) + wide-tile rule: parity, step A/B
mkdir -p gpurun_out/c39
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_kernels.py -k "not attention" > gpurun_out/c39/pytest.log 2>&1
echo rc=$? >> gpurun_out/c39/pytest.log
VARS="TP_DW_STREAMS=2 TP_DW_STREAMS=1 TP_LIB=paper_2102_07988_b200/libtp_base.so" SLICING=2048 scripts/env_ab.sh 4 > gpurun_out/c39/ab.txt 2>&1
