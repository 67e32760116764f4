# wide pair tiles only for MN-major (dW) GEMMs: GEMM tests, shapes, step A/B vs the previous rule (libtp_base.so)
mkdir -p gpurun_out/c38
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "gemm" > gpurun_out/c38/pytest_gemm.log 2>&1
echo rc=$? >> gpurun_out/c38/pytest_gemm.log
VARS="TP_LIB=paper_2102_07988_b200/libtp.so TP_LIB=paper_2102_07988_b200/libtp_base.so" SLICING=2048 scripts/env_ab.sh 4 > gpurun_out/c38/ab.txt 2>&1
timeout 600 python scripts/bench_kernels.py --which gemm --filter "13b" > gpurun_out/c38/gemm13b_new.jsonl 2>&1
TP_LIB=paper_2102_07988_b200/libtp_base.so timeout 600 python scripts/bench_kernels.py --which gemm --filter "13b" > gpurun_out/c38/gemm13b_old.jsonl 2>&1
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c38/pytest.log 2>&1
echo rc=$? >> gpurun_out/c38/pytest.log
