mkdir -p gpurun_out/c7
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_kernels.py tests/test_gpu_parity.py -x > gpurun_out/c7/pytest.log 2>&1
echo rc=$? >> gpurun_out/c7/pytest.log
VARS="X=1" scripts/env_ab.sh 2 > gpurun_out/c7/ab.txt 2>&1
python scripts/bench_kernels.py --which gemm > gpurun_out/c7/gemm.jsonl 2>&1
