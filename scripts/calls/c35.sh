# GEMM: 32-bit stream-K index math (no 64-bit division helper calls) -> uniform-datapath MMA issue:
# GEMM tests (incl. stream-K), GEMM shapes, step A/B vs the previous commit's build (libtp_base.so)
mkdir -p gpurun_out/c35
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "gemm" > gpurun_out/c35/pytest_gemm.log 2>&1
echo rc=$? >> gpurun_out/c35/pytest_gemm.log
for lib in libtp.so libtp_base.so; do
  TP_LIB=paper_2102_07988_b200/$lib timeout 600 python scripts/bench_kernels.py --which gemm --filter "T=16384" > gpurun_out/c35/gemm_$lib.jsonl 2>&1
done
VARS="TP_LIB=paper_2102_07988_b200/libtp.so TP_LIB=paper_2102_07988_b200/libtp_base.so" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c35/ab.txt 2>&1
