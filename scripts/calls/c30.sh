# default forward dispatch (64-key two-tile kernel when >= 2 waves): tests, step A/B vs the two-tile 128-key kernel, ncu
mkdir -p gpurun_out/c30
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py -k "attention" > gpurun_out/c30/pytest_k.log 2>&1
echo rc=$? >> gpurun_out/c30/pytest_k.log
VARS="TP_ATTN_FWD=0 TP_ATTN_FWD=2" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c30/ab.txt 2>&1
TP_ATTN_FWD=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd3 -c 1 -o gpurun_out/c30/fwd3 \
  python scripts/attn_bench.py 128 2048 0 2048 1 > gpurun_out/c30/ncu_fwd3.log 2>&1
