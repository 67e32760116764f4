mkdir -p gpurun_out/c11
for f in 1 2; do
  echo "TP_ATTN_FWD=$f" >> gpurun_out/c11/attn.txt
  TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c11/attn.txt 2>&1
  TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c11/attn.txt 2>&1
  TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py 80 2048 1536 512 20 >> gpurun_out/c11/attn.txt 2>&1
done
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py tests/test_gpu_parity.py > gpurun_out/c11/pytest.log 2>&1
echo rc=$? >> gpurun_out/c11/pytest.log
VARS="TP_ATTN_FWD=1 TP_ATTN_FWD=2 TP_GEMM_STREAMK=0" scripts/env_ab.sh 2 > gpurun_out/c11/ab.txt 2>&1
timeout 600 python scripts/bench_kernels.py --which gemm > gpurun_out/c11/gemm.jsonl 2>&1
