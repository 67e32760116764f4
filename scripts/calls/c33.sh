# uniform-datapath MMA issue (warp index via shuffle, warp-uniform role branches, no printf in the
# mbarrier watchdog): attention kernel timing, kernel + parity tests, one bench line
mkdir -p gpurun_out/c33
for f in 3 2 1; do
  echo "TP_ATTN_FWD=$f" >> gpurun_out/c33/attn.txt
  for shp in "128 2048 0 2048" "128 2048 576 1472" "128 2048 0 576" "80 2048 1536 512"; do
    TP_ATTN_FWD=$f timeout 120 python scripts/attn_bench.py $shp 20 >> gpurun_out/c33/attn.txt 2>&1
  done
done
TP_ATTN_TRACE=1 TP_ATTN_FWD=3 timeout 120 python scripts/attn_bench.py 128 2048 0 2048 2 > gpurun_out/c33/trace.txt 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_kernels.py > gpurun_out/c33/pytest_k.log 2>&1
echo rc=$? >> gpurun_out/c33/pytest_k.log
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 300 tests/test_gpu_parity.py tests/test_gpu_benchsize.py > gpurun_out/c33/pytest.log 2>&1
echo rc=$? >> gpurun_out/c33/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/c33/bench.json 2> gpurun_out/c33/bench.err
timeout 600 python scripts/bench_kernels.py --which gemm --filter "T=16384" > gpurun_out/c33/gemm.jsonl 2>&1
