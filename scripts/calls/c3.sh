mkdir -p gpurun_out/c3
python scripts/attn_bench.py 128 2048 576 1472 20 > gpurun_out/c3/attn.txt 2>&1
python scripts/attn_bench.py 128 2048 0 576 20 >> gpurun_out/c3/attn.txt 2>&1
python scripts/attn_bench.py 128 2048 0 2048 20 >> gpurun_out/c3/attn.txt 2>&1
TP_ATTN_TRACE=1 python scripts/attn_bench.py 128 2048 576 1472 1 > gpurun_out/c3/trace.txt 2>&1
