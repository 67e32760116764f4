mkdir -p gpurun_out/c32
TP_ATTN_TRACE=1 TP_ATTN_FWD=3 timeout 120 python scripts/attn_bench.py 128 2048 0 2048 2 > gpurun_out/c32/fwd3_trace.txt 2>&1
