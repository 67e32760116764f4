mkdir -p gpurun_out/c15
TP_ATTN_BWD_SPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c15/split_launches.csv python scripts/attn_bench.py 128 2048 576 1472 3 > gpurun_out/c15/split.log 2>&1
TP_ATTN_BWD_SPLIT=1 TP_ATTN_TRACE=1 timeout 120 python scripts/attn_bench.py 128 2048 576 1472 1 > gpurun_out/c15/split_trace.txt 2>&1
