mkdir -p gpurun_out/c17
TP_ATTN_BWD_SPLIT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd" -s 2 -c 2 -o gpurun_out/c17/split python scripts/attn_bench.py 128 2048 576 1472 2 > gpurun_out/c17/ncu.log 2>&1
