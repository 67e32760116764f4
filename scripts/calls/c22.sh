mkdir -p gpurun_out/c22
for sp in 1 0; do
  echo "TP_ATTN_BWD_SPLIT=$sp" >> gpurun_out/c22/attn.txt
  TP_ATTN_BWD_SPLIT=$sp timeout 120 python scripts/attn_bench.py 128 2048 576 1472 20 >> gpurun_out/c22/attn.txt 2>&1
done
TP_ATTN_BWD_SPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c22/split_launches.csv python scripts/attn_bench.py 128 2048 576 1472 3 > gpurun_out/c22/split.log 2>&1
