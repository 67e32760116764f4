# step A/B on one box: uniform-datapath MMA issue build (libtp.so) vs the previous commit (libtp_base.so)
mkdir -p gpurun_out/c34
VARS="TP_LIB=paper_2102_07988_b200/libtp.so TP_LIB=paper_2102_07988_b200/libtp_base.so" SLICING=2048 scripts/env_ab.sh 3 > gpurun_out/c34/ab.txt 2>&1
for lib in libtp.so libtp_base.so; do
  echo "TP_LIB=$lib" >> gpurun_out/c34/attn.txt
  TP_LIB=paper_2102_07988_b200/$lib timeout 120 python scripts/attn_bench.py 128 2048 0 2048 20 >> gpurun_out/c34/attn.txt 2>&1
done
