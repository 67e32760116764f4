# GEMM-only A/B: libtp.so (uniform-datapath GEMM MMA issue, 32-bit stream-K math) vs libtp_base.so (same
# tree with the previous gemm_sm100.cu)
mkdir -p gpurun_out/c36
VARS="TP_LIB=paper_2102_07988_b200/libtp.so TP_LIB=paper_2102_07988_b200/libtp_base.so" SLICING=2048 scripts/env_ab.sh 5 > gpurun_out/c36/ab.txt 2>&1
for lib in libtp.so libtp_base.so libtp.so libtp_base.so; do
  TP_LIB=paper_2102_07988_b200/$lib timeout 600 python scripts/bench_kernels.py --which gemm --filter "T=16384" > gpurun_out/c36/gemm_$lib.$RANDOM.jsonl 2>&1
done
