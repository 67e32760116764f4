# GEMM shapes of the default bench plan (T = 16384) vs cuBLAS; ncu --set full of the fc1 forward GEMM
mkdir -p gpurun_out/c28
timeout 600 python scripts/bench_kernels.py --which gemm --filter "T=16384" > gpurun_out/c28/gemm.jsonl 2>&1
timeout 600 python scripts/bench_kernels.py --which gemm --filter "b=8 l=1472" >> gpurun_out/c28/gemm.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100 -c 1 -o gpurun_out/c28/gemm_fc1 \
  python scripts/bench_kernels.py --which gemm --filter "T=16384 fc1 fwd" > gpurun_out/c28/ncu.log 2>&1
