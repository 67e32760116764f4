mkdir -p gpurun_out/c6
python scripts/bench_kernels.py --which gemm > gpurun_out/c6/gemm.jsonl 2>&1
B="python bench.py --steps 1 --warmup 3 --slicing 576,1472 --batch-slices 8 --no-gpipe --no-cpu-baseline"
# job 2 (b=8 x 1472) layer 0: QKV is the 5th K-major GEMM of job 2 ... capture QKV (launch 97 = first GEMM of job 2? use kernel regex + skip)
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"gemm_sm100" --launch-skip 98 -c 4 -o gpurun_out/c6/gemm_job2 $B > gpurun_out/c6/ncu1.log 2>&1
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"gemm_sm100_kernel<2, 256, true, true" -c 4 -o gpurun_out/c6/gemm_dw $B > gpurun_out/c6/ncu2.log 2>&1
