# 1 x B200: stream-K A/B, GEMM microbench, cost-model study (dense table + Fig. 4), K = 4 / 8
# predictions, the default bench line, and the ncu metrics pass of one step
mkdir -p gpurun_out/c13
timeout 1200 python -m pytest -q -p no:cacheprovider --timeout 600 tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_fullsize.py > gpurun_out/c13/pytest.log 2>&1
echo rc=$? >> gpurun_out/c13/pytest.log
VARS="TP_ATTN_DKV_FUSED=1 TP_ATTN_DKV_FUSED=0" scripts/env_ab.sh 2 > gpurun_out/c13/ab_dkv.txt 2>&1
VARS="TP_GEMM_STREAMK=1 TP_GEMM_STREAMK=0" scripts/env_ab.sh 2 > gpurun_out/c13/ab_sk.txt 2>&1
timeout 600 python scripts/bench_kernels.py --which gemm > gpurun_out/c13/gemm.jsonl 2>&1
timeout 1500 python scripts/cost_model_study.py --config gpt3-13b --layers 10 --out gpurun_out/c13/cost_model_13b.json > gpurun_out/c13/cost_model.log 2>&1
TP_COMM_ALPHA_NS=12500 TP_COMM_GBS=600 timeout 1800 python scripts/predict_stages.py --config gpt3-13b --stages 4,8 --out gpurun_out/c13/predict_13b.jsonl > gpurun_out/c13/predict.log 2>&1
timeout 600 python bench.py > gpurun_out/c13/bench_n1.json 2> gpurun_out/c13/bench_n1.err
B="python bench.py --steps 1 --warmup 3 --slicing 576,1472 --batch-slices 8 --no-gpipe --no-cpu-baseline"
TP_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/c13/metrics.csv $B > gpurun_out/c13/ncu_metrics.log 2>&1
