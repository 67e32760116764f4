# 4 x B200: multi-GPU parity, N = 2 / 4 bench lines, the 13B pipeline (DP vs GPipe), p2p / schedule A/Bs
mkdir -p gpurun_out/c10
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_multi.py tests/test_gpu_parity.py -k "multi or nccl or p2p or 1f1b or profile" > gpurun_out/c10/pytest_multi.log 2>&1
echo rc=$? >> gpurun_out/c10/pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29555"
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/c10/bench_n2.json 2> gpurun_out/c10/bench_n2.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/c10/bench_n4.json 2> gpurun_out/c10/bench_n4.err
TP_DEVICE_P2P=1 timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/c10/bench_n4_p2p.json 2> gpurun_out/c10/bench_n4_p2p.err
TP_SCHEDULE=1f1b timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/c10/bench_n4_1f1b.json 2> gpurun_out/c10/bench_n4_1f1b.err
for v in "" "TP_DEVICE_P2P=1"; do
  env $v timeout 1200 $TR --nproc-per-node 4 bench.py --gpus 4 --config gpt3-13b --steps 3 --warmup 2 --no-cpu-baseline \
    > gpurun_out/c10/pipe_13b_n4${v:+_p2p}.json 2> gpurun_out/c10/pipe_13b_n4${v:+_p2p}.err
done
timeout 1500 $TR --nproc-per-node 4 scripts/pipeline_sweep.py --config gpt3-13b-8k --uniform 1,2,4,8,16 \
  > gpurun_out/c10/sweep_13b8k_n4.jsonl 2> gpurun_out/c10/sweep_13b8k_n4.err
