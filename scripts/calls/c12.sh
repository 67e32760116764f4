# 4 x B200: balanced-partition parity (1 GPU + NCCL + device p2p), then the N = 2 / 4 bench lines with
# the new defaults (device p2p, balanced partition) and the uniform / NCCL A/B
mkdir -p gpurun_out/c12
timeout 1500 python -m pytest -q -p no:cacheprovider --timeout 600 tests/test_gpu_multi.py tests/test_gpu_parity.py -k "balanced or device or 1f1b" > gpurun_out/c12/pytest.log 2>&1
echo rc=$? >> gpurun_out/c12/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29556"
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/c12/bench_n2.json 2> gpurun_out/c12/bench_n2.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/c12/bench_n4.json 2> gpurun_out/c12/bench_n4.err
TP_PARTITION=uniform timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/c12/bench_n4_uniform.json 2> gpurun_out/c12/bench_n4_uniform.err
# 13B K = 4: DP vs GPipe with the new defaults (device p2p; balanced = uniform for 13B)
timeout 1200 $TR --nproc-per-node 4 bench.py --gpus 4 --config gpt3-13b --steps 3 --warmup 2 --no-cpu-baseline \
  > gpurun_out/c12/pipe_13b_n4.json 2> gpurun_out/c12/pipe_13b_n4.err
timeout 1500 $TR --nproc-per-node 4 bench.py --gpus 4 --config gpt3-175b-24l --steps 3 --warmup 2 --no-cpu-baseline \
  > gpurun_out/c12/pipe_175b_n4.json 2> gpurun_out/c12/pipe_175b_n4.err
