# final 4-GPU lines: multi-GPU tests, N = 2 / 4 bench (defaults), 13B K = 4 DP vs GPipe
mkdir -p gpurun_out/final4
timeout 1500 python -m pytest -q -p no:cacheprovider --timeout 600 tests/test_gpu_multi.py > gpurun_out/final4/pytest_multi.log 2>&1
echo rc=$? >> gpurun_out/final4/pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29557"
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/final4/bench_n2.json 2> gpurun_out/final4/bench_n2.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/final4/bench_n4.json 2> gpurun_out/final4/bench_n4.err
timeout 1200 $TR --nproc-per-node 4 bench.py --gpus 4 --config gpt3-13b --steps 3 --warmup 2 --no-cpu-baseline \
  > gpurun_out/final4/pipe_13b_n4.json 2> gpurun_out/final4/pipe_13b_n4.err
# 1F1B bounds the stage buffers: B = 32 in buffers sized for 8 sequences (vs GPipe store-all)
timeout 900 $TR --nproc-per-node 4 bench.py --gpus 4 --batch 32 --batch-slices 1,2 --no-gpipe --no-cpu-baseline --steps 3 \
  > gpurun_out/final4/gpipe_b32.json 2> gpurun_out/final4/gpipe_b32.err
TP_SCHEDULE=1f1b timeout 900 $TR --nproc-per-node 4 bench.py --gpus 4 --batch 32 --max-batch 8 --batch-slices 1,2 --no-gpipe \
  --no-cpu-baseline --steps 3 > gpurun_out/final4/1f1b_b32_mb8.json 2> gpurun_out/final4/1f1b_b32_mb8.err
