# final-tree refresh of the other north-star configurations at K = 4: 175B-24L (B = 2) and 13B-8k (B = 2)
mkdir -p gpurun_out/final4b
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29563"
timeout 1200 $TR --nproc-per-node 4 bench.py --gpus 4 --config gpt3-175b-24l --steps 3 --warmup 2 --no-cpu-baseline \
  > gpurun_out/final4b/pipe_175b_n4.json 2> gpurun_out/final4b/pipe_175b_n4.err
timeout 1200 $TR --nproc-per-node 4 bench.py --gpus 4 --config gpt3-13b-8k --steps 3 --warmup 2 --no-cpu-baseline \
  > gpurun_out/final4b/pipe_13b8k_n4.json 2> gpurun_out/final4b/pipe_13b8k_n4.err
