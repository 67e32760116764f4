# clock sampler check at N = 4 (short timed region) and N = 1
mkdir -p gpurun_out/c42
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29561"
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/c42/bench_n4.json 2> gpurun_out/c42/bench_n4.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c42/bench_n1.json 2> gpurun_out/c42/bench_n1.err
