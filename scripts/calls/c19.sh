# 4 x B200: DP vs uniform sweeps with the final defaults (device p2p), and the 1F1B memory bound
mkdir -p gpurun_out/c19
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29558"
timeout 1500 $TR --nproc-per-node 4 scripts/pipeline_sweep.py --config gpt3-13b-8k --uniform 1,2,4,8,16 \
  > gpurun_out/c19/sweep_13b8k_n4.jsonl 2> gpurun_out/c19/sweep_13b8k_n4.err
timeout 1500 $TR --nproc-per-node 4 scripts/pipeline_sweep.py --config gpt3-175b-24l --uniform 1,2,4,8,16 \
  > gpurun_out/c19/sweep_175b_n4.jsonl 2> gpurun_out/c19/sweep_175b_n4.err
timeout 900 $TR --nproc-per-node 4 bench.py --gpus 4 --batch 32 --batch-slices 1,2 --no-gpipe --no-cpu-baseline --steps 3 \
  > gpurun_out/c19/gpipe_b32.json 2> gpurun_out/c19/gpipe_b32.err
TP_SCHEDULE=1f1b timeout 900 $TR --nproc-per-node 4 bench.py --gpus 4 --batch 32 --max-batch 8 --batch-slices 1,2 --no-gpipe \
  --no-cpu-baseline --steps 3 > gpurun_out/c19/1f1b_b32_mb8.json 2> gpurun_out/c19/1f1b_b32_mb8.err
