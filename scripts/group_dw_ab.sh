mkdir -p gpurun_out
python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/gdw_tests.log 2>&1; echo pytest=$? >> gpurun_out/gdw_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["value"], d["clocks"]["sm_mhz"])'
for rep in 1 2; do for g in 0 1 2 4; do
  echo -n "1b g=$g " >> gpurun_out/gdw_ab.txt
  TP_GROUP_DW=$g timeout 300 $TR bench.py --gpus 4 --steps 10 --warmup 3 --slicing 2048 --batch-slices 1 --no-gpipe --no-cpu-baseline 2>>gpurun_out/gdw_err.txt | python -c "$P" >> gpurun_out/gdw_ab.txt 2>&1
done; done
S13=128,192,192,192,192,192,192,192,192,192,192
for g in 0 1 0 1; do
  echo -n "13b g=$g " >> gpurun_out/gdw_ab.txt
  TP_GROUP_DW=$g timeout 400 $TR bench.py --config gpt3-13b --gpus 4 --steps 4 --warmup 3 --slicing $S13 --batch-slices 4 --no-gpipe --no-cpu-baseline 2>>gpurun_out/gdw_err.txt | python -c "$P" >> gpurun_out/gdw_ab.txt 2>&1
done
