mkdir -p gpurun_out/c1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1/smi.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/c1/smoke.log 2>&1
echo smoke rc=$? >> gpurun_out/c1/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/c1/pytest.log 2>&1
echo pytest rc=$? >> gpurun_out/c1/pytest.log
VARS="TP_GEMM_GROUP=2048 TP_GEMM_GROUP=100000" scripts/env_ab.sh 2 > gpurun_out/c1/ab_group.txt 2>&1
timeout 600 python bench.py > gpurun_out/c1/bench.json 2> gpurun_out/c1/bench.err
