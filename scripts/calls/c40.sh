# final N = 1 bench line (default arguments) on the final tree, twice
mkdir -p gpurun_out/c40
timeout 900 python bench.py > gpurun_out/c40/bench_n1.json 2> gpurun_out/c40/bench_n1.err
timeout 900 python bench.py > gpurun_out/c40/bench_n1_b.json 2> gpurun_out/c40/bench_n1_b.err
