mkdir -p gpurun_out
HSDE_TIMING=1 timeout 600 python bench.py --no-extras --no-cpu > gpurun_out/bench_quick_t.json 2> gpurun_out/bench_quick_t.err
