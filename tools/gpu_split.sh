mkdir -p gpurun_out
timeout 300 python tools/split_check.py --config 4 --iters 220 > gpurun_out/split_c4_v1.log 2>&1
timeout 300 python bench.py --no-extras --no-e2e --no-cpu > gpurun_out/bench_quick.json 2>&1
