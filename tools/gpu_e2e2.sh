mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
HSDE_TIMING=1 timeout 600 python tools/e2e_profile.py 4 > gpurun_out/e2e_timing.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu > gpurun_out/bench_quick.json 2>&1
