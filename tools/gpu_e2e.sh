mkdir -p gpurun_out
HSDE_TIMING=1 timeout 600 python tools/e2e_profile.py 4 > gpurun_out/e2e_timing.log 2>&1
timeout 300 python tools/setup_profile.py 4 > gpurun_out/setup_profile.log 2>&1
