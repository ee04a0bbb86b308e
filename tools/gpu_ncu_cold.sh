# ncu --set full of the cold path (k_cone_cold on all 400 cliques of config 4, iteration 5) with source
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cone_cold" -s 8 -c 1 -o gpurun_out/full_cold python tools/profile_run.py --config 4 --iters 8 > gpurun_out/ncu_cold.log 2>&1
tail -3 gpurun_out/ncu_cold.log
