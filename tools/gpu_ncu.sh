mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cone_split|k_ua_half|k_spmv_half|k_rhs|k_xupd|k_pair_sum|k_schur|k_scalars|k_rowsum" -s 1800 -c 9 -o gpurun_out/full_r01d python tools/profile_run.py --config 4 --iters 220 > gpurun_out/ncu_full.log 2>&1
