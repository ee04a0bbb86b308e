set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1800 -c 200 --csv --log-file gpurun_out/launches_steady.csv python tools/profile_run.py --config 4 --iters 220 > gpurun_out/ncu_launch2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cone_split|k_ua_half|k_spmv_half|k_rhs|k_xupd|k_pair_sum|k_schur|k_scalars|k_rowsum" -s 1800 -c 9 -o gpurun_out/full_r01f python tools/profile_run.py --config 4 --iters 220 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
