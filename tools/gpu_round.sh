# One full GPU evidence pass: tests, smoke, both bench arms, launch lists, one ncu --set full capture.
# Usage (from the repo root, through gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r02}
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/small_profile.py > gpurun_out/small_profile_$TAG.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1800 -c 200 --csv --log-file gpurun_out/launches_steady_$TAG.csv python tools/profile_run.py --config 4 --iters 220 > gpurun_out/ncu_launch2.log 2>&1
for c in 0 1 2 3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rhs|k_pair_sum|k_spmv|k_rowsum|k_schur|k_ua|k_scalars|k_cone|k_xupd|k_sep|k_zero" -s 300 -c 150 --csv --log-file gpurun_out/launches_cfg${c}_$TAG.csv python tools/profile_run.py --config $c --iters 80 > gpurun_out/ncu_launch_cfg$c.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cone|k_cold|k_ua_half|k_spmv_half|k_rhs|k_xupd|k_pair_sum|k_schur|k_scalars|k_rowsum" -s 1800 -c 12 -o gpurun_out/full_$TAG python tools/profile_run.py --config 4 --iters 220 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
