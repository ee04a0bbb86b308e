# quick check: cold / hot-path parity tests, early-iteration timings, bench (no extras)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cold or adversarial or long_pin or config_fixed or to_tolerance or large_cliques or split" > gpurun_out/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.log
timeout 300 python tools/cold_phases.py > gpurun_out/cold_phases.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
HSDE_SPLIT_PREFETCH=0 timeout 300 python bench.py --steps 200 --warmup 220 --no-extras --no-cpu --no-e2e > gpurun_out/bench_steady_nopf.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 220 --no-extras --no-cpu --no-e2e > gpurun_out/bench_steady.json 2>&1
