mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "adversarial or first_iteration or large_cliques" > gpurun_out/pytest_adv.log 2>&1; echo "exit $?" >> gpurun_out/pytest_adv.log
timeout 300 python tools/cfg0diag.py > gpurun_out/cfg0diag.txt 2>&1
timeout 300 python tools/cold_phases.py > gpurun_out/cold_phases.txt 2>&1
timeout 300 python tools/early_iters.py --iters 45 > gpurun_out/early_iters.txt 2>&1
timeout 300 python tools/split_check.py --iters 60 > gpurun_out/split_check.txt 2>&1
