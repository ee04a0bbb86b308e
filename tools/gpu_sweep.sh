# grid-knob sweep of the streaming kernels on config 4 (kernel ms per iteration from bench.py)
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/sweep.txt; env "$@" timeout 180 python bench.py --steps 200 --warmup 20 --no-extras --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernel_ms_per_iteration']; print(round(d['value'],1), {x: round(k[x]*1e3,1) for x in ('k_rhs','k_xupd','k_ua','k_spmv_seg')})" >> gpurun_out/sweep.txt 2>&1; }
run X=0
for r in 592 2368 4736 9472; do run HSDE_RHS_CTAS=$r; done
for r in 592 2368 4736; do run HSDE_XUPD_CTAS=$r; done
for r in 1184 3552 4736; do run HSDE_UA_CTAS=$r; done
for t in 1024 4096; do run HSDE_RT_TILE=$t; done
for t in 1 4; do run HSDE_RT_SPLIT=$t; done
run X=0
