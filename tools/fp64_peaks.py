"""Measure the fp64 peaks used as the eigensolver roofline denominator.

    python tools/fp64_peaks.py > profiles/fp64_peaks.json

* fp64_tflops_dgemm: cuBLAS DGEMM (torch.matmul, float64) 8192^3, best of 10,
  CUDA events (the same recipe as MEASURED_PEAKS.json's bf16 entry);
* fp64_tflops_ffma: tools/fp64_fma_bench (plain DFMA chains on every SM).
fp64_tflops = max of the two.
"""
import json
import subprocess
import sys
from pathlib import Path

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
dgemm = 2 * n ** 3 / (best / 1e3) / 1e12
here = Path(__file__).resolve().parent
exe = here / "fp64_fma_bench"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe),
                str(here / "fp64_fma_bench.cu")], check=True)
ffma = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout)
out = {"fp64_tflops_dgemm": round(dgemm, 3), "fp64_tflops_ffma": ffma["fp64_tflops_ffma"],
       "fp64_tflops": round(max(dgemm, ffma["fp64_tflops_ffma"]), 3),
       "gpu": torch.cuda.get_device_name(0),
       "how": "DGEMM: torch.matmul float64 8192^3 best of 10 (CUDA events); "
              "FFMA: 148x8 CTAs x 256 threads x 8 independent DFMA chains, best of 5"}
print(json.dumps(out, indent=1))
