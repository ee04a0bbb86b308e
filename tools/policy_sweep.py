"""Cold / warm policy thresholds (HSDE_POL_F2C, HSDE_POL_C2F: read once per process):
per-iteration graph time of config 4's iterations 1..40 and the window 6..25 mean.

    HSDE_POL_F2C=0.16 HSDE_POL_C2F=0.5 python tools/policy_sweep.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

h = _lib.Handle(make_config(4))
ms, fast = [], []
for i in range(40):
    ms.append(h.time_iterations(1))
    st = h.stats()
    fast.append(st["split_done"])
win = sum(ms[5:25]) / 20
print(f"F2C={os.environ.get('HSDE_POL_F2C', '0.1225')} C2F={os.environ.get('HSDE_POL_C2F', '0.36')}: "
      f"window 6..25 mean {win:.3f} ms, 1..40 sum {sum(ms):.2f} ms; fast fraction per iteration "
      + " ".join(f"{f:.1f}" for f in fast), flush=True)
h.close()
