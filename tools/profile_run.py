"""Short driver for ncu / compute-sanitizer: K iterations of a BASELINE config.

    python tools/profile_run.py --config 4 --iters 8 [--cold] [--eager]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--cold", action="store_true")
ap.add_argument("--eager", action="store_true", help="eager launches (profile hook) instead of graphs")
a = ap.parse_args()
cp = make_config(a.config)
h = _lib.Handle(cp, flags=_lib.HSDE_FLAG_COLD_EIG if a.cold else 0)
t = time.time()
if a.eager:
    prof, n = h.profile_iterations(a.iters)
    print({k: round(v / a.iters, 4) for k, v in prof.items() if v})
else:
    h.iterate(a.iters)
    h.sync()
print("iters", a.iters, "wall", time.time() - t, h.stats())
h.close()
