"""Per-kernel time per iteration (CUDA events, eager launches) and graph-replay
rate for BASELINE configs 0-3 after a warm-up.

    python tools/small_profile.py [--warm 200]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warm", type=int, default=200)
ap.add_argument("--configs", default="0,1,2,3")
a = ap.parse_args()
for cfg in map(int, a.configs.split(",")):
    h = _lib.Handle(make_config(cfg))
    h.time_iterations(a.warm)
    ms = h.time_iterations(200) / 200
    prof, nl = h.profile_iterations(20)
    print(f"config {cfg}: graph {ms * 1e3:.1f} us/it ({1.0 / ms * 1e3:.0f} it/s), launches/it {nl / 20:.0f}; eager us/it:",
          {k: round(v / 20 * 1e3, 1) for k, v in prof.items() if v}, flush=True)
    h.close()
