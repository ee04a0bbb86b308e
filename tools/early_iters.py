"""Per-iteration graph time and fast-path statistics of the first iterations.

    python tools/early_iters.py [--config 4] [--iters 40]
"""
import os

os.environ.setdefault("HSDE_DEBUG", "1")  # diagnostics buffer (hsde_debug_jacobi)
import argparse
import sys

import numpy as np
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=40)
a = ap.parse_args()
h = _lib.Handle(make_config(a.config))
for i in range(a.iters):
    ms = h.time_iterations(1)
    st = h.stats()
    print(i + 1, round(ms, 3), {k: round(v, 3) for k, v in st.items() if k in (
        "mean_sweeps_large", "split_done", "split_fp_iters", "split_resumed", "handoff_off", "handoff_stall")},
        flush=True)
    dbg = h.debug_jacobi(0)
    nh = int(np.frombuffer(dbg[23:24].tobytes(), dtype=np.uint64)[0])
    if nh:
        print("   stalls", nh, [tuple(float('%.3g' % x) for x in dbg[24 + 7 * i:31 + 7 * i]) for i in range(min(nh, 4))], flush=True)
h.close()
