"""Phase clock of the cold path (k_cone_cold / k_cone_split cold branch) on
config 4: clock64 stamps of CTA 0 (W.dbg[32..39]) after project_cone (plain
mode, all 400 cliques cold) and after hot iterations 1..3.

    python tools/cold_phases.py
"""
import os

os.environ.setdefault("HSDE_DEBUG", "1")  # diagnostics buffer (hsde_debug_jacobi)
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

names = ["load", "tridiag", "bisect", "twisted", "backtr", "newton-schulz", "P"]
cp = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = _lib.Handle(cp)
rng = np.random.default_rng(1)
v = rng.normal(size=h.total)
for rep in range(3):
    t = time.perf_counter()
    h.project_cone(v)
    dt = time.perf_counter() - t
    st = h.debug_jacobi(0)[32:40]
    cyc = [int(st[i + 1] - st[i]) for i in range(7)]
    print("plain", f"{dt * 1e3:.2f} ms wall (incl. copies)", dict(zip(names, cyc)), "total", int(st[7] - st[0]), flush=True)
    dd = h.debug_jacobi(0)[16:21]
    print("   tridiag step 20 (warp 1): producer wait", int(dd[1] - dd[0]), "partials", int(dd[2] - dd[1]),
          "barrier", int(dd[3] - dd[2]), "reduce+update", int(dd[4] - dd[3]), flush=True)
for i in range(3):
    ms = h.time_iterations(1)
    st = h.debug_jacobi(0)[32:40]
    cyc = [int(st[k + 1] - st[k]) for k in range(7)]
    print("hot it", i + 1, f"{ms:.3f} ms", dict(zip(names, cyc)), "total", int(st[7] - st[0]), flush=True)
h.close()
