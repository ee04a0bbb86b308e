"""Cold-path phase clock vs. cliques per SM: project_cone (plain mode) on
block-arrow problems with 148 / 296 / 444 cliques of order 80.

    python tools/cold_contention.py
"""
import os

os.environ.setdefault("HSDE_DEBUG", "1")  # diagnostics buffer (hsde_debug_jacobi)
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import block_arrow  # noqa: E402

names = ["load", "tridiag", "bisect", "twisted", "backtr", "newton-schulz", "P"]
for p in (148, 296, 444):
    cp = block_arrow(p, 40, 40, 50, 0.02, 4, f"arrow{p}")
    h = _lib.Handle(cp)
    v = np.random.default_rng(1).normal(size=h.total)
    for _ in range(2):
        h.project_cone(v)
    st = h.debug_jacobi(0)[32:40]
    cyc = [int(st[i + 1] - st[i]) for i in range(7)]
    print(p, "cliques:", dict(zip(names, cyc)), "total", int(st[7] - st[0]), flush=True)
    h.close()
