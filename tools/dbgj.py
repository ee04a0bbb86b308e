"""Jacobi off-norm history (relative to |A|_F) per sweep for a few cliques, at a
few iteration counts.  python tools/dbgj.py [config] [clique ...]"""
import os

os.environ.setdefault("HSDE_DEBUG", "1")  # diagnostics buffer (hsde_debug_jacobi)
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cliques = [int(x) for x in sys.argv[2:]] or [0]
cp = make_config(cfg)
for q in cliques:
    h = _lib.Handle(cp)
    h.debug_jacobi(q)  # select the clique (takes effect from the next launch)
    done = 0
    for it in [1, 2, 3, 5, 10, 20, 40, 80, 150, 300]:
        h.iterate(it - done)
        done = it
        d = h.debug_jacobi(q)
        vals = [v for v in d[1:40] if v >= 0]
        pn = [v for v in d[40:60] if v >= 0]
        print(q, it, "warm" if d[0] else "cold", " ".join(f"{v:.1e}" for v in vals),
              f"| PN {' '.join(f'{v:.1e}' for v in pn)} | g {d[63]:.1e} | split it {d[60]:.0f} off/g {d[62]:.2e}",
              flush=True)
    h.close()
