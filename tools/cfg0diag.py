import os

os.environ.setdefault("HSDE_DEBUG", "1")  # diagnostics buffer (hsde_debug_jacobi)
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1611_01828_b200 import _lib
from paper_1611_01828_b200.synthetic import make_config
h = _lib.Handle(make_config(0))
for i in range(12):
    ms = h.time_iterations(20)
    st = h.stats()
    dbg = h.debug_jacobi(0)
    stamps = dbg[48:57]
    print((i + 1) * 20, round(ms / 20 * 1e3, 1), "us/it", {k: round(v, 3) for k, v in st.items()},
          "phases", [int(stamps[j + 1] - stamps[j]) for j in range(8)], flush=True)
h.close()
