import sys, numpy as np
sys.path.insert(0, '.')
from paper_1611_01828_b200 import _lib
from paper_1611_01828_b200.synthetic import make_config
cp = make_config(4)
ha = _lib.Handle(cp)
hb = _lib.Handle(cp, flags=_lib.HSDE_FLAG_COLD_EIG)
for it in range(1, 6):
    ha.iterate(1); hb.iterate(1)
    ua, _ = ha.get_state(); ub, _ = hb.get_state()
    d = ha.debug_jacobi(0)
    print(it, "rel diff", np.linalg.norm(ua - ub) / np.linalg.norm(ub),
          "seg", [float(np.linalg.norm(ua[sl] - ub[sl]) / max(np.linalg.norm(ub[sl]), 1e-300)) for sl in (cp.sl_x, cp.sl_s, cp.sl_y, cp.sl_v)])
    print("   dbg", np.array2string(d[:21], precision=1), ha.stats())
