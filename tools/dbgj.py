import sys, numpy as np
sys.path.insert(0, '.')
from paper_1611_01828_b200 import _lib
from paper_1611_01828_b200.synthetic import make_config
cp = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = _lib.Handle(cp)
for it in [1, 2, 3, 5, 10, 20, 40, 80, 150, 300]:
    prev = getattr(h, "_it", 0)
    h.iterate(it - prev); h._it = it
    d = h.debug_jacobi(0)
    vals = [v for v in d[1:] if v >= 0]
    print(it, "warm" if d[0] else "cold", " ".join(f"{v:.1e}" for v in vals))
