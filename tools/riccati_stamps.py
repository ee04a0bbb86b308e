"""Fine clock64 stamps of one Riccati pass (pass 2, CTA 0) of k_cone_split on config 4."""
import os
os.environ.setdefault("HSDE_DEBUG", "1")
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_01828_b200 import _lib
from paper_1611_01828_b200.synthetic import make_config
h = _lib.Handle(make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4))
h.iterate(220); h.sync()
for rep in range(4):
    ms = h.time_iterations(1)
    d = h.debug_jacobi(0)
    st = d[1:8]
    ph = d[48:57]
    print(f"{ms:.3f} ms; pass 2: X products {int(st[1]-st[0])}, Y products {int(st[2]-st[1])}, barrier {int(st[3]-st[2])}, "
          f"update {int(st[4]-st[3])}, reduce+barrier {int(st[5]-st[4])}, decide {int(st[6]-st[5])}; total {int(st[6]-st[0])}; "
          f"phases {[int(ph[i+1]-ph[i]) for i in range(8)]} passes {d[47]}", flush=True)
h.close()
