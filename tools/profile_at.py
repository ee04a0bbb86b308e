"""Per-phase eager profile of k iterations after advancing the solve by w
iterations (graph replay): python tools/profile_at.py [config] [w] [k]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = int(sys.argv[2]) if len(sys.argv) > 2 else 200
k = int(sys.argv[3]) if len(sys.argv) > 3 else 10
h = _lib.Handle(make_config(cfg))
h.iterate(w)
h.sync()
prof, n = h.profile_iterations(k)
print({a: round(b / k, 4) for a, b in prof.items() if b}, h.stats())
