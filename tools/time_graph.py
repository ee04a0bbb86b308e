"""Graph-replay iterations/s per BASELINE config (device-resident, no extras).

    python tools/time_graph.py [config ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

for c in [int(x) for x in sys.argv[1:]] or [0, 1, 2, 3, 4]:
    cp = make_config(c)
    h = _lib.Handle(cp)
    h.iterate(20)
    h.sync()
    n = 200 if c == 4 else 400
    ms = h.time_iterations(n)
    print(f"config {c}: {n / ms * 1e3:9.1f} it/s  ({ms / n * 1e3:7.1f} us/it)  {h.stats()}", flush=True)
    h.close()
