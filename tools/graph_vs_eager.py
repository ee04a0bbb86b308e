"""Graph-replay time per iteration vs the eager per-phase sum at the same point."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

h = _lib.Handle(make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4))
h.iterate(200)
h.sync()
for rep in range(2):
    ms = h.time_iterations(40)
    prof, n = h.profile_iterations(40)
    tot = sum(prof.values())
    print(f"graph {ms / 40 * 1e3:7.1f} us/it   eager phases {tot / 40 * 1e3:7.1f} us/it", flush=True)
