"""Mean / max Jacobi sweeps of the CTA cliques at a few iteration counts."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

cp = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = _lib.Handle(cp)
done = 0
for it in [1, 2, 5, 10, 20, 30, 40, 60, 80, 100, 120, 150, 200, 220, 250, 300]:
    h.iterate(it - done)
    done = it
    st = h.stats()
    print(it, round(st["mean_sweeps"], 2), st["max_sweeps"], flush=True)
