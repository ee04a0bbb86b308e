"""Create the config-N handle a few times with HSDE_TIMING phase output."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("HSDE_TIMING", "1")
from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

cp = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
for rep in range(5):
    t = time.perf_counter()
    h = _lib.Handle(cp)
    t1 = time.perf_counter()
    h.close()
    print(f"create {t1 - t:.3f}s close {time.perf_counter() - t1:.3f}s", file=sys.stderr, flush=True)
