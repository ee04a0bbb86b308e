"""Phase timing of the public solve path (solve_decomposed) on a BASELINE config.

    python tools/e2e_profile.py [config]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1611_01828_b200 as H  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cp = make_config(cfg)
H.solve_decomposed(make_config(0), H.SolverSettings())  # CUDA context, library load
H.solve_decomposed(make_config(4 if cfg != 4 else 3), H.SolverSettings())  # warm the device pool
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
rep = H.solve_decomposed(cp, H.SolverSettings())  # first solve of this problem (report caches cold)
pr.disable()
wall = time.perf_counter() - t
print(f"wall {wall:.3f}s setup {rep.timing.setup_s:.3f}s loop {rep.timing.iterations_s:.3f}s "
      f"iters {rep.iterations} status {rep.status}")
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
