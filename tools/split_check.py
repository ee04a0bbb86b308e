"""k_cone_split vs the Jacobi-only CTA path: iterates, stats, timing.

    python tools/split_check.py [--config 4] [--iters 200]
"""
import os

os.environ.setdefault("HSDE_DEBUG", "1")  # diagnostics buffer (hsde_debug_jacobi)
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.synthetic import block_arrow, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
cp = block_arrow(12, 24, 16, 50, 0.05, 7, "ctapath") if a.config == "cta" else make_config(int(a.config))
res = {}
for name, flags in (("split", 0), ("jacobi", _lib.HSDE_FLAG_NO_SPLIT)):
    h = _lib.Handle(cp, flags=flags)
    t0 = time.time()
    hist = []
    done = 0
    while done < a.iters:
        step = min(20, a.iters - done)
        ms_chunk = h.time_iterations(step) / step
        done += step
        st = h.stats()
        if name == "split":
            dbg = h.debug_jacobi(0)
            nh = int(np.frombuffer(dbg[23:24].tobytes(), dtype=np.uint64)[0])
            if nh:
                print("   handovers at", done, nh, [tuple(round(float(x), 5) for x in dbg[24 + 3 * i:27 + 3 * i]) for i in range(min(nh, 8))], flush=True)
            dbg[23] = 0.0
            h.clear_debug() if hasattr(h, "clear_debug") else None
        hist.append((done, round(ms_chunk, 3), round(st["split_done"], 3), round(st["split_fp_iters"], 2), round(st["handoff_off"], 3),
                     round(st["handoff_rn"], 3), round(st["handoff_stall"], 3), round(st["split_resumed"], 3), round(st["mean_sweeps_large"], 2)))
    h.sync()
    u, w = h.get_state()
    res[name] = (u, w)
    ms = h.time_iterations(50) / 50 if hasattr(h, "time_iterations") else float("nan")
    prof, n = h.profile_iterations(10)
    print(name, "wall", round(time.time() - t0, 2), "ms/it(graph)", ms,
          {k: round(v / 10, 4) for k, v in prof.items() if v}, flush=True)
    dbg = h.debug_jacobi(0)
    st_ = dbg[48:57]
    if name == "split":
        print("  phase cycles:", [int(st_[i + 1] - st_[i]) for i in range(8)], "fp iters", dbg[47], flush=True)
    print("  (iter, ms/it, done, fp_iters, h_off, h_rn, h_stall, resumed, sweeps_large):", hist, flush=True)
    h.close()
du = np.linalg.norm(res["split"][0] - res["jacobi"][0]) / np.linalg.norm(res["jacobi"][0])
dw = np.linalg.norm(res["split"][1] - res["jacobi"][1]) / np.linalg.norm(res["jacobi"][1])
print(f"rel diff u {du:.3e} w {dw:.3e}")
