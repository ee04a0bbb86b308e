"""Per-shard kernel times of config 4 with G = 1, 2, 4, 8 clique shards emulated on
one GPU (same kernels as the NCCL path; reductions by a device sum): the eager
profile sums each phase over the shards, so phase / G is what one rank would spend
on it (no overlap between ranks is emulated; the all-reduces are device sums).

    python tools/shard_profile.py [--config 4] [--warm 230]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1611_01828_b200 import _lib  # noqa: E402
from paper_1611_01828_b200.shard import make_shards  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--warm", type=int, default=230)
a = ap.parse_args()
cp = make_config(a.config)
for G in (1, 2, 4, 8):
    sh = make_shards(cp, G) if G > 1 else None
    h = _lib.Handle(cp, shards=sh)
    h.iterate(a.warm)
    h.sync()
    n = 10
    prof, _ = h.profile_iterations(n)
    per = {k: round(1e3 * v / n / G, 1) for k, v in prof.items() if v}
    tot = sum(per.values())
    cl = [len(s.problem.sizes) for s in sh] if sh else [cp.p]
    print(f"G={G}: cliques per shard {cl}; half passes {h.half_passes}; per-shard us per iteration {per}; sum {tot:.0f} us",
          flush=True)
    h.close()
