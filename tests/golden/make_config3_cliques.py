"""Generate tests/golden/config3_cliques.npz with the LIVE reference.

Config 3's chordal extension is the reference's greedy minimum-degree fill
(graphs.py:121-163) followed by maximal_cliques (graphs.py:259-271).  This
script runs those reference functions once, in the build container (where
/root/reference exists), and commits the resulting clique list so the GPU box
(no reference there) builds the identical problem.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_config3_cliques.py
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

from chordalsdp.graphs import SparsityPattern, chordal_extend, maximal_cliques  # noqa: E402

from paper_1611_01828_b200.synthetic import maxcut_graph  # noqa: E402

n = 5000
edges = maxcut_graph(n, 3)
g = SparsityPattern.from_edges(n, [tuple(e) for e in edges])
ext = chordal_extend(g)
dec = maximal_cliques(ext)
nodes = np.concatenate([np.asarray(c, dtype=np.int32) for c in dec.cliques])
sizes = np.asarray(dec.sizes, dtype=np.int32)
h = hashlib.sha256(edges.tobytes()).hexdigest()
out = Path(__file__).with_name("config3_cliques.npz")
np.savez_compressed(out, nodes=nodes, sizes=sizes, edges_sha256=np.array(h))
print(f"edges={len(edges)} cliques={len(sizes)} sizes {sizes.min()}..{sizes.max()} "
      f"n_d={int((sizes.astype(np.int64)**2).sum())} -> {out}")
