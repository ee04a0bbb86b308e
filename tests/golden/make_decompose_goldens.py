"""Golden fixtures for the host decomposition, made by
running the LIVE reference in the build container:

    python tests/golden/make_decompose_goldens.py

* random sparsity patterns (chordal and not) -> the reference's
  ``chordal_extend`` fill edges and ``maximal_cliques`` cliques
  (graphs.py:73-184, 217-220);
* small seeded multi-block SDP problems (reference ``SdpProblem`` /
  ``SymMatrix``) -> ``decompose`` (decompose.py:106-176), stored in the
  compressed layout (covered coordinates, c, A in CSR, cliques).

Writes ``tests/golden/decompose.npz``.  The GPU box never runs this.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

from chordalsdp.decompose import decompose  # noqa: E402
from chordalsdp.graphs import SparsityPattern, chordal_extend, is_chordal, maximal_cliques  # noqa: E402
from chordalsdp.sdpa import SdpProblem  # noqa: E402
from chordalsdp.symmat import SymMatrix  # noqa: E402

from paper_1611_01828_b200.problem import compress  # noqa: E402


def random_pattern(rng, n, p):
    iu = np.triu_indices(n, 1)
    keep = rng.random(iu[0].size) < p
    return [(int(i), int(j)) for i, j in zip(iu[0][keep], iu[1][keep])]


def random_sym(rng, dim, density):
    ent = []
    for i in range(dim):
        for j in range(i, dim):
            if i == j or rng.random() < density:
                if rng.random() < 0.9:
                    ent.append((i, j, float(rng.normal())))
    return SymMatrix(dim, tuple(ent))


def main():
    out = {}
    rng = np.random.default_rng(20261020)
    cases = [(12, 0.3), (30, 0.1), (30, 0.25), (60, 0.05), (80, 0.08), (120, 0.03), (200, 0.02)]
    for t, (n, p) in enumerate(cases):
        edges = random_pattern(rng, n, p)
        g = SparsityPattern.from_edges(n, edges)
        chordal, _ = is_chordal(g)
        ext = chordal_extend(g)
        dec = maximal_cliques(ext)
        fill = sorted(ext.edges - g.edges)
        pre = f"g{t}_"
        out[pre + "n"] = n
        out[pre + "edges"] = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        out[pre + "chordal"] = int(chordal)
        out[pre + "fill"] = np.asarray(fill, dtype=np.int32).reshape(-1, 2)
        out[pre + "clique_nodes"] = np.concatenate([np.asarray(c, np.int32) for c in dec.cliques])
        out[pre + "clique_sizes"] = np.asarray([len(c) for c in dec.cliques], np.int32)
    out["n_graphs"] = len(cases)
    # small SDP problems: two PSD blocks and one diagonal block
    probs = [((8, 6, -3), 5, 0.25), ((10, 12), 7, 0.15), ((15,), 4, 0.2)]
    for t, (dims, m, dens) in enumerate(probs):
        blocks = [abs(d) for d in dims]

        def mat(k):
            mats = []
            for d, dd in zip(blocks, dims):
                if dd < 0:  # diagonal block
                    mats.append(SymMatrix(d, tuple((i, i, float(rng.normal())) for i in range(d))))
                else:
                    mats.append(random_sym(rng, d, dens))
            return tuple(mats)

        C = mat(-1)
        A = tuple(mat(i) for i in range(m))
        b = rng.normal(size=m)
        prob = SdpProblem(m=m, block_dims=tuple(dims), b=b, C=C, A=A)
        dp = decompose(prob)
        cp = compress(dp)
        pre = f"p{t}_"
        out[pre + "dims"] = np.asarray(dims, np.int32)
        out[pre + "m"] = m
        out[pre + "b"] = b
        # the problem entries: (matrix id (0 = C, 1 + i = A_i), block, i, j, value)
        rows = []
        for mid, mats in enumerate((C,) + A):
            for blk, sm in enumerate(mats):
                for i, j, v in sm.entries:
                    rows.append((mid, blk, i, j, v))
        rows = np.asarray(rows, dtype=float)
        out[pre + "entries"] = rows
        out[pre + "covered"] = cp.covered
        out[pre + "c"] = cp.c
        out[pre + "A_data"] = cp.A.data
        out[pre + "A_indices"] = cp.A.indices
        out[pre + "A_indptr"] = cp.A.indptr
        out[pre + "clique_nodes"] = np.concatenate([np.asarray(c, np.int64) for c in cp.cliques])
        out[pre + "clique_sizes"] = np.asarray(cp.sizes, np.int64)
        out[pre + "slot_cov"] = cp.slot_cov
        out[pre + "aggregate_edges"] = cp.aggregate_edges
    out["n_problems"] = len(probs)
    np.savez_compressed(HERE / "decompose.npz", **out)
    print("wrote", HERE / "decompose.npz", {k: np.asarray(v).shape for k, v in out.items() if k.endswith("fill")})


if __name__ == "__main__":
    main()
