"""Seeded synthetic SDPs of BASELINE.json's five configs, built directly in
the compressed layout.

The RNG call order follows SURVEY.md section 8(d) ("Exact RNG call order of
the survey generator"), so the same problems feed the reference (via
``problem.expand_to_mirror``) and this package:

* block-arrow / band: ``rng = default_rng(seed)``; ``slots`` = sorted pattern
  pairs (i <= j); ``k = round(f * len(slots))``; per constraint
  ``pick = rng.choice(len(slots), k, replace=False)`` then
  ``vals = rng.normal(size=k)``; then ``y0 = rng.normal(size=m)``;
  ``b = A vec(I)``, ``c = vec(I) + A' y0``.  Config 1 appends a copy of row 0
  with ``b[0] + 1``.
* max-cut: ``pts = rng.random((5000, 2))``, unit-disk graph of radius
  ``sqrt(6 / (pi (n - 1)))``, ``C = -L/4``, ``diag(X) = 1``.  Its chordal
  extension (the reference's greedy min-degree, graphs.py:121-163) is read
  from the committed fixture ``tests/golden/config3_cliques.npz`` generated
  by ``tests/golden/make_goldens.py`` with the live reference.

These stand in for no public dataset: BASELINE.json's configs are synthetic.
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import scipy.sparse as sp

from .problem import CompressedProblem, OBJECTIVE_SIGN, selector_flat

_REPO = Path(__file__).resolve().parent.parent
CONFIG3_CLIQUES = _REPO / "tests" / "golden" / "config3_cliques.npz"

CONFIG_NAMES = {
    0: "blockarrow_l20_d10_h10_m100_seed0",
    1: "infeasible_blockarrow_l10_d8_h8_m61_seed1",
    2: "band_n2000_w10_m200_seed2",
    3: "maxcut_rgg_n5000_seed3",
    4: "blockarrow_l400_d40_h40_m1000_seed4",
}


def _structure(n: int, cliques: list[np.ndarray]):
    """Upper slots (sorted), covered flats, slot->covered map for the cliques."""
    ups = []
    for c in cliques:
        c = np.asarray(c, dtype=np.int64)
        ii, jj = np.triu_indices(len(c))
        ups.append(c[ii] * n + c[jj])            # encode (i, j), i <= j, as i*n + j
    code = np.unique(np.concatenate(ups))
    si, sj = code // n, code % n                   # lexicographic (i, j) order
    flats = np.unique(np.concatenate([sj * n + si, si * n + sj]))
    return si, sj, flats


def _assemble(n, cliques, si, sj, covered, rows, b=None, c=None, name="",
              aggregate_edges=None, m=None):
    """rows: list of (slot_ids, vals) per constraint (symmetric A_i on slots)."""
    m = len(rows) if m is None else m
    p1 = np.searchsorted(covered, sj * n + si)     # flat j*n+i
    p2 = np.searchsorted(covered, si * n + sj)     # flat i*n+j (mirror)
    r_idx, c_idx, vals = [], [], []
    for r, (pick, val) in enumerate(rows):
        off = si[pick] != sj[pick]
        r_idx.append(np.full(pick.size + int(off.sum()), r, dtype=np.int64))
        c_idx.append(np.concatenate([p1[pick], p2[pick][off]]))
        vals.append(np.concatenate([val, val[off]]))
    if rows:
        A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(r_idx), np.concatenate(c_idx))),
                          shape=(m, covered.size), dtype=float)
    else:
        A = sp.csr_matrix((m, covered.size), dtype=float)
    A.sum_duplicates()
    A.sort_indices()
    cl = tuple(np.asarray(sorted(c), dtype=np.int64) for c in
               sorted(cliques, key=lambda c: (min(c), tuple(sorted(c)))))
    sizes = np.array([len(c) for c in cl], dtype=np.int64)
    offsets = np.zeros(len(cl) + 1, dtype=np.int64)
    np.cumsum(sizes * sizes, out=offsets[1:])
    gi = np.concatenate([selector_flat(c_, n) for c_ in cl])
    slot_cov = np.searchsorted(covered, gi).astype(np.int32)
    return CompressedProblem(
        n=n, m=m, covered=covered, c=c, A=A, b=b, cliques=cl, sizes=sizes,
        offsets=offsets, slot_cov=slot_cov, block_dims=(n,),
        objective_sign=OBJECTIVE_SIGN, aggregate_edges=aggregate_edges, name=name)


def _random_pattern_problem(n, cliques, m, frac, seed, name, extra_dup_row=False):
    rng = np.random.default_rng(seed)
    si, sj, covered = _structure(n, cliques)
    nslots = si.size
    k = int(round(frac * nslots))
    rows = []
    for _ in range(m):
        pick = rng.choice(nslots, size=k, replace=False)
        vals = rng.normal(size=k)
        rows.append((pick, vals))
    y0 = rng.normal(size=m)
    m_tot = m + (1 if extra_dup_row else 0)
    if extra_dup_row:
        rows.append(rows[0])
    cp = _assemble(n, cliques, si, sj, covered, rows, name=name, m=m_tot,
                   aggregate_edges=np.stack([si[si != sj], sj[si != sj]], axis=1))
    diag = (covered // n) == (covered % n)
    e = diag.astype(float)                          # vec(I) on covered coordinates
    b = cp.A @ e
    c = e + cp.A[:m].T @ y0
    if extra_dup_row:
        b[m] = b[0] + 1.0
    cp.b = np.asarray(b, dtype=float)
    cp.c = np.asarray(c, dtype=float)
    return cp


def block_arrow(l: int, d: int, h: int, m: int, frac: float, seed: int, name: str = "",
                infeasible: bool = False) -> CompressedProblem:
    """l diagonal blocks of size d plus a trailing arrow head of width h."""
    n = l * d + h
    head = np.arange(l * d, n)
    cliques = [np.concatenate([np.arange(k * d, (k + 1) * d), head]) for k in range(l)]
    return _random_pattern_problem(n, cliques, m, frac, seed, name, extra_dup_row=infeasible)


def band(n: int, w: int, m: int, frac: float, seed: int, name: str = "") -> CompressedProblem:
    cliques = [np.arange(i, i + w + 1) for i in range(n - w)]
    return _random_pattern_problem(n, cliques, m, frac, seed, name)


def maxcut_graph(n: int = 5000, seed: int = 3) -> np.ndarray:
    """Edges (i<j, sorted) of the seeded random geometric graph (config 3)."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = np.sqrt(6.0 / (np.pi * (n - 1)))
    pairs = sorted(cKDTree(pts).query_pairs(r))
    return np.asarray(pairs, dtype=np.int64).reshape(-1, 2)


def load_config3_cliques(path: Path = CONFIG3_CLIQUES) -> list[np.ndarray]:
    z = np.load(path)
    nodes, sizes = z["nodes"], z["sizes"]
    out, pos = [], 0
    for s in sizes:
        out.append(nodes[pos: pos + s])
        pos += s
    return out


def maxcut(n: int = 5000, seed: int = 3, cliques: list[np.ndarray] | None = None,
           name: str = "") -> CompressedProblem:
    edges = maxcut_graph(n, seed)
    if cliques is None:
        cliques = load_config3_cliques()
    si, sj, covered = _structure(n, cliques)
    # A_i = e_i e_i': one entry at flat i*n+i.
    diag_pos = np.searchsorted(covered, np.arange(n, dtype=np.int64) * (n + 1))
    A = sp.csr_matrix((np.ones(n), diag_pos, np.arange(n + 1)), shape=(n, covered.size))
    cp = _assemble(n, cliques, si, sj, covered, [], name=name, m=n, aggregate_edges=edges)
    cp.A = A
    deg = np.bincount(edges.ravel(), minlength=n).astype(float)
    c = np.zeros(covered.size)
    c[diag_pos] = -deg / 4.0                          # C = -L/4: diagonal -deg/4
    ei, ej = edges[:, 0], edges[:, 1]
    c[np.searchsorted(covered, ej * n + ei)] = 0.25   # off-diagonal -(-1)/4
    c[np.searchsorted(covered, ei * n + ej)] = 0.25
    cp.c = c
    cp.b = np.ones(n)
    return cp


def make_config(idx: int) -> CompressedProblem:
    """BASELINE.json configs[idx] as a CompressedProblem."""
    name = CONFIG_NAMES[idx]
    if idx == 0:
        return block_arrow(20, 10, 10, 100, 0.10, 0, name)
    if idx == 1:
        return block_arrow(10, 8, 8, 60, 0.10, 1, name, infeasible=True)
    if idx == 2:
        return band(2000, 10, 200, 0.05, 2, name)
    if idx == 3:
        return maxcut(5000, 3, name=name)
    if idx == 4:
        return block_arrow(400, 40, 40, 1000, 0.02, 4, name)
    raise ValueError(f"unknown config {idx}")


def config_stats(cp: CompressedProblem) -> dict:
    return {
        "n": cp.n, "m": cp.m, "N_c": cp.N_c, "p": cp.p, "n_d": cp.n_d,
        "nnz_A": int(cp.A.nnz), "clique_min": int(cp.sizes.min()),
        "clique_max": int(cp.sizes.max()),
        "sum_d3": int((cp.sizes.astype(np.int64) ** 3).sum()),
    }
