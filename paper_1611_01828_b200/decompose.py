"""Host decomposition: parsed SDP -> compressed problem.

Mirrors the reference's ``decompose`` (chordalsdp/decompose.py:106-176) but
builds the covered-coordinate layout (:class:`CompressedProblem`) directly,
without the reference's n**2-dense ``c`` and cover counts.  The graph work
(chordality test, minimum-degree chordal extension, maximal cliques) runs in
C++ in ``libhsde.so`` (``hsde_pattern_*``) with the reference's orderings and
tie-breaking (graphs.py:73-184, 217-220), so the cliques -- and therefore the
slot layout and every iterate -- are identical to the reference's.

Input: :func:`paper_1611_01828_b200.sdpa.parse_sdpa`'s ``SdpProblem`` (flat
``entry_table`` arrays, the fast path), the reference's ``SdpProblem``
(sdpa.py:58-91) or any object with ``m``, ``block_dims``, ``b``, ``C[blk]``
and ``A[i][blk]`` whose blocks carry upper-triangle ``entries`` (i, j, value).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _lib
from .problem import OBJECTIVE_SIGN, CompressedProblem

__all__ = ["chordal_cliques", "decompose"]


def chordal_cliques(n: int, edges, extend: bool = True):
    """Maximal cliques of the chordal extension of the pattern ``edges`` on
    nodes 0..n-1 (graphs.py:155-164 ``chordal_extend`` + :258-271
    ``maximal_cliques``).

    Returns ``(cliques, fill, was_chordal)``: cliques in the reference's order
    (by min node, then sorted nodes), the added fill edges (a < b) in
    elimination order, and whether the input was already chordal.  With
    ``extend=False`` a non-chordal pattern raises ``ValueError`` (NotChordal).
    """
    lib = _lib.load()
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    ei = np.ascontiguousarray(e[:, 0], dtype=np.int32)
    ej = np.ascontiguousarray(e[:, 1], dtype=np.int32)
    h = C.c_void_p()
    i32 = C.POINTER(C.c_int32)
    rc = lib.hsde_pattern_decompose(int(n), int(e.shape[0]), ei.ctypes.data_as(i32),
                                    ej.ctypes.data_as(i32), 1 if extend else 0, C.byref(h))
    if rc != 0:
        raise ValueError("pattern is not chordal; extend it first" if not extend
                         else "invalid sparsity pattern")
    try:
        nc, nn, nf = C.c_int64(), C.c_int64(), C.c_int64()
        ch = C.c_int32()
        lib.hsde_pattern_sizes(h, C.byref(nc), C.byref(nn), C.byref(nf), C.byref(ch))
        ptr = np.empty(nc.value + 1, dtype=np.int64)
        nodes = np.empty(max(nn.value, 1), dtype=np.int32)
        lib.hsde_pattern_cliques(h, ptr.ctypes.data_as(C.POINTER(C.c_int64)), nodes.ctypes.data_as(i32))
        fi = np.empty(max(nf.value, 1), dtype=np.int32)
        fj = np.empty(max(nf.value, 1), dtype=np.int32)
        lib.hsde_pattern_fill(h, fi.ctypes.data_as(i32), fj.ctypes.data_as(i32))
    finally:
        lib.hsde_pattern_destroy(h)
    cliques = [nodes[ptr[k]:ptr[k + 1]].astype(np.int64) for k in range(nc.value)]
    fill = np.stack([fi[:nf.value], fj[:nf.value]], axis=1).astype(np.int64)
    return cliques, fill, bool(ch.value)


def _entries(sym) -> np.ndarray:
    ent = getattr(sym, "entries", ())
    if len(ent) == 0:
        return np.zeros((0, 3))
    return np.asarray(ent, dtype=float).reshape(-1, 3)


def _object_entries(problem, dims, offs, m):
    """(global i, global j, value, matrix id) of every stored entry of an
    object-view problem (``C[blk]`` / ``A[i][blk]`` with ``entries``)."""
    mats = [problem.C] + [problem.A[i] for i in range(m)]
    gi_l, gj_l, v_l, who_l = [], [], [], []
    for mid, blocks in enumerate(mats):
        for blk in range(len(dims)):
            e = _entries(blocks[blk])
            if e.shape[0] == 0:
                continue
            gi_l.append(e[:, 0].astype(np.int64) + offs[blk])
            gj_l.append(e[:, 1].astype(np.int64) + offs[blk])
            v_l.append(e[:, 2])
            who_l.append(np.full(e.shape[0], mid, dtype=np.int64))
    gi = np.concatenate(gi_l) if gi_l else np.zeros(0, np.int64)
    gj = np.concatenate(gj_l) if gj_l else np.zeros(0, np.int64)
    vv = np.concatenate(v_l) if v_l else np.zeros(0)
    who = np.concatenate(who_l) if who_l else np.zeros(0, np.int64)
    return gi, gj, vv, who


def decompose(problem, split_cones: bool = True) -> CompressedProblem:
    """Decomposed standard form of a parsed problem, in the compressed layout
    (decompose.py:106-176): c = -vec(F0) (OBJECTIVE_SIGN), A rows vec(F_i)
    over both triangles, cliques of each block's extended aggregate pattern
    (or one clique per block with ``split_cones=False``)."""
    dims = tuple(int(d) for d in problem.block_dims)
    sizes = [abs(d) for d in dims]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offs[-1])
    m = int(problem.m)
    table = getattr(problem, "entry_table", None)
    if table is not None:
        # flat arrays from parse_sdpa (C++ reader): no per-entry Python objects
        mat, blk, ii, jj, vv = table
        gi = ii.astype(np.int64) + offs[blk]
        gj = jj.astype(np.int64) + offs[blk]
        vv = np.asarray(vv, dtype=float)
        who = mat.astype(np.int64)
    else:
        gi, gj, vv, who = _object_entries(problem, dims, offs, m)
    # aggregate pattern (decompose.py:85-103): off-diagonal entries of F0 and
    # every F_i, explicit zeros included
    off = gi != gj
    agg = np.unique(np.minimum(gi[off], gj[off]) * n + np.maximum(gi[off], gj[off]))
    agg_edges = np.stack([agg // n, agg % n], axis=1)
    cliques = []
    for blk, d in enumerate(sizes):
        o = offs[blk]
        sel = (agg_edges[:, 0] >= o) & (agg_edges[:, 1] < o + d)
        local = agg_edges[sel] - o
        if split_cones:
            cl, _, _ = chordal_cliques(d, local)
            cliques.extend(c + o for c in cl)
        else:
            cliques.append(np.arange(o, o + d, dtype=np.int64))
    cliques.sort(key=lambda c: (int(c[0]), tuple(int(x) for x in c)))
    csz = np.asarray([len(c) for c in cliques], dtype=np.int64)
    coffs = np.concatenate([[0], np.cumsum(csz * csz)]).astype(np.int64)
    slots = (np.concatenate([np.add.outer(c * n, c).ravel() for c in cliques])
             if cliques else np.zeros(0, np.int64))
    # c (both triangles) and A rows (both triangles; duplicates summed as the
    # reference's csr_matrix construction does)
    isc = who == 0
    c_idx = np.concatenate([gj[isc] * n + gi[isc], gi[isc] * n + gj[isc]])
    c_val = np.concatenate([vv[isc], vv[isc]]) * OBJECTIVE_SIGN
    ia = ~isc
    row = who[ia] - 1
    a_cols = [gj[ia] * n + gi[ia]]
    a_rows = [row]
    a_vals = [vv[ia]]
    offd = ia & off
    a_cols.append(gi[offd] * n + gj[offd])
    a_rows.append(who[offd] - 1)
    a_vals.append(vv[offd])
    a_cols = np.concatenate(a_cols)
    a_rows = np.concatenate(a_rows)
    a_vals = np.concatenate(a_vals)
    covered = np.unique(np.concatenate([slots, a_cols, c_idx[c_val != 0.0]]))
    pos = np.searchsorted(covered, a_cols)
    A = sp.csr_matrix((a_vals, (a_rows, pos)), shape=(m, covered.size))
    A.sum_duplicates()
    A.sort_indices()
    c = np.zeros(covered.size)
    cp_ = np.searchsorted(covered, c_idx)
    keep = (cp_ < covered.size)
    keep[keep] &= covered[cp_[keep]] == c_idx[keep]
    c[cp_[keep]] = c_val[keep]  # c[gj n + gi] = c[gi n + gj] = sign v (last write wins, same value)
    slot_cov = np.searchsorted(covered, slots).astype(np.int32)
    return CompressedProblem(
        n=n, m=m, covered=covered, c=c, A=A, b=np.asarray(problem.b, dtype=float).copy(),
        cliques=tuple(cliques), sizes=csz, offsets=coffs, slot_cov=slot_cov, block_dims=dims,
        objective_sign=OBJECTIVE_SIGN, aggregate_edges=agg_edges)
