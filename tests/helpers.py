"""Test helpers: rebuild golden toy problems, dense oracles of the embedding.

The dense oracles restate the reference's test oracles
(pkg/tests/helpers.py:174-223): the explicit skew matrix Q and the inner
block system, materialised for tiny problems.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem


def toy_problem(z, pre: str = "") -> DecomposedProblem:
    n, m = int(z[pre + "n"]), int(z[pre + "m"])
    nodes, sizes = z[pre + "clique_nodes"], z[pre + "clique_sizes"]
    cl, pos = [], 0
    for s in sizes:
        cl.append(list(map(int, nodes[pos: pos + s])))
        pos += s
    dec = CliqueDecomposition.build(n, cl)
    A = sp.csr_matrix(np.asarray(z[pre + "A"], dtype=float).reshape(m, n * n))
    return DecomposedProblem(n=n, m=m, c=np.asarray(z[pre + "c"], float), A=A,
                             b=np.asarray(z[pre + "b"], float), dec=dec, block_dims=(n,))


def dense_selector(dp) -> np.ndarray:
    n2 = dp.n * dp.n
    gi = np.asarray(dp.dec.gather_index)
    h = np.zeros((gi.size, n2))
    h[np.arange(gi.size), gi] = 1.0
    return h


def dense_embedding(dp) -> np.ndarray:
    """Explicit skew-symmetric Q (reference tests/helpers.py:184-208)."""
    n2, nd, m = dp.n * dp.n, dp.n_d, dp.m
    h = dense_selector(dp)
    a = dp.A.toarray()
    T = n2 + nd + m + nd + 1
    q = np.zeros((T, T))
    ix, is_ = slice(0, n2), slice(n2, n2 + nd)
    iy, iv = slice(n2 + nd, n2 + nd + m), slice(n2 + nd + m, T - 1)
    q[ix, iy] = -a.T
    q[ix, iv] = -h.T
    q[ix, -1] = dp.c
    q[is_, iv] = np.eye(nd)
    q[iy, ix] = a
    q[iy, -1] = -dp.b
    q[iv, ix] = h
    q[iv, is_] = -np.eye(nd)
    q[-1, ix] = -dp.c
    q[-1, iy] = dp.b
    return q


def dense_inner(dp) -> np.ndarray:
    """[[I, B'], [-B, I]] with B = [[-A, 0], [-H, I]] (reference helpers.py:211-223)."""
    m, nd, n2 = dp.m, dp.n_d, dp.n * dp.n
    h = dense_selector(dp)
    bhat = np.block([[-dp.A.toarray(), np.zeros((m, nd))], [-h, np.eye(nd)]])
    return np.block([[np.eye(n2 + nd), bhat.T], [-bhat, np.eye(m + nd)]])


def rel(a, b) -> float:
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def fixture_state(z, cp, prefix: str = "fixed_"):
    """Full compressed (u, w) of a config fixture (tests/golden/make_goldens.py),
    or None when the fixture holds only samples.  w is stored on its nonzero
    segments (z and kappa); its x / y / v parts are exactly 0."""
    if prefix + "u" not in z.files:
        return None
    u = np.asarray(z[prefix + "u"], float)
    if prefix + "w" in z.files:
        return u, np.asarray(z[prefix + "w"], float)
    w = np.zeros_like(u)
    w[cp.sl_s] = z[prefix + "w_z"]
    w[-1] = float(z[prefix + "w_kappa"])
    return u, w


def gen_hash(cp) -> str:
    """SHA-256 over a generated problem's arrays (the same digest
    tests/golden/make_goldens.py records as ``gen_hash``)."""
    import hashlib

    h = hashlib.sha256()
    for arr in (cp.covered, cp.A.indptr, cp.A.indices, cp.A.data, cp.c, cp.b,
                cp.sizes, np.concatenate([np.asarray(c) for c in cp.cliques])):
        a = np.ascontiguousarray(arr)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()
