"""Host decomposition against the reference's outputs.

Fixtures: ``tests/golden/decompose.npz`` (made by make_decompose_goldens.py
from the live reference: chordal_extend / maximal_cliques of random patterns,
decompose() of small multi-block SDPs) and ``config3_cliques.npz`` (the
reference's cliques of config 3's random geometric graph).  CPU only: the
graph code is host C++ in libhsde.so.
"""
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1611_01828_b200.decompose import chordal_cliques, decompose
from paper_1611_01828_b200.synthetic import load_config3_cliques, maxcut_graph


def _split(nodes, sizes):
    out, pos = [], 0
    for s in sizes:
        out.append([int(v) for v in nodes[pos: pos + s]])
        pos += s
    return out


def test_chordal_cliques_match_reference(golden_dir):
    z = np.load(golden_dir / "decompose.npz")
    for t in range(int(z["n_graphs"])):
        pre = f"g{t}_"
        cl, fill, chordal = chordal_cliques(int(z[pre + "n"]), z[pre + "edges"])
        assert chordal == bool(z[pre + "chordal"]), t
        assert [list(map(int, c)) for c in cl] == _split(z[pre + "clique_nodes"], z[pre + "clique_sizes"]), t
        assert set(map(tuple, fill.tolist())) == set(map(tuple, z[pre + "fill"].tolist())), t


def test_config3_cliques_match_reference():
    """3,493 cliques of the min-degree extension of config 3's graph."""
    cl, fill, chordal = chordal_cliques(5000, maxcut_graph(5000, 3))
    assert not chordal and fill.shape[0] > 0
    ref = load_config3_cliques()
    assert len(cl) == len(ref)
    assert all(np.array_equal(a, b) for a, b in zip(cl, ref))


def test_not_chordal_without_extension():
    with pytest.raises(ValueError):
        chordal_cliques(4, [(0, 1), (1, 2), (2, 3), (0, 3)], extend=False)  # 4-cycle
    cl, fill, chordal = chordal_cliques(4, [(0, 1), (1, 2), (2, 3), (0, 3)])
    assert not chordal and fill.shape[0] == 1


def _problem(z, pre):
    dims = tuple(int(d) for d in z[pre + "dims"])
    m = int(z[pre + "m"])
    ent = z[pre + "entries"]
    mats = [[SimpleNamespace(entries=[]) for _ in dims] for _ in range(m + 1)]
    for mid, blk, i, j, v in ent:
        mats[int(mid)][int(blk)].entries.append((int(i), int(j), float(v)))
    return SimpleNamespace(m=m, block_dims=dims, b=z[pre + "b"], C=mats[0], A=mats[1:])


def test_decompose_matches_reference_compressed(golden_dir):
    z = np.load(golden_dir / "decompose.npz")
    for t in range(int(z["n_problems"])):
        pre = f"p{t}_"
        cp = decompose(_problem(z, pre))
        assert np.array_equal(cp.covered, z[pre + "covered"]), t
        assert np.array_equal(cp.c, z[pre + "c"]), t
        assert np.array_equal(cp.A.indptr, z[pre + "A_indptr"]), t
        assert np.array_equal(cp.A.indices, z[pre + "A_indices"]), t
        assert np.array_equal(cp.A.data, z[pre + "A_data"]), t
        assert np.array_equal(np.concatenate(cp.cliques), z[pre + "clique_nodes"]), t
        assert np.array_equal(cp.sizes, z[pre + "clique_sizes"]), t
        assert np.array_equal(cp.slot_cov, z[pre + "slot_cov"]), t
        assert np.array_equal(cp.aggregate_edges, z[pre + "aggregate_edges"]), t


def test_report_pattern_index_matches_numpy(golden_dir):
    """The library's pattern index (hsde_pattern_index) equals the numpy
    restatement of solver.py:443-452 on the reference's multi-block problems."""
    from paper_1611_01828_b200 import solver as S

    z = np.load(golden_dir / "decompose.npz")
    for t in range(int(z["n_problems"])):
        cp = decompose(_problem(z, f"p{t}_"))
        n = cp.n
        edges = cp.aggregate_edges if cp.aggregate_edges is not None else np.zeros((0, 2), np.int64)
        diag = np.arange(n, dtype=np.int64)
        pairs = np.concatenate([np.asarray(edges, dtype=np.int64).reshape(-1, 2), np.stack([diag, diag], 1)])
        code = np.unique(pairs[:, 0] * n + pairs[:, 1])
        gi, gj = code // n, code % n
        flat = gj * n + gi
        pos = np.searchsorted(cp.covered, flat)
        pos_c = np.minimum(pos, max(cp.N_c - 1, 0))
        hit = (pos < cp.N_c) & (cp.covered[pos_c] == flat)
        starts = np.concatenate([[0], np.cumsum(np.abs(np.asarray(cp.block_dims or (n,))))])
        bi = np.searchsorted(starts, gi, side="right") - 1
        bj = np.searchsorted(starts, gj, side="right") - 1
        want = (bi + 1, gi - starts[bi] + 1, gj - starts[bj] + 1, pos_c, hit)
        got = S._pattern_index(cp, cp)
        for a, b in zip(got[:4], want[:4]):
            assert np.array_equal(a, b), t
        if got[4] is None:  # every row covered
            assert want[4].all(), t
        else:
            assert np.array_equal(got[4], want[4]), t
