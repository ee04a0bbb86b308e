"""CPU tests of the boundary and host logic (no GPU, no compute calls)."""
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1611_01828_b200 import _lib
from paper_1611_01828_b200.problem import compress, expand_to_mirror
from paper_1611_01828_b200.report import (Residuals, SolverReport, Timing, ProblemStats,
                                          emit_report, read_report)
from paper_1611_01828_b200.solver import SolverSettings, _cert_decision, _MeritTracker
from paper_1611_01828_b200.synthetic import (config_stats, load_config3_cliques, make_config,
                                             maxcut_graph)

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "hsde.h").read_text()
    declared = set(re.findall(r"\b(hsde_[a-z_]+)\s*\(", header))
    lib = _lib.load()  # loads libhsde.so (no compute call without a GPU)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_lib.EXPORTED)


# SURVEY.md section 8 table (measured with the reference decomposition)
EXPECTED = {
    0: dict(n=210, m=100, N_c=6100, p=20, n_d=8000, nnz_A=61099),
    1: dict(n=88, m=61, N_c=1984, p=10, n_d=2560, nnz_A=12127),
    2: dict(n=2000, m=200, N_c=41890, p=1990, n_d=240790, nnz_A=418703),
    3: dict(n=5000, m=5000, N_c=56506, p=3493, n_d=140792, nnz_A=5000, clique_min=1,
            clique_max=29),
}


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_generator_matches_survey_sizes(cfg):
    st = config_stats(make_config(cfg))
    for k, v in EXPECTED[cfg].items():
        assert st[k] == v, (k, st[k], v)


def test_config3_fixture_matches_regenerated_graph(golden_dir):
    z = np.load(golden_dir / "config3_cliques.npz")
    edges = maxcut_graph(5000, 3)
    assert hashlib.sha256(edges.tobytes()).hexdigest() == str(z["edges_sha256"])
    assert len(edges) == 14737
    cl = load_config3_cliques()
    assert len(cl) == 3493


def test_compress_expand_roundtrip():
    cp = make_config(1)
    mir = expand_to_mirror(cp)
    cp2 = compress(mir)
    assert np.array_equal(cp2.covered, cp.covered)
    assert np.array_equal(cp2.slot_cov, cp.slot_cov)
    assert np.array_equal(cp2.c, cp.c)
    assert (cp2.A != cp.A).nnz == 0
    rng = np.random.default_rng(0)
    v = rng.normal(size=cp.total)
    full = cp.expand_vector(v)
    assert np.array_equal(cp.compress_vector(full), v)
    # gather / scatter are adjoint (graphs.py:245-252)
    x = rng.normal(size=cp.N_c)
    s = rng.normal(size=cp.n_d)
    assert np.isclose(cp.gather(x) @ s, x @ cp.scatter(s), rtol=1e-12)
    assert np.array_equal(mir.dec.gather(cp.expand_x(x)), cp.gather(x))


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_library_cover_layout_matches_numpy(cfg):
    """problem.compress through the library (hsde_cover_*: bit mask + popcount ranks
    on host threads) equals its numpy restatement on the reference layout, and
    recovers the generator's covered set; unsorted / duplicated A entries and int64
    column ids go through the same path."""
    import scipy.sparse as sp

    cp = make_config(cfg)
    dp = expand_to_mirror(cp)
    a, b = compress(dp), compress(dp, _numpy_only=True)
    assert np.array_equal(a.covered, cp.covered) and np.array_equal(a.covered, b.covered)
    assert np.array_equal(a.c, b.c) and np.array_equal(a.slot_cov, b.slot_cov)
    for x, y in ((a.A, b.A), (a.A, cp.A)):
        assert np.array_equal(x.indptr, y.indptr) and np.array_equal(x.indices, y.indices)
        assert np.array_equal(x.data, y.data)
    # a COO input with shuffled, split entries: canonicalised first, same result
    coo = dp.A.tocoo()
    perm = np.random.default_rng(0).permutation(coo.nnz)
    rows = np.concatenate([coo.row[perm], coo.row[perm[:7]]])
    cols = np.concatenate([coo.col[perm], coo.col[perm[:7]]]).astype(np.int64)
    vals = np.concatenate([coo.data[perm], np.zeros(7)])
    vals[:7] *= 0.5
    vals[-7:] = vals[:7]
    dp2 = type(dp)(n=dp.n, m=dp.m, c=dp.c, A=sp.coo_matrix((vals, (rows, cols)), shape=dp.A.shape), b=dp.b,
                   dec=dp.dec, aggregate=None, block_dims=dp.block_dims, objective_sign=dp.objective_sign)
    c2 = compress(dp2)
    assert np.array_equal(c2.covered, a.covered) and np.array_equal(c2.A.indices, a.A.indices)
    assert np.allclose(c2.A.data, a.A.data, rtol=1e-15, atol=0)


def test_edges_array_matches_sorted_tuples():
    """problem.edges_array turns the reference's aggregate pattern (graphs.py:37, a
    frozenset of (i, j) tuples) into the array `sorted(edges)` gives, without the
    Python-level sort; already sorted arrays pass through."""
    from paper_1611_01828_b200.problem import edges_array

    class Agg:
        pass

    rng = np.random.default_rng(5)
    n = 300
    pairs = {tuple(sorted(map(int, rng.integers(0, n, 2)))) for _ in range(5000)}
    a = Agg()
    a.edges = frozenset(pairs)
    want = np.asarray(sorted(a.edges), dtype=np.int64).reshape(-1, 2)
    assert np.array_equal(edges_array(a, n), want)
    a.edges = want[::-1].copy()  # an array, unsorted
    assert np.array_equal(edges_array(a, n), want)
    a.edges = frozenset()
    assert edges_array(a, n).shape == (0, 2)
    assert edges_array(None, n) is None


def test_library_cover_layout_rejects_bad_ids():
    with pytest.raises(ValueError):
        _lib.cover_layout(16, np.zeros(16), np.array([3, 16], dtype=np.int64), np.array([1], dtype=np.int32))
    with pytest.raises(ValueError):
        _lib.cover_layout(16, np.zeros(16), np.array([3], dtype=np.int64), np.array([-1], dtype=np.int64))
    cov, cc, pos, sc = _lib.cover_layout(16, np.eye(4).ravel(), np.array([1, 5], dtype=np.int64),
                                         np.array([15, 2], dtype=np.int64))
    assert cov.tolist() == [0, 1, 2, 5, 10, 15] and cc.tolist() == [1, 0, 0, 1, 1, 1]
    assert pos.tolist() == [5, 2] and sc.tolist() == [1, 3]


def test_full_layout_compress_keeps_all_coordinates():
    cp = make_config(1)
    mir = expand_to_mirror(cp)
    full = compress(mir, full=True)
    assert full.N_c == cp.n * cp.n
    assert np.array_equal(full.covered[full.slot_cov], mir.dec.gather_index)


def test_settings_validation():
    with pytest.raises(ValueError):
        SolverSettings(tol=0)
    with pytest.raises(ValueError):
        SolverSettings(alpha=2.0)
    with pytest.raises(ValueError):
        SolverSettings(max_iters=0)
    with pytest.raises(ValueError):
        SolverSettings(check_interval=0)
    s = SolverSettings()
    assert (s.tol, s.max_iters, s.alpha, s.check_interval, s.normalize) == (1e-4, 2000, 1.6, 20, True)


def test_certificate_decision_rules():
    nan = float("nan")
    assert _cert_decision(np.array([1.0, 0.5, 1e-6, -1e-6, nan, nan, nan]), 1e-4) == "DualInfeasible"
    assert _cert_decision(np.array([1.0, 0.5, 1e-3, 0.0, nan, nan, nan]), 1e-4) is None
    assert _cert_decision(np.array([-1.0, -2.0, nan, nan, 1e-6, 1e-6, 0.0]), 1e-4) == "PrimalInfeasible"
    assert _cert_decision(np.array([-1.0, -2.0, nan, nan, 1e-6, 1e-3, 0.0]), 1e-4) is None


def test_pattern_entries_behave_as_rows():
    """Solution rows held as arrays serialise exactly like the reference's lists."""
    import json

    from paper_1611_01828_b200.report import PatternEntries

    rows = [[1, 1, 1, 0.5], [1, 2, 1, -0.25], [2, 3, 3, 1e-300]]
    pe = PatternEntries(*zip(*rows))
    assert len(pe) == 3 and pe[1] == rows[1] and pe[1:] == rows[1:] and list(pe) == rows
    assert pe == rows and rows == pe and pe == PatternEntries(*zip(*rows))
    timing, stats = Timing(0.1, 0.2, 0.3, 0.01), ProblemStats(3, 1, [3], 1, 3, 3, 9)
    mk = lambda e: SolverReport(status="Optimal", objective_primal=1.0, objective_dual=1.0,
                                iterations=20, residuals=Residuals(1e-5, 1e-5, 1e-5),
                                timing=timing, problem=stats, tol=1e-4,
                                solution={"x_entries": e, "y": [1.0]})
    assert emit_report(mk(pe)) == emit_report(mk(rows))
    assert json.loads(emit_report(mk(pe)))["solution"]["x_entries"] == rows
    assert read_report(emit_report(mk(pe))) == mk(pe)


def test_report_json_roundtrip():
    rep = SolverReport(status="Optimal", objective_primal=1.0, objective_dual=1.0, iterations=20,
                       residuals=Residuals(1e-5, 1e-5, 1e-5), timing=Timing(0.1, 0.2, 0.3, 0.01),
                       problem=ProblemStats(3, 1, [3], 1, 3, 3, 9), tol=1e-4,
                       solution={"y": [1.0]})
    assert read_report(emit_report(rep)) == rep
    with pytest.raises(ValueError):
        SolverReport(status="Optimal", objective_primal=1.0, objective_dual=1.0, iterations=1,
                     residuals=Residuals(1.0, 0, 0), timing=Timing(0, 0, 0, 0),
                     problem=ProblemStats(3, 1, [3], 1, 3, 3, 9), tol=1e-4)


def test_merit_tracker_warns(caplog):
    tr = _MeritTracker()
    with caplog.at_level("WARNING"):
        for k, v in [(20, 1.0), (40, 0.9), (60, 2.0), (80, 2.0), (100, 2.0), (120, 3.0)]:
            tr.record(k, v)
    assert any("fixed-point residual rose" in r.message for r in caplog.records)


def _so_projection(lam, E):
    """Second-order Daleckii-Krein projection of diag(lam) + E (E off-diagonal),
    the formula of hsde_eig.cuh's cta_rebuild_perturbative (order 2)."""
    p = lam > 0
    diff = p[:, None] != p[None, :]
    den = lam[:, None] - lam[None, :]
    G = np.where(diff, E / np.where(diff, den, 1.0), 0.0)
    ES = np.where(~diff, E, 0.0)
    T1 = G @ (np.abs(lam)[:, None] * G)
    T2, T3 = ES @ G, G @ ES
    M = np.where(p[:, None] & p[None, :], ES, 0.0) - np.where(~diff, T1, 0.0)
    M[np.diag_indices_from(M)] = np.maximum(lam, 0.0) - np.diag(T1)
    pn = p[:, None] & ~p[None, :]
    mpn = lam[:, None] * G + (-lam[None, :] * T2 + lam[:, None] * T3) / np.where(pn, den, 1.0)
    M = np.where(pn, mpn, M)
    M = np.where(pn.T, mpn.T, M)
    return M


def test_second_order_projection_formula():
    """P(D + E) by the second-order expansion: error O(|E|^3), against eigh."""
    rng = np.random.default_rng(3)
    n = 16
    lam = np.concatenate([rng.uniform(0.3, 2.0, 9), -rng.uniform(0.3, 2.0, 7)])
    errs = []
    for eps in (1e-2, 1e-3, 1e-4):
        E = rng.normal(size=(n, n))
        E = (E + E.T) / 2
        np.fill_diagonal(E, 0.0)
        E *= eps
        w, v = np.linalg.eigh(np.diag(lam) + E)
        exact = (v * np.maximum(w, 0.0)) @ v.T
        errs.append(np.abs(_so_projection(lam, E) - exact).max())
    assert errs[2] < 1e-11
    assert errs[0] / errs[1] > 300 and errs[1] / errs[2] > 300  # cubic
