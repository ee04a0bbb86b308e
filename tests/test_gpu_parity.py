"""GPU parity tests: the CUDA path (through libhsde.so's C ABI) vs the
reference's golden outputs, the dense oracles, and the CPU oracle.

Tolerances (written per test) follow BASELINE.json's north_star: iterates
after a fixed iteration count within 1e-8 relative; at termination the same
status / certificate type, iteration count +-2 and objective within 1e-6
relative.  Unit-level operators match the reference's own oracle
tolerances (test_solver_oracles.py: 1e-10 dense solve, 1e-12 cone, 1e-14
golden first iteration).
"""
import math

import numpy as np
import pytest

import paper_1611_01828_b200 as H
from helpers import dense_embedding, dense_inner, rel, toy_problem
from oracle import hsde_oracle as O
from paper_1611_01828_b200.problem import compress
from paper_1611_01828_b200.synthetic import make_config

pytestmark = pytest.mark.gpu


def test_golden_first_iteration(golden_dir):
    z = np.load(golden_dir / "first_iteration.npz")
    dp = toy_problem(z)
    cache = H.setup_cache(dp)
    _, layout = H.build_hsde(dp)
    st = H.iterate(H.initial_state(layout), cache, layout, H.SolverSettings(alpha=1.0, normalize=False))
    assert np.allclose(st.u, z["u"], atol=1e-14, rtol=0)
    assert np.allclose(st.w_dual, z["w"], atol=1e-14, rtol=0)


def _toys(golden_dir):
    z = np.load(golden_dir / "toys.npz")
    for t in range(int(z["count"])):
        yield t, z, f"t{t}_"


def test_affine_and_inner_match_dense_and_reference(golden_dir):
    """test_solver_oracles.py:201-219 and acceptance criterion 6 (<= 1e-9)."""
    worst = [0.0] * 4
    for t, z, pre in _toys(golden_dir):
        dp = toy_problem(z, pre)
        cache = H.setup_cache(dp)
        assert cache.factored_dims == (dp.m,)
        w = z[pre + "aff_in"]
        got = H.affine_project(cache, w)
        ref = np.linalg.solve(np.eye(w.size) + dense_embedding(dp), w)
        worst[0] = max(worst[0], rel(got, ref))
        worst[1] = max(worst[1], rel(got, z[pre + "aff_out"]))
        n12a = dp.n * dp.n + dp.n_d
        w2 = z[pre + "inner_in"]
        u1, u2 = H.solve_inner(cache, w2[:n12a], w2[n12a:])
        got2 = np.concatenate([u1, u2])
        worst[2] = max(worst[2], rel(got2, np.linalg.solve(dense_inner(dp), w2)))
        worst[3] = max(worst[3], rel(got2, z[pre + "inner_out"]))
    assert worst[0] <= 1e-10 and worst[2] <= 1e-9, worst
    assert worst[1] <= 1e-11 and worst[3] <= 1e-11, worst


def test_affine_inner_product_identity(golden_dir):
    """(I + Q) u = w with skew Q forces u'w = |u|^2 (test_solver_oracles.py:221-231)."""
    z = np.load(golden_dir / "toys.npz")
    dp = toy_problem(z, "t3_")
    cache = H.setup_cache(dp)
    rng = np.random.default_rng(11)
    _, layout = H.build_hsde(dp)
    for _ in range(20):
        w = rng.normal(size=layout.total)
        u = H.affine_project(cache, w)
        assert u @ w >= 0
        assert np.isclose(u @ w, u @ u, rtol=1e-9)


def test_project_cone_matches_reference(golden_dir):
    worst = 0.0
    for t, z, pre in _toys(golden_dir):
        dp = toy_problem(z, pre)
        _, layout = H.build_hsde(dp)
        got = H.project_cone(z[pre + "cone_in"], layout)
        worst = max(worst, rel(got, z[pre + "cone_out"]))
        # free blocks pass through bit for bit (test_solver_oracles.py:270-273)
        assert np.array_equal(got[layout.sl_x], z[pre + "cone_in"][layout.sl_x])
        assert np.array_equal(got[layout.sl_v], z[pre + "cone_in"][layout.sl_v])
    assert worst <= 1e-12


def test_project_cone_fixed_point_and_tau_clamp(golden_dir):
    z = np.load(golden_dir / "toys.npz")
    dp = toy_problem(z, "t5_")
    _, layout = H.build_hsde(dp)
    rng = np.random.default_rng(13)
    u = rng.normal(size=layout.total)
    for k in range(dp.p):
        d = int(dp.dec.sizes[k])
        g = rng.normal(size=(d, d))
        u[layout.sl_s][dp.dec.offsets[k]: dp.dec.offsets[k + 1]] = (g @ g.T).ravel()
    u[layout.idx_tau] = -1.0
    got = H.project_cone(u, layout)
    assert got[layout.idx_tau] == 0.0
    assert np.allclose(got[layout.sl_s], u[layout.sl_s], atol=1e-12)


def test_iterate_matches_reference_from_random_starts(golden_dir):
    worst = 0.0
    for t, z, pre in _toys(golden_dir):
        dp = toy_problem(z, pre)
        cache = H.setup_cache(dp)
        _, layout = H.build_hsde(dp)
        st = H.iterate(H.HsdeState(z[pre + "it_u0"], z[pre + "it_w0"]), cache, layout, H.SolverSettings())
        worst = max(worst, rel(st.u, z[pre + "it_u1"]), rel(st.w_dual, z[pre + "it_w1"]))
        # dual-side zero blocks exactly zero (test_solver_oracles.py:396-399)
        assert not st.w_dual[layout.sl_x].any()
        assert not st.w_dual[layout.sl_y].any()
        assert not st.w_dual[layout.sl_v].any()
        # Moreau: complementarity, tau/kappa >= 0
        scale = max(np.linalg.norm(st.u) * np.linalg.norm(st.w_dual), 1e-30)
        assert abs(st.u @ st.w_dual) <= 1e-9 * scale
        assert st.u[-1] >= 0 and st.w_dual[-1] >= 0
    assert worst <= 1e-10


def test_toy_solves_match_reference(golden_dir):
    for t, z, pre in _toys(golden_dir):
        dp = toy_problem(z, pre)
        rep = H.solve_decomposed(dp, H.SolverSettings(max_iters=400, check_interval=20))
        assert rep.status == str(z[pre + "solve_status"]), t
        assert abs(rep.iterations - int(z[pre + "solve_iters"])) <= 2, t
        ref = z[pre + "solve_obj"]
        if rep.objective_primal is not None and not math.isnan(ref[0]):
            assert abs(rep.objective_primal - ref[0]) <= 1e-6 * (1 + abs(ref[0])), t


def test_residuals_and_tauzero(golden_dir):
    z = np.load(golden_dir / "toys.npz")
    dp = toy_problem(z, "t2_")
    _, layout = H.build_hsde(dp)
    rng = np.random.default_rng(22)
    u = rng.normal(size=layout.total)
    u[-1] = 1.3
    cp = compress(dp, full=True)
    want = O.residuals(cp, cp.compress_vector(u))
    got = H.residuals(H.HsdeState(u, np.zeros_like(u)), dp)
    assert np.allclose([got.primal, got.dual, got.gap], want, rtol=1e-12)
    u[-1] = 0.0
    with pytest.raises(H.TauZero):
        H.residuals(H.HsdeState(u, np.zeros_like(u)), dp)


def test_factorization_failure_on_bad_data():
    from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem
    import scipy.sparse as sp

    dec = CliqueDecomposition.build(2, [[0, 1]])
    dp = DecomposedProblem(n=2, m=1, c=np.zeros(4), A=sp.csr_matrix(np.array([[np.inf, 0, 0, 1.0]])),
                           b=np.array([1.0]), dec=dec, block_dims=(2,))
    with pytest.raises(H.FactorizationFailure):
        H.setup_cache(dp)


def test_malformed_constraint_matrix_rejected():
    """Column indices out of order (validated on the device after the upload)."""
    import dataclasses

    from paper_1611_01828_b200 import _lib

    cp = make_config(0)
    A = cp.A.copy()
    row = 3
    b, e = A.indptr[row], A.indptr[row + 1]
    A.indices[b:e] = A.indices[b:e][::-1].copy()
    bad = dataclasses.replace(cp, A=A, _cache={})
    with pytest.raises(ValueError, match="row 3"):
        _lib.Handle(bad)


def test_eigen_failure_on_nan():
    from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem
    import scipy.sparse as sp

    dec = CliqueDecomposition.build(3, [[0, 1, 2]])
    dp = DecomposedProblem(n=3, m=1, c=np.zeros(9), A=sp.csr_matrix(np.eye(3).reshape(1, 9)),
                           b=np.array([1.0]), dec=dec, block_dims=(3,))
    _, layout = H.build_hsde(dp)
    u = np.ones(layout.total)
    u[layout.sl_s][4] = np.nan
    with pytest.raises(H.EigenFailure):
        H.project_cone(u, layout)


# --------------------------------------------------------------------------
# BASELINE configs vs the live-reference fixtures


def _fixed_run(cfg, iters):
    cp = make_config(cfg)
    states = {}
    logs = []

    def cb(info):
        logs.append((info.iteration, info.pres, info.dres, info.gap, info.tau, info.kappa))
        if info.iteration == iters:
            states["u"], states["w"] = info.state.u.copy(), info.state.w_dual.copy()

    H.solve_decomposed(cp, H.SolverSettings(max_iters=iters, tol=1e-300), iteration_callback=cb)
    return cp, states, np.array(logs)


def _compare_state(z, cp, u, w, tol, prefix="fixed_"):
    from helpers import fixture_state

    full = fixture_state(z, cp, prefix)
    if full is not None:
        assert rel(u, full[0]) <= tol
        assert rel(w, full[1]) <= tol
        return
    # large configs: 4096 seeded sample entries + per-segment norms
    for name, vec in (("u", u), ("w", w)):
        idx, val = z[f"{prefix}{name}_idx"], z[f"{prefix}{name}_val"]
        assert rel(vec[idx], val) <= tol, name
        norms = np.array([np.linalg.norm(vec[sl]) for sl in (cp.sl_x, cp.sl_s, cp.sl_y, cp.sl_v)]
                         + [vec[-1]])
        ref = z[f"{prefix}{name}_norms"]
        scale = np.linalg.norm(ref)
        assert np.all(np.abs(norms - ref) <= tol * scale), (name, norms, ref)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_config_fixed_iterations(golden_dir, cfg):
    """Iterates after 500 iterations within 1e-8 relative of the reference."""
    z = np.load(golden_dir / f"cfg{cfg}_reference.npz")
    iters = int(z["fixed_iters"])
    cp, st, logs = _fixed_run(cfg, iters)
    _compare_state(z, cp, st["u"], st["w"], 1e-8)
    ref = z["fixed_log"]
    assert np.array_equal(logs[:, 0], ref[:, 0])
    finite = np.isfinite(ref[:, 1])
    assert np.array_equal(np.isfinite(logs[:, 1]), finite)
    assert np.allclose(logs[finite, 1:4], ref[finite, 1:4], rtol=1e-6)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_config_to_tolerance(golden_dir, cfg):
    z = np.load(golden_dir / f"cfg{cfg}_reference.npz")
    rep = H.solve_decomposed(make_config(cfg), H.SolverSettings())
    assert rep.status == str(z["tol_status"])
    assert abs(rep.iterations - int(z["tol_iters"])) <= 2
    if rep.certificate is not None:
        assert rep.certificate["ray"] == str(z["cert_ray"])
        assert rep.certificate["b_dot_y"] == 1.0
        assert np.allclose(rep.certificate["y"], z["cert_y"], rtol=1e-6, atol=1e-9)
        assert rep.certificate["residual"] <= 1e-4
        assert rep.certificate["min_block_eigenvalue"] >= -1e-4
    else:
        ref = z["tol_obj"]
        assert abs(rep.objective_primal - ref[0]) <= 1e-6 * abs(ref[0])
        assert abs(rep.objective_dual - ref[1]) <= 1e-6 * abs(ref[1])


def test_runs_are_bitwise_reproducible():
    cp = make_config(0)
    out = []
    for _ in range(2):
        got = {}

        def cb(info):
            if info.iteration == 100:
                got["u"] = info.state.u.copy()

        H.solve_decomposed(cp, H.SolverSettings(max_iters=100, tol=1e-300), iteration_callback=cb)
        out.append(got["u"])
    assert np.array_equal(out[0], out[1])


def test_exact_uy_flag_matches_identity_path():
    """uy by an explicit A ua pass (solver.py:241) vs the identity A ua = S^-1 A t."""
    from paper_1611_01828_b200 import _lib

    cp = make_config(0)
    res = []
    for flags in (0, _lib.HSDE_FLAG_EXACT_UY):
        h = _lib.Handle(cp, flags=flags)
        h.iterate(200)
        res.append(h.get_state()[0])
        h.close()
    assert rel(res[1], res[0]) <= 1e-10


def test_warm_started_eigensolves_match_cold_and_oracle():
    """CTA-team cliques (d = 40 > 32) with and without the warm start, vs the
    CPU oracle after 200 iterations (1e-8 relative)."""
    from paper_1611_01828_b200 import _lib
    from paper_1611_01828_b200.synthetic import block_arrow

    cp = block_arrow(12, 24, 16, 50, 0.05, 7, "ctapath")
    res = []
    for flags in (0, _lib.HSDE_FLAG_COLD_EIG):
        h = _lib.Handle(cp, flags=flags)
        h.iterate(200)
        res.append(h.get_state())
        st = h.stats()
        assert st["warm_start"] == (flags == 0)
        h.close()
    assert rel(res[0][0], res[1][0]) <= 1e-9
    ref = {}

    def cb(k, p, d, g, tau, kap, u, w):
        if k == 200:
            ref["u"] = u.copy()

    O.solve(cp, O.OracleSettings(max_iters=200, tol=1e-300), callback=cb)
    assert rel(res[0][0], ref["u"]) <= 1e-8


def test_project_cone_clique_orders():
    """PSD projection of random symmetric blocks over the clique orders the two
    Jacobi teams cover (warp d <= 32, CTA d > 32, odd and even, up to the
    shared-memory limit) against numpy's eigh projection (symmat.py:153-165)."""
    import scipy.sparse as sp

    from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem

    sizes = [2, 3, 7, 16, 17, 31, 32, 33, 40, 47, 64, 80, 81, 96, 111]
    n = sum(sizes)
    cl, o = [], 0
    for d in sizes:
        cl.append(list(range(o, o + d)))
        o += d
    dec = CliqueDecomposition.build(n, cl)
    A = sp.csr_matrix(([1.0], ([0], [0])), shape=(1, n * n))
    dp = DecomposedProblem(n=n, m=1, c=np.eye(n).ravel(), A=A, b=np.ones(1), dec=dec,
                           block_dims=(n,))
    _, layout = H.build_hsde(dp)
    rng = np.random.default_rng(5)
    u = rng.normal(size=layout.total)
    got = H.project_cone(u, layout)
    s_in, s_out = u[layout.sl_s], got[layout.sl_s]
    for k, d in enumerate(sizes):
        o0, o1 = dec.offsets[k], dec.offsets[k + 1]
        b = s_in[o0:o1].reshape(d, d)
        w, v = np.linalg.eigh(0.5 * (b + b.T))
        want = (v * np.maximum(w, 0.0)) @ v.T
        assert rel(s_out[o0:o1], want.ravel()) <= 1e-12, d


@pytest.mark.parametrize("cfg", [0, 2, 4])
def test_half_passes_match_full_passes(cfg, monkeypatch):
    """A passes over mirror pairs (symmetric constraint matrices) vs the
    full-column passes: same iterate after 60 iterations to 1e-10."""
    from paper_1611_01828_b200 import _lib

    cp = make_config(cfg)
    res = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("HSDE_NO_HALF", "1")
        h = _lib.Handle(cp)
        assert h.half_passes == (not off)
        h.iterate(60)
        res.append(h.get_state()[0])
        h.close()
    assert rel(res[0], res[1]) <= 1e-10


def test_half_passes_off_for_nonsymmetric_columns():
    """One A_ij != A_ji entry disables the half passes; the result still
    matches the oracle."""
    import dataclasses

    from paper_1611_01828_b200 import _lib

    cp = make_config(0)
    A = cp.A.copy()
    A.data[5] += 0.25
    bad = dataclasses.replace(cp, A=A, _cache={})
    h = _lib.Handle(bad)
    assert not h.half_passes
    h.iterate(100)
    u = h.get_state()[0]
    h.close()
    ref = {}

    def cb(k, p, d, g, tau, kap, uu, w):
        if k == 100:
            ref["u"] = uu.copy()

    O.solve(bad, O.OracleSettings(max_iters=100, tol=1e-300), callback=cb)
    assert rel(u, ref["u"]) <= 1e-9


def test_project_cone_nearly_diagonal():
    """Blocks D + E with small E hit the perturbative exits (first / second
    order, CTA and warp teams) before any rotation; eigh projection at 1e-13."""
    import scipy.sparse as sp

    from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem

    sizes = [24, 40, 80, 80, 33]
    n = sum(sizes)
    cl, o = [], 0
    for d in sizes:
        cl.append(list(range(o, o + d)))
        o += d
    dec = CliqueDecomposition.build(n, cl)
    A = sp.csr_matrix(([1.0], ([0], [0])), shape=(1, n * n))
    dp = DecomposedProblem(n=n, m=1, c=np.eye(n).ravel(), A=A, b=np.ones(1), dec=dec,
                           block_dims=(n,))
    _, layout = H.build_hsde(dp)
    rng = np.random.default_rng(11)
    u = rng.normal(size=layout.total)
    s_in = u[layout.sl_s]
    for k, d in enumerate(sizes):
        lam = rng.uniform(0.5, 2.0, d) * rng.choice([-1.0, 1.0], d)
        e = rng.normal(size=(d, d))
        eps = [1e-9, 1e-7, 1e-7, 1e-12, 1e-6][k]
        b = np.diag(lam) + eps * (e + e.T) / 2 * (1 - np.eye(d))
        s_in[dec.offsets[k]: dec.offsets[k + 1]] = b.ravel()
    u[layout.sl_s] = s_in
    got = H.project_cone(u, layout)[layout.sl_s]
    for k, d in enumerate(sizes):
        o0, o1 = dec.offsets[k], dec.offsets[k + 1]
        b = s_in[o0:o1].reshape(d, d)
        w, v = np.linalg.eigh(0.5 * (b + b.T))
        want = (v * np.maximum(w, 0.0)) @ v.T
        assert rel(got[o0:o1], want.ravel()) <= 1e-13, d


@pytest.mark.gpu
def test_solve_from_sdpa_text():
    """parse_sdpa -> solve (solver.py:775-789): C++ reader + C++ decomposition
    + device iterations, on a max-cut SDP written as SDPA text."""
    from paper_1611_01828_b200.synthetic import maxcut_graph
    n = 300
    edges = maxcut_graph(n, 11)
    deg = np.bincount(edges.ravel(), minlength=n)
    lines = [f"{n} = mDIM", "1 = nBLOCK", f"{n}", " ".join(["1.0"] * n)]
    lines += [f"0 1 {i + 1} {i + 1} {float(0.25 * deg[i])!r}" for i in range(n) if deg[i]]
    lines += [f"0 1 {j + 1} {i + 1} -0.25" for i, j in edges]  # lower triangle on purpose
    lines += [f"{i + 1} 1 {i + 1} {i + 1} 1.0" for i in range(n)]
    prob = H.parse_sdpa("\n".join(lines) + "\n")
    st = H.SolverSettings(max_iters=4000)
    rep = H.solve(prob, st)
    assert rep.status == H.STATUS_OPTIMAL
    assert abs(rep.objective_primal - rep.objective_dual) <= 1e-3 * abs(rep.objective_primal)
    rep2 = H.solve_decomposed(H.decompose(prob), st)
    assert rep2.iterations == rep.iterations and rep2.objective_primal == rep.objective_primal
    assert rep.problem.n == n and rep.problem.m == n and rep.problem.p > 1


def test_split_fast_path_matches_jacobi_path():
    """k_cone_split (Riccati invariant-subspace projection on DMMA blocks, V
    rotated onto the new subspaces) against the Jacobi-only CTA path on config
    4 (400 cliques of order 80): iterates agree to rounding after 120
    iterations, and the fast path finishes nearly every clique."""
    from paper_1611_01828_b200 import _lib

    cp = make_config(4)
    res, stats = [], []
    for flags in (0, _lib.HSDE_FLAG_NO_SPLIT):
        h = _lib.Handle(cp, flags=flags)
        h.iterate(120)
        res.append(h.get_state())
        stats.append(h.stats())
        h.close()
    assert rel(res[0][0], res[1][0]) <= 1e-11
    assert rel(res[0][1], res[1][1]) <= 1e-11
    assert stats[0]["split_done"] >= 0.9
    assert 1 <= stats[0]["split_fp_iters"] <= 24
    assert stats[1]["split_done"] == 0.0


def test_report_vectors_match_host_path():
    """The report's device vectors (u_x, u_y and H' vt summed in slot order,
    hsde_report_vectors) equal the host restatement (unscale, divide,
    np.bincount: solver.py:668-687, graphs.py:251) bit for bit."""
    from paper_1611_01828_b200 import _lib

    cp = make_config(2)
    h = _lib.Handle(cp)
    h.iterate(60)
    u, _ = h.get_state()
    tau = float(u[-1])
    x, y, hv = h.report_vectors(tau)
    h.close()
    assert np.array_equal(x, u[cp.sl_x])
    assert np.array_equal(y, u[cp.sl_y])
    v = u[cp.sl_v]
    if h.sigma_c != 1.0:
        v = v / h.sigma_c
    assert np.array_equal(hv, cp.scatter(v / tau))


def _entries(pe):
    return np.column_stack([pe.block, pe.i, pe.j, pe.value]).astype(float)


def _compare_entries(got, ref, tol):
    assert got.shape == ref.shape
    assert np.array_equal(got[:, :3], ref[:, :3])  # block, i, j: same pattern rows, same order
    scale = np.linalg.norm(ref[:, 3])
    assert np.linalg.norm(got[:, 3] - ref[:, 3]) <= tol * max(scale, 1e-300)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_report_entries_match_reference(golden_dir, cfg):
    """Solution entries x_entries / z_entries / y (solver.py:553-556) and the
    certificate's entry list (solver.py:472-503) against the reference report
    of the same to-tolerance solve: identical [block, i, j] rows, values within
    1e-6 relative (the final iterates agree to ~1e-10)."""
    z = np.load(golden_dir / f"cfg{cfg}_reference.npz")
    rep = H.solve_decomposed(make_config(cfg), H.SolverSettings())
    assert rep.status == str(z["tol_status"])
    if "sol_x_entries" in z.files:
        _compare_entries(_entries(rep.solution["x_entries"]), z["sol_x_entries"], 1e-6)
        _compare_entries(_entries(rep.solution["z_entries"]), z["sol_z_entries"], 1e-6)
        assert rel(np.array(rep.solution["y"]), z["sol_y"]) <= 1e-6
    else:
        assert "cert_slack_entries" in z.files or "cert_ray_entries" in z.files
        key = "slack_entries" if "cert_slack_entries" in z.files else "ray_entries"
        _compare_entries(_entries(rep.certificate[key]), z[f"cert_{key}"], 1e-6)


def test_recover_matches_solve_report(golden_dir):
    """recover (solver.py:608-617) on the final iterate of an un-normalised
    solve gives the same status, objectives and solution entries as the solve."""
    cp = make_config(0)
    st = H.SolverSettings(normalize=False)
    last = {}

    def cb(info):
        last["state"] = info.state

    rep = H.solve_decomposed(cp, st, iteration_callback=cb)
    s = last["state"]
    rec = H.recover(H.HsdeState(s.u.copy(), s.w_dual.copy()), cp, st, rep.iterations, rep.timing)
    assert rec.status == rep.status == "Optimal"
    assert rec.iterations == rep.iterations
    assert abs(rec.objective_primal - rep.objective_primal) <= 1e-12 * abs(rep.objective_primal)
    assert abs(rec.objective_dual - rep.objective_dual) <= 1e-12 * abs(rep.objective_dual)
    _compare_entries(_entries(rec.solution["x_entries"]), _entries(rep.solution["x_entries"]), 1e-12)
    _compare_entries(_entries(rec.solution["z_entries"]), _entries(rep.solution["z_entries"]), 1e-12)


@pytest.mark.parametrize("at", ["mid", "fixed"])
def test_config4_long_pin(golden_dir, at):
    """Config 4 iterated 100 / 200 iterations (tol = 1e-300) against the
    reference's own iterates (tests/golden/cfg4_long_reference.npz, ~50 min of
    reference CPU time): 4096 seeded entries + segment norms within 1e-8."""
    path = golden_dir / "cfg4_long_reference.npz"
    if not path.exists():
        pytest.skip("cfg4_long_reference.npz not generated")
    z = np.load(path)
    from helpers import gen_hash

    cp = make_config(4)
    assert gen_hash(cp) == str(z["gen_hash"])
    iters = int(z[f"{at}_iters"])
    _, st, logs = _fixed_run(4, iters)
    _compare_state(z, cp, st["u"], st["w"], 1e-8, prefix=f"{at}_")


@pytest.mark.parametrize("d,h", [(57, 40), (71, 40), (40, 40)])
def test_large_cliques_hot_path(d, h):
    """Cliques of order 97 and 111 (above the fast path's and the cold path's
    register tiles: the Jacobi path) and 80 (fast + cold path) through 80 hot
    iterations against the CPU oracle at 1e-8 (orders 97-112)."""
    from oracle import hsde_oracle as O
    from paper_1611_01828_b200.synthetic import block_arrow

    cp = block_arrow(3, d, h, 30, 0.05, 11, f"arrow_{d}_{h}")
    assert int(cp.sizes.max()) == d + h
    got = {}

    def cb(info):
        if info.iteration == 80:
            got["u"] = info.state.u.copy()

    H.solve_decomposed(cp, H.SolverSettings(max_iters=80, tol=1e-300), iteration_callback=cb)
    ref = {}

    def ocb(k, p, dd, g, tau, kap, u, w):
        if k == 80:
            ref["u"] = u.copy()

    O.solve(cp, O.OracleSettings(max_iters=80, tol=1e-300), callback=ocb)
    assert rel(got["u"], ref["u"]) <= 1e-8


def test_cold_path_matches_jacobi_path():
    """Config 4's first 30 iterations -- all cliques on the tridiagonal cold
    path (hsde_cold.cuh), then the fast path -- against the Jacobi-only
    eigensolver (HSDE_FLAG_JACOBI): same iterate to 1e-10."""
    from paper_1611_01828_b200 import _lib

    cp = make_config(4)
    st = []
    for flags in (0, _lib.HSDE_FLAG_JACOBI):
        h = _lib.Handle(cp, flags=flags)
        h.iterate(30)
        st.append(h.get_state())
        if flags == 0:
            stats = h.stats()
        h.close()
    assert rel(st[0][0], st[1][0]) <= 1e-10
    assert rel(st[0][1], st[1][1]) <= 1e-10
    assert stats["cold_failed"] == 0.0


def _adversarial_blocks(rng, d):
    q, _ = np.linalg.qr(rng.normal(size=(d, d)))
    lam = np.ones(d)
    lam[: d // 3] = -2.0
    x = rng.normal(size=d)
    tight = np.concatenate([1 + 1e-9 * rng.normal(size=d // 2), -1 + 1e-9 * rng.normal(size=d - d // 2)])
    near0 = np.linspace(-1, 1, d)
    nz = min(5, d - d // 2)
    near0[d // 2: d // 2 + nz] = 1e-13 * np.arange(nz)
    return {
        "two_values": (q * lam) @ q.T, "identity": np.eye(d), "zero": np.zeros((d, d)),
        "diag": np.diag(rng.normal(size=d)), "rank1": np.outer(x, x) - 0.5 * np.eye(d),
        "tight_clusters": (q * tight) @ q.T, "near_zero_cluster": (q * near0) @ q.T,
        "graded": (q * np.logspace(-12, 0, d) * np.sign(rng.normal(size=d))) @ q.T,
    }


@pytest.mark.parametrize("kind", ["two_values", "identity", "zero", "diag", "rank1", "tight_clusters",
                                  "near_zero_cluster", "graded"])
def test_project_cone_adversarial_spectra(kind):
    """The cold eigensolver (warp d <= 32, CTA d <= 96, Jacobi beyond) on
    repeated, clustered, zero and graded spectra: 1e-12 of numpy's eigh
    projection (symmat.py:153-165)."""
    import scipy.sparse as sp

    from paper_1611_01828_b200.problem import CliqueDecomposition, DecomposedProblem

    sizes = [5, 16, 29, 33, 64, 80, 96, 111]
    n = sum(sizes)
    cl, o = [], 0
    for d in sizes:
        cl.append(list(range(o, o + d)))
        o += d
    dec = CliqueDecomposition.build(n, cl)
    A = sp.csr_matrix(([1.0], ([0], [0])), shape=(1, n * n))
    dp = DecomposedProblem(n=n, m=1, c=np.eye(n).ravel(), A=A, b=np.ones(1), dec=dec, block_dims=(n,))
    _, layout = H.build_hsde(dp)
    rng = np.random.default_rng(17)
    u = rng.normal(size=layout.total)
    s_in = u[layout.sl_s].copy()
    for k, d in enumerate(sizes):
        s_in[dec.offsets[k]:dec.offsets[k + 1]] = _adversarial_blocks(rng, d)[kind].ravel()
    u[layout.sl_s] = s_in
    got = H.project_cone(u, layout)[layout.sl_s]
    for k, d in enumerate(sizes):
        o0, o1 = dec.offsets[k], dec.offsets[k + 1]
        b = s_in[o0:o1].reshape(d, d)
        w, v = np.linalg.eigh(0.5 * (b + b.T))
        want = ((v * np.maximum(w, 0.0)) @ v.T).ravel()
        assert np.linalg.norm(got[o0:o1] - want) <= 1e-12 * max(np.linalg.norm(b), 1e-300), (kind, d)
