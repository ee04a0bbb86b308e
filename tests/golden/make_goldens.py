"""Generate golden fixtures by running the LIVE reference (build container only).

    python tests/golden/make_goldens.py first toys cfg0 cfg1 cfg2 [cfg3] [cfg4] [cfg4long]

Imports ``chordalsdp`` from /root/reference/pkg/src (read-only, never copied)
and writes ``tests/golden/*.npz``.  The GPU box never runs this; it only reads
the committed fixtures.  Sections:

* ``first`` -- the reference's first-iteration golden problem
  (test_solver_oracles.py:33-43, :349-373) re-run through the reference.
* ``toys``  -- random decomposed toy problems from the reference's own test
  builders (tests/helpers.py:245-297) with the reference's outputs of
  ``affine_project``, ``solve_inner``, ``project_cone``, ``iterate``,
  ``residuals`` on seeded inputs.
* ``cfgK``  -- BASELINE config K (paper_1611_01828_b200.synthetic) solved by
  the reference: iterate at a fixed iteration count (500; config 4: 40) with
  tol=1e-300, the per-check log, and the default-settings to-tolerance report.
  Configs 0-3 store the full compressed state (w only on its nonzero z/kappa
  segments); config 4 a summary (segment norms + 4096 seeded sample entries).
  The to-tolerance report's solution entries (x_entries / z_entries, solver.py:
  553-556) or certificate entry lists (solver.py:472-503) are stored too.
* ``cfg4long`` -- config 4 iterated by the reference to a fixed 200 iterations
  (tol=1e-300): summaries at iterations 100 and 200 plus the check log (SURVEY
  section 7.1's long pin; about an hour of CPU).

Every config fixture records ``gen_hash``: a SHA-256 over the generated
problem's arrays, so a generator change is detected by the tests.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, str(HERE.parents[1]))

import scipy.sparse as sp  # noqa: E402
from chordalsdp.decompose import DecomposedProblem as RDP  # noqa: E402
from chordalsdp.graphs import CliqueDecomposition as RCD  # noqa: E402
from chordalsdp.graphs import SparsityPattern, maximal_cliques  # noqa: E402
from chordalsdp import solver as R  # noqa: E402

from paper_1611_01828_b200.problem import expand_to_mirror  # noqa: E402
from paper_1611_01828_b200.synthetic import make_config  # noqa: E402

FULL_STATE_MAX = 600_000  # store the whole compressed state below this length
N_SAMPLES = 4096


def to_reference(cp):
    mir = expand_to_mirror(cp)
    pat = SparsityPattern(cp.n, frozenset(map(tuple, cp.aggregate_edges.tolist())))
    dec = RCD.build(cp.n, [list(map(int, c)) for c in cp.cliques], pat)
    return RDP(n=cp.n, m=cp.m, c=mir.c, A=mir.A, b=cp.b.copy(), dec=dec,
               aggregate=pat, block_dims=(cp.n,))


def gen_hash(cp) -> str:
    import hashlib
    h = hashlib.sha256()
    for arr in (cp.covered, cp.A.indptr, cp.A.indices, cp.A.data, cp.c, cp.b,
                cp.sizes, np.concatenate([np.asarray(c) for c in cp.cliques])):
        a = np.ascontiguousarray(arr)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def entries_array(rows) -> np.ndarray:
    return np.array(rows, dtype=np.float64).reshape(-1, 4)


def sample_index(total: int) -> np.ndarray:
    return np.sort(np.random.default_rng(12345).choice(total, size=min(N_SAMPLES, total),
                                                       replace=False))


def state_summary(cp, u, w, prefix):
    out = {}
    segs = {"x": cp.sl_x, "s": cp.sl_s, "y": cp.sl_y, "v": cp.sl_v}
    for name, vec in (("u", u), ("w", w)):
        out[f"{prefix}{name}_norms"] = np.array([np.linalg.norm(vec[sl]) for sl in segs.values()]
                                                + [vec[-1]])
        if cp.total <= FULL_STATE_MAX and name == "w":
            # the x / y / v parts of w are exactly 0
            out[f"{prefix}w_z"] = vec[cp.sl_s]
            out[f"{prefix}w_kappa"] = np.float64(vec[-1])
        elif cp.total <= FULL_STATE_MAX:
            out[f"{prefix}{name}"] = vec
        else:
            idx = sample_index(cp.total)
            out[f"{prefix}{name}_idx"] = idx
            out[f"{prefix}{name}_val"] = vec[idx]
    return out


def pack_problem(dp, prefix=""):
    cl = [np.asarray(c, dtype=np.int64) for c in dp.dec.cliques]
    return {
        f"{prefix}n": np.int64(dp.n), f"{prefix}m": np.int64(dp.m),
        f"{prefix}c": np.asarray(dp.c, float), f"{prefix}A": dp.A.toarray(),
        f"{prefix}b": np.asarray(dp.b, float),
        f"{prefix}clique_nodes": np.concatenate(cl) if cl else np.zeros(0, np.int64),
        f"{prefix}clique_sizes": np.array([len(c) for c in cl], dtype=np.int64),
    }


def section_first():
    dec = maximal_cliques(SparsityPattern.complete(2))
    a = sp.csr_matrix(np.array([[1.0, 0.0, 0.0, 1.0]]))
    dp = RDP(n=2, m=1, c=np.array([1.0, 0.5, 0.5, -0.25]), A=a, b=np.array([1.0]), dec=dec,
             aggregate=SparsityPattern.complete(2), block_dims=(2,))
    cache = R.setup_cache(dp)
    _, layout = R.build_hsde(dp)
    st = R.iterate(R.initial_state(layout), cache, layout, R.SolverSettings(alpha=1.0, normalize=False))
    np.savez(HERE / "first_iteration.npz", **pack_problem(dp), u=st.u, w=st.w_dual)
    print("first_iteration: u", st.u[:4], "...")


def section_toys():
    from helpers import known_solution_decomposed, random_decomposed

    rng = np.random.default_rng(2024)
    data = {}
    count = 0
    for kind in ("random", "known"):
        for _ in range(20):
            n = int(rng.integers(2, 7))
            m = int(rng.integers(1, 5))
            if kind == "random":
                dp = random_decomposed(rng, n, m)
            else:
                dp, _ = known_solution_decomposed(rng, max(n, 3), m)
            cache = R.setup_cache(dp)
            _, lay = R.build_hsde(dp)
            pre = f"t{count}_"
            data.update(pack_problem(dp, pre))
            w = rng.normal(size=lay.total)
            data[pre + "aff_in"] = w
            data[pre + "aff_out"] = R.affine_project(cache, w)
            n12a = dp.n * dp.n + dp.n_d
            w_in = rng.normal(size=lay.total - 1)
            u1, u2 = R.solve_inner(cache, w_in[:n12a], w_in[n12a:])
            data[pre + "inner_in"] = w_in
            data[pre + "inner_out"] = np.concatenate([u1, u2])
            cin = rng.normal(size=lay.total)
            data[pre + "cone_in"] = cin
            data[pre + "cone_out"] = R.project_cone(cin, lay)
            u0, w0 = rng.normal(size=lay.total), rng.normal(size=lay.total)
            st = R.iterate(R.HsdeState(u0.copy(), w0.copy()), cache, lay, R.SolverSettings())
            data[pre + "it_u0"], data[pre + "it_w0"] = u0, w0
            data[pre + "it_u1"], data[pre + "it_w1"] = st.u, st.w_dual
            rep = R.solve_decomposed(dp, R.SolverSettings(max_iters=400, check_interval=20))
            data[pre + "solve_status"] = np.array(rep.status)
            data[pre + "solve_iters"] = np.int64(rep.iterations)
            data[pre + "solve_obj"] = np.array([
                np.nan if rep.objective_primal is None else rep.objective_primal,
                np.nan if rep.objective_dual is None else rep.objective_dual])
            count += 1
    data["count"] = np.int64(count)
    np.savez_compressed(HERE / "toys.npz", **data)
    print(f"toys: {count} problems")


def section_cfg(idx: int):
    cp = make_config(idx)
    t = time.time()
    dp = to_reference(cp)
    print(f"cfg{idx}: built reference problem in {time.time() - t:.1f}s")
    fixed = 40 if idx == 4 else 500
    out = {"fixed_iters": np.int64(fixed), "gen_hash": np.array(gen_hash(cp))}
    log = []

    def cb(info):
        log.append((info.iteration, info.pres, info.dres, info.gap, info.tau, info.kappa))
        if info.iteration == fixed:
            out.update(state_summary(cp, cp.compress_vector(info.state.u),
                                     cp.compress_vector(info.state.w_dual), "fixed_"))

    if idx != 4:
        t = time.time()
        R.solve_decomposed(dp, R.SolverSettings(max_iters=fixed, tol=1e-300), iteration_callback=cb)
        out["fixed_log"] = np.array(log)
        out["fixed_wall_s"] = np.float64(time.time() - t)
        print(f"cfg{idx}: fixed {fixed} in {time.time() - t:.1f}s; last check {log[-1]}")
        log.clear()
    tol_log = []

    def cb2(info):
        tol_log.append((info.iteration, info.pres, info.dres, info.gap, info.tau, info.kappa))
        if idx == 4:
            cb(info)

    t = time.time()
    rep = R.solve_decomposed(dp, R.SolverSettings(), iteration_callback=cb2)
    out["tol_wall_s"] = np.float64(time.time() - t)
    out["tol_log"] = np.array(tol_log)
    if idx == 4:
        out["fixed_log"] = np.array(log)
    out["tol_status"] = np.array(rep.status)
    out["tol_iters"] = np.int64(rep.iterations)
    out["tol_setup_s"] = np.float64(rep.timing.setup_s)
    out["tol_per_iteration_s"] = np.float64(rep.timing.per_iteration_s)
    out["tol_obj"] = np.array([
        np.nan if rep.objective_primal is None else rep.objective_primal,
        np.nan if rep.objective_dual is None else rep.objective_dual])
    if rep.residuals is not None:
        out["tol_res"] = np.array([rep.residuals.primal, rep.residuals.dual, rep.residuals.gap])
    if rep.certificate is not None:
        cert = rep.certificate
        out["cert_ray"] = np.array(cert["ray"])
        out["cert_residual"] = np.float64(cert["residual"])
        out["cert_min_eig"] = np.float64(cert["min_block_eigenvalue"])
        if "y" in cert:
            out["cert_y"] = np.array(cert["y"])
        for key in ("slack_entries", "ray_entries"):
            if key in cert:
                out[f"cert_{key}"] = entries_array(cert[key])
    if rep.solution is not None:
        out["sol_x_entries"] = entries_array(rep.solution["x_entries"])
        out["sol_z_entries"] = entries_array(rep.solution["z_entries"])
        out["sol_y"] = np.array(rep.solution["y"], dtype=np.float64)
    np.savez_compressed(HERE / f"cfg{idx}_reference.npz", **out)
    print(f"cfg{idx}: {rep.status} it={rep.iterations} obj={out['tol_obj']} "
          f"tol run {time.time() - t:.1f}s")


def section_cfg4long(fixed: int = 200, mid: int = 100):
    cp = make_config(4)
    t = time.time()
    dp = to_reference(cp)
    print(f"cfg4long: built reference problem in {time.time() - t:.1f}s", flush=True)
    out = {"fixed_iters": np.int64(fixed), "mid_iters": np.int64(mid),
           "gen_hash": np.array(gen_hash(cp))}
    log = []

    def cb(info):
        log.append((info.iteration, info.pres, info.dres, info.gap, info.tau, info.kappa))
        print(f"cfg4long: check {log[-1]} at {time.time() - t:.0f}s", flush=True)
        if info.iteration in (mid, fixed):
            pre = "fixed_" if info.iteration == fixed else "mid_"
            out.update(state_summary(cp, cp.compress_vector(info.state.u),
                                     cp.compress_vector(info.state.w_dual), pre))

    t = time.time()
    R.solve_decomposed(dp, R.SolverSettings(max_iters=fixed, tol=1e-300), iteration_callback=cb)
    out["fixed_log"] = np.array(log)
    out["fixed_wall_s"] = np.float64(time.time() - t)
    np.savez_compressed(HERE / "cfg4_long_reference.npz", **out)
    print(f"cfg4long: {fixed} iterations in {time.time() - t:.1f}s")


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        if arg == "first":
            section_first()
        elif arg == "toys":
            section_toys()
        elif arg == "cfg4long":
            section_cfg4long()
        elif arg.startswith("cfg"):
            section_cfg(int(arg[3:]))
        else:
            raise SystemExit(f"unknown section {arg}")
