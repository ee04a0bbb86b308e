"""CPU tests: pin the oracle (oracle/hsde_oracle.py) to the reference.

The fixtures in tests/golden/ were produced by running the LIVE reference
(tests/golden/make_goldens.py); nothing here imports /root/reference.
"""
import numpy as np
import pytest

from helpers import rel, toy_problem, dense_embedding, dense_inner
from oracle import hsde_oracle as O
from paper_1611_01828_b200.problem import compress


def test_golden_first_iteration(golden_dir):
    """Reference golden vectors (test_solver_oracles.py:349-373), atol 1e-14."""
    z = np.load(golden_dir / "first_iteration.npz")
    dp = toy_problem(z)
    cp = compress(dp, full=True)
    cache = O.setup_cache(cp)
    u0, w0 = O.initial_state(cp)
    u, w = O.iterate(cp, cache, u0, w0, alpha=1.0)
    assert np.allclose(u, z["u"], atol=1e-14, rtol=0)
    assert np.allclose(w, z["w"], atol=1e-14, rtol=0)


def _toys(golden_dir):
    z = np.load(golden_dir / "toys.npz")
    for t in range(int(z["count"])):
        yield t, z, f"t{t}_"


def test_toy_operators_match_reference(golden_dir):
    worst = {"aff": 0.0, "inner": 0.0, "cone": 0.0, "it_u": 0.0, "it_w": 0.0, "dense": 0.0}
    for t, z, pre in _toys(golden_dir):
        dp = toy_problem(z, pre)
        cp = compress(dp, full=True)
        cache = O.setup_cache(cp)
        got = O.affine_project(cp, cache, z[pre + "aff_in"])
        worst["aff"] = max(worst["aff"], rel(got, z[pre + "aff_out"]))
        T = cp.total
        ref = np.linalg.solve(np.eye(T) + dense_embedding(dp), z[pre + "aff_in"])
        worst["dense"] = max(worst["dense"], rel(got, ref))
        n12a = cp.N_c + cp.n_d
        w_in = z[pre + "inner_in"]
        u1, u2 = O.solve_inner(cp, cache, w_in[:n12a], w_in[n12a:])
        worst["inner"] = max(worst["inner"], rel(np.concatenate([u1, u2]), z[pre + "inner_out"]))
        got = O.project_cone(cp, z[pre + "cone_in"])
        worst["cone"] = max(worst["cone"], rel(got, z[pre + "cone_out"]))
        u1, w1 = O.iterate(cp, cache, z[pre + "it_u0"].copy(), z[pre + "it_w0"].copy(), 1.6)
        worst["it_u"] = max(worst["it_u"], rel(u1, z[pre + "it_u1"]))
        worst["it_w"] = max(worst["it_w"], rel(w1, z[pre + "it_w1"]))
    assert worst["aff"] <= 1e-12, worst
    assert worst["dense"] <= 1e-10, worst
    assert worst["inner"] <= 1e-12, worst
    assert worst["cone"] <= 1e-12, worst
    assert worst["it_u"] <= 1e-10 and worst["it_w"] <= 1e-10, worst


def test_toy_solves_match_reference(golden_dir):
    for t, z, pre in _toys(golden_dir):
        dp = toy_problem(z, pre)
        cp = compress(dp)
        out = O.solve(cp, O.OracleSettings(max_iters=400, check_interval=20))
        assert out["status"] == str(z[pre + "solve_status"]), t
        assert out["iterations"] == int(z[pre + "solve_iters"]), t
        if out["status"] in ("Optimal", "MaxItersReached") and "objective_primal" in out:
            ref = z[pre + "solve_obj"]
            assert abs(out["objective_primal"] - ref[0]) <= 1e-6 * (1 + abs(ref[0])), t


@pytest.mark.parametrize("cfg", [0, 1])
def test_config_fixed_iterations_match_reference(golden_dir, cfg):
    """Iterate after 500 iterations within 1e-8 relative of the reference."""
    from paper_1611_01828_b200.synthetic import make_config

    z = np.load(golden_dir / f"cfg{cfg}_reference.npz")
    cp = make_config(cfg)
    states = {}

    def cb(k, p, d, g, tau, kap, u, w):
        states[k] = (u.copy(), w.copy())

    O.solve(cp, O.OracleSettings(max_iters=500, tol=1e-300), callback=cb)
    from helpers import fixture_state

    u, w = states[500]
    ru, rw = fixture_state(z, cp)
    assert rel(u, ru) <= 1e-8
    assert rel(w, rw) <= 1e-8


@pytest.mark.parametrize("cfg", [0, 1])
def test_config_to_tolerance_matches_reference(golden_dir, cfg):
    from paper_1611_01828_b200.synthetic import make_config

    z = np.load(golden_dir / f"cfg{cfg}_reference.npz")
    out = O.solve(make_config(cfg))
    assert out["status"] == str(z["tol_status"])
    assert abs(out["iterations"] - int(z["tol_iters"])) <= 2
    if "cert_ray" in z.files:
        assert out["certificate"]["ray"] == str(z["cert_ray"])
        assert np.allclose(out["certificate"]["y"], z["cert_y"], rtol=1e-6, atol=1e-9)
    else:
        ref = z["tol_obj"]
        assert abs(out["objective_primal"] - ref[0]) <= 1e-6 * abs(ref[0])
        assert abs(out["objective_dual"] - ref[1]) <= 1e-6 * abs(ref[1])


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_generator_hash_matches_fixture(golden_dir, cfg):
    """The synthetic generator still produces the problems the reference
    fixtures were computed on (tests/golden/make_goldens.py gen_hash)."""
    from helpers import gen_hash
    from paper_1611_01828_b200.synthetic import make_config

    z = np.load(golden_dir / f"cfg{cfg}_reference.npz")
    assert gen_hash(make_config(cfg)) == str(z["gen_hash"])
