"""CPU oracle for the HSDE-ADMM hot path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference algorithm (package ``chordalsdp``,
``/root/reference/pkg/src/chordalsdp``) in the compressed covered-coordinate
layout of ``paper_1611_01828_b200.problem.CompressedProblem``.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import it, and only as the checker or the timed
CPU baseline -- never as the product path.

Parity pin: the restatement is checked against the live reference (fixtures
in ``tests/golden/`` produced by ``tests/golden/make_goldens.py``, which
imports the reference in the build container) and against the reference's
own golden first-iteration vectors (test_solver_oracles.py:349-373).

Operation order follows the reference step for step (cited per function);
the one deliberate change is the layout: x holds only covered coordinates.
Off-pattern coordinates of x stay exactly zero from the zero start
(SURVEY.md 0.6), so the iterates are the reference's restricted to the
covered set; dot products differ from the reference only in summation order.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import scipy.linalg

STATUS_OPTIMAL = "Optimal"
STATUS_PRIMAL_INFEASIBLE = "PrimalInfeasible"
STATUS_DUAL_INFEASIBLE = "DualInfeasible"
STATUS_MAX_ITERS = "MaxItersReached"


class OracleFactorizationFailure(RuntimeError):
    pass


class OracleEigenFailure(RuntimeError):
    pass


class OracleTauZero(RuntimeError):
    pass


@dataclass
class OracleSettings:
    """solver.py:82-89 defaults."""

    tol: float = 1e-4
    max_iters: int = 2000
    alpha: float = 1.6
    infeas_tau_tol: float = 1e-9
    infeas_kappa_tol: float = 1e-6
    check_interval: int = 20
    normalize: bool = True


@dataclass
class OracleCache:
    """solver.py:184-200 (KktCache), compressed."""

    p_inv: np.ndarray
    schur: tuple
    zeta: np.ndarray
    minv_zeta: np.ndarray
    zeta_scale: float


def _inner(cp, p_inv, schur, w1, w2):
    """solver.py:203-245 (_solve_inner_parts)."""
    Nc, m = cp.N_c, cp.m
    wa, wb = w1[:Nc], w1[Nc:]
    wy, wv = w2[:m], w2[m:]
    gb = wb - wv                                            # :222
    r = cp.scatter(gb)                                      # :223
    r *= 0.5                                                # :224
    r += cp.scatter(wv)                                     # :225
    r += cp.AT @ wy                                         # :226
    r += wa                                                 # :227
    t = r * p_inv                                           # :230-231
    q = scipy.linalg.cho_solve(schur, cp.A @ t, check_finite=False)
    corr = (cp.AT @ q) * p_inv                              # :232-233
    ua = t - corr                                           # :234-235
    hua = cp.gather(ua)                                     # :236
    ub = 0.5 * (gb + hua)                                   # :237-239
    uy = wy - cp.A @ ua                                     # :240-241
    uv = (ub - hua) + wv                                    # :242-244
    return np.concatenate([ua, ub]), np.concatenate([uy, uv])


def setup_cache(cp) -> OracleCache:
    """solver.py:248-283."""
    p_inv = 1.0 / (1.0 + 0.5 * cp.D)                        # :250
    scaled = cp.A.multiply(p_inv).tocsr()                   # :251
    schur_mat = (scaled @ cp.A.T).toarray()                 # :252
    schur_mat[np.diag_indices_from(schur_mat)] += 1.0       # :253
    try:
        schur = scipy.linalg.cho_factor(schur_mat, lower=True, check_finite=False)
    except (scipy.linalg.LinAlgError, ValueError) as exc:  # :254-259
        raise OracleFactorizationFailure(str(exc)) from exc
    if not np.all(np.isfinite(schur[0])):
        raise OracleFactorizationFailure("non-finite Cholesky factor")
    Nc, nd = cp.N_c, cp.n_d
    zeta = np.concatenate([cp.c, np.zeros(nd), -cp.b, np.zeros(nd)])   # :264
    z1, z2 = _inner(cp, p_inv, schur, zeta[: Nc + nd], zeta[Nc + nd:])  # :265-267
    minv_zeta = np.concatenate([z1, z2])
    zeta_scale = 1.0 + zeta @ minv_zeta                     # :269
    if not zeta_scale > 0:                                  # :270-273
        raise OracleFactorizationFailure(f"rank-one scale {zeta_scale}")
    return OracleCache(p_inv, schur, zeta, minv_zeta, float(zeta_scale))


def solve_inner(cp, cache, w1, w2):
    """solver.py:286-293."""
    return _inner(cp, cache.p_inv, cache.schur, w1, w2)


def affine_project(cp, cache, w):
    """solver.py:296-318: (I + Q) u = w."""
    n12a = cp.N_c + cp.n_d
    w12, w3 = w[:-1], w[-1]
    rho = w12 - w3 * cache.zeta                             # :301
    u1, u2 = _inner(cp, cache.p_inv, cache.schur, rho[:n12a], rho[n12a:])
    u12 = np.concatenate([u1, u2])
    shift = (cache.zeta @ u12) / cache.zeta_scale           # :315
    u12 -= shift * cache.minv_zeta                          # :316
    out = np.empty(w.shape[0])
    out[:-1] = u12
    out[-1] = w3 + cache.zeta @ u12                         # :317
    return out


def project_psd_batch(blocks):
    """symmat.py:153-165."""
    if blocks.shape[-1] == 1:
        return np.maximum(blocks, 0.0)
    sym = 0.5 * (blocks + np.swapaxes(blocks, -1, -2))
    try:
        w, q = np.linalg.eigh(sym)
    except np.linalg.LinAlgError as exc:
        raise OracleEigenFailure(str(exc)) from exc
    if not np.all(np.isfinite(w)):
        raise OracleEigenFailure("non-finite eigenvalues")
    np.maximum(w, 0.0, out=w)
    return np.einsum("kij,kj,klj->kil", q, w, q)


def _groups(cp):
    g = cp._cache.get("oracle_groups")
    if g is None:
        g = []
        for d in np.unique(cp.sizes):                        # solver.py:139-152
            ids = np.flatnonzero(cp.sizes == d)
            idx = cp.offsets[ids][:, None] + np.arange(d * d)[None, :]
            g.append((int(d), idx))
        cp._cache["oracle_groups"] = g
    return g


def project_cone(cp, u_raw, copy=True):
    """solver.py:321-355 (threads=1)."""
    out = u_raw.copy() if copy else u_raw
    s = out[cp.sl_s]
    for d, idx in _groups(cp):
        if d == 1:
            s[idx] = np.maximum(s[idx], 0.0)
            continue
        blocks = s[idx].reshape(idx.shape[0], d, d)
        s[idx] = project_psd_batch(blocks).reshape(idx.shape[0], d * d)
    tau = out[cp.idx_tau]
    out[cp.idx_tau] = tau if tau > 0.0 else 0.0
    return out


def initial_state(cp):
    """solver.py:366-372."""
    u = np.zeros(cp.total)
    w = np.zeros(cp.total)
    u[-1] = 1.0
    w[-1] = 1.0
    return u, w


def iterate(cp, cache, u, w, alpha):
    """solver.py:375-395."""
    u_hat = affine_project(cp, cache, u + w)
    if alpha != 1.0:
        u_hat *= alpha
        u_hat += (1.0 - alpha) * u
    arg = u_hat - w
    u_new = project_cone(cp, arg, copy=False)
    w_new = w - u_hat
    w_new += u_new
    return u_new, w_new


def residuals(cp, u, tau_tol=1e-9):
    """solver.py:398-429 -> (pres, dres, gap)."""
    tau = u[cp.idx_tau]
    if tau <= tau_tol:
        raise OracleTauZero(f"tau = {tau}")
    xt = u[cp.sl_x] / tau
    st = u[cp.sl_s] / tau
    yt = u[cp.sl_y] / tau
    vt = u[cp.sl_v] / tau
    pa = np.linalg.norm(cp.A @ xt - cp.b) / (1.0 + np.linalg.norm(cp.b))
    pc = np.linalg.norm(cp.gather(xt) - st) / (1.0 + np.linalg.norm(st))
    dres = np.linalg.norm(cp.AT @ yt + cp.scatter(vt) - cp.c) / (1.0 + np.linalg.norm(cp.c))
    ctx, bty = cp.c @ xt, cp.b @ yt
    gap = abs(ctx - bty) / (1.0 + abs(ctx) + abs(bty))
    return float(max(pa, pc)), float(dres), float(gap)


def clique_min_eig(cp, s):
    """solver.py:432-440."""
    worst = np.inf
    for k in range(cp.p):
        d = int(cp.sizes[k])
        blk = s[cp.offsets[k]: cp.offsets[k + 1]].reshape(d, d)
        sym = 0.5 * (blk + blk.T)
        worst = min(worst, float(np.linalg.eigvalsh(sym)[0]) if d > 1 else float(sym[0, 0]))
    return worst


def try_certificates(cp, u, tol):
    """solver.py:455-505 on an unscaled iterate with original data ``cp``."""
    x, s, y, v = u[cp.sl_x], u[cp.sl_s], u[cp.sl_y], u[cp.sl_v]
    by = cp.b @ y
    cx = cp.c @ x
    if by > 0:
        yt, vt = y / by, v / by
        resid = float(np.linalg.norm(cp.AT @ yt + cp.scatter(vt)))
        me = clique_min_eig(cp, vt)
        if resid <= tol and me >= -tol:
            return STATUS_DUAL_INFEASIBLE, {"ray": "dual", "y": yt, "b_dot_y": 1.0,
                                            "residual": resid, "min_block_eigenvalue": me}
    if cx < 0:
        scale = -cx
        xt, st = x / scale, s / scale
        resid = float(np.linalg.norm(cp.A @ xt))
        cons = float(np.linalg.norm(cp.gather(xt) - st))
        me = clique_min_eig(cp, cp.gather(xt))
        if resid <= tol and cons <= tol and me >= -tol:
            return STATUS_PRIMAL_INFEASIBLE, {"ray": "primal", "x": xt, "c_dot_x": -1.0,
                                              "residual": resid, "min_block_eigenvalue": me}
    return None


def normalization_scales(cp, enabled):
    """solver.py:659-665."""
    if not enabled:
        return 1.0, 1.0
    nc, nb = float(np.linalg.norm(cp.c)), float(np.linalg.norm(cp.b))
    return (1.0 / nc if nc > 0 else 1.0, 1.0 / nb if nb > 0 else 1.0)


def unscale(cp, u, w, sc, sb):
    """solver.py:668-687."""
    if sc == 1.0 and sb == 1.0:
        return u, w
    u, w = u.copy(), w.copy()
    for vec in (u, w):
        vec[cp.sl_x] /= sb
        vec[cp.sl_s] /= sb
        vec[cp.sl_y] /= sc
        vec[cp.sl_v] /= sc
    return u, w


def solve(cp, settings: OracleSettings | None = None, callback=None, max_wall_s=None):
    """solver.py:690-772 loop + _classify (:521-605), summarised as a dict.

    ``callback(k, pres, dres, gap, tau, kappa, u, w)`` at every check.
    ``max_wall_s`` bounds a CPU-baseline sample (stops after that many seconds).
    """
    import time

    st = settings or OracleSettings()
    sc, sb = normalization_scales(cp, st.normalize)
    cpi = cp if (sc == 1.0 and sb == 1.0) else cp.with_data(c=sc * cp.c, b=sb * cp.b)
    t0 = time.perf_counter()
    cache = setup_cache(cpi)
    u, w = initial_state(cpi)
    setup_s = time.perf_counter() - t0
    log = []
    t1 = time.perf_counter()
    k = 0
    for k in range(1, st.max_iters + 1):
        pu, pw = u, w
        u, w = iterate(cpi, cache, u, w, st.alpha)
        if max_wall_s is not None and time.perf_counter() - t1 > max_wall_s:
            break
        if k % st.check_interval and k != st.max_iters:
            continue
        merit = float(np.linalg.norm(u - pu) + np.linalg.norm(w - pw))
        tau, kappa = u[-1], w[-1]
        if tau > st.infeas_tau_tol:
            pres, dres, gap = residuals(cpi, u, st.infeas_tau_tol)
            log.append((k, pres, dres, gap, float(tau), float(kappa), merit))
            if callback:
                callback(k, pres, dres, gap, float(tau), float(kappa), u, w)
            if max(pres, dres, gap) <= st.tol:
                break
        else:
            inf = float("inf")
            log.append((k, inf, inf, inf, float(tau), float(kappa), merit))
            if callback:
                callback(k, inf, inf, inf, float(tau), float(kappa), u, w)
            if kappa > st.infeas_kappa_tol:
                uu, _ = unscale(cpi, u, w, sc, sb)
                if try_certificates(cp, uu, st.tol) is not None:
                    break
    loop_s = time.perf_counter() - t1
    out = {"iterations": k, "setup_s": setup_s, "loop_s": loop_s, "log": log,
           "u": u, "w": w}
    tau, kappa = u[-1], w[-1]
    uu, _ = unscale(cpi, u, w, sc, sb)
    if tau > st.infeas_tau_tol:
        res = residuals(cpi, u, st.infeas_tau_tol)
        xt, yt = uu[cp.sl_x] / tau, uu[cp.sl_y] / tau
        out.update(status=STATUS_OPTIMAL if max(res) <= st.tol else STATUS_MAX_ITERS,
                   residuals=res,
                   objective_primal=cp.objective_sign * float(cp.c @ xt),
                   objective_dual=cp.objective_sign * float(cp.b @ yt))
        return out
    if kappa > st.infeas_kappa_tol:
        found = try_certificates(cp, uu, st.tol)
        if found is not None:
            out.update(status=found[0], certificate=found[1])
            return out
    out.update(status=STATUS_MAX_ITERS)
    return out
