"""Drop-in HSDE-ADMM solver entry points, computed on the B200.

Mirrors the public API of the reference module ``chordalsdp/solver.py``
(same names, signatures, argument meaning, exceptions and report schema):
``SolverSettings`` (:68-99), ``VariableLayout`` (:102-152), ``QOperator``
(:155-175), ``build_hsde`` (:178-181), ``setup_cache`` (:248-283),
``solve_inner`` (:286-293), ``affine_project`` (:296-318), ``project_cone``
(:321-355), ``HsdeState`` / ``initial_state`` (:358-372), ``iterate``
(:375-395), ``residuals`` (:398-429), ``recover`` (:608-617),
``IterationInfo`` (:620-631), ``solve_decomposed`` (:690-772).

Every arithmetic step of the iteration runs in libhsde.so (hand-written
sm_100a CUDA, see csrc/).  Python here only converts layouts, drives the
loop (one device sync per residual check), and assembles the report the way
the reference's Python does.  There is no CPU fallback: without the library
or a GPU every entry point raises.
"""

from __future__ import annotations

import logging
import math
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import EigenFailure, FactorizationFailure, TauZero
from .problem import CompressedProblem, compress, edges_array
from .report import (STATUS_DUAL_INFEASIBLE, STATUS_MAX_ITERS, STATUS_OPTIMAL,
                     STATUS_PRIMAL_INFEASIBLE, PatternEntries, ProblemStats, Residuals, SolverReport,
                     Timing)

logger = logging.getLogger(__name__)

#: unit-level API calls keep every n**2 coordinate on the device below this size
FULL_LAYOUT_MAX = 1 << 22

__all__ = [
    "SolverSettings", "VariableLayout", "QOperator", "build_hsde", "KktCache", "setup_cache",
    "solve_inner", "affine_project", "project_cone", "HsdeState", "initial_state", "iterate",
    "residuals", "recover", "IterationInfo", "solve", "solve_decomposed", "FactorizationFailure",
    "TauZero", "EigenFailure",
]


@dataclass
class SolverSettings:
    """Termination and algorithm parameters (solver.py:68-99, same defaults)."""

    tol: float = 1e-4
    max_iters: int = 2000
    alpha: float = 1.6
    infeas_tau_tol: float = 1e-9
    infeas_kappa_tol: float = 1e-6
    check_interval: int = 20
    normalize: bool = True
    threads: int = 1
    device: int | None = None  # CUDA device ordinal (extension; default LOCAL_RANK / 0)

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if not 1.0 <= self.alpha < 2.0:
            raise ValueError("alpha must lie in [1, 2)")
        if self.check_interval < 1:
            raise ValueError("check_interval must be at least 1")


@dataclass(frozen=True, eq=False)
class VariableLayout:
    """Reference stacked layout (solver.py:102-152): x is n**2 long."""

    n: int
    m: int
    n_d: int
    dec: object

    @property
    def n2(self) -> int:
        return self.n * self.n

    @property
    def total(self) -> int:
        return self.n2 + 2 * self.n_d + self.m + 1

    @property
    def sl_x(self) -> slice:
        return slice(0, self.n2)

    @property
    def sl_s(self) -> slice:
        return slice(self.n2, self.n2 + self.n_d)

    @property
    def sl_y(self) -> slice:
        return slice(self.n2 + self.n_d, self.n2 + self.n_d + self.m)

    @property
    def sl_v(self) -> slice:
        return slice(self.n2 + self.n_d + self.m, self.total - 1)

    @property
    def idx_tau(self) -> int:
        return self.total - 1

    def size_groups(self):
        sizes = np.asarray(self.dec.sizes)
        out = []
        for size in np.unique(sizes):
            ids = np.nonzero(sizes == size)[0]
            base = np.asarray(self.dec.offsets)[ids]
            out.append((int(size), base[:, None] + np.arange(size * size)[None, :]))
        return out


@dataclass(frozen=True, eq=False)
class QOperator:
    """Implicit skew embedding operator (solver.py:155-175).

    Test utility only (the reference uses it only in tests); evaluated with
    numpy on the host, never on the solve path.
    """

    dp: object
    layout: VariableLayout

    def apply(self, u: np.ndarray) -> np.ndarray:
        lay, dp = self.layout, self.dp
        x, s, y, v = u[lay.sl_x], u[lay.sl_s], u[lay.sl_y], u[lay.sl_v]
        tau = u[lay.idx_tau]
        gi = np.asarray(dp.dec.gather_index)
        out = np.empty_like(u)
        out[lay.sl_x] = -(dp.A.T @ y) - np.bincount(gi, weights=v, minlength=lay.n2) + tau * dp.c
        out[lay.sl_s] = v
        out[lay.sl_y] = dp.A @ x - tau * dp.b
        out[lay.sl_v] = x[gi] - s
        out[lay.idx_tau] = -(dp.c @ x) + dp.b @ y
        return out


def build_hsde(dp):
    """(QOperator, VariableLayout) of a reference-layout problem (solver.py:178-181)."""
    layout = VariableLayout(n=dp.n, m=dp.m, n_d=dp.n_d, dec=dp.dec)
    return QOperator(dp, layout), layout


@dataclass
class HsdeState:
    """One ADMM iterate (solver.py:358-363)."""

    u: np.ndarray
    w_dual: np.ndarray


def initial_state(layout) -> HsdeState:
    """u = w = 0 with tau = kappa = 1 (solver.py:366-372)."""
    u = np.zeros(layout.total)
    w = np.zeros(layout.total)
    u[layout.idx_tau] = 1.0
    w[layout.idx_tau] = 1.0
    return HsdeState(u, w)


# ---------------------------------------------------------------------------
# layout conversion between reference vectors and device (compressed) vectors


class _Mapper:
    """Reference-layout <-> compressed-layout conversion for one problem."""

    def __init__(self, cp: CompressedProblem, n2: int):
        self.cp = cp
        self.n2 = n2
        self.full = cp.N_c == n2
        self._off = None

    @property
    def off(self) -> np.ndarray:
        """Off-pattern flat ids (built on first use: n^2 long scans, 2.6e8 for config 4,
        that a plain solve never needs)."""
        if self._off is None:
            mask = np.ones(self.n2, dtype=bool)
            mask[self.cp.covered] = False
            self._off = np.flatnonzero(mask)
        return self._off

    def down(self, full_vec: np.ndarray) -> np.ndarray:
        full_vec = np.asarray(full_vec, dtype=float)
        if self.full:
            return np.ascontiguousarray(full_vec)
        return self.cp.compress_vector(full_vec)

    def up(self, comp: np.ndarray, off_values: np.ndarray | None = None) -> np.ndarray:
        if self.full:
            return comp
        out = np.empty(self.n2 + comp.shape[0] - self.cp.N_c)
        out[: self.n2] = 0.0
        if off_values is not None:
            out[self.off] = off_values
        out[self.cp.covered] = comp[: self.cp.N_c]
        out[self.n2:] = comp[self.cp.N_c:]
        return out


def _api_problem(dp) -> tuple[CompressedProblem, _Mapper]:
    if isinstance(dp, CompressedProblem):
        return dp, _Mapper(dp, dp.N_c)
    n2 = int(dp.n) * int(dp.n)
    cp = compress(dp, full=n2 <= FULL_LAYOUT_MAX)
    return cp, _Mapper(cp, n2 if not isinstance(dp, CompressedProblem) else cp.N_c)


def _device(settings: SolverSettings | None = None) -> int:
    if settings is not None and settings.device is not None:
        return int(settings.device)
    return _lib.default_device()


class KktCache:
    """Device-resident counterpart of the reference KktCache (solver.py:184-200).

    Holds the factored m x m Schur inverse, P^{-1}, zeta and M^{-1} zeta on the
    device.  ``factored_dims == (m,)``: the only factorisation is m x m.
    """

    def __init__(self, dp, handle: _lib.Handle, cp: CompressedProblem, mapper: _Mapper):
        self.dp = dp
        self.handle = handle
        self.cp = cp
        self.mapper = mapper
        self.zeta_scale = handle.zeta_scale
        self.factored_dims = (int(dp.m),)

    @property
    def p_inv(self) -> np.ndarray:
        d = np.bincount(np.asarray(self.dp.dec.gather_index, dtype=np.int64),
                        minlength=int(self.dp.n) ** 2).astype(float)
        return 1.0 / (1.0 + 0.5 * d)

    @property
    def zeta(self) -> np.ndarray:
        return np.concatenate([np.asarray(self.dp.c, float), np.zeros(self.dp.n_d),
                               -np.asarray(self.dp.b, float), np.zeros(self.dp.n_d)])

    @property
    def minv_zeta(self) -> np.ndarray:
        mz = self.handle.minv_zeta()
        return self.mapper.up(np.concatenate([mz, [0.0]]))[:-1]


def setup_cache(dp) -> KktCache:
    """Factor the m x m reduced system on the device (solver.py:248-283)."""
    cp, mapper = _api_problem(dp)
    h = _lib.Handle(cp, normalize=False, device=_device())
    return KktCache(dp, h, cp, mapper)


def solve_inner(cache: KktCache, w1: np.ndarray, w2: np.ndarray):
    """Solve [[I, B'], [-B, I]] (u1, u2) = (w1, w2) (solver.py:286-293)."""
    mp, cp = cache.mapper, cache.cp
    n12a = mp.n2 + int(cache.dp.n_d) if not isinstance(cache.dp, CompressedProblem) else cp.N_c + cp.n_d
    w = np.concatenate([np.asarray(w1, float), np.asarray(w2, float), [0.0]])
    wc = mp.down(w)
    u12 = cache.handle.solve_inner(wc[:-1])
    # off-support x coordinates: ua = wa exactly (no clique, column or cost there)
    full = mp.up(np.concatenate([u12, [0.0]]), None if mp.full else w[mp.off])[:-1]
    return full[:n12a].copy(), full[n12a:].copy()


def affine_project(cache: KktCache, w: np.ndarray) -> np.ndarray:
    """Solve (I + Q) u_hat = w on the device (solver.py:296-318)."""
    mp = cache.mapper
    w = np.asarray(w, dtype=float)
    u = cache.handle.affine_project(mp.down(w))
    return mp.up(u, None if mp.full else w[mp.off])


_cone_handles: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _cone_handle(layout):
    """NO_FACTOR handle carrying only the clique structure of a layout."""
    try:
        hit = _cone_handles.get(layout)
    except TypeError:
        hit = None
    if hit is not None:
        return hit
    if isinstance(layout, CompressedProblem):
        cp = layout.with_data()
        cp.A = sp.csr_matrix((cp.m, cp.N_c))
        cp.c = np.zeros(cp.N_c)
        cp.b = np.zeros(cp.m)
        mapper = _Mapper(cp, cp.N_c)
    else:
        n = int(layout.n)
        n2 = n * n
        gi = np.asarray(layout.dec.gather_index, dtype=np.int64)
        full = n2 <= FULL_LAYOUT_MAX
        covered = np.arange(n2, dtype=np.int64) if full else np.unique(gi)
        cp = CompressedProblem(
            n=n, m=int(layout.m), covered=covered, c=np.zeros(covered.size),
            A=sp.csr_matrix((int(layout.m), covered.size)), b=np.zeros(int(layout.m)),
            cliques=tuple(np.asarray(c, dtype=np.int64) for c in layout.dec.cliques),
            sizes=np.asarray(layout.dec.sizes, dtype=np.int64),
            offsets=np.asarray(layout.dec.offsets, dtype=np.int64),
            slot_cov=np.searchsorted(covered, gi).astype(np.int32))
        mapper = _Mapper(cp, n2)
    h = _lib.Handle(cp, normalize=False, flags=_lib.HSDE_FLAG_NO_FACTOR, device=_device())
    hit = (h, mapper)
    try:
        _cone_handles[layout] = hit
    except TypeError:
        pass
    return hit


def project_cone(u_raw: np.ndarray, layout, threads: int = 1, copy: bool = True) -> np.ndarray:
    """Blockwise cone projection on the device (solver.py:321-355).

    x, y, v pass through, clique blocks of s are projected onto their PSD
    cones (one warp / CTA per clique), tau is clamped.  ``threads`` is
    accepted for signature compatibility; the result never depends on it.
    """
    h, mp = _cone_handle(layout)
    u_raw = np.asarray(u_raw, dtype=float)
    out = mp.up(h.project_cone(mp.down(u_raw)), None if mp.full else u_raw[mp.off])
    if not copy:
        u_raw[...] = out
        return u_raw
    return out


def iterate(state: HsdeState, cache: KktCache, layout, settings: SolverSettings) -> HsdeState:
    """One ADMM sweep on the device (solver.py:375-395)."""
    mp = cache.mapper
    h = cache.handle
    h.set_alpha(settings.alpha)
    u = np.asarray(state.u, dtype=float)
    w = np.asarray(state.w_dual, dtype=float)
    h.set_state(mp.down(u), mp.down(w))
    h.iterate(1)
    un, wn = h.get_state()
    if mp.full:
        return HsdeState(un, wn)
    # off-support x coordinates carry no coupling: u_hat = u + w there
    uo, wo = u[mp.off], w[mp.off]
    uh = uo + wo
    if settings.alpha != 1.0:
        uh = settings.alpha * uh + (1.0 - settings.alpha) * uo
    xn = uh - wo
    return HsdeState(mp.up(un, xn), mp.up(wn, (wo - uh) + xn))


_resid_handles: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def residuals(state: HsdeState, dp, tau_tol: float = 1e-9) -> Residuals:
    """Scaled primal/dual/gap residuals on the device (solver.py:398-429)."""
    lay_total = (dp.N_c if isinstance(dp, CompressedProblem) else int(dp.n) ** 2) \
        + 2 * int(dp.n_d) + int(dp.m) + 1
    u = np.asarray(state.u, dtype=float)
    if u.shape != (lay_total,):
        raise ValueError(f"state length {u.shape} does not match the problem ({lay_total})")
    tau = u[-1]
    if tau <= tau_tol:
        raise TauZero(f"tau = {tau} is numerically zero")
    hit = None
    try:
        hit = _resid_handles.get(dp)
    except TypeError:
        pass
    if hit is None:
        cp, mp = _api_problem(dp)
        h = _lib.Handle(cp, normalize=False, infeas_tau_tol=-math.inf,
                        flags=_lib.HSDE_FLAG_NO_FACTOR, device=_device())
        hit = (h, mp)
        try:
            _resid_handles[dp] = hit
        except TypeError:
            pass
    h, mp = hit
    r = h.residuals(mp.down(u))
    return Residuals(primal=float(r[0]), dual=float(r[1]), gap=float(r[2]))


# ---------------------------------------------------------------------------
# the solve driver


@dataclass
class IterationInfo:
    """Snapshot handed to the iteration callback at every check (solver.py:620-631).

    ``state`` is fetched from the device (and expanded to the reference
    layout) only when the callback reads it.
    """

    iteration: int
    pres: float
    dres: float
    gap: float
    tau: float
    kappa: float
    _fetch: object = None
    layout: object = None

    @property
    def state(self) -> HsdeState:
        return self._fetch()


class _MeritTracker:
    """Warns when the fixed-point residual rises across 50-iteration windows
    (solver.py:634-656)."""

    window = 50

    def __init__(self):
        self._minima: dict[int, float] = {}

    def record(self, iteration: int, merit: float) -> None:
        bucket = (iteration - 1) // self.window
        self._minima[bucket] = min(self._minima.get(bucket, math.inf), merit)
        if bucket >= 2:
            older, newer = self._minima.get(bucket - 2), self._minima.get(bucket - 1)
            if older is not None and newer is not None and newer > older * (1 + 1e-9):
                logger.warning("fixed-point residual rose across windows %d -> %d (%.3e -> %.3e)",
                               bucket - 2, bucket - 1, older, newer)
                self._minima.pop(bucket - 2, None)


def _cert_decision(cert: np.ndarray, tol: float):
    """Acceptance rules of _try_certificates (solver.py:472-503)."""
    by, cx, dres, dmin, pres, pcons, pmin = (float(v) for v in cert)
    if by > 0 and dres <= tol and dmin >= -tol:
        return STATUS_DUAL_INFEASIBLE
    if cx < 0 and pres <= tol and pcons <= tol and pmin >= -tol:
        return STATUS_PRIMAL_INFEASIBLE
    return None


class _Session:
    """One device handle driven through a solve (shared by solve/recover).

    ``shards``: run the clique-sharded algorithm -- an int G
    emulates G shards on this device; ``comm=(world, rank, nccl_id)`` runs this
    rank's shard of ``shard.make_shards(cp, world)`` with NCCL.
    """

    def __init__(self, dp, settings: SolverSettings, normalize: bool, shards=None, comm=None):
        from .shard import make_shards

        self.dp = dp
        self.cp = dp if isinstance(dp, CompressedProblem) else compress(dp, with_edges=False)
        self.n2 = self.cp.N_c if isinstance(dp, CompressedProblem) else int(dp.n) ** 2
        self.mapper = _Mapper(self.cp, self.n2)
        self.settings = settings
        self.shards = None
        self.comm = comm
        # The report's pattern index (solver.py:443-452) depends on the problem only:
        # it is built on a host thread during the device setup and the iterations
        # (numpy and the library release the GIL), and joined in _classify.
        self.index_thread = threading.Thread(target=_pattern_index, args=(self.cp, dp), daemon=True)
        self.index_thread.start()
        kw = dict(alpha=settings.alpha, tol=settings.tol, infeas_tau_tol=settings.infeas_tau_tol,
                  infeas_kappa_tol=settings.infeas_kappa_tol,
                  check_interval=settings.check_interval, normalize=normalize,
                  device=_device(settings))
        if comm is not None:
            world, rank = int(comm[0]), int(comm[1])
            self.shards = make_shards(self.cp, world)
            self.h = _lib.Handle(self.cp, shards=[self.shards[rank]], comm=comm, **kw)
        elif shards:
            self.shards = make_shards(self.cp, int(shards))
            self.h = _lib.Handle(self.cp, shards=self.shards, **kw)
        else:
            self.h = _lib.Handle(self.cp, **kw)
        self.sigma_c, self.sigma_b = self.h.sigma_c, self.h.sigma_b

    def raw_state(self):
        """Global compressed (u, w) of the normalised problem."""
        from .shard import gather_state

        if self.shards is None:
            return self.h.get_state()
        if self.comm is None:
            parts = [self.h.get_state(g) for g in range(len(self.shards))]
        elif int(self.comm[0]) == 1:
            parts = [self.h.get_state(0)]
        else:
            import torch.distributed as dist

            mine = self.h.get_state(0)
            parts = [None] * int(self.comm[0])
            dist.all_gather_object(parts, mine)
        u = gather_state(self.cp, self.shards, [p[0] for p in parts])
        w = gather_state(self.cp, self.shards, [p[1] for p in parts])
        return u, w

    def state_ref_layout(self) -> HsdeState:
        u, w = self.raw_state()
        return HsdeState(self.mapper.up(u), self.mapper.up(w))

    def unscaled(self):
        """Compressed unscaled u (solver.py:668-687; the report reads u only)."""
        u = self.h.get_u() if self.shards is None else self.raw_state()[0]
        cp = self.cp
        if self.sigma_c != 1.0 or self.sigma_b != 1.0:
            u[cp.sl_x] /= self.sigma_b
            u[cp.sl_s] /= self.sigma_b
            u[cp.sl_y] /= self.sigma_c
            u[cp.sl_v] /= self.sigma_c
        return u


def _pattern_index(cp: CompressedProblem, dp):
    """Block-local (block, i, j) of the aggregate pattern plus the diagonal
    (solver.py:443-452), and where each entry sits in the covered vector.
    Cached on ``cp``: x and z share it."""
    key = "pattern_index"
    if key in cp._cache:
        return cp._cache[key]
    n = cp.n
    if isinstance(dp, CompressedProblem) or getattr(dp, "aggregate", None) is None:
        edges = cp.aggregate_edges if cp.aggregate_edges is not None else np.zeros((0, 2), np.int64)
    else:
        edges = edges_array(dp.aggregate, n)
        if edges is None:
            edges = np.zeros((0, 2), np.int64)
    diag = np.arange(n, dtype=np.int64)
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    ecode = edges[:, 0] * n + edges[:, 1]
    dcode = diag * (n + 1)
    if ecode.size and bool(np.all(ecode[1:] > ecode[:-1])):
        # sorted, unique edge codes (the usual case): merge the diagonal in O(N)
        at = np.searchsorted(ecode, dcode)
        present = ecode[np.minimum(at, ecode.size - 1)] == dcode
        code = np.insert(ecode, at[~present], dcode[~present])
    else:
        code = np.unique(np.concatenate([ecode, dcode]))
    dims = np.abs(np.asarray(cp.block_dims or (n,), dtype=np.int64))
    starts = np.concatenate([[0], np.cumsum(dims)])
    # block, block-local (i, j), and the covered position of the flat id
    # gj * n + gi (= np.searchsorted(cp.covered, gj * n + gi)), in the library
    b, i, j, pos_c, hit = _lib.pattern_index(cp.covered, n, code, starts)
    out = (b, i, j, pos_c, None if bool(hit.all()) else hit)  # hit None: every row is covered
    cp._cache[key] = out
    return out


def _pattern_entries(cp: CompressedProblem, dp, xc: np.ndarray) -> PatternEntries:
    """[block, i, j, value] rows (1-based, block-local) on the aggregate pattern
    plus the diagonal (solver.py:443-452); ``xc`` is a covered-coordinate vector."""
    b, i, j, pos_c, hit = _pattern_index(cp, dp)
    if hit is None:
        vals = xc[pos_c]
    else:
        vals = np.where(hit, xc[pos_c] if cp.N_c else 0.0, 0.0)
    return PatternEntries(b, i, j, vals)


def _problem_stats(cp: CompressedProblem, dp) -> ProblemStats:
    sizes = cp.sizes
    return ProblemStats(
        n=int(cp.n), m=int(cp.m), blocks=[int(d) for d in (cp.block_dims or (cp.n,))],
        p=int(cp.p), clique_max=int(sizes.max()) if len(sizes) else 0,
        clique_min=int(sizes.min()) if len(sizes) else 0, n_d=int(cp.n_d))


def _classify(sess: _Session, chk: np.ndarray, iterations: int, timing: Timing) -> SolverReport:
    """solver.py:521-605 on the device iterate."""
    st, cp, dp = sess.settings, sess.cp, sess.dp
    th = getattr(sess, "index_thread", None)
    if th is not None:
        th.join()
        sess.index_thread = None
    stats = _problem_stats(cp, dp)
    sign = float(getattr(dp, "objective_sign", cp.objective_sign))
    tau, kappa = float(chk[3]), float(chk[4])
    if tau > st.infeas_tau_tol:
        res = Residuals(primal=float(chk[0]), dual=float(chk[1]), gap=float(chk[2]))
        hvt = None
        if sess.shards is None:
            # x, y and H' vt straight from the device (no full-state copy, no host bincount)
            ux, uy, hvt = sess.h.report_vectors(tau)
            if sess.sigma_b != 1.0:
                ux /= sess.sigma_b
            if sess.sigma_c != 1.0:
                uy /= sess.sigma_c
            xt, yt = ux / tau, uy / tau
        else:
            u = sess.unscaled()
            xt = u[cp.sl_x] / tau
            yt = u[cp.sl_y] / tau
        # (einsum's own loops, not BLAS ddot: OpenBLAS workers keep spinning after a
        # threaded call and slowed the next solve's staged H2D copies by ~40 ms)
        obj_p = sign * float(np.einsum("i,i->", cp.c, xt))
        obj_d = sign * float(np.einsum("i,i->", cp.b, yt))
        if res.max() <= st.tol:
            if hvt is None:
                hvt = cp.scatter(u[cp.sl_v] / tau)
            solution = {
                "x_entries": _pattern_entries(cp, dp, xt),
                "y": [float(t) for t in yt],
                "z_entries": _pattern_entries(cp, dp, hvt),
            }
            return SolverReport(status=STATUS_OPTIMAL, objective_primal=obj_p,
                                objective_dual=obj_d, iterations=iterations, residuals=res,
                                timing=timing, problem=stats, tol=st.tol, solution=solution)
        return SolverReport(status=STATUS_MAX_ITERS, objective_primal=obj_p,
                            objective_dual=obj_d, iterations=iterations, residuals=res,
                            timing=timing, problem=stats, tol=st.tol)
    if kappa > st.infeas_kappa_tol:
        cert = sess.h.certificate()
        status = _cert_decision(cert, st.tol)
        if status is not None:
            u = sess.unscaled()
            if status == STATUS_DUAL_INFEASIBLE:
                by = float(cert[0])
                yt, vt = u[cp.sl_y] / by, u[cp.sl_v] / by
                certificate = {
                    "ray": "dual", "y": [float(t) for t in yt],
                    "slack_entries": _pattern_entries(cp, dp, cp.scatter(vt)),
                    "b_dot_y": 1.0, "residual": float(cert[2]),
                    "min_block_eigenvalue": float(cert[3]),
                }
            else:
                scale = -float(cert[1])
                xt = u[cp.sl_x] / scale
                certificate = {
                    "ray": "primal", "ray_entries": _pattern_entries(cp, dp, xt),
                    "c_dot_x": -1.0, "residual": float(cert[4]),
                    "min_block_eigenvalue": float(cert[6]),
                }
            return SolverReport(status=status, objective_primal=None, objective_dual=None,
                                iterations=iterations, residuals=None, timing=timing,
                                problem=stats, tol=st.tol, certificate=certificate)
    return SolverReport(status=STATUS_MAX_ITERS, objective_primal=None, objective_dual=None,
                        iterations=iterations, residuals=None, timing=timing, problem=stats,
                        tol=st.tol)


def solve_decomposed(dp, settings: SolverSettings | None = None, iteration_callback=None,
                     setup_elapsed: float = 0.0, *, shards: int | None = None,
                     comm=None) -> SolverReport:
    """Run the ADMM loop on the B200 (solver.py:690-772).

    ``dp`` is a reference-layout ``DecomposedProblem`` (the reference's own or
    :class:`paper_1611_01828_b200.problem.DecomposedProblem`) or a
    :class:`CompressedProblem`.  Iterations run back to back on the device
    (CUDA-graph replay); the host syncs once per ``check_interval``.

    Extensions (keyword-only): ``comm=(world, rank, nccl_id)`` runs this rank's
    clique shard with NCCL all-reduce (one process per GPU, see
    paper_1611_01828_b200.multigpu); ``shards=G`` emulates G shards on one GPU.
    """
    settings = settings or SolverSettings()
    t0 = time.perf_counter()
    sess = _Session(dp, settings, settings.normalize, shards=shards, comm=comm)
    setup_s = setup_elapsed + (time.perf_counter() - t0)
    layout = sess.cp if isinstance(dp, CompressedProblem) else build_hsde(dp)[1]
    tracker = _MeritTracker()
    ci = settings.check_interval
    t1 = time.perf_counter()
    k = 0
    chk = None
    while k < settings.max_iters:
        step = min(ci - (k % ci), settings.max_iters - k)
        sess.h.iterate(step)
        k += step
        chk = sess.h.check()
        pres, dres, gap, tau, kappa, merit = (float(v) for v in chk[:6])
        tracker.record(k, merit)
        fetch = sess.state_ref_layout
        if tau > settings.infeas_tau_tol:
            if iteration_callback is not None:
                iteration_callback(IterationInfo(k, pres, dres, gap, tau, kappa, fetch, layout))
            if max(pres, dres, gap) <= settings.tol:
                break
        else:
            if iteration_callback is not None:
                inf = float("inf")
                iteration_callback(IterationInfo(k, inf, inf, inf, tau, kappa, fetch, layout))
            if kappa > settings.infeas_kappa_tol:
                if _cert_decision(sess.h.certificate(), settings.tol) is not None:
                    break
    loop_s = time.perf_counter() - t1
    timing = Timing(setup_s=setup_s, iterations_s=loop_s, total_s=setup_s + loop_s,
                    per_iteration_s=loop_s / max(k, 1))
    report = _classify(sess, chk, k, timing)
    sess.h.close()
    return report


def solve(problem, settings: SolverSettings | None = None, split_cones: bool = True,
          iteration_callback=None) -> SolverReport:
    """Decompose, embed, iterate and classify a parsed problem (solver.py:775-789):
    host decomposition in C++ (:func:`paper_1611_01828_b200.decompose`), then
    :func:`solve_decomposed` on the B200; decomposition time counts as setup."""
    from .decompose import decompose
    t0 = time.perf_counter()
    cp = decompose(problem, split_cones=split_cones)
    return solve_decomposed(cp, settings=settings, iteration_callback=iteration_callback,
                            setup_elapsed=time.perf_counter() - t0)


def recover(state: HsdeState, dp, settings: SolverSettings, iterations: int,
            timing: Timing) -> SolverReport:
    """Classify a final iterate of ``dp`` (solver.py:608-617), no normalisation."""
    sess = _Session(dp, settings, normalize=False)
    sess.h.set_state(sess.mapper.down(state.u), sess.mapper.down(state.w_dual))
    chk = sess.h.check()
    report = _classify(sess, chk, iterations, timing)
    sess.h.close()
    return report
