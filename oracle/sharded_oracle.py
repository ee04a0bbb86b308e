"""Sharded CPU restatement of the HSDE iteration -- TEST INFRASTRUCTURE ONLY.

Checks the multi-GPU algorithm of paper_1611_01828_b200.shard (SURVEY.md
section 8(e)) on the CPU: each shard runs the reference iteration
(chordalsdp/solver.py:203-245, 296-318, 375-395, restated as in
hsde_oracle.py) on its local cliques / coordinates and meets the others at
exactly the three all-reduce points the CUDA path uses:

  1. separator pull-scatter partials   (|S| doubles)
  2. partial A t over owned columns     (m doubles)
  3. partial c.ua over owned coordinates (1 double)

plus the setup reductions (|c|^2, the m x m Schur matrix, zeta.M zeta) and
the residual-check reductions.  The per-rank algorithm is a generator that
yields ('sum', array) at every reduction point; a driver sends the reduced
array back -- in-process (sum in rank order) or across processes with
torch.distributed (gloo).  Only tests/ import this module.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from .hsde_oracle import project_psd_batch


def _reduce(arr):
    out = yield ("sum", np.asarray(arr, dtype=float))
    return out


class ShardRun:
    """Per-rank state of the sharded oracle."""

    def __init__(self, sh, alpha=1.6, normalize=True):
        self.sh = sh
        self.lp = sh.problem
        self.alpha = alpha
        self.normalize = normalize
        lp = self.lp
        self.p_inv = 1.0 / (1.0 + 0.5 * sh.D)
        self.AT = lp.A.T.tocsr()
        self.A_own = lp.A[:, np.flatnonzero(sh.owned)].tocsr()
        self.own_idx = np.flatnonzero(sh.owned)
        self.groups = []
        for d in np.unique(lp.sizes):
            ids = np.flatnonzero(lp.sizes == d)
            self.groups.append((int(d), lp.offsets[ids][:, None] + np.arange(d * d)[None, :]))

    # -- pieces ---------------------------------------------------------------
    def scatter(self, s):
        return np.bincount(self.lp.slot_cov, weights=s, minlength=self.lp.N_c)

    def _sep_exchange(self, part):
        sh = self.sh
        buf = np.zeros(sh.n_sep)
        buf[sh.sep_pos] = part[sh.sep_local]
        full = yield from _reduce(buf)
        part = part.copy()
        part[sh.sep_local] = full[sh.sep_pos]
        return part

    def inner(self, rx, rs, ry, rv):
        """_solve_inner_parts (solver.py:203-245), sharded; uy by the identity A ua = q'."""
        gb = rs - rv
        part = self.scatter(gb) * 0.5 + self.scatter(rv)
        part = yield from self._sep_exchange(part)
        r = (part + self.AT @ ry) + rx
        t = r * self.p_inv
        qpart = self.A_own @ t[self.own_idx]
        q = yield from _reduce(qpart)
        qp = scipy.linalg.cho_solve(self.schur, q, check_finite=False)
        ua = t - (self.AT @ qp) * self.p_inv
        hua = ua[self.lp.slot_cov]
        ub = 0.5 * (gb + hua)
        uy = ry - qp
        uv = (ub - hua) + rv
        return ua, ub, uy, uv

    # -- setup (solver.py:248-283, 659-665) ------------------------------------------------
    def setup(self):
        lp, sh = self.lp, self.sh
        if self.normalize:
            nc2 = yield from _reduce(np.array([float(lp.c[self.own_idx] @ lp.c[self.own_idx])]))
            nc = float(np.sqrt(nc2[0]))
            nb = float(np.linalg.norm(lp.b))
            self.sc = 1.0 / nc if nc > 0 else 1.0
            self.sb = 1.0 / nb if nb > 0 else 1.0
        else:
            self.sc = self.sb = 1.0
        self.c = self.sc * lp.c
        self.b = self.sb * lp.b
        scaled = self.A_own.multiply(self.p_inv[self.own_idx]).tocsr()
        spart = (scaled @ self.A_own.T).toarray()
        S = yield from _reduce(spart)
        S[np.diag_indices_from(S)] += 1.0
        self.schur = scipy.linalg.cho_factor(S, lower=True, check_finite=False)
        zs, zv = np.zeros(lp.n_d), np.zeros(lp.n_d)
        ua, ub, uy, uv = yield from self.inner(self.c, zs, -self.b, zv)
        self.mz = (ua, ub, uy, uv)
        zpart = float(self.c[self.own_idx] @ ua[self.own_idx])
        zmz = yield from _reduce(np.array([zpart]))
        self.zmz = float(zmz[0] - self.b @ uy)
        self.zeta_scale = 1.0 + self.zmz
        u = np.zeros(lp.total)
        w = np.zeros(lp.total)
        u[-1] = w[-1] = 1.0
        self.u, self.w = u, w

    # -- one iteration (solver.py:375-395) --------------------------------------------------
    def iterate(self):
        lp, a = self.lp, self.alpha
        u, w = self.u, self.w
        atau = u[-1] + w[-1]
        rx = (u[lp.sl_x] + w[lp.sl_x]) - atau * self.c
        rs = u[lp.sl_s] + w[lp.sl_s]
        ry = (u[lp.sl_y] + w[lp.sl_y]) + atau * self.b
        rv = u[lp.sl_v] + w[lp.sl_v]
        ua, ub, uy, uv = yield from self.inner(rx, rs, ry, rv)
        cpart = float(self.c[self.own_idx] @ ua[self.own_idx])
        cua = yield from _reduce(np.array([cpart]))
        zu = float(cua[0] - self.b @ uy)
        shift = zu / self.zeta_scale
        mx, ms, my, mv = self.mz
        uh = np.empty(lp.total)
        uh[lp.sl_x] = ua - shift * mx
        uh[lp.sl_s] = ub - shift * ms
        uh[lp.sl_y] = uy - shift * my
        uh[lp.sl_v] = uv - shift * mv
        uh[-1] = atau + (zu - shift * self.zmz)
        if a != 1.0:
            uh = a * uh + (1.0 - a) * u
        arg = uh - w
        s = arg[lp.sl_s]
        for d, idx in self.groups:
            if d == 1:
                s[idx] = np.maximum(s[idx], 0.0)
            else:
                s[idx] = project_psd_batch(s[idx].reshape(-1, d, d)).reshape(-1, d * d)
        arg[-1] = arg[-1] if arg[-1] > 0.0 else 0.0
        w_new = (w - uh) + arg
        self.u, self.w = arg, w_new

    # -- residual check (solver.py:398-429) ----------------------------------------------------
    def residuals(self):
        lp, sh = self.lp, self.sh
        u = self.u
        tau = u[-1]
        xt, st, yt, vt = u[lp.sl_x] / tau, u[lp.sl_s] / tau, u[lp.sl_y] / tau, u[lp.sl_v] / tau
        ax = yield from _reduce(self.A_own @ xt[self.own_idx])
        hx = xt[lp.slot_cov] - st
        cons = yield from _reduce(np.array([hx @ hx, st @ st]))
        hv = yield from self._sep_exchange(self.scatter(vt))
        dr = (self.AT @ yt + hv) - self.c
        dr2 = yield from _reduce(np.array([dr[self.own_idx] @ dr[self.own_idx],
                                           self.c[self.own_idx] @ xt[self.own_idx]]))
        nb = np.linalg.norm(self.b)
        nc2 = yield from _reduce(np.array([self.c[self.own_idx] @ self.c[self.own_idx]]))
        pres = max(np.linalg.norm(ax - self.b) / (1 + nb),
                   np.sqrt(cons[0]) / (1 + np.sqrt(cons[1])))
        dres = np.sqrt(dr2[0]) / (1 + np.sqrt(nc2[0]))
        ctx, bty = dr2[1], self.b @ yt
        gap = abs(ctx - bty) / (1 + abs(ctx) + abs(bty))
        return float(pres), float(dres), float(gap)


def rank_program(run: ShardRun, iters: int, check_every: int = 20):
    """Generator of one rank: setup, `iters` iterations, residual checks."""
    yield from run.setup()
    log = []
    for k in range(1, iters + 1):
        yield from run.iterate()
        if k % check_every == 0 and run.u[-1] > 1e-9:
            res = yield from run.residuals()
            log.append((k,) + res)
    return log


def drive_in_process(gens):
    """Run rank generators in lockstep; reductions sum in rank order."""
    results = [None] * len(gens)
    pending = [next(g) for g in gens]
    while True:
        arrays = [p[1] for p in pending]
        total = arrays[0].copy()
        for a in arrays[1:]:
            total = total + a
        nxt = []
        done = 0
        for i, g in enumerate(gens):
            try:
                nxt.append(g.send(total.copy()))
            except StopIteration as stop:
                results[i] = stop.value
                nxt.append(None)
                done += 1
        if done == len(gens):
            return results
        if done:
            raise RuntimeError("ranks disagree on the number of reductions")
        pending = nxt


def drive_torch_dist(gen):
    """Run one rank generator with torch.distributed all_reduce (any backend)."""
    import torch
    import torch.distributed as dist

    try:
        req = next(gen)
        while True:
            t = torch.from_numpy(np.ascontiguousarray(req[1], dtype=np.float64))
            dist.all_reduce(t)
            req = gen.send(t.numpy().copy())
    except StopIteration as stop:
        return stop.value
