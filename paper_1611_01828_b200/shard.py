"""Clique sharding of the HSDE hot path across GPUs.

The cone step is independent per clique, so cliques are cut, in the
reference's clique order (graphs.py:217-220), into G contiguous ranges of
balanced load (sum of d^3 for the eigensolve plus d^2 for the streaming
work).  Every covered coordinate l gets exactly one *owner* rank (the rank of
the first clique covering it; coordinates no clique covers go round-robin),
which alone contributes l to the sums over columns (A t, c.ua, norms).  A rank
keeps every coordinate its cliques touch; coordinates touched by cliques of
more than one rank are *separators* (the arrow head of a block-arrow
pattern, the overlaps of a band at the cuts) and are replicated on every
touching rank.

Per iteration the shards then exchange (all-reduce, sum):
  1. the partial pull-scatter 0.5 H'(rho_s - rho_v) + H' rho_v of the separator
     coordinates (|S| doubles, S the global separator list);
  2. the partial A t over owned columns (m doubles);
  3. the partial c.ua over owned coordinates (1 double).
The m x m Schur solve, the rank-one correction, tau/kappa and y are
replicated.  Everything else is shard-local.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .problem import CompressedProblem


@dataclass(eq=False)
class Shard:
    rank: int
    world: int
    clique_ids: np.ndarray      # global clique indices of this shard (contiguous)
    covered: np.ndarray         # global covered positions kept locally (ascending)
    owned: np.ndarray           # bool per local covered coordinate
    slot_global: np.ndarray     # global slot index of each local slot (ascending)
    sep_local: np.ndarray       # local covered index of each separator coordinate touched
    sep_pos: np.ndarray         # its position in the global separator list
    n_sep: int                  # |S|
    D: np.ndarray               # GLOBAL cover counts of the local covered coordinates
    problem: CompressedProblem  # local sub-problem (local covered layout / cliques)


def partition_cliques(sizes: np.ndarray, world: int) -> list[np.ndarray]:
    """Contiguous clique ranges of balanced weight d^3 + 8 d^2."""
    sizes = np.asarray(sizes, dtype=np.float64)
    w = sizes ** 3 + 8.0 * sizes ** 2
    cum = np.cumsum(w)
    total = cum[-1] if len(cum) else 0.0
    cuts = [0]
    for g in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * g / world, side="left")) + 1)
    cuts.append(len(sizes))
    cuts = np.maximum.accumulate(np.minimum(np.array(cuts), len(sizes)))
    return [np.arange(cuts[g], cuts[g + 1]) for g in range(world)]


def make_shards(cp: CompressedProblem, world: int) -> list[Shard]:
    """Partition `cp` into `world` shards (host-side, once per problem)."""
    p = cp.p
    ranges = partition_cliques(cp.sizes, world)
    clique_rank = np.empty(p, dtype=np.int64)
    for g, r in enumerate(ranges):
        clique_rank[r] = g
    # slot -> clique
    slot_clique = np.repeat(np.arange(p), cp.sizes * cp.sizes)
    slot_rank = clique_rank[slot_clique]
    # owner of each covered coordinate: rank of the first covering clique
    owner = np.full(cp.N_c, -1, dtype=np.int64)
    order = np.argsort(cp.slot_cov, kind="stable")           # ascending slot per coordinate
    first = np.ones(len(order), dtype=bool)
    sc = cp.slot_cov[order]
    first[1:] = sc[1:] != sc[:-1]
    owner[sc[first]] = slot_rank[order[first]]
    unc = np.flatnonzero(owner < 0)
    owner[unc] = unc % world
    # touch matrix: which ranks touch each coordinate via slots
    touch = sp.csr_matrix((np.ones(cp.n_d), (cp.slot_cov, slot_rank)), shape=(cp.N_c, world))
    touch.data[:] = 1.0
    touch.sum_duplicates()
    ntouch = np.asarray((touch > 0).sum(axis=1)).ravel()
    sep_global = np.flatnonzero(ntouch > 1)
    D = cp.D
    A_csc = cp.A.tocsc()
    shards = []
    for g in range(world):
        cids = ranges[g]
        slots = np.flatnonzero(slot_rank == g)
        touched = np.unique(cp.slot_cov[slots]) if slots.size else np.zeros(0, np.int64)
        loc = np.union1d(touched, np.flatnonzero(owner == g)).astype(np.int64)
        owned = owner[loc] == g
        pos_in_loc = np.full(cp.N_c, -1, dtype=np.int64)
        pos_in_loc[loc] = np.arange(loc.size)
        sep_mask = np.isin(sep_global, touched)
        sep_pos = np.flatnonzero(sep_mask)
        sep_local = pos_in_loc[sep_global[sep_mask]]
        # local sub-problem
        A_loc = A_csc[:, loc].tocsr()
        A_loc.sort_indices()
        cl = tuple(cp.cliques[k] for k in cids)
        sizes = cp.sizes[cids]
        offsets = np.zeros(len(cids) + 1, dtype=np.int64)
        np.cumsum(sizes * sizes, out=offsets[1:])
        slot_cov_loc = pos_in_loc[cp.slot_cov[slots]].astype(np.int32)
        sub = CompressedProblem(
            n=cp.n, m=cp.m, covered=cp.covered[loc], c=cp.c[loc].copy(), A=A_loc,
            b=cp.b.copy(), cliques=cl, sizes=sizes, offsets=offsets, slot_cov=slot_cov_loc,
            block_dims=cp.block_dims, objective_sign=cp.objective_sign,
            aggregate_edges=None, name=f"{cp.name}[{g}/{world}]")
        shards.append(Shard(rank=g, world=world, clique_ids=cids, covered=loc, owned=owned,
                            slot_global=slots, sep_local=sep_local.astype(np.int32),
                            sep_pos=sep_pos.astype(np.int32), n_sep=int(sep_global.size),
                            D=D[loc].copy(), problem=sub))
    return shards


def scatter_state(cp: CompressedProblem, shards: list[Shard], u: np.ndarray):
    """Global compressed vector -> per-shard local vectors."""
    out = []
    for sh in shards:
        lp = sh.problem
        v = np.empty(lp.total)
        v[lp.sl_x] = u[cp.sl_x][sh.covered]
        v[lp.sl_s] = u[cp.sl_s][sh.slot_global]
        v[lp.sl_y] = u[cp.sl_y]
        v[lp.sl_v] = u[cp.sl_v][sh.slot_global]
        v[-1] = u[-1]
        out.append(v)
    return out


def gather_state(cp: CompressedProblem, shards: list[Shard], parts: list[np.ndarray]) -> np.ndarray:
    """Per-shard local vectors -> global compressed vector (owned x, local slots)."""
    u = np.zeros(cp.total)
    for sh, v in zip(shards, parts):
        lp = sh.problem
        u[cp.sl_x][sh.covered[sh.owned]] = v[lp.sl_x][sh.owned]
        u[cp.sl_s][sh.slot_global] = v[lp.sl_s]
        u[cp.sl_v][sh.slot_global] = v[lp.sl_v]
    u[cp.sl_y] = parts[0][shards[0].problem.sl_y]
    u[-1] = parts[0][-1]
    return u
