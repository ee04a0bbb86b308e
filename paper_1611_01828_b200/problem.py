"""Problem data for the HSDE hot path.

Two representations live here:

* ``DecomposedProblem`` / ``CliqueDecomposition`` -- minimal mirrors of the
  reference's input types (``chordalsdp/decompose.py:40-79`` and
  ``chordalsdp/graphs.py:190-252``): x is a dense column-stacked length-n**2
  vector, ``A`` is CSR over n**2 columns, the clique selectors are
  ``gather_index`` (``graphs.py:184-187``).  ``solve_decomposed`` accepts these
  (or the reference's own objects -- duck typing, same field names).

* ``CompressedProblem`` -- the layout the device works in.  Only *covered*
  coordinates are kept: flat indices that some clique selects (``D > 0``) plus
  any column touched by ``A`` or ``c``.  Everything else evolves trivially
  (off-pattern entries stay exactly 0 from the zero
  start), so compression is exact.  Covered coordinates are kept in ascending
  flat order, which keeps the reference's CSR/CSC accumulation order
  (SURVEY.md Appendix B).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np
import scipy.sparse as sp

OBJECTIVE_SIGN = -1.0  # decompose.py:31


# ---------------------------------------------------------------------------
# mirrors of the reference input types


def selector_flat(clique: np.ndarray, n: int) -> np.ndarray:
    """Flat (column-stacked) indices a clique selector picks, local row-major.

    Local slot a*d + b <-> ambient flat C[a]*n + C[b] (graphs.py:184-187).
    """
    c = np.asarray(clique, dtype=np.int64)
    return (c[:, None] * n + c[None, :]).ravel()


@dataclass(frozen=True, eq=False)
class CliqueDecomposition:
    """Clique list plus stacked selector (mirror of graphs.py:190-252)."""

    n: int
    cliques: tuple
    sizes: np.ndarray
    offsets: np.ndarray
    n_d: int
    gather_index: np.ndarray
    extended_pattern: object = None
    _cover: list = field(default_factory=list, repr=False)

    @classmethod
    def build(cls, n: int, cliques: Iterable[Iterable[int]], extended_pattern=None):
        # Same canonical order as graphs.py:217-220: by (min, sorted tuple).
        ordered = sorted((sorted(int(v) for v in c) for c in cliques),
                         key=lambda c: (c[0], tuple(c)))
        cl = tuple(np.asarray(c, dtype=np.int64) for c in ordered)
        sizes = np.array([len(c) for c in cl], dtype=np.int64)
        offsets = np.zeros(len(cl) + 1, dtype=np.int64)
        np.cumsum(sizes * sizes, out=offsets[1:])
        gi = (np.concatenate([selector_flat(c, n) for c in cl])
              if cl else np.zeros(0, dtype=np.int64))
        return cls(n=n, cliques=cl, sizes=sizes, offsets=offsets,
                   n_d=int(offsets[-1]), gather_index=gi,
                   extended_pattern=extended_pattern)

    @property
    def p(self) -> int:
        return len(self.cliques)

    @property
    def cover_counts(self) -> np.ndarray:
        if not self._cover:
            self._cover.append(
                np.bincount(self.gather_index, minlength=self.n * self.n).astype(float))
        return self._cover[0]

    def gather(self, x: np.ndarray) -> np.ndarray:
        return x[self.gather_index]

    def scatter(self, s: np.ndarray) -> np.ndarray:
        return np.bincount(self.gather_index, weights=s, minlength=self.n * self.n)

    def block(self, s: np.ndarray, k: int) -> np.ndarray:
        return s[self.offsets[k]: self.offsets[k + 1]]


@dataclass(frozen=True, eq=False)
class DecomposedProblem:
    """Mirror of chordalsdp.decompose.DecomposedProblem (decompose.py:40-79)."""

    n: int
    m: int
    c: np.ndarray
    A: sp.csr_matrix
    b: np.ndarray
    dec: CliqueDecomposition
    aggregate: object = None
    block_dims: tuple = ()
    objective_sign: float = OBJECTIVE_SIGN

    @property
    def n_d(self) -> int:
        return self.dec.n_d

    @property
    def D(self) -> np.ndarray:
        return self.dec.cover_counts

    @property
    def p(self) -> int:
        return self.dec.p


# ---------------------------------------------------------------------------
# the compressed layout


@dataclass(eq=False)
class CompressedProblem:
    """Problem in the covered-coordinate layout the device iterates on.

    Stacked HSDE vector (compressed): ``[x N_c | s n_d | y m | v n_d | tau]``
    -- the reference layout of solver.py:119-137 with x restricted to the
    covered coordinates.
    """

    n: int
    m: int
    covered: np.ndarray          # int64[N_c] ascending flat indices (col*n+row)
    c: np.ndarray                # float64[N_c]
    A: sp.csr_matrix             # m x N_c, sorted indices, fp64
    b: np.ndarray                # float64[m]
    cliques: tuple               # sorted node arrays, reference clique order
    sizes: np.ndarray            # int64[p]
    offsets: np.ndarray          # int64[p+1]
    slot_cov: np.ndarray         # int32[n_d]: covered position of each clique slot
    block_dims: tuple = ()
    objective_sign: float = OBJECTIVE_SIGN
    aggregate_edges: np.ndarray | None = None  # (E, 2) i<j, report extraction only
    name: str = ""
    _cache: dict = field(default_factory=dict, repr=False)

    # -- sizes ---------------------------------------------------------------
    @property
    def N_c(self) -> int:
        return int(self.covered.shape[0])

    @property
    def n_d(self) -> int:
        return int(self.offsets[-1])

    @property
    def p(self) -> int:
        return len(self.cliques)

    @property
    def total(self) -> int:
        return self.N_c + 2 * self.n_d + self.m + 1

    @property
    def sl_x(self):
        return slice(0, self.N_c)

    @property
    def sl_s(self):
        return slice(self.N_c, self.N_c + self.n_d)

    @property
    def sl_y(self):
        return slice(self.N_c + self.n_d, self.N_c + self.n_d + self.m)

    @property
    def sl_v(self):
        return slice(self.N_c + self.n_d + self.m, self.total - 1)

    @property
    def idx_tau(self) -> int:
        return self.total - 1

    # -- derived data (cached) -------------------------------------------------
    @property
    def D(self) -> np.ndarray:
        """Cover counts on covered coordinates (graphs.py:228)."""
        if "D" not in self._cache:
            self._cache["D"] = np.bincount(self.slot_cov, minlength=self.N_c).astype(float)
        return self._cache["D"]

    @property
    def cover_ptr_slots(self) -> tuple[np.ndarray, np.ndarray]:
        """CSR of covered -> slots (ascending slot order: bincount's order)."""
        if "cover" not in self._cache:
            order = np.argsort(self.slot_cov, kind="stable").astype(np.int32)
            counts = np.bincount(self.slot_cov, minlength=self.N_c)
            ptr = np.zeros(self.N_c + 1, dtype=np.int64)
            np.cumsum(counts, out=ptr[1:])
            self._cache["cover"] = (ptr, order)
        return self._cache["cover"]

    @property
    def AT(self) -> sp.csr_matrix:
        """A transposed as CSR over covered rows == CSC of A (solver.py:262)."""
        if "AT" not in self._cache:
            at = self.A.T.tocsr()
            at.sort_indices()
            self._cache["AT"] = at
        return self._cache["AT"]

    def gather(self, x: np.ndarray) -> np.ndarray:
        return x[self.slot_cov]

    def scatter(self, s: np.ndarray) -> np.ndarray:
        return np.bincount(self.slot_cov, weights=s, minlength=self.N_c)

    def with_data(self, c: np.ndarray | None = None, b: np.ndarray | None = None):
        """Copy with replaced objective / right-hand side (shares structure)."""
        out = CompressedProblem(
            n=self.n, m=self.m, covered=self.covered,
            c=self.c if c is None else np.asarray(c, dtype=float),
            A=self.A, b=self.b if b is None else np.asarray(b, dtype=float),
            cliques=self.cliques, sizes=self.sizes, offsets=self.offsets,
            slot_cov=self.slot_cov, block_dims=self.block_dims,
            objective_sign=self.objective_sign,
            aggregate_edges=self.aggregate_edges, name=self.name)
        for k in ("D", "cover", "AT"):
            if k in self._cache:
                out._cache[k] = self._cache[k]
        return out

    # -- layout conversion -------------------------------------------------------
    def compress_vector(self, full: np.ndarray) -> np.ndarray:
        """Reference stacked vector (length n**2+2n_d+m+1) -> compressed."""
        n2 = self.n * self.n
        full = np.asarray(full, dtype=float)
        out = np.empty(self.total)
        out[: self.N_c] = full[self.covered]
        out[self.N_c:] = full[n2:]
        return out

    def expand_vector(self, comp: np.ndarray, off_pattern: np.ndarray | None = None) -> np.ndarray:
        """Compressed stacked vector -> reference layout; off-pattern x from
        ``off_pattern`` (a full-length vector) or zero."""
        n2 = self.n * self.n
        out = np.zeros(n2 + self.total - self.N_c)
        if off_pattern is not None:
            out[:n2] = off_pattern[:n2]
        out[self.covered] = comp[: self.N_c]
        out[n2:] = comp[self.N_c:]
        return out

    def expand_x(self, xc: np.ndarray) -> np.ndarray:
        out = np.zeros(self.n * self.n)
        out[self.covered] = xc
        return out


def edges_array(agg, n: int):
    """The aggregate pattern's (i, j) pairs (graphs.py:37: a frozenset of tuples) as a
    lexicographically sorted (E, 2) int64 array -- the order of ``sorted(agg.edges)``,
    without a Python-level sort of up to millions of tuples."""
    if agg is None or getattr(agg, "edges", None) is None:
        return None
    ed = agg.edges
    if isinstance(ed, np.ndarray):
        e = np.asarray(ed, dtype=np.int64).reshape(-1, 2)
    else:
        import itertools

        e = np.fromiter(itertools.chain.from_iterable(ed), dtype=np.int64, count=2 * len(ed)).reshape(-1, 2)
    if e.shape[0] > 1:
        code = e[:, 0] * max(int(n), int(e[:, 1].max(initial=0)) + 1) + e[:, 1]
        if not bool(np.all(code[1:] > code[:-1])):
            e = e[np.argsort(code, kind="stable")]
    return e


def compress(dp, full: bool = False, _numpy_only: bool = False, with_edges: bool = True) -> CompressedProblem:
    """Build the covered layout from a reference-style DecomposedProblem.

    ``dp`` may be the reference's own object or the mirror above.  Covered =
    clique-selected coordinates (D > 0) + A's column support + c's support.
    ``full=True`` keeps all n**2 coordinates (the unit-level API uses it for
    small problems so arbitrary reference-layout vectors run on the device).
    ``with_edges=False`` skips the aggregate pattern's edge list (the report's
    pattern index then takes it from ``dp`` itself, off the critical path).
    """
    n, m = int(dp.n), int(dp.m)
    n2 = n * n
    gi = np.asarray(dp.dec.gather_index, dtype=np.int64)
    A = dp.A if (sp.issparse(dp.A) and dp.A.format == "csr" and dp.A.dtype == np.float64) else sp.csr_matrix(dp.A, dtype=float)
    if not A.has_canonical_format:
        A = A.copy()
        A.sum_duplicates()
        A.sort_indices()
    c_full = np.asarray(dp.c, dtype=float)
    c_cov = None
    if full:
        covered = np.arange(n2, dtype=np.int64)
        pos, slot_cov = A.indices.astype(np.int64), gi.astype(np.int32)
    elif 0 < n2 and not _numpy_only:
        # bit mask over n^2 + popcount ranks in the library, on the host's threads
        # (config 4, n^2 = 2.6e8, nnz(A) = 3.8e7: 3.9 s with numpy sorts -> ~0.3 s)
        from . import _lib

        covered, c_cov, pos, slot_cov = _lib.cover_layout(n2, c_full, gi, A.indices)
    elif 0 < n2 < 2 ** 31:
        # numpy restatement (byte mask + int32 rank map): the check of the library path
        mark = c_full != 0.0
        mark[gi] = True
        mark[A.indices] = True
        covered = np.flatnonzero(mark)
        rank = np.cumsum(mark, dtype=np.int32)
        rank -= 1
        pos = rank[A.indices]
        slot_cov = rank[gi]
        del mark, rank
    else:
        parts = [gi, A.indices.astype(np.int64), np.flatnonzero(c_full)]
        covered = np.unique(np.concatenate(parts)) if n2 else np.zeros(0, np.int64)
        pos = np.searchsorted(covered, A.indices.astype(np.int64))
        slot_cov = np.searchsorted(covered, gi).astype(np.int32)
    # ranks are order-preserving: the compressed CSR is canonical as built (values
    # and row pointers shared with the input, which is never written)
    Ac = sp.csr_matrix((A.data, pos, A.indptr), shape=(m, covered.shape[0]), copy=False)
    Ac.has_sorted_indices = True
    Ac.has_canonical_format = True
    if c_cov is None:
        c_cov = c_full[covered].copy()
    cliques = tuple(np.asarray(c, dtype=np.int64) for c in dp.dec.cliques)
    sizes = np.asarray(dp.dec.sizes, dtype=np.int64)
    offsets = np.asarray(dp.dec.offsets, dtype=np.int64)
    edges = edges_array(getattr(dp, "aggregate", None), n) if with_edges else None
    return CompressedProblem(
        n=n, m=m, covered=covered, c=c_cov, A=Ac,
        b=np.asarray(dp.b, dtype=float).copy(), cliques=cliques, sizes=sizes,
        offsets=offsets, slot_cov=slot_cov,
        block_dims=tuple(getattr(dp, "block_dims", (n,))),
        objective_sign=float(getattr(dp, "objective_sign", OBJECTIVE_SIGN)),
        aggregate_edges=edges)


def expand_to_mirror(cp: CompressedProblem) -> DecomposedProblem:
    """Compressed problem -> reference-layout mirror (small problems only)."""
    n, n2 = cp.n, cp.n * cp.n
    c = np.zeros(n2)
    c[cp.covered] = cp.c
    A = sp.csr_matrix((cp.A.data, cp.covered[cp.A.indices], cp.A.indptr), shape=(cp.m, n2))
    A.sort_indices()
    dec = CliqueDecomposition.build(n, [list(c_) for c_ in cp.cliques])
    return DecomposedProblem(n=n, m=cp.m, c=c, A=A, b=cp.b.copy(), dec=dec,
                             aggregate=None, block_dims=cp.block_dims or (n,),
                             objective_sign=cp.objective_sign)


def size_groups(sizes: Sequence[int]) -> list[tuple[int, np.ndarray]]:
    """Cliques grouped by size, ascending (solver.py:139-152)."""
    sizes = np.asarray(sizes)
    return [(int(d), np.flatnonzero(sizes == d)) for d in np.unique(sizes)]
