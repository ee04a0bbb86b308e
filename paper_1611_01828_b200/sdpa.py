"""SDPA sparse-format reader.

Same entry point, result fields and errors as the reference's
``parse_sdpa`` (chordalsdp/sdpa.py:94-234); the text scan runs in C++ in
``libhsde.so`` (``hsde_sdpa_*``, csrc/hsde_sdpa.cpp) and returns flat entry
arrays, so a 10^6-entry file never materialises per-entry Python tuples.
``SdpProblem.C`` / ``.A`` (per-block ``SymMatrix`` objects, upper triangle,
0-based, sorted by (i, j)) are built lazily for code that wants the
reference's object view; :func:`paper_1611_01828_b200.decompose` reads the
flat arrays directly (``entry_table``).

Matrices are stored verbatim in the file's convention: ``C`` holds F0,
``A[i]`` holds F(i+1) (sdpa.py:1-20); explicit zeros are kept (structural).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from functools import cached_property
from pathlib import Path
from typing import IO

import numpy as np

from . import _lib

__all__ = ["DuplicateEntry", "ParseError", "SdpProblem", "SymMatrix", "parse_sdpa"]


class ParseError(ValueError):
    """Malformed SDPA input; carries the 1-based line number (sdpa.py:44-50)."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


class DuplicateEntry(ParseError):
    """The same (matno, blkno, i, j) coordinate appeared twice (sdpa.py:53-54)."""


@dataclass(frozen=True)
class SymMatrix:
    """Upper-triangle coordinates of a symmetric block (mirror of
    chordalsdp/symmat.py:25-50: ``dim``, ``entries`` = ((i, j, v), ...))."""

    dim: int
    entries: tuple

    def get(self, i: int, j: int) -> float:
        if i > j:
            i, j = j, i
        for a, b, v in self.entries:
            if a == i and b == j:
                return v
        return 0.0

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.dim, self.dim))
        for i, j, v in self.entries:
            out[i, j] = v
            out[j, i] = v
        return out


@dataclass(frozen=True, eq=False)
class SdpProblem:
    """Parsed SDPA problem (mirror of sdpa.py:57-91).

    ``block_dims`` keeps the signed sizes (negative = diagonal block).
    ``entry_table`` = (mat, blk, i, j, val): matrix number (0 = F0), 0-based
    block, 0-based i <= j within the block, value; sorted by (mat, blk, i, j).
    """

    m: int
    block_dims: tuple
    b: np.ndarray
    entry_table: tuple = field(repr=False)

    @property
    def block_sizes(self) -> tuple:
        return tuple(abs(d) for d in self.block_dims)

    @property
    def block_offsets(self) -> tuple:
        offs = [0]
        for d in self.block_sizes:
            offs.append(offs[-1] + d)
        return tuple(offs)

    @property
    def n_total(self) -> int:
        return sum(self.block_sizes)

    def entry_count(self) -> int:
        return int(self.entry_table[4].size)

    @cached_property
    def _blocks(self):
        mat, blk, ii, jj, vv = self.entry_table
        nb = len(self.block_dims)
        key = mat.astype(np.int64) * nb + blk
        bounds = np.searchsorted(key, np.arange((self.m + 1) * nb + 1))
        sizes = self.block_sizes
        ii_l, jj_l, vv_l = ii.tolist(), jj.tolist(), vv.tolist()

        def block(mid, b):
            k = mid * nb + b
            lo, hi = int(bounds[k]), int(bounds[k + 1])
            return SymMatrix(sizes[b], tuple(zip(ii_l[lo:hi], jj_l[lo:hi], vv_l[lo:hi])))

        return tuple(tuple(block(mid, b) for b in range(nb)) for mid in range(self.m + 1))

    @property
    def C(self) -> tuple:
        return self._blocks[0]

    @property
    def A(self) -> tuple:
        return self._blocks[1:]


def _text(source) -> bytes:
    if isinstance(source, Path):
        text = source.read_text()
    elif isinstance(source, bytes):
        text = source.decode()
    elif isinstance(source, str):
        text = source
    else:
        raw = source.read()
        text = raw.decode() if isinstance(raw, bytes) else raw
    return text.encode()


def parse_sdpa(source: "str | bytes | Path | IO") -> SdpProblem:
    """Parse SDPA sparse format from text, bytes, a path, or an open stream
    (sdpa.py:94-234).  Raises :class:`ParseError` (with ``.line``) or
    :class:`DuplicateEntry` exactly where the reference does."""
    lib = _lib.load()
    data = _text(source)
    h = C.c_void_p()
    rc = lib.hsde_sdpa_parse(data, len(data), C.byref(h))
    if rc != 0:
        line, dup = C.c_int64(), C.c_int32()
        msg = lib.hsde_sdpa_error(C.byref(line), C.byref(dup)).decode()
        raise (DuplicateEntry if dup.value else ParseError)(int(line.value), msg)
    try:
        m, nb, ne = C.c_int32(), C.c_int32(), C.c_int64()
        lib.hsde_sdpa_sizes(h, C.byref(m), C.byref(nb), C.byref(ne))
        dims = np.empty(nb.value, np.int32)
        b = np.empty(m.value, np.float64)
        cols = [np.empty(ne.value, np.int32) for _ in range(4)]
        val = np.empty(ne.value, np.float64)
        i32 = C.POINTER(C.c_int32)
        f64 = C.POINTER(C.c_double)
        lib.hsde_sdpa_data(h, dims.ctypes.data_as(i32), b.ctypes.data_as(f64),
                           *(c.ctypes.data_as(i32) for c in cols), val.ctypes.data_as(f64))
    finally:
        lib.hsde_sdpa_destroy(h)
    return SdpProblem(m=int(m.value), block_dims=tuple(int(d) for d in dims), b=b,
                      entry_table=(cols[0], cols[1], cols[2], cols[3], val))
