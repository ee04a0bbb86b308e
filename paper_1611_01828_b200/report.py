"""Report schema of the reference (chordalsdp/sdpa.py:29-44, 237-319).

Same dataclasses, field names, status labels and JSON serialisation, so a
report produced here is interchangeable with the reference's.
"""

from __future__ import annotations

import json
from collections.abc import Sequence
from dataclasses import asdict, dataclass

import numpy as np

STATUS_OPTIMAL = "Optimal"
STATUS_PRIMAL_INFEASIBLE = "PrimalInfeasible"
STATUS_DUAL_INFEASIBLE = "DualInfeasible"
STATUS_MAX_ITERS = "MaxItersReached"
STATUSES = (STATUS_OPTIMAL, STATUS_PRIMAL_INFEASIBLE, STATUS_DUAL_INFEASIBLE, STATUS_MAX_ITERS)


@dataclass
class Residuals:
    primal: float
    dual: float
    gap: float

    def max(self) -> float:
        return max(self.primal, self.dual, self.gap)


@dataclass
class Timing:
    setup_s: float
    iterations_s: float
    total_s: float
    per_iteration_s: float


@dataclass
class ProblemStats:
    n: int
    m: int
    blocks: list
    p: int
    clique_max: int
    clique_min: int
    n_d: int


class PatternEntries(Sequence):
    """The ``[block, i, j, value]`` rows of a solution or certificate matrix on
    the aggregate pattern (sdpa.py:280-290), held as arrays.

    Behaves as the reference's list of rows (indexing, iteration, ``len``,
    equality with a list) and serialises to the same JSON; rows are built
    only when read, so a large solve does not pay for a million Python lists
    it may never look at."""

    __slots__ = ("block", "i", "j", "value")

    def __init__(self, block, i, j, value):
        self.block = np.asarray(block, dtype=np.int64)
        self.i = np.asarray(i, dtype=np.int64)
        self.j = np.asarray(j, dtype=np.int64)
        self.value = np.asarray(value, dtype=np.float64)

    def __len__(self):
        return int(self.value.size)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[q] for q in range(*k.indices(len(self)))]
        return [int(self.block[k]), int(self.i[k]), int(self.j[k]), float(self.value[k])]

    def __iter__(self):
        return iter(self.tolist())

    def tolist(self) -> list:
        return [list(r) for r in zip(self.block.tolist(), self.i.tolist(), self.j.tolist(),
                                     self.value.tolist())]

    def __eq__(self, other):
        if isinstance(other, PatternEntries):
            return (np.array_equal(self.block, other.block) and np.array_equal(self.i, other.i)
                    and np.array_equal(self.j, other.j)
                    and np.array_equal(self.value, other.value))
        if isinstance(other, (list, tuple)):
            return self.tolist() == [list(r) for r in other]
        return NotImplemented

    def __repr__(self):
        return f"PatternEntries({len(self)} rows)"

    def __deepcopy__(self, memo):
        return self  # immutable view; dataclasses.asdict deep-copies values


def _json_default(o):
    if isinstance(o, PatternEntries):
        return o.tolist()
    raise TypeError(f"{type(o).__name__} is not JSON serialisable")


@dataclass
class SolverReport:
    """Outcome of a solve (sdpa.py:266-294): statuses in the file convention."""

    status: str
    objective_primal: float | None
    objective_dual: float | None
    iterations: int
    residuals: Residuals | None
    timing: Timing
    problem: ProblemStats
    tol: float
    solution: dict | None = None
    certificate: dict | None = None

    def __post_init__(self):
        if self.status not in STATUSES:
            raise ValueError(f"unknown status {self.status!r}")
        if self.status == STATUS_OPTIMAL:
            if self.residuals is None or self.residuals.max() > self.tol:
                raise ValueError("Optimal status requires residuals within tolerance")


def emit_report(report: SolverReport) -> str:
    """Deterministic JSON (sorted keys, 2-space indent), as sdpa.py:297-299."""
    return json.dumps(asdict(report), sort_keys=True, indent=2, default=_json_default) + "\n"


def read_report(text: str | bytes) -> SolverReport:
    if isinstance(text, bytes):
        text = text.decode()
    raw = json.loads(text)
    res = Residuals(**raw["residuals"]) if raw["residuals"] is not None else None
    return SolverReport(
        status=raw["status"], objective_primal=raw["objective_primal"],
        objective_dual=raw["objective_dual"], iterations=raw["iterations"], residuals=res,
        timing=Timing(**raw["timing"]), problem=ProblemStats(**raw["problem"]), tol=raw["tol"],
        solution=raw["solution"], certificate=raw["certificate"])
