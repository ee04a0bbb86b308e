"""Report schema of the reference (chordalsdp/sdpa.py:29-44, 237-319).

Same dataclasses, field names, status labels and JSON serialisation, so a
report produced here is interchangeable with the reference's.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass

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
    return json.dumps(asdict(report), sort_keys=True, indent=2) + "\n"


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
