"""B200-native (sm_100a, fp64) HSDE-ADMM hot path for chordally decomposed SDPs.

Drop-in for the solve path of the reference package ``chordalsdp``
(arXiv:1611.01828): the names below keep the reference's signatures
(chordalsdp/__init__.py:30-44 and solver.py), but every iteration runs in
hand-written CUDA kernels of ``libhsde.so`` (csrc/, C ABI in include/hsde.h).
"""

from .decompose import chordal_cliques, decompose
from .errors import EigenFailure, FactorizationFailure, TauZero
from .sdpa import DuplicateEntry, ParseError, SdpProblem, SymMatrix, parse_sdpa
from .problem import (CliqueDecomposition, CompressedProblem, DecomposedProblem, compress,
                      expand_to_mirror)
from .report import (STATUS_DUAL_INFEASIBLE, STATUS_MAX_ITERS, STATUS_OPTIMAL,
                     STATUS_PRIMAL_INFEASIBLE, PatternEntries, ProblemStats, Residuals,
                     SolverReport, Timing, emit_report, read_report)
from .solver import (HsdeState, IterationInfo, KktCache, QOperator, SolverSettings,
                     VariableLayout, affine_project, build_hsde, initial_state, iterate,
                     project_cone, recover, residuals, setup_cache, solve, solve_decomposed,
                     solve_inner)

__version__ = "0.1.0"

__all__ = [
    "CliqueDecomposition", "CompressedProblem", "DecomposedProblem", "EigenFailure",
    "chordal_cliques", "decompose", "DuplicateEntry", "ParseError", "SdpProblem", "SymMatrix",
    "parse_sdpa", "solve",
    "FactorizationFailure", "HsdeState", "IterationInfo", "KktCache", "ProblemStats",
    "PatternEntries", "QOperator", "Residuals", "STATUS_DUAL_INFEASIBLE", "STATUS_MAX_ITERS", "STATUS_OPTIMAL",
    "STATUS_PRIMAL_INFEASIBLE", "SolverReport", "SolverSettings", "TauZero", "Timing",
    "VariableLayout", "affine_project", "build_hsde", "compress", "emit_report",
    "expand_to_mirror", "initial_state", "iterate", "project_cone", "read_report", "recover",
    "residuals", "setup_cache", "solve_decomposed", "solve_inner",
]
