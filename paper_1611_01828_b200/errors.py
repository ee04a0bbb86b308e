"""Exception types of the reference API (same names, same meaning).

* ``FactorizationFailure`` -- chordalsdp/solver.py:60-61
* ``TauZero``              -- chordalsdp/solver.py:64-65
* ``EigenFailure``         -- chordalsdp/symmat.py:21-22
"""


class FactorizationFailure(RuntimeError):
    """The m x m system could not be factorized (rank-deficient or ill-scaled data)."""


class TauZero(RuntimeError):
    """Raised by :func:`residuals` when the scaling variable tau is numerically zero."""


class EigenFailure(RuntimeError):
    """Raised when the symmetric eigensolver does not converge / is non-finite."""
