"""Exception classes of the reference API and the status-code -> exception mapping.

Classes mirror gradfem: InvertedElementError (elements.py:34-35), InvertedDeformationError
(materials.py:19-24), KernelEvaluationError (autodiff.py:27-32), ConflictingConstraintError
(assembly.py:32-33), LinearSolverError / BreakdownError / NonConvergenceError
(solvers.py:22-37).  UnsupportedKernelError is new: a problem the device path cannot
evaluate (user flux/source overrides, foreign materials) fails before any device work.
"""

from __future__ import annotations

from . import _lib
from .elements import InvertedElementError
from .materials import InvertedDeformationError


class KernelEvaluationError(RuntimeError):
    """Non-finite intermediate produced by a kernel evaluation."""

    def __init__(self, message, bad_mask=None):
        super().__init__(message)
        self.bad_mask = bad_mask


class ConflictingConstraintError(ValueError):
    """Two Dirichlet specs prescribe different values on one DOF."""


class LinearSolverError(RuntimeError):
    def __init__(self, message, iterations=None, residual=None):
        super().__init__(message)
        self.iterations = iterations
        self.residual = residual


class BreakdownError(LinearSolverError):
    pass


class NonConvergenceError(RuntimeError):
    def __init__(self, message, residual_norms=None, step=None):
        super().__init__(message)
        self.residual_norms = residual_norms or []
        self.step = step


class UnsupportedKernelError(NotImplementedError):
    """The problem uses a flux/source map the sm_100a kernels do not implement."""


def raise_for(status: int, err: "_lib.Error | None" = None, where: str = ""):
    """Map a libb200fem status to the reference exception class (no-op on OK)."""
    if status == _lib.OK:
        return
    msg = err.message if err is not None and err.msg else f"{where}: status {status}"
    if status == _lib.E_INVERTED_ELEMENT:
        raise InvertedElementError(msg)
    if status == _lib.E_INVERTED_DEFORMATION:
        raise InvertedDeformationError(msg)
    if status in (_lib.E_NONFINITE_VALUE, _lib.E_NONFINITE_DERIV):
        raise KernelEvaluationError(msg)
    if status == _lib.E_BREAKDOWN:
        raise BreakdownError(msg, iterations=int(err.iterations), residual=float(err.value))
    if status == _lib.E_LINEAR_SOLVER:
        raise LinearSolverError(msg, iterations=int(err.iterations), residual=float(err.value))
    if status == _lib.E_ZERO_DIAGONAL:
        raise LinearSolverError(msg)
    if status == _lib.E_UNSUPPORTED:
        raise UnsupportedKernelError(msg)
    if status == _lib.E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"libb200fem failure ({where}): {msg}")
