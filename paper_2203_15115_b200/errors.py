"""Exception hierarchy of the voxel topology-optimization hot path.

Mirrors the reference's error types (``topovox/errors.py:1-66``) so callers
that catch ``NoConvergence`` / ``SingularSystem`` / ``DimensionMismatch`` keep
working. The C-ABI returns integer status codes; ``raise_for_status`` maps
them onto these classes (see ``include/topovox_b200.h``).
"""

from __future__ import annotations


class TopovoxError(Exception):
    """Root of every error raised by this package."""


class BadDimension(TopovoxError):
    """Grid with a non-positive element count or edge length."""


class EmptyDomain(TopovoxError):
    """The design mask selects no element."""


class EmptyLoadRegion(TopovoxError):
    """A load selector matched no node."""


class DimensionMismatch(TopovoxError):
    """A vector does not have the operator's DOF (or element) count."""


class NoConvergence(TopovoxError):
    """Iterative solve stopped at its iteration cap.

    ``residual`` is the last relative residual, ``iterations`` the cap.
    ``u`` (an addition to the reference's exception, None unless the solver
    set it) is the iterate after the last iteration -- what a fixed-iteration
    parity check compares.
    """

    def __init__(self, message, residual=None, iterations=None, u=None):
        super().__init__(message)
        self.residual = residual
        self.iterations = iterations
        self.u = u


class SingularSystem(TopovoxError):
    """Loaded free DOF whose stiffness diagonal is zero."""


class MissingAnalysis(TopovoxError):
    """A constraint refers to an analysis that was not evaluated."""


class AllWeightsZero(TopovoxError):
    """Every augmented-Lagrangian weight is zero (SPEC combine fallback)."""


class SemanticError(TopovoxError):
    """Well-formed but meaningless input (e.g. a selector id out of range)."""


class ConfigRejected(SemanticError):
    """Constraint set-up that would stop the optimizer at its first step."""


class NoPositiveFactor(TopovoxError):
    """Buckling: no positive load factor below the search cap (structure in
    pure tension). solve_buckling reports it as the P = +inf
    sentinel instead of raising; the class names the outcome."""


class ZeroMassSubspace(UserWarning):
    """Modal analysis: free DOFs with zero lumped mass; they
    are reported and excluded from the eigen subspace."""


class CudaError(TopovoxError):
    """The CUDA runtime reported an error inside the native library."""


# C-ABI status codes (keep in sync with include/topovox_b200.h).
STATUS_OK = 0
STATUS_BAD_DIMS = 1
STATUS_CUDA = 2
STATUS_NOT_SPD = 3
STATUS_NO_CONVERGENCE = 4
STATUS_SINGULAR = 5
STATUS_BAD_ARG = 6
STATUS_WORKSPACE = 7


def raise_for_status(code: int, what: str, detail: str = "") -> None:
    """Translate a nonzero native status into the matching exception."""
    if code == STATUS_OK:
        return
    msg = f"{what}: {detail}" if detail else what
    if code == STATUS_BAD_DIMS:
        raise DimensionMismatch(msg)
    if code == STATUS_SINGULAR:
        raise SingularSystem(msg)
    if code == STATUS_NO_CONVERGENCE:
        raise NoConvergence(msg)
    if code == STATUS_CUDA:
        raise CudaError(msg)
    if code in (STATUS_BAD_ARG, STATUS_WORKSPACE):
        raise ValueError(msg)
    raise TopovoxError(f"{msg} (native status {code})")
