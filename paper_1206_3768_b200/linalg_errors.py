"""Typed errors of the dense kernels — same classes and meaning as the
reference (`spectral_chain/linalg.py:28-49`)."""

from __future__ import annotations

__all__ = [
    "NotHermitianError",
    "NotPositiveDefiniteError",
    "RankDeficientError",
    "EigenSolverError",
]


class NotHermitianError(ValueError):
    """Matrix fails the Hermitian symmetry check."""


class NotPositiveDefiniteError(ValueError):
    """Cholesky pivot is non-positive; the matrix is not a valid overlap."""


class RankDeficientError(ValueError):
    """Orthonormalization found (numerically) dependent columns; ``indices``
    holds the offending column positions."""

    def __init__(self, indices):
        self.indices = tuple(int(i) for i in indices)
        super().__init__(f"rank-deficient columns at {self.indices}")


class EigenSolverError(RuntimeError):
    """The dense eigensolver failed to converge (pathological input)."""
