"""Exception types of the reference API, same names, fields and messages.

CholeskyBreakdown / TriangularSingularError: reference kernels.py:25-47.
ShiftAttemptLimitError: reference algorithms.py:47-56.
"""

from __future__ import annotations


class CholeskyBreakdown(Exception):
    """Factorization hit a pivot that is not strictly positive (or NaN)."""

    def __init__(self, pivot_index, pivot_value):
        super().__init__(
            f"cholesky breakdown at pivot {pivot_index}: "
            f"schur diagonal {pivot_value:.6e} <= 0"
        )
        self.pivot_index = pivot_index
        self.pivot_value = pivot_value


class TriangularSingularError(Exception):
    """Triangular matrix cannot be inverted because a diagonal entry is zero."""

    def __init__(self, index):
        super().__init__(f"triangular matrix is singular: zero diagonal at index {index}")
        self.index = index


class ShiftAttemptLimitError(Exception):
    """Even the escalated shifted factorizations kept breaking down."""

    def __init__(self, attempts, last_shift):
        super().__init__(
            f"factorization still breaks down after {attempts} shifted "
            f"attempts (last shift {last_shift:.3e})"
        )
        self.attempts = attempts
        self.last_shift = last_shift
