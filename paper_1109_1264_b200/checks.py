"""Scalar loop references and access counting, as the reference exports them
(lanevec/oracle.py:1-70, __init__.py:43-46) — for callers whose own tests
check results against `lanevec.oracle_dot(...)` and friends.

These are naive left-to-right Python loops over any indexable sequence, in
the element type of the inputs (pass NumPy scalars of the target type for
exact comparisons).  They are NOT used by the GPU path and do not import
the repository's oracle/ test infrastructure; they exist so that code
written against the reference's public surface keeps working.
"""

from .counting import CountingVector

__all__ = ["CountingVector", "oracle_dot", "oracle_sum", "oracle_scal", "oracle_axpy",
           "oracle_scaled_copy", "kahan_sum"]


def _same_length(x, y):
    if len(x) != len(y):
        raise ValueError(f"length mismatch: {len(x)} vs {len(y)}")


def oracle_dot(x, y):
    """sum_i x[i] * y[i], accumulated left to right from integer 0."""
    _same_length(x, y)
    total = 0
    for k in range(len(x)):
        total = total + x[k] * y[k]
    return total


def oracle_sum(x):
    total = 0
    for k in range(len(x)):
        total = total + x[k]
    return total


def oracle_scal(alpha, x) -> list:
    return [alpha * x[k] for k in range(len(x))]


def oracle_scaled_copy(alpha, x) -> list:
    return [alpha * x[k] for k in range(len(x))]


def oracle_axpy(alpha, x, y) -> list:
    """[y[i] + alpha * x[i]] (the sum's left operand is y, as in the reference)."""
    _same_length(x, y)
    return [y[k] + alpha * x[k] for k in range(len(x))]


def kahan_sum(values):
    """Neumaier-compensated left-to-right sum in the inputs' element type."""
    s = 0
    c = 0
    for v in values:
        t = s + v
        # the compensation takes the low part of whichever operand is smaller
        c = c + (((s - t) + v) if abs(s) >= abs(v) else ((v - t) + s))
        s = t
    return s + c
