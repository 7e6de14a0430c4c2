"""Exact error columns for the benchmark report (the semantics of the
reference's verify::max_rel_err / digit_loss, verify.cpp:21-39, over its
exact dyadic oracle, oracle.cpp:163-193).

The reference's oracle needs Boost cpp_int; binary64 components are exact
dyadic rationals, so Python's Fraction is an exact stand-in.  Used only for
the max_rel_err / digits_lost CSV columns at small n (n <= --oracle-max),
never on the compute path.
"""
from __future__ import annotations

import math
from fractions import Fraction


def _value(components) -> Fraction:
    s = Fraction(0)
    for v in components:
        s += Fraction(float(v))
    return s


def rel_err(approx, exact: Fraction) -> float:
    """o_rel_err: |approx - exact| / |exact|, rounded once (oracle.cpp:163-174)."""
    a = _value(approx)
    if exact == 0:
        if a == 0:
            return 0.0
        raise ZeroDivisionError("relative error against exact zero is undefined; compare absolutely")
    d = a - exact
    return 0.0 if d == 0 else float(abs(d) / abs(exact))


def exact_matmul(A, B, K: int, n: int):
    """o_matmul (oracle.cpp:176-193) over (W, rows, ld) plane arrays."""
    m = A.shape[1]
    a = [[_value(A[:, i, k]) for k in range(K)] for i in range(m)]
    b = [[_value(B[:, k, j]) for j in range(n)] for k in range(K)]
    return [[sum((a[i][k] * b[k][j] for k in range(K)), Fraction(0)) for j in range(n)] for i in range(m)]


def max_rel_err(C, exact, cols: int) -> float:
    """verify::max_rel_err (verify.cpp:21-31)."""
    worst = 0.0
    for i, row in enumerate(exact):
        for j in range(cols):
            worst = max(worst, rel_err(C[:, i, j], row[j]))
    return worst


def digit_loss(worst: float, eps: float) -> float:
    """verify::digit_loss (verify.cpp:33-39)."""
    if worst == 0.0:
        return 0.0
    return max(0.0, math.log10(worst) - math.log10(eps))
