"""Exact dyadic-rational oracle (TEST INFRASTRUCTURE ONLY).

Restates the semantics of the reference's Boost-based exact oracle
(/root/reference/proj/src/oracle.cpp, include/mpfkit/oracle.hpp) with Python
integers, which is enough for error-bound checks (Boost is absent here):

  from_double       oracle.cpp:83-91   value = sig * 2^exp, exact
  add / mul         oracle.cpp:97-117  exact
  o_round_to_binary64 / o_div_to_binary64  oracle.cpp:27-56, 133-161  RN-even
  o_rel_err         oracle.cpp:163-174 |approx - exact| / |exact| rounded once
  o_matmul          oracle.cpp:176-193 exact sum of exact products
  max_rel_err / digit_loss  verify.cpp:21-39

Values are (sig, exp) pairs with sig an int (canonical: odd or zero).
"""
from __future__ import annotations

import math
from fractions import Fraction


def from_double(v: float) -> Fraction:
    if not math.isfinite(v):
        raise ValueError("oracle: NaN/Inf has no dyadic value")
    return Fraction(v)  # exact for binary64


def from_components(c) -> Fraction:
    s = Fraction(0)
    for v in c:
        s += Fraction(float(v))
    return s


def round_to_binary64(x: Fraction) -> float:
    """RN-even rounding of an exact rational (oracle.cpp:27-56 semantics)."""
    if x == 0:
        return 0.0
    neg = x < 0
    x = -x if neg else x
    # float(Fraction) is correctly rounded (RN-even) in CPython
    r = float(x)
    return -r if neg else r


def rel_err(approx, exact: Fraction) -> float:
    """o_rel_err, oracle.cpp:163-174."""
    a = from_components(approx)
    if exact == 0:
        if a == 0:
            return 0.0
        raise ZeroDivisionError("oracle: relative error against exact zero is undefined")
    d = a - exact
    if d == 0:
        return 0.0
    return float(abs(d) / abs(exact))


def matmul_exact(A, B, K: int, n: int, rows=None):
    """o_matmul over plane arrays (W, m, lda), (W, K, ldb) -> list of rows of
    Fractions.  rows=(r0, r1) limits the rows computed."""
    W, m, _ = A.shape
    r0, r1 = (0, m) if rows is None else rows
    a = [[from_components(A[:, i, k]) for k in range(K)] for i in range(r0, r1)]
    b = [[from_components(B[:, k, j]) for j in range(n)] for k in range(K)]
    out = []
    for ai in a:
        out.append([sum((ai[k] * b[k][j] for k in range(K)), Fraction(0)) for j in range(n)])
    return out


def max_rel_err(Cm, exact, rows=None) -> float:
    """verify::max_rel_err, verify.cpp:21-31 (C as (W, m, ldc) planes)."""
    r0 = 0 if rows is None else rows[0]
    worst = 0.0
    for ii, row in enumerate(exact):
        i = r0 + ii
        for j, ex in enumerate(row):
            worst = max(worst, rel_err(Cm[:, i, j], ex))
    return worst


def digit_loss(worst: float, eps: float) -> float:
    """verify::digit_loss, verify.cpp:33-39."""
    if worst == 0.0:
        return 0.0
    return max(0.0, math.log10(worst) - math.log10(eps))
