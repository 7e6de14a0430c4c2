"""MPFK_LEAN arithmetic (csrc/mpf_lean.cuh) compiled for the host
(tests/_build/libarith_host.so) against the exact dyadic oracle: the lean
multiply-accumulate chain of a GEMM element must stay within the north
star's normwise 4*k*u_p on the BASELINE distributions and on adversarial
inputs (positive growth, cancellation, wide range, sparse, continuation), its
renormalisations must not change the value, and its results must be
canonical normalised values.  It is NOT compared bitwise with the reference:
the lean form is the tolerance mode.  The reference-order chain with the
product's bit-exact arithmetic runs beside it as the accuracy yardstick."""
import ctypes as C
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from tests.helpers import special_matrix

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libarith_host.so")
pytestmark = pytest.mark.skipif(not os.path.exists(SO), reason="host arith shim not built")

U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}  # north star


@pytest.fixture(scope="module")
def H():
    L = C.CDLL(SO)
    L.hst_lean_dot_batch.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t,
                                     C.c_void_p, C.c_void_p]
    L.hst_ref_dot_batch.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hst_lean_renorm_batch.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_void_p, C.c_void_p]
    L.hst_lean_gemm.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                                C.c_size_t, C.c_void_p, C.c_size_t]
    return L


def frac(c):
    return sum((Fraction(float(v)) for v in c), Fraction(0))


def chains(H, W, a, b, every=16, init=None):
    """a, b: (count, k, W) -> lean results, reference-order results, exact sums"""
    count, k, _ = a.shape
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    lean, ref = np.zeros((count, W)), np.zeros((count, W))
    ip = None if init is None else np.ascontiguousarray(init).ctypes.data
    assert H.hst_lean_dot_batch(W, count, k, a.ctypes.data, b.ctypes.data, every, ip, lean.ctypes.data) == 0
    assert H.hst_ref_dot_batch(W, count, k, a.ctypes.data, b.ctypes.data, ref.ctypes.data) == 0
    exact = []
    for c in range(count):
        e = Fraction(0) if init is None else frac(init[c])
        for i in range(k):
            e += frac(a[c, i]) * frac(b[c, i])
        exact.append(e)
    return lean, ref, exact


def normwise(got, exact):
    den = max(abs(e) for e in exact)
    return float(max(abs(frac(g) - e) for g, e in zip(got, exact)) / den)


def is_canonical(v):
    """each component at most half an ulp of the one before; zeros last"""
    seen_zero = False
    for w in range(len(v)):
        if v[w] == 0:
            seen_zero = True
            continue
        if seen_zero:
            return False
        if w and abs(v[w]) > np.spacing(abs(v[w - 1])) / 2:
            return False
    return True


def baseline_pairs(W, count, k, seed, wide):
    A = O.orc_fill_baseline(W, count, k, seed, wide=wide)[:, :, :k]
    B = O.orc_fill_baseline(W, count, k, seed + 1, wide=wide)[:, :, :k]
    return A.transpose(1, 2, 0).copy(), B.transpose(1, 2, 0).copy()


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("wide", [False, True])
def test_lean_chain_within_tolerance_baseline(H, W, wide):
    k = 1500
    a, b = baseline_pairs(W, 16, k, 40 + W, wide)
    lean, ref, exact = chains(H, W, a, b)
    tol = 4 * k * U_P[W]
    e_lean, e_ref = normwise(lean, exact), normwise(ref, exact)
    assert e_ref <= tol
    assert e_lean <= 0.02 * tol, (e_lean / tol, e_ref / tol)  # measured 2e-4 .. 4e-3 of the tolerance
    assert all(is_canonical(v) for v in lean)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_chain_positive_inputs_componentwise(H, W):
    """no cancellation: the error is also small relative to every element
    (test_linalg.cpp:250-268's criterion, n*4*eps against the oracle)"""
    k = 1200
    a, b = baseline_pairs(W, 12, k, 70 + W, False)
    # positive values: flip every operand whose leading component is negative
    a = a * np.sign(a[:, :, :1])
    b = b * np.sign(b[:, :, :1])
    lean, ref, exact = chains(H, W, a, b)
    tol = 4 * k * U_P[W]
    worst = max(float(abs(frac(g) - e) / abs(e)) for g, e in zip(lean, exact))
    assert worst <= 0.02 * tol, worst / tol
    assert all(is_canonical(v) for v in lean)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_chain_cancellation_and_sparse(H, W):
    """chains whose partial sums cancel to (near) zero and come back, zeros
    and signed zeros in the operands, single-component values"""
    k = 640
    a, b = baseline_pairs(W, 8, k, 90 + W, True)
    # second half cancels the first exactly, then a last small term
    a[:4, k // 2:k - 1] = a[:4, :k // 2 - 1]
    b[:4, k // 2:k - 1] = -b[:4, :k // 2 - 1]
    # sparse: zero out most operands of two chains, signed zeros included
    a[4:6, ::3] = 0.0
    a[4:6, 1::3] = -0.0
    # single-component values
    b[6:, :, 1:] = 0.0
    lean, ref, exact = chains(H, W, a, b)
    # the error is relative to the largest partial sum of the chain (as for
    # any floating accumulation), which the first half reaches
    scale = []
    for c in range(8):
        s, mx = Fraction(0), Fraction(0)
        for i in range(k):
            s += frac(a[c, i]) * frac(b[c, i])
            mx = max(mx, abs(s))
        scale.append(mx)
    tol = 4 * k * U_P[W]
    for c in range(8):
        if scale[c] == 0:
            assert frac(lean[c]) == 0
            continue
        err = float(abs(frac(lean[c]) - exact[c]) / scale[c])
        assert err <= 0.02 * tol, (c, err / tol)
        assert is_canonical(lean[c]), lean[c]


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_chain_special_values(H, W):
    """zeros, integers, powers of two, non-normalised operands (what drives
    the reference's renorm5 paths B/C/D): exact or within tolerance"""
    k = 200
    A = special_matrix(W, 10, k, 300 + W)[:, :, :k]
    B = special_matrix(W, 10, k, 400 + W)[:, :, :k]
    a, b = A.transpose(1, 2, 0).copy(), B.transpose(1, 2, 0).copy()
    lean, ref, exact = chains(H, W, a, b)
    tol = 4 * k * U_P[W]
    for c in range(10):
        s, mx = Fraction(0), Fraction(0)
        for i in range(k):
            s += abs(frac(a[c, i]) * frac(b[c, i]))
        if s == 0:
            assert frac(lean[c]) == 0
            continue
        assert float(abs(frac(lean[c]) - exact[c]) / s) <= tol
        assert is_canonical(lean[c]), lean[c]


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_renorm_is_exact_and_orders_levels(H, W):
    """renorm_loose and finish never change the value of the levels, for any
    overlap, order or cancellation between them"""
    rng = np.random.default_rng(5 + W)
    count = 4000
    x = rng.standard_normal((count, W)) * np.ldexp(1.0, rng.integers(-60, 60, size=(count, W)))
    # overlapping levels of comparable magnitude, cancelling leaders, zeros
    x[::5, 1] = -x[::5, 0] * (1 + 2.0 ** -30)
    x[1::7, 0] = 0.0
    x[2::11] = 0.0
    x[3::13, W - 1] = x[3::13, 0] * 2.0 ** 40
    for finish in (0, 1):
        out = np.zeros_like(x)
        assert H.hst_lean_renorm_batch(W, finish, count, x.ctypes.data, out.ctypes.data) == 0
        for c in range(0, count, 7):
            assert frac(out[c]) == frac(x[c]), (finish, x[c], out[c])
        if finish:
            assert all(is_canonical(v) for v in out)
    # levels that overlap heavily but whose leader does not cancel (what a
    # k-tile of the GEMM produces): one loose pass leaves each level within an
    # ulp of the one above
    y = np.zeros((count, W))
    y[:, 0] = rng.standard_normal(count) * np.ldexp(1.0, rng.integers(-30, 30, size=count))
    for w in range(1, W):
        y[:, w] = y[:, w - 1] * 2.0 ** -40 * rng.standard_normal(count)
    out = np.zeros_like(y)
    assert H.hst_lean_renorm_batch(W, 0, count, y.ctypes.data, out.ctypes.data) == 0
    for c in range(0, count, 3):
        assert frac(out[c]) == frac(y[c])
        for w in range(1, W):
            if out[c, w - 1] != 0:
                assert abs(out[c, w]) <= np.spacing(abs(out[c, w - 1])), (c, w, y[c], out[c])


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_continuation_from_a_value(H, W):
    """K panels: a chain continued from a normalised value (C reloaded) stays
    within tolerance of the exact total"""
    k = 700
    a, b = baseline_pairs(W, 6, k, 120 + W, False)
    h = 320
    first, _, _ = chains(H, W, a[:, :h], b[:, :h])
    total, _, exact = chains(H, W, a[:, h:], b[:, h:], init=first)
    whole = [sum((frac(a[c, i]) * frac(b[c, i]) for i in range(k)), Fraction(0)) for c in range(6)]
    tol = 4 * k * U_P[W]
    assert normwise(total, whole) <= 0.02 * tol


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_gemm_host_matches_chains(H, W):
    """hst_lean_gemm (the kernel's element order: k-tiles of 16, renormalise at
    each tile end, finish) is the chain of hst_lean_dot_batch"""
    m, k, n = 3, 37, 5
    A = O.orc_fill_baseline(W, m, k, 7, wide=True)
    B = O.orc_fill_baseline(W, k, n, 8, wide=True)
    Cm = O.planes(W, m, n)
    assert H.hst_lean_gemm(W, m, k, n, A.ctypes.data, A.shape[2], B.ctypes.data, B.shape[2], Cm.ctypes.data,
                           Cm.shape[2]) == 0
    for i in range(m):
        for j in range(n):
            a = A[:, i, :k].T.copy()[None]
            b = B[:, :k, j].T.copy()[None]
            lean, _, exact = chains(H, W, a, b)
            assert np.array_equal(lean[0].view(np.uint64), Cm[:, i, j].copy().view(np.uint64))
            assert float(abs(frac(lean[0]) - exact[0])) <= 4 * k * U_P[W] * float(abs(exact[0])) + 1e-300
