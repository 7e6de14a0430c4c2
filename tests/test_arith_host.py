"""The product's device arithmetic (csrc/mpf_arith.cuh), compiled for the host
(tests/_build/libarith_host.so, -ffp-contract=off), against the reference
build on the CPU: the branch-free renorm5/vseb restatements and every width
kernel must be bit-identical on random, wide-range and special inputs.  The
device build uses __dadd_rn & co. with the same IEEE semantics; the GPU
tests (test_gemm_gpu.py) close that last step on the B200.
"""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed, special_matrix

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libarith_host.so")

pytestmark = [pytest.mark.skipif(not os.path.exists(SO), reason="host arith shim not built"),
              pytest.mark.skipif(not O.ref_available(), reason="reference build absent")]


@pytest.fixture(scope="module")
def H():
    L = C.CDLL(SO)
    L.hst_binop_batch.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hst_renorm5_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p]
    L.hst_vseb23_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p]
    L.hst_gemm.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                           C.c_size_t, C.c_void_p, C.c_size_t]
    return L


def _pairs(W, count, seed):
    st = (C.c_uint64 * 1)(seed)
    x = np.zeros((count, W))
    for i in range(count):
        O.ref().ref_random_normalized(W, C.cast(st, C.c_void_p), 1, x[i].ctypes.data)
    return x


def _special_values(W, count, seed):
    """mixtures of +-0, integers, powers of two and normalized values per
    component slot -- including non-normalized combinations that drive every
    renorm5 path."""
    rng = np.random.default_rng(seed)
    pool = np.array([0.0, -0.0, 1.0, -1.0, 2.0, 0.5, 3.0, -3.0, 2.0 ** -53, -2.0 ** -53, 2.0 ** -106,
                     2.0 ** -159, 2.0 ** 30, 1.0 + 2.0 ** -52, 7.0, -2.0 ** -1074])
    x = rng.choice(pool, size=(count, W))
    norm = _pairs(W, count, seed + 1)
    pick = rng.integers(0, 3, size=(count, 1))
    return np.where(pick == 0, norm, x)


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("op", ["add", "mul"])
def test_width_kernels_random(H, W, op):
    n = 40000
    x = _pairs(W, n, 10 + W)
    y = _pairs(W, n, 20 + W) * np.ldexp(1.0, np.random.default_rng(W).integers(-80, 80, (n, 1)))
    y[::7] = -x[::7] * (1 + 2.0 ** -40)  # near cancellation
    r = np.empty_like(x)
    H.hst_binop_batch(W, {"add": 0, "mul": 1}[op], n, x.ctypes.data, y.ctypes.data, r.ctypes.data)
    want = O.ref_binop_batch(W, op, x, y)
    assert not (r.view(np.uint64) != want.view(np.uint64)).any()


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("op", ["add", "mul"])
def test_width_kernels_special(H, W, op):
    n = 40000
    x = _special_values(W, n, 30 + W)
    y = _special_values(W, n, 40 + W)
    r = np.empty_like(x)
    H.hst_binop_batch(W, {"add": 0, "mul": 1}[op], n, x.ctypes.data, y.ctypes.data, r.ctypes.data)
    want = O.ref_binop_batch(W, op, x, y)
    bad = (r.view(np.uint64) != want.view(np.uint64)).any(axis=1)
    assert not bad.any(), (x[bad][:3], y[bad][:3], r[bad][:3], want[bad][:3])


def test_td_add_folds_are_identities(H):
    """td_add_q with the constant-lane folds == the literal zero-extend +
    qd_add sequence == the reference, on signed-zero-heavy inputs."""
    H.hst_td_add_unfolded_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    n = 60000
    x = _special_values(3, n, 91)
    y = _special_values(3, n, 92)
    y[::3] = -x[::3]
    folded = np.empty_like(x)
    unfolded = np.empty_like(x)
    H.hst_binop_batch(3, 0, n, x.ctypes.data, y.ctypes.data, folded.ctypes.data)
    H.hst_td_add_unfolded_batch(n, x.ctypes.data, y.ctypes.data, unfolded.ctypes.data)
    want = O.ref_binop_batch(3, "add", x, y)
    assert not (folded.view(np.uint64) != unfolded.view(np.uint64)).any()
    assert not (folded.view(np.uint64) != want.view(np.uint64)).any()


def test_renorm5_all_paths(H):
    """Branch-free fast path + verbatim fallback vs eft.hpp:241-288 on inputs
    hitting paths A-D and the zero corners."""
    rng = np.random.default_rng(5)
    n = 100000
    c = np.zeros((n, 5))
    c[:, 0] = 1.0 + rng.random(n)
    for i in range(1, 5):
        c[:, i] = (rng.random(n) * 2 - 1) * np.ldexp(2.0, -53 * i)
    # zero out random subsets of tail terms, and plant exact cancellations
    mask = rng.random((n, 5)) < 0.3
    mask[:, 0] = False
    c[mask] = 0.0
    c[::11, 2] = -c[::11, 1]
    c[::13, 4] = -0.0
    out = np.zeros((n, 4))
    H.hst_renorm5_batch(n, c.ctypes.data, out.ctypes.data)
    want = np.zeros((n, 4))
    for i in range(n):
        O.ref().ref_renorm5(c[i].ctypes.data, want[i].ctypes.data)
    assert not (out.view(np.uint64) != want.view(np.uint64)).any()


def test_vseb_2_3(H):
    """vseb with k = 2, n = 3 (td_mul's use, mpf.hpp:162) vs eft.hpp:205-225."""
    rng = np.random.default_rng(6)
    n = 60000
    e = np.zeros((n, 3))
    e[:, 0] = rng.random(n) * 2 - 1
    e[:, 1] = (rng.random(n) * 2 - 1) * 2.0 ** -53
    e[:, 2] = (rng.random(n) * 2 - 1) * 2.0 ** -106
    z = rng.random((n, 3)) < 0.25
    e[z] = 0.0
    e[::9, 2] = -0.0
    e[::5, 1] = 0.0
    out = np.zeros((n, 2))
    H.hst_vseb23_batch(n, e.ctypes.data, out.ctypes.data)
    want = np.zeros((n, 2))
    for i in range(n):
        assert O.ref().ref_vseb(e[i].ctypes.data, 3, want[i].ctypes.data, 2) == 0
    assert not (out.view(np.uint64) != want.view(np.uint64)).any()


@pytest.mark.parametrize("W", [2, 3, 4])
def test_gemm_order_on_host(H, W):
    """The kernel's per-element order (mul, then add(C, p) ascending k) with
    the product arithmetic == the reference GEMM."""
    for (m, k, n), gen in [((17, 23, 19), random_signed), ((20, 20, 20), special_matrix)]:
        A = gen(W, m, k, 60 + m)
        B = gen(W, k, n, 70 + n)
        Cm = O.planes(W, m, n)
        H.hst_gemm(W, m, k, n, A.ctypes.data, A.shape[2], B.ctypes.data, B.shape[2], Cm.ctypes.data, Cm.shape[2])
        assert mismatches(Cm, O.ref_gemm(A, B, k, n)) == 0


def test_td_add_merge_host(H):
    """merge6 + vec_sum<6> + vseb(3 of 6) (mpf.hpp:125-131) vs the reference,
    on sorted, unsorted and zero-laden inputs."""
    H.hst_td_add_merge_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    n = 40000
    x = np.concatenate([_pairs(3, n // 2, 51), _special_values(3, n // 2, 52)])
    y = np.concatenate([_pairs(3, n // 2, 53) * np.ldexp(1.0, np.random.default_rng(3).integers(-70, 70, (n // 2, 1))),
                        _special_values(3, n // 2, 54)])
    y[::5] = -x[::5]
    r = np.empty_like(x)
    H.hst_td_add_merge_batch(n, x.ctypes.data, y.ctypes.data, r.ctypes.data)
    want = np.empty_like(x)
    O.ref().ref_td_add_merge_batch(n, x.ctypes.data, y.ctypes.data, want.ctypes.data)
    assert not (r.view(np.uint64) != want.view(np.uint64)).any()
    # the ranked merge + straight-line compress (the device ew kernel's form)
    H.hst_td_add_merge_ranked_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    r2 = np.empty_like(x)
    H.hst_td_add_merge_ranked_batch(n, x.ctypes.data, y.ctypes.data, r2.ctypes.data)
    assert not (r2.view(np.uint64) != want.view(np.uint64)).any()


def test_td_add_merge_ranked_ties_and_orders(H):
    """Ranked merge vs the reference on magnitude ties across the operands
    (|x[i]| == |y[j]| with either sign, zeros of both signs), equal
    components, unsorted operands and zero residuals."""
    H.hst_td_add_merge_ranked_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(77)
    n = 60000
    pool = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, 2.0 ** -53, -2.0 ** -53, 2.0 ** -106, 3.0, 0.75, 2.0 ** -60])
    x = rng.choice(pool, size=(n, 3))
    y = rng.choice(pool, size=(n, 3))
    # a third sorted by magnitude (the ranked path), a third with y = +-x, the rest as drawn
    srt = lambda a: np.take_along_axis(a, np.argsort(-np.abs(a), axis=1, kind="stable"), axis=1)
    x[: n // 3] = srt(x[: n // 3])
    y[: n // 3] = srt(y[: n // 3])
    y[n // 3: 2 * n // 3] = x[n // 3: 2 * n // 3] * rng.choice([1.0, -1.0], size=(n // 3, 1))
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    r = np.empty_like(x)
    H.hst_td_add_merge_ranked_batch(n, x.ctypes.data, y.ctypes.data, r.ctypes.data)
    want = np.empty_like(x)
    O.ref().ref_td_add_merge_batch(n, x.ctypes.data, y.ctypes.data, want.ctypes.data)
    assert not (r.view(np.uint64) != want.view(np.uint64)).any()


def test_two_sum_sorted_equals_knuth(H):
    """The 3-FP64-op two-sum (operands ordered by exponent on the integer
    pipes, then Dekker's fast two-sum, mpf_arith.cuh:two_sum_sorted) returns
    the same bits as Knuth's 6-op two_sum (eft.hpp:46-51) -- sum, error and
    the sign of a zero error -- on signed zeros, subnormals, equal and
    distant exponents, exact cancellation and random pairs."""
    H.hst_two_sum_pair_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(2101)
    pool = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, 1.5, 3.0, -3.0, 2.0 ** -53, -2.0 ** -53, 2.0 ** -1074,
                     -2.0 ** -1074, 2.0 ** -1022, -2.0 ** -1022, 2.0 ** -1023, 1.0 + 2.0 ** -52, -(1.0 + 2.0 ** -52),
                     2.0 ** 52, 2.0 ** 53 + 2, 2.0 ** 1000, -2.0 ** 1000, 2.0 ** -1000, np.nextafter(1.0, 0.0)])
    n = 400_000
    a = rng.choice(pool, n) * np.where(rng.integers(0, 2, n) == 1, 1.0, -1.0)
    b = rng.choice(pool, n)
    # random pairs: exponents near (cancellation), far, and subnormal
    m = n // 4
    r = rng.uniform(-1, 1, m)
    a[:m] = r
    b[:m] = -r * (1 + rng.integers(-8, 9, m) * 2.0 ** -52)
    a[m:2 * m] = rng.uniform(-1, 1, m) * np.ldexp(1.0, rng.integers(-60, 61, m))
    b[m:2 * m] = rng.uniform(-1, 1, m) * np.ldexp(1.0, rng.integers(-60, 61, m))
    a[2 * m:2 * m + m // 2] = rng.integers(-2 ** 40, 2 ** 40, m // 2) * 2.0 ** -1074
    b[2 * m:2 * m + m // 2] = rng.integers(-2 ** 40, 2 ** 40, m // 2) * 2.0 ** -1074
    # same-magnitude pairs (key ties) in both orders
    a[-1000:] = b[-1000:]
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    out = np.zeros((n, 4))
    H.hst_two_sum_pair_batch(n, a.ctypes.data, b.ctypes.data, out.ctypes.data)
    knuth = out[:, :2].view(np.uint64)
    fast = out[:, 2:].view(np.uint64)
    assert np.array_equal(knuth, fast), np.nonzero((knuth != fast).any(axis=1))[0][:10]
    # and both orders of every pair
    H.hst_two_sum_pair_batch(n, b.ctypes.data, a.ctypes.data, out.ctypes.data)
    assert np.array_equal(out[:, :2].view(np.uint64), out[:, 2:].view(np.uint64))


@pytest.mark.parametrize("W", [3, 4])
@pytest.mark.parametrize("level", [1, 2])
def test_fast_forms_flag_every_departure(H, W, level):
    """The GEMM fast pass (TileCfg::FASTR): acc = add(acc, mul(a, b)) in the
    branch-free forms equals the exact forms whenever the `rare` accumulator
    stayed clear, for both accumulators; RareMin (FMNMX3 minimum of high
    words) is conservative -- set whenever RareBool (exact zero tests) is."""
    H.hst_fast_mac_batch.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p]
    n = 60000
    a = np.concatenate([_pairs(W, n // 2, 300 + W), _special_values(W, n // 2, 310 + W)])
    b = np.concatenate([_pairs(W, n // 2, 320 + W), _special_values(W, n // 2, 330 + W)])
    acc = np.concatenate([_pairs(W, n // 2, 340 + W), _special_values(W, n // 2, 350 + W)])
    acc[::5] *= 2.0 ** -40
    # exact cancellations of the leading terms and subnormal residues below
    # 2^-1042 (zero high word, nonzero low word: RareMin reads them as zero)
    p = O.ref_binop_batch(W, "mul", a, b)
    acc[1::9] = -p[1::9]
    acc[2::9, 1:] = 2.0 ** -1060
    out = np.empty_like(a)
    flags = np.zeros((n, 2), dtype=np.int32)
    assert H.hst_fast_mac_batch(W, level, n, a.ctypes.data, b.ctypes.data, acc.ctypes.data, out.ctypes.data,
                                flags.ctypes.data) == 0
    assert (flags >= 0).all(), "the accumulator type changed the arithmetic"
    want = O.ref_binop_batch(W, "add", acc, p)
    clear = flags[:, 0] == 0
    bad = (out.view(np.uint64) != want.view(np.uint64)).any(axis=1) & clear
    assert not bad.any(), (a[bad][:3], b[bad][:3], acc[bad][:3])
    assert not ((flags[:, 0] == 1) & (flags[:, 1] == 0)).any(), "RareMin missed a departure"
    assert clear.sum() > 5000 and (~clear).sum() > 100  # both sides exercised


def test_two_sum_ordered_equals_knuth_when_the_order_holds(H):
    """The fast pass's ordered two-sum (3 operations, first operand assumed
    at least in the second's binade): identical bits to Knuth's form whenever
    its order test (mag_ge: one compare of the high words) did not flag --
    including signed zeros, ties, subnormals and cancelling pairs -- and the
    test flags every pair whose exponents are the other way round."""
    H.hst_two_sum_ordered_batch.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(77)
    n = 400000
    a = rng.standard_normal(n) * np.ldexp(1.0, rng.integers(-40, 41, size=n))
    b = rng.standard_normal(n) * np.ldexp(1.0, rng.integers(-40, 41, size=n))
    special = np.array([0.0, -0.0, 1.0, -1.0, 2.0 ** -1074, -2.0 ** -1074, 2.0 ** -1060, 1.0 + 2.0 ** -52,
                        2.0 ** 52, 2.0 ** 53 + 2.0, 0.5, -0.5, 3.0, 2.0 ** -1022, 2.0 ** 1000, -2.0 ** 1000])
    a[:65536] = np.repeat(special, 4096)[:65536]
    b[:65536] = np.tile(np.repeat(special, 256), 16)[:65536]
    a[65536:70000] = -b[65536:70000]                      # exact cancellation
    a[70000:80000] = b[70000:80000] * (1 + 2.0 ** -30)    # near ties
    out = np.zeros((n, 4))
    flag = np.zeros(n, dtype=np.int32)
    H.hst_two_sum_ordered_batch(n, a.ctypes.data, b.ctypes.data, out.ctypes.data, flag.ctypes.data)
    clear = flag == 0
    k, o = out[:, :2].view(np.uint64), out[:, 2:].view(np.uint64)
    bad = (k != o).any(axis=1) & clear
    assert not bad.any(), (a[bad][:5], b[bad][:5])
    # the sum is the same rounded sum either way
    assert np.array_equal(k[:, 0], o[:, 0])
    # every pair with exponent(a) < exponent(b) is flagged (finite values)
    ea, eb = np.frexp(a)[1], np.frexp(b)[1]
    must = (ea < eb) & (b != 0) & (np.abs(a) >= 2.0 ** -1022) & (np.abs(b) >= 2.0 ** -1022)
    assert flag[must].all()
    assert clear.sum() > 100000 and (~clear).sum() > 100000
