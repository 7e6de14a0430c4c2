"""The oracle is pinned before it is trusted (CPU, no GPU needed):

  * the C restatement (oracle/_build) is bit-identical to the reference
    itself (oracle/_ref: the unmodified mpfkit compiled here) on every kernel,
    generator and GEMM case below;
  * both reproduce the reference's own frozen test cases (test_eft.cpp,
    test_mpf.cpp, test_linalg.cpp known answers);
  * both match the committed golden fixtures (tests/golden/, generated from the
    reference build by tests/golden/make_golden.py).
The reference build only exists where /root/reference could be compiled; on
the GPU box the prebuilt .so travels with the repo.
"""
import ctypes as C
import glob
import os

import numpy as np
import pytest

import oracle as O
from oracle import dyadic
from tests.helpers import mismatches, random_signed, special_matrix

HERE = os.path.dirname(os.path.abspath(__file__))
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) absent")


def pair(fn, a, b):
    s = C.c_double()
    e = C.c_double()
    fn(a, b, C.addressof(s), C.addressof(e))
    return s.value, e.value


def arr(*v):
    return np.array(v, dtype=np.float64)


def call2(f, W, x, y):
    x, y = arr(*x), arr(*y)
    r = np.zeros(W)
    f(W, x.ctypes.data, y.ctypes.data, r.ctypes.data)
    return tuple(r)


# ---- test_eft.cpp frozen cases -------------------------------------------------

@pytest.mark.parametrize("lib", ["orc", "ref"])
def test_eft_frozen_cases(lib):
    if lib == "ref" and not O.ref_available():
        pytest.skip("no reference build")
    L = O.orc() if lib == "orc" else O.ref()
    p = lib + "_"
    ts, qts, tp = getattr(L, p + "two_sum"), getattr(L, p + "quick_two_sum"), getattr(L, p + "two_prod")
    assert pair(ts, 1.5, 2.25) == (3.75, 0.0)                      # test_eft.cpp:41-44
    assert pair(ts, 1.0, 2.0 ** -53) == (1.0, 2.0 ** -53)          # :45-47 tie to even
    assert pair(ts, 2.0 ** 53, 1.0) == (2.0 ** 53, 1.0)            # :48-50
    assert pair(qts, 2.0, 1.0) == (3.0, 0.0)                       # :63-66
    assert pair(qts, 1.0, 2.0 ** -53) == (1.0, 2.0 ** -53)
    assert pair(qts, 0.0, 0.0) == (0.0, 0.0)
    assert pair(tp, 1.5, 2.0) == (3.0, 0.0)                        # :90-105
    f = 2.0 ** 27 + 1.0
    assert pair(tp, f, f) == (2.0 ** 54 + 2.0 ** 28, 1.0)


@pytest.mark.parametrize("lib", ["orc", "ref"])
def test_renorm5_and_vseb_frozen_cases(lib):
    if lib == "ref" and not O.ref_available():
        pytest.skip("no reference build")
    L = O.orc() if lib == "orc" else O.ref()
    rn = getattr(L, lib + "_renorm5")
    vs = getattr(L, lib + "_vseb")
    for c, want in [((1, 0, 0, 0, 0), (1, 0, 0, 0)),                                   # test_eft.cpp:317-322
                    ((1.0, 2 ** -60, 2 ** -120, 2 ** -180, 0.0), (1.0, 2 ** -60, 2 ** -120, 2 ** -180))]:
        c = arr(*c)
        r = np.zeros(4)
        rn(c.ctypes.data, r.ctypes.data)
        assert tuple(r) == want
    for e, want in [((1.0, 2 ** -55, 2 ** -110), (1.0, 2 ** -55, 2 ** -110)),          # test_eft.cpp:200-218
                    ((0, 0, 0, 0, 0, 0), (0, 0, 0)),
                    ((1.0, 2 ** -60, 0, 0, 0, 0), (1.0, 2 ** -60, 0.0))]:
        e = arr(*e)
        out = np.zeros(3)
        assert vs(e.ctypes.data, len(e), out.ctypes.data, 3) == 0
        assert tuple(out) == want
    e = arr(1.0, 2.0)
    out = np.zeros(4)
    assert vs(e.ctypes.data, 2, out.ctypes.data, 0) != 0   # k < 1 rejected (eft.hpp:208)
    assert vs(e.ctypes.data, 2, out.ctypes.data, 4) != 0   # n < k rejected (eft.hpp:209)


@pytest.mark.parametrize("lib", ["orc", "ref"])
def test_mpf_frozen_cases(lib):
    """test_mpf.cpp:92-135."""
    if lib == "ref" and not O.ref_available():
        pytest.skip("no reference build")
    if lib == "orc":
        add = lambda W, x, y: call2(O.orc().orc_add, W, x, y)
        mul = lambda W, x, y: call2(O.orc().orc_mul, W, x, y)
    else:
        add = lambda W, x, y: call2(lambda W_, a, b, r: O.ref().ref_binop(W_, 0, a, b, r), W, x, y)
        mul = lambda W, x, y: call2(lambda W_, a, b, r: O.ref().ref_binop(W_, 1, a, b, r), W, x, y)
    x = (1.5, 2 ** -55)
    assert add(2, x, (0, 0)) == x
    assert add(2, x, (-1.5, -2 ** -55)) == (0.0, 0.0)
    s = add(2, (1.0, 2 ** -54), (2 ** -54, 0))
    assert dyadic.from_components(s) == dyadic.from_components((1.0, 2 ** -53))
    y = (1.25, 2 ** -54)
    assert mul(2, (1.0, 0.0), y) == y
    assert mul(2, (2.0, 0.0), (0.5, 0.0)) == (1.0, 0.0)
    assert mul(2, (2 ** 10, 0.0), y) == (2 ** 10 * 1.25, 2 ** -44)
    t = (1.5, 2 ** -55, 2 ** -110)
    assert add(3, t, (0, 0, 0)) == t
    assert mul(3, (1, 0, 0), t) == t
    q = (1.5, 2 ** -55, 2 ** -110, 2 ** -165)
    assert add(4, q, (0, 0, 0, 0)) == q
    assert mul(4, (1, 0, 0, 0), q) == q
    assert add(4, (1, 0, 0, 0), (1, 0, 0, 0)) == (2, 0, 0, 0)
    assert mul(4, (2 ** 7, 0, 0, 0), q) == (2 ** 7 * 1.5, 2 ** -48, 2 ** -103, 2 ** -158)


def _random_pairs(W, count, seed, signed=True):
    st = (C.c_uint64 * 1)(seed)
    x = np.zeros((count, W))
    for i in range(count):
        if O.ref_available():
            O.ref().ref_random_normalized(W, C.cast(st, C.c_void_p), int(signed), x[i].ctypes.data)
        else:
            O.orc().orc_random_normalized(W, C.cast(st, C.c_void_p), x[i].ctypes.data)
    return x


@needs_ref
@pytest.mark.parametrize("W", [2, 3, 4])
def test_oracle_kernels_match_reference(W):
    x = _random_pairs(W, 5000, 100 + W)
    y = _random_pairs(W, 5000, 200 + W) * np.ldexp(1.0, np.random.default_rng(W).integers(-60, 60, (5000, 1)))
    for op in ("add", "mul"):
        a = O.orc_binop_batch(W, op, x, y)
        b = O.ref_binop_batch(W, op, x, y)
        assert not (a.view(np.uint64) != b.view(np.uint64)).any()


@needs_ref
@pytest.mark.parametrize("W", [2, 3, 4])
def test_oracle_generators_match_reference(W):
    a = O.orc_fill_random(W, 9, 13, 4242 + W)
    b = O.ref_fill_random(W, 9, 13, 4242 + W)
    assert mismatches(a, b) == 0 and not (a.view(np.uint64) != b.view(np.uint64)).any()
    pa, pb = O.orc_gen_paper(W, 37)
    ra, rb = O.ref_gen_paper(W, 37)
    assert mismatches(pa, ra) == 0 and mismatches(pb, rb) == 0


@needs_ref
@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("shape", [(1, 1, 1), (4, 4, 4), (8, 8, 8), (33, 33, 33), (7, 12, 9), (5, 0, 6)])
def test_oracle_gemm_matches_reference(W, shape):
    m, k, n = shape
    A = random_signed(W, m, k, 10 * m + k)
    B = random_signed(W, k, n, 10 * n + k + 1)
    want = O.ref_gemm(A, B, k, n)
    assert mismatches(O.orc_gemm(A, B, k, n), want) == 0
    # every reference algorithm/variant agrees bitwise (linalg.hpp:338-344)
    for variant in (0, 1, 2):
        for n_min in (4, 8, 32):
            assert mismatches(O.ref_gemm(A, B, k, n, workers=3, n_min=n_min, variant=variant), want) == 0
    assert mismatches(O.ref_gemm(A, B, k, n, naive=True, variant=0), want) == 0


@needs_ref
@pytest.mark.parametrize("W", [2, 3, 4])
def test_oracle_gemm_special_values_match_reference(W):
    A = special_matrix(W, 30, 30, 77)
    B = special_matrix(W, 30, 30, 78)
    assert mismatches(O.orc_gemm(A, B, 30, 30), O.ref_gemm(A, B, 30, 30)) == 0


@needs_ref
def test_reference_error_messages_and_counters():
    """linalg.hpp:279-294, :409 messages; count_matmul (test_linalg.cpp:347-363)."""
    R = O.ref()
    cases = [((3, 4, 5, 2, 3, 2, 32, 0, 1), "matmul: inner dimensions differ"),
             ((3, 4, 4, 2, 3, 3, 32, 0, 1), "matmul: result shape mismatch"),
             ((3, 4, 4, 2, 3, 2, 0, 0, 1), "matmul: n_min must be at least 1"),
             ((3, 4, 4, 2, 3, 2, 5, 1, 1), "matmul: SIMD variants need n_min divisible by 4"),
             ((3, 4, 4, 2, 3, 2, 32, 0, 0), "matmul: workers must be at least 1")]
    for args, msg in cases:
        assert R.ref_gemm_shapes(2, *args) != 0
        assert R.ref_last_error().decode() == msg
    R.ref_op_counters_reset()
    A = random_signed(2, 4, 4, 530)
    B = random_signed(2, 4, 4, 531)
    O.ref_gemm(A, B, 4, 4, naive=True, variant=0)
    adds, muls = C.c_uint64(), C.c_uint64()
    R.ref_op_counts(C.addressof(adds), C.addressof(muls))
    assert (muls.value, adds.value) == (64, 48)


def test_dyadic_oracle_bound_on_oracle_gemm():
    """test_linalg.cpp:250-268 analog on the C restatement: within
    n*4*format_eps of the exact product (positive inputs)."""
    for W, eps in ((2, 2.0 ** -104), (3, 2.0 ** -157), (4, 2.0 ** -209)):
        n = 8
        # bench::fill_random values are positive (lead in [1, 2))
        A = O.orc_fill_random(W, n, n, 470 + W)
        B = O.orc_fill_random(W, n, n, 480 + W)
        Cm = O.orc_gemm(A, B, n, n)
        exact = dyadic.matmul_exact(A, B, n, n)
        assert dyadic.max_rel_err(Cm, exact) <= n * 4 * eps
        assert dyadic.digit_loss(dyadic.max_rel_err(Cm, exact), eps) < 2.5


GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


@pytest.mark.skipif(not GOLDEN, reason="no golden fixtures")
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_golden(path):
    """Fixtures produced by the reference build (tests/golden/make_golden.py)."""
    z = np.load(path)
    W, k, n = int(z["W"]), int(z["k"]), int(z["n"])
    assert mismatches(O.orc_gemm(z["A"], z["B"], k, n), z["C"]) == 0
