"""Strassen top levels on the GPU with block-GEMM
leaves, bit-identical to the reference's matmul_strassen[_parallel]
(linalg.hpp:472-617).  Mirrors test_linalg.cpp:270-306 (cutoff delegation,
7^k leaf law, odd padding, errors) and acceptance.cpp criterion 6."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed, to_mp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,k,n,cutoff", [(40, 40, 40, 8), (33, 33, 33, 8), (17, 30, 23, 4), (64, 64, 64, 16),
                                          (9, 70, 5, 2), (100, 100, 100, 24)])
def test_strassen_bitwise_vs_reference(gpu_lib, W, m, k, n, cutoff):
    P = gpu_lib
    A = random_signed(W, m, k, 500 + m + W)
    B = random_signed(W, k, n, 600 + n + W)
    want = O.ref_strassen(A, B, k, n, cutoff=cutoff, n_min=4)
    got = P.matmul_strassen(to_mp(A, k), to_mp(B, n), cutoff, 4)
    assert mismatches(got.data, want) == 0
    assert not got.data[:, :, n:].view(np.uint64).any()
    par = P.matmul_strassen_parallel(to_mp(A, k), to_mp(B, n), cutoff, 4, P.KernelVariant.NORMAL, 4)
    assert mismatches(par.data, want) == 0
    if W == 3:
        assert mismatches(O.ref_strassen(A, B, k, n, cutoff=cutoff, n_min=4, workers=4), want) == 0


def test_strassen_delegation_and_leaf_law(gpu_lib):
    """test_linalg.cpp:270-290; acceptance.cpp criterion 6 (7^k law)."""
    P = gpu_lib
    a = to_mp(random_signed(2, 32, 32, 500), 32)
    b = to_mp(random_signed(2, 32, 32, 501), 32)
    assert P.bits_equal(P.matmul_strassen(a, b, 64, 32), P.matmul_block(a, b, 32))
    leaves = {}
    for n in (32, 64, 128, 256):
        A = P.fill_random(2, n, n, 6000 + n)
        B = P.fill_random(2, n, n, 6001 + n)
        P.op_counters_reset()
        P.matmul_strassen(A, B, 32, 32)
        leaves[n] = P.op_counters_read().leaf_multiplies
    assert leaves[32] == 1 and leaves[64] == 7 and leaves[128] == 49 and leaves[256] == 343


def test_strassen_counters_match_reference(gpu_lib):
    P = gpu_lib
    A = random_signed(3, 45, 45, 70)
    B = random_signed(3, 45, 45, 71)
    O.ref().ref_op_counters_reset()
    O.ref_strassen(A, B, 45, 45, cutoff=8, n_min=4)
    import ctypes as C
    adds, muls = C.c_uint64(), C.c_uint64()
    O.ref().ref_op_counts(C.addressof(adds), C.addressof(muls))
    P.op_counters_reset()
    P.matmul_strassen(to_mp(A, 45), to_mp(B, 45), 8, 4)
    c = P.op_counters_read()
    assert (c.adds, c.muls, c.leaf_multiplies) == (adds.value, muls.value, O.ref().ref_leaf_multiplies())


def test_strassen_odd_padding_accuracy_and_errors(gpu_lib):
    """test_linalg.cpp:292-305: odd sizes pad per level; result shape is the
    true shape; error within 33*64*eps of the exact product."""
    P = gpu_lib
    from oracle import dyadic
    a = O.ref_fill_random(2, 33, 33, 506)
    b = O.ref_fill_random(2, 33, 33, 507)
    s = P.matmul_strassen(to_mp(a, 33), to_mp(b, 33), 8, 4)
    assert (s.rows(), s.cols()) == (33, 33)
    assert not s.data[:, :, 33:].view(np.uint64).any()
    exact = dyadic.matmul_exact(a, b, 33, 33, rows=(0, 4))
    assert dyadic.max_rel_err(s.data, exact, rows=(0, 4)) <= 33 * 64.0 * P.format_eps(2)
    x = to_mp(random_signed(2, 32, 32, 500), 32)
    with pytest.raises(ValueError, match="matmul: cutoff must be at least 1"):
        P.matmul_strassen(x, x, 0, 32)
    with pytest.raises(ValueError, match="matmul: workers must be at least 1"):
        P.matmul_strassen_parallel(x, x, 64, 32, P.KernelVariant.SIMD_SET, 0)
    with pytest.raises(ValueError, match="matmul: inner dimensions differ"):
        P.matmul_strassen(x, P.MPMatrix(2, 31, 32))


def test_strassen_depth_first_fallback_bitwise(gpu_lib, monkeypatch):
    """With no scratch budget every level runs depth-first (children one at a
    time, strided product views); the bits and counters must not change."""
    P = gpu_lib
    A = random_signed(4, 37, 41, 900)
    B = random_signed(4, 41, 29, 901)
    want = O.ref_strassen(A, B, 41, 29, cutoff=6, n_min=4)
    P.op_counters_reset()
    fast = P.matmul_strassen(to_mp(A, 41), to_mp(B, 29), 6, 4)
    c_fast = P.op_counters_read()
    monkeypatch.setenv("MPFK_STRASSEN_BUDGET_BYTES", "1")
    P.op_counters_reset()
    slow = P.matmul_strassen(to_mp(A, 41), to_mp(B, 29), 6, 4)
    assert P.op_counters_read() == c_fast
    assert mismatches(fast.data, want) == 0 and mismatches(slow.data, want) == 0


def test_strassen_device_entry(gpu_lib):
    import torch
    P = gpu_lib
    W, m, k, n = 2, 130, 96, 70
    A = random_signed(W, m, k, 910)
    B = random_signed(W, k, n, 911)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros((W, m, B.shape[2]), dtype=torch.float64, device="cuda")
    launches = P.strassen_device(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), B.shape[2],
                                 k * B.shape[2], dC.data_ptr(), B.shape[2], m * B.shape[2], cutoff=16)
    torch.cuda.synchronize()
    assert launches < 20  # level-synchronous: a handful of launches, not 7^depth
    assert mismatches(dC.cpu().numpy(), O.ref_strassen(A, B, k, n, cutoff=16, n_min=4)) == 0
