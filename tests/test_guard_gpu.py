"""Guard bands around every device entry point (the box has no
compute-sanitizer): operands are windows inside larger buffers whose margins
hold NaN (A, B) or a sentinel (C).  Any read of a margin that reaches a
result shows up as a bit mismatch against the reference; any write outside
the m x n window of C shows up as a changed sentinel."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed

pytestmark = pytest.mark.gpu

SENT = 7.25


def window(P, torch, W, rows, cols, fill, data=None, r0=3, c0=4, extra_cols=6, extra_rows=5):
    """A (W, rows, cols) window at (r0, c0) of a buffer with margins; ld even."""
    ld = cols + c0 + extra_cols
    ld += ld & 1
    R = rows + r0 + extra_rows
    buf = torch.full((W, R, ld), fill, dtype=torch.float64, device="cuda")
    if data is not None:
        buf[:, r0:r0 + rows, c0:c0 + cols] = torch.from_numpy(np.ascontiguousarray(data[:, :rows, :cols])).cuda()
    ptr = buf.data_ptr() + 8 * (r0 * ld + c0)
    return buf, ptr, ld, R * ld


def outside_untouched(buf, rows, cols, r0=3, c0=4):
    b = buf.cpu().numpy().copy()
    b[:, r0:r0 + rows, c0:c0 + cols] = SENT
    return bool(np.all(b == SENT))


CASES = [(2, 37, 29, 41), (3, 64, 64, 64), (4, 33, 70, 130), (2, 130, 33, 600), (3, 9, 5, 3000)]


@pytest.mark.parametrize("W,m,n,k", CASES)
def test_guard_gemm_device_acc_fast(gpu_lib, W, m, n, k):
    import torch
    P = gpu_lib
    A = random_signed(W, m, k, 500 + m)
    B = random_signed(W, k, n, 600 + n)
    want = O.ref_gemm(A, B, k, n)
    bA, pA, lda, pa = window(P, torch, W, m, k, float("nan"), A)
    bB, pB, ldb, pb = window(P, torch, W, k, n, float("nan"), B)
    # one shot
    bC, pC, ldc, pc = window(P, torch, W, m, n, SENT)
    P.gemm_device(W, m, n, k, pA, lda, pa, pB, ldb, pb, pC, ldc, pc)
    torch.cuda.synchronize()
    got = bC.cpu().numpy()[:, 3:3 + m, 4:4 + n]
    assert mismatches(got, want[:, :, :n]) == 0
    assert outside_untouched(bC, m, n)
    # two K panels (continuation)
    h = max(16, (k // 2) // 16 * 16) if k > 16 else k
    bC2, pC2, _, _ = window(P, torch, W, m, n, SENT)
    P.gemm_device(W, m, n, h, pA, lda, pa, pB, ldb, pb, pC2, ldc, pc)
    if k > h:
        P.gemm_device_acc(W, m, n, k - h, pA + 8 * h, lda, pa, pB + 8 * h * ldb, ldb, pb, pC2, ldc, pc)
    torch.cuda.synchronize()
    assert mismatches(bC2.cpu().numpy()[:, 3:3 + m, 4:4 + n], want[:, :, :n]) == 0
    assert outside_untouched(bC2, m, n)
    # FAST (split-K where planned)
    bC3, pC3, _, _ = window(P, torch, W, m, n, SENT)
    P.gemm_device_ex(W, m, n, k, pA, lda, pa, pB, ldb, pb, pC3, ldc, pc, P.FAST)
    torch.cuda.synchronize()
    got3 = bC3.cpu().numpy()[:, 3:3 + m, 4:4 + n]
    assert np.all(np.isfinite(got3))
    if P.splitk_segments(W, m, n, k) == 1:
        assert mismatches(got3, want[:, :, :n]) == 0
    assert outside_untouched(bC3, m, n)
    # LEAN (tolerance mode): the same windows -- a margin read would put a NaN
    # into the result, a stray write would change a sentinel; every cell is
    # the host chain of the same source (tests/csrc/arith_host.cpp)
    import ctypes as C
    import os
    H = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libarith_host.so"))
    H.hst_lean_gemm.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                                C.c_size_t, C.c_void_p, C.c_size_t]
    chain = np.zeros((W, m, n))
    assert H.hst_lean_gemm(W, m, k, n, A.ctypes.data, A.shape[2], B.ctypes.data, B.shape[2], chain.ctypes.data, n) == 0
    bC4, pC4, _, _ = window(P, torch, W, m, n, SENT)
    P.gemm_device_ex(W, m, n, k, pA, lda, pa, pB, ldb, pb, pC4, ldc, pc, P.LEAN)
    torch.cuda.synchronize()
    assert mismatches(bC4.cpu().numpy()[:, 3:3 + m, 4:4 + n], chain) == 0
    assert outside_untouched(bC4, m, n)


@pytest.mark.parametrize("W,m,n,k", CASES[:3])
def test_guard_pull_and_strassen(gpu_lib, W, m, n, k):
    import torch
    P = gpu_lib
    A = random_signed(W, m, k, 700 + m)
    B = random_signed(W, k, n, 800 + n)
    bA, pA, lda, pa = window(P, torch, W, m, k, float("nan"), A)
    # fused pull: B's destination is a window too (its margins must survive)
    cut = k // 3 + 1
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1, :])).cuda() for r0, r1 in ((0, cut), (cut, k))]
    # the pull copies whole rows of ldb doubles from the slices into B (the
    # slices' row stride); B sits 4 rows into a sentinel buffer
    ldb = B.shape[2]
    bB = torch.full((W, k + 8, ldb), SENT, dtype=torch.float64, device="cuda")
    pB = bB.data_ptr() + 8 * 4 * ldb
    bC, pC, ldc, pc = window(P, torch, W, m, n, SENT)
    P.gemm_device_pull(W, m, n, k, pA, lda, pa, pB, ldb, (k + 8) * ldb, pC, ldc, pc,
                       [t.data_ptr() for t in slices], [0, cut, k], 16, 4)
    torch.cuda.synchronize()
    want = O.ref_gemm(A, B, k, n)
    assert mismatches(bC.cpu().numpy()[:, 3:3 + m, 4:4 + n], want[:, :, :n]) == 0
    assert outside_untouched(bC, m, n)
    hb = bB.cpu().numpy()
    assert np.all(hb[:, :4] == SENT) and np.all(hb[:, 4 + k:] == SENT)  # rows around B untouched
    # device Strassen on windows
    bB2, pB2, ldb2, pb2 = window(P, torch, W, k, n, float("nan"), B)
    bC2, pC2, _, _ = window(P, torch, W, m, n, SENT)
    P.strassen_device(W, m, n, k, pA, lda, pa, pB2, ldb2, pb2, pC2, ldc, pc, 16)
    torch.cuda.synchronize()
    wantS = O.ref_strassen(A, B, k, n, cutoff=16)
    assert mismatches(bC2.cpu().numpy()[:, 3:3 + m, 4:4 + n], wantS[:, :, :n]) == 0
    assert outside_untouched(bC2, m, n)


@pytest.mark.parametrize("W,op", [(2, 0), (3, 1), (4, 0), (3, 2)])
def test_guard_ew_device(gpu_lib, W, op):
    import torch
    P = gpu_lib
    rows, cols = 19, 37
    X = random_signed(W, rows, cols, 900)
    Y = random_signed(W, rows, cols, 901)
    bX, pX, ldx, px = window(P, torch, W, rows, cols, float("nan"), X)
    bY, pY, ldy, py = window(P, torch, W, rows, cols, float("nan"), Y)
    bO, pO, ldo, po = window(P, torch, W, rows, cols, SENT)
    P.ew_device(W, op, rows, cols, pO, ldo, po, pX, ldx, px, pY, ldy, py)
    torch.cuda.synchronize()
    want = O.ref_ew(W, {0: "add", 1: "mul", 2: "add_merge"}[op], X, Y, cols)
    assert mismatches(bO.cpu().numpy()[:, 3:3 + rows, 4:4 + cols], want[:, :, :cols]) == 0
    assert outside_untouched(bO, rows, cols)
