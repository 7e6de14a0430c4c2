"""The drop-in boundary under less friendly callers (GPU):
  * host matrices with arbitrary row strides (odd, > pad4) and plane strides
    (gaps between planes) -- the C ABI repacks them, results stay bit-exact
    and cells outside rows x cols of C are left alone except the row pads;
  * several host threads calling concurrently (ctypes releases the GIL);
  * very long K (one chain of 10^5 multiply-adds per element);
  * the device API on offset (16-byte aligned) sub-matrices.
"""
import ctypes as C
import threading

import numpy as np
import pytest

import oracle as O
from paper_2101_06584_b200 import _native as N
from tests.helpers import mismatches, random_signed, to_mp

pytestmark = pytest.mark.gpu


def _mat(arr, rows, cols, stride, plane):
    return N.MpfkMat(arr.ctypes.data, rows, cols, stride, plane)


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("sa,sb,sc,gap", [(13, 11, 9, 0), (29, 40, 33, 7), (12, 8, 8, 3)])
def test_arbitrary_host_strides(gpu_lib, W, sa, sb, sc, gap):
    m, k, n = 9, 11, 8
    A = random_signed(W, m, k, 40 + W)
    B = random_signed(W, k, n, 50 + W)
    pa, pb, pc = m * sa + gap, k * sb + gap, m * sc + gap
    ha = np.full(W * pa, np.nan)
    hb = np.full(W * pb, np.nan)
    hc = np.full(W * pc, 5.0)
    for w in range(W):
        for i in range(m):
            ha[w * pa + i * sa: w * pa + i * sa + k] = A[w, i, :k]
        for i in range(k):
            hb[w * pb + i * sb: w * pb + i * sb + n] = B[w, i, :n]
    a, b, c = _mat(ha, m, k, sa, pa), _mat(hb, k, n, sb, pb), _mat(hc, m, n, sc, pc)
    N.check(N.lib().mpfk_matmul_block_parallel_into(W, C.byref(c), C.byref(a), C.byref(b), 32, 0, 1))
    want = O.ref_gemm(A, B, k, n)
    for w in range(W):
        for i in range(m):
            row = hc[w * pc + i * sc: w * pc + i * sc + sc]
            assert np.array_equal(row[:n].view(np.uint64), want[w, i, :n].view(np.uint64))
            assert not row[n:].view(np.uint64).any()  # C's row pads end +0 (zero_pads)
        assert (hc[w * pc + m * sc: w * pc + pc] == 5.0).all()  # the plane gap is not C's


def test_concurrent_host_callers(gpu_lib):
    P = gpu_lib
    cases = []
    for t in range(6):
        W, n = 2 + t % 3, 45 + t
        A = random_signed(W, 70 + t, 50, 60 + t)
        B = random_signed(W, 50, n, 70 + t)
        cases.append((W, n, A, B, O.ref_gemm(A, B, 50, n)))
    errors = []

    def run(case):
        W, n, A, B, want = case
        try:
            for _ in range(3):
                got = P.matmul_block_parallel(to_mp(A, 50), to_mp(B, n), 32, P.KernelVariant.NORMAL, 1)
                if mismatches(got.data, want) != 0:
                    errors.append("mismatch")
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ths = [threading.Thread(target=run, args=(c,)) for c in cases]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("W", [2, 4])
def test_very_long_k_chain(gpu_lib, W):
    """1 x K . K x 2 with K = 100003 (odd): a single chain of 10^5 adds."""
    P = gpu_lib
    k = 100003
    A = random_signed(W, 1, k, 80 + W)
    B = random_signed(W, k, 2, 90 + W)
    got = P.matmul_block(to_mp(A, k), to_mp(B, 2))
    assert mismatches(got.data, O.orc_gemm(A, B, k, 2)) == 0


def test_device_api_on_submatrices(gpu_lib):
    """A window of a larger device matrix (offset rows/cols, 16-byte aligned)."""
    import torch
    P = gpu_lib
    W = 3
    big = random_signed(W, 40, 48, 95)
    dbig = torch.from_numpy(big).cuda()
    ld = big.shape[2]
    r0, c0 = 3, 6  # even column offset keeps 16-byte alignment
    m, k = 20, 30
    B = random_signed(W, k, 17, 96)
    dB = torch.from_numpy(B).cuda()
    dC = torch.zeros((W, m, B.shape[2]), dtype=torch.float64, device="cuda")
    P.gemm_device(W, m, 17, k, dbig.data_ptr() + 8 * (r0 * ld + c0), ld, 40 * ld, dB.data_ptr(), B.shape[2],
                  k * B.shape[2], dC.data_ptr(), B.shape[2], m * B.shape[2])
    torch.cuda.synchronize()
    sub = np.ascontiguousarray(big[:, r0:r0 + m, c0:c0 + k])
    want = O.ref_gemm(sub, B, k, 17)
    assert mismatches(dC.cpu().numpy(), want) == 0


def test_set_device_mirrors_torch(gpu_lib):
    import torch
    P = gpu_lib
    torch.cuda.set_device(0)
    assert P.get_device() == 0
    P.set_device(0)
    assert P.get_device() == 0
    with pytest.raises(ValueError, match="device index out of range"):
        P.set_device(P.device_count())


@pytest.mark.parametrize("W,m,n,k", [(2, 2048, 5000, 64), (4, 700, 3000, 900)])
def test_pageable_staging_multi_piece(gpu_lib, W, m, n, k):
    """Pageable host operands go through libmpfk's pinned staging ring
    (16 MiB slots, copy-outs deferred until a slot is reused): rows wider
    than a slot's share, several pieces per plane and ring wrap-around must
    give the same bits as page-locked operands and as the reference."""
    P = gpu_lib
    A = P.fill_baseline(W, m, k, 7, wide=True)
    B = P.fill_baseline(W, k, n, 8, wide=True)
    Cpage = P.MPMatrix(W, m, n)
    Cpage.data[...] = 9.0
    P.matmul_block_parallel_into(Cpage, A, B)
    Ap, Bp = A.copy(pinned=True), B.copy(pinned=True)
    Cpin = P.MPMatrix(W, m, n, pinned=True)
    P.matmul_block_parallel_into(Cpin, Ap, Bp)
    assert P.bits_equal(Cpage, Cpin)
    rows = [0, m // 3, m - 1]
    want = O.ref_gemm(np.ascontiguousarray(A.data[:, rows]), B.data, k, n)
    assert mismatches(Cpage.data[:, rows], want) == 0


@pytest.mark.parametrize("W,m,n,k", [(2, 700, 300, 1100), (3, 257, 129, 2000), (4, 100, 40, 5000),
                                     (2, 33, 7, 17), (3, 1, 1, 600)])
def test_gated_host_path_bitwise(gpu_lib, W, m, n, k, monkeypatch):
    """Page-locked host operands on one GPU take the copy-engine-gated single
    launch when it pays (K panels flagged by stream memory writes, row bands
    downloaded on stream wait-values); it must give the reference's bits and
    the same bits as the row-chunked path (MPFK_CHUNKED_HOST=1)."""
    P = gpu_lib
    A = P.fill_baseline(W, m, k, 11, wide=True, pinned=True)
    B = P.fill_baseline(W, k, n, 12, wide=True, pinned=True)
    Cg = P.MPMatrix(W, m, n, pinned=True)
    Cg.data[...] = 5.0
    P.matmul_block_parallel_into(Cg, A, B)
    gated = P.last_stats()["kernel_launches"] == 1
    monkeypatch.setenv("MPFK_CHUNKED_HOST", "1")
    Cc = P.MPMatrix(W, m, n, pinned=True)
    P.matmul_block_parallel_into(Cc, A, B)
    assert P.bits_equal(Cg, Cc)
    want = O.ref_gemm(A.data, B.data, k, n)
    assert mismatches(Cg.data, want) == 0
    assert gated or k < 256  # these shapes are small enough for the gated path


def test_out_of_memory_is_memory_error(gpu_lib):
    """an impossible allocation maps to MPFK_ENOMEM -> MemoryError (the
    reference's std::bad_alloc, linalg.hpp:116), and the library stays usable"""
    P = gpu_lib
    with pytest.raises(MemoryError):
        P.device_alloc(1 << 50)
    A = P.fill_baseline(2, 40, 30, 1)
    B = P.fill_baseline(2, 30, 20, 2)
    assert mismatches(P.matmul_block(A, B).data, O.ref_gemm(A.data, B.data, 30, 20)) == 0


def test_shutdown_and_reinitialise(gpu_lib):
    """mpfk_shutdown releases every device resource (streams, events, buffers,
    staging ring, flag buffers); the next call initialises again and gives the
    same bits, for the host, device, gated and staged paths"""
    import torch
    P = gpu_lib
    W, m, n, k = 3, 300, 200, 700
    A = P.fill_baseline(W, m, k, 5, wide=True, pinned=True)
    B = P.fill_baseline(W, k, n, 6, wide=True, pinned=True)
    Ap = P.fill_baseline(W, m, k, 5, wide=True)  # pageable copies
    Bp = P.fill_baseline(W, k, n, 6, wide=True)
    want = O.ref_gemm(A.data, B.data, k, n)
    for _ in range(2):
        C1 = P.MPMatrix(W, m, n, pinned=True)
        P.matmul_block_parallel_into(C1, A, B)
        C2 = P.matmul_block(Ap, Bp)
        assert mismatches(C1.data, want) == 0 and mismatches(C2.data, want) == 0
        dA, dB = torch.from_numpy(A.data).cuda(), torch.from_numpy(B.data).cuda()
        dC = torch.zeros((W, m, B.stride()), dtype=torch.float64, device="cuda")
        P.gemm_device(W, m, n, k, dA.data_ptr(), A.stride(), m * A.stride(), dB.data_ptr(), B.stride(),
                      k * B.stride(), dC.data_ptr(), B.stride(), m * B.stride())
        torch.cuda.synchronize()
        assert mismatches(dC.cpu().numpy(), want) == 0
        N.lib().mpfk_shutdown()
