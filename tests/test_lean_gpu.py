"""MPFK_LEAN on the B200 (csrc/mpf_lean.cuh through the GEMM kernels): the
tolerance mode of the north star -- fewer FP64 instructions per
multiply-add, NOT bit-identical to the reference.  What must hold:
  * every element is exactly the chain the same source computes on the host
    (tests/csrc/arith_host.cpp: hst_lean_gemm), for ragged shapes, edges and
    k-tile remainders -- so the result does not depend on tiles, grids or
    row shards;
  * the result is within the north star's normwise 4*k*u_p of the exact
    product (dyadic oracle) and of the bit-exact GEMM at the BASELINE sizes;
  * canonical values, +0 pads, op counters, flags validation, and
    MPFK_BIT_EXACT untouched by any of it."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from oracle import dyadic
from tests.helpers import mismatches

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}  # north star


@pytest.fixture(scope="module")
def H():
    L = C.CDLL(os.path.join(HERE, "_build", "libarith_host.so"))
    L.hst_lean_gemm.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                                C.c_size_t, C.c_void_p, C.c_size_t]
    return L


def device_lean(P, W, A, B, m, n, k, flags=None, sentinel=None):
    import torch
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ldc = n + (n & 1) + 2
    fill = 0.0 if sentinel is None else sentinel
    dC = torch.full((W, m, ldc), fill, dtype=torch.float64, device="cuda")
    launches = P.gemm_device_ex(W, m, n, k, dA.data_ptr(), A.shape[2], A.shape[1] * A.shape[2], dB.data_ptr(),
                                B.shape[2], B.shape[1] * B.shape[2], dC.data_ptr(), ldc, m * ldc,
                                P.LEAN if flags is None else flags)
    torch.cuda.synchronize()
    return dC.cpu().numpy(), launches


def host_lean(H, W, A, B, m, n, k):
    Cm = np.zeros((W, m, n))
    assert H.hst_lean_gemm(W, m, k, n, A.ctypes.data, A.shape[2], B.ctypes.data, B.shape[2], Cm.ctypes.data, n) == 0
    return Cm


SHAPES = [(37, 41, 29), (64, 64, 64), (70, 130, 33), (9, 5, 300), (130, 33, 47), (33, 70, 16), (1, 1, 1)]


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_lean_device_is_the_host_chain(gpu_lib, H, W, m, n, k):
    P = gpu_lib
    A = O.orc_fill_baseline(W, m, k, 31 + m, wide=True)
    B = O.orc_fill_baseline(W, k, n, 32 + n, wide=True)
    got, launches = device_lean(P, W, A, B, m, n, k, sentinel=5.0)
    assert launches == 1
    want = host_lean(H, W, A, B, m, n, k)
    assert mismatches(got[:, :, :n], want) == 0
    assert np.all(got[:, :, n:] == 5.0)  # only the m x n cells are written
    # and it is not the reference's arithmetic: the bit-exact path still is
    ref = O.ref_gemm(A, B, k, n) if O.ref_available() else O.orc_gemm(A, B, k, n)
    exact, _ = device_lean(P, W, A, B, m, n, k, flags=P.BIT_EXACT)
    assert mismatches(exact[:, :, :n], ref[:, :, :n]) == 0


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_special_values_host_chain(gpu_lib, H, W):
    """zeros of both signs, integers, powers of two, non-normalised operands"""
    from tests.helpers import special_matrix
    P = gpu_lib
    m, n, k = 40, 36, 50
    A = special_matrix(W, m, k, 11 + W)
    B = special_matrix(W, k, n, 21 + W)
    got, _ = device_lean(P, W, A, B, m, n, k)
    assert mismatches(got[:, :, :n], host_lean(H, W, A, B, m, n, k)) == 0


def normwise_err(Cm, exact, rows, cols):
    num = den = 0.0
    for i in range(rows):
        for j in range(cols):
            ex = exact[i][j]
            num = max(num, abs(float(dyadic.from_components(Cm[:, i, j]) - ex)))
            den = max(den, abs(float(ex)))
    return num / den


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("wide", [False, True])
def test_lean_within_tolerance_of_exact(gpu_lib, W, wide):
    P = gpu_lib
    m, n, k = 6, 5, 3000
    A = O.orc_fill_baseline(W, m, k, 11, wide=wide)
    B = O.orc_fill_baseline(W, k, n, 12, wide=wide)
    got, _ = device_lean(P, W, A, B, m, n, k)
    exact = dyadic.matmul_exact(A, B, k, n)
    err = normwise_err(got, exact, m, n)
    assert err <= 4 * k * U_P[W], err
    assert err <= 0.02 * 4 * k * U_P[W], err / (4 * k * U_P[W])  # measured: 2e-4 .. 4e-3 of the tolerance
    # canonical values: each component at most half an ulp of the one before
    for w in range(1, W):
        hi, lo = np.abs(got[w - 1, :, :n]), np.abs(got[w, :, :n])
        assert np.all(lo <= np.spacing(hi) / 2)


def planes_diff(a, b, W, n):
    """max |a - b| / max |b| summing component differences from the smallest
    up (the leading components cancel exactly where the results agree)"""
    d = a[W - 1] - b[W - 1]
    for w in range(W - 2, -1, -1):
        d = d + (a[w] - b[w])
    return float(np.abs(d[:, :n]).max() / np.abs(b[0][:, :n]).max())


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_vs_bit_exact_n1024(gpu_lib, W):
    """BASELINE configs[0-2] (n = 1024): lean vs the bit-exact product, itself
    verified against the reference elsewhere; both are within 4*k*u_p of the
    exact product, so they differ by at most twice that -- measured ~1e-3"""
    import torch
    P = gpu_lib
    n = 1024
    A = P.fill_baseline(W, n, n, 1).data
    B = P.fill_baseline(W, n, n, 2).data
    lean, _ = device_lean(P, W, A, B, n, n, n)
    exact, _ = device_lean(P, W, A, B, n, n, n, flags=P.BIT_EXACT)
    d = planes_diff(lean, exact, W, n)
    assert 0 < d <= 0.05 * 4 * n * U_P[W], d / (4 * n * U_P[W])
    # deterministic
    again, _ = device_lean(P, W, A, B, n, n, n)
    assert mismatches(lean, again) == 0
    # independent of the row shard: rows [320, 711) on their own
    r0, r1 = 320, 711
    part, _ = device_lean(P, W, np.ascontiguousarray(A[:, r0:r1]), B, r1 - r0, n, n)
    assert mismatches(part[:, :, :n], lean[:, r0:r1, :n]) == 0
    torch.cuda.empty_cache()


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_host_api(gpu_lib, H, W):
    """mpfk_gemm(flags = MPFK_LEAN) with host matrices: the same chains, +0
    pads, op counters like count_matmul; chunked rows and K panels of the
    host pipeline stay within tolerance of the one-shot chain"""
    P = gpu_lib
    m, k, n = 70, 45, 37
    A = P.MPMatrix.from_planes(O.orc_fill_baseline(W, m, k, 3, wide=True)[:, :, :k])
    B = P.MPMatrix.from_planes(O.orc_fill_baseline(W, k, n, 4, wide=True)[:, :, :n])
    P.op_counters_reset()
    Cm = P.gemm(A, B, flags=P.LEAN)
    c = P.op_counters_read()
    assert (c.muls, c.adds) == (m * n * k, m * n * (k - 1))
    want = host_lean(H, W, np.ascontiguousarray(A.data), np.ascontiguousarray(B.data), m, n, k)
    assert mismatches(np.ascontiguousarray(Cm.data[:, :, :n]), want) == 0
    assert np.all(Cm.data[:, :, n:] == 0) and not np.any(np.signbit(Cm.data[:, :, n:]))
    # a shape the host pipeline cuts into row chunks and K panels
    n2 = 1536
    A2, B2 = P.fill_baseline(W, n2, n2, 5), P.fill_baseline(W, n2, n2, 6)
    C2 = P.gemm(A2, B2, flags=P.LEAN)
    E2 = P.matmul_block(A2, B2)
    d = planes_diff(C2.data, E2.data, W, n2)
    assert d <= 0.05 * 4 * n2 * U_P[W], d / (4 * n2 * U_P[W])
    assert np.all(C2.data[:, :, n2:] == 0)


def test_lean_flags(gpu_lib):
    P = gpu_lib
    W, m, n, k = 2, 8, 8, 1 << 13
    A = O.orc_fill_baseline(W, m, k, 1)
    B = O.orc_fill_baseline(W, k, n, 2)
    assert P.splitk_segments(W, m, n, k) > 1
    # FAST | LEAN where FAST splits K: the FAST result (segments keep the reference's arithmetic)
    both, l_both = device_lean(P, W, A, B, m, n, k, flags=P.FAST | P.LEAN)
    fast, l_fast = device_lean(P, W, A, B, m, n, k, flags=P.FAST)
    assert l_both == l_fast == 2 and mismatches(both, fast) == 0
    # ... and where it does not: the LEAN result
    m2 = n2 = 300
    k2 = 200
    A2 = O.orc_fill_baseline(W, m2, k2, 3)
    B2 = O.orc_fill_baseline(W, k2, n2, 4)
    assert P.splitk_segments(W, m2, n2, k2) == 1
    both, _ = device_lean(P, W, A2, B2, m2, n2, k2, flags=P.FAST | P.LEAN)
    lean, _ = device_lean(P, W, A2, B2, m2, n2, k2, flags=P.LEAN)
    assert mismatches(both, lean) == 0
    with pytest.raises(ValueError, match="unknown flags"):
        device_lean(P, W, A2, B2, m2, n2, k2, flags=4)
    # k == 0: +0
    dC, _ = device_lean(P, W, A2, B2, m2, n2, 0, sentinel=3.0)
    assert np.all(dC[:, :, :n2] == 0)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_paper_matrices_digit_loss(gpu_lib, W):
    """acceptance criterion 5 (acceptance.cpp:286-337) for the tolerance mode:
    the paper's generator matrices (exactly representable entries that drive
    the reference's renorm5 paths B/C/D) lose at most 2.5 digits against the
    exact product, componentwise, like the reference's own algorithms"""
    P = gpu_lib
    for n in (64, 256):
        rows = (0, 8) if n == 256 else (0, n)
        A, B = P.gen_paper_matrices(W, n)
        exact = dyadic.matmul_exact(A.data, B.data, n, n, rows=rows)
        Cm = P.gemm(A, B, flags=P.LEAN)
        dl = dyadic.digit_loss(dyadic.max_rel_err(Cm.data, exact, rows=rows), P.format_eps(W))
        assert dl <= 2.5, (n, dl)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_k_panels_and_staged_gather(gpu_lib, W):
    """MPFK_LEAN through the K-panel continuation (mpfk_gemm_device_acc_ex) and
    the staged all-gather -> GEMM (mpfk_gemm_device_staged_ex): the staged
    call equals its panel schedule replayed by hand, bitwise; a panelled lean
    product is within the tolerance of the bit-exact one (each panel ends
    with the lean form's normalisation, so it is not the one-shot chain)."""
    import torch
    from tests.test_staged_gpu import expected_panels
    P = gpu_lib
    m, k, n = 70, 1000, 66
    cuts = [0, 1, 100, 500, 930, 1000]
    A = O.orc_fill_baseline(W, m, k, 41, wide=True)
    B = O.orc_fill_baseline(W, k, n, 42, wide=True)
    ld = B.shape[2]
    dA, dBfull = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    dB = torch.full((W, k, ld), float("nan"), dtype=torch.float64, device="cuda")
    dC = torch.full((W, m, ld), 7.0, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        launches = P.gemm_device_staged(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld,
                                        k * ld, dC.data_ptr(), ld, m * ld, [t.data_ptr() for t in slices], cuts,
                                        16, s.cuda_stream, flags=P.LEAN)
    s.synchronize()
    panels = expected_panels(k, 16)
    assert launches == len(panels) - 1
    assert np.array_equal(dB.cpu().numpy().view(np.uint64), B.view(np.uint64))
    # the same schedule by hand
    dH = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    for p, (k0, k1) in enumerate(zip(panels, panels[1:])):
        a_ptr, b_ptr = dA.data_ptr() + 8 * k0, dBfull.data_ptr() + 8 * k0 * ld
        if p == 0:
            P.gemm_device_ex(W, m, n, k1 - k0, a_ptr, A.shape[2], m * A.shape[2], b_ptr, ld, k * ld, dH.data_ptr(),
                             ld, m * ld, P.LEAN)
        else:
            P.gemm_device_acc(W, m, n, k1 - k0, a_ptr, A.shape[2], m * A.shape[2], b_ptr, ld, k * ld, dH.data_ptr(),
                              ld, m * ld, flags=P.LEAN)
    torch.cuda.synchronize()
    got, hand = dC.cpu().numpy(), dH.cpu().numpy()
    assert mismatches(got[:, :, :n], hand[:, :, :n]) == 0
    assert (got[:, :, n:] == 7.0).all()
    ref = O.ref_gemm(A, B, k, n)
    d = planes_diff(got, ref, W, n)
    assert d <= 0.05 * 4 * k * U_P[W], d / (4 * k * U_P[W])
    with pytest.raises(ValueError, match="MPFK_LEAN only"):
        P.gemm_device_acc(W, m, n, 16, dA.data_ptr(), A.shape[2], m * A.shape[2], dBfull.data_ptr(), ld, k * ld,
                          dH.data_ptr(), ld, m * ld, flags=P.FAST)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_lean_edge_shapes_exact_small_values(gpu_lib, W):
    """empty and one-element shapes through the host API; products of small
    exactly representable values are exact in both modes, so they agree
    bitwise, pads +0"""
    P = gpu_lib
    for (m, k, n) in [(0, 5, 3), (4, 0, 3), (4, 5, 0), (1, 1, 1), (33, 1, 2), (2, 17, 1)]:
        A, B = P.MPMatrix(W, m, k), P.MPMatrix(W, k, n)
        if m and k:
            A.data[0, :, :k] = 1.5
        if k and n:
            B.data[0, :, :n] = -2.0
        Cm = P.gemm(A, B, flags=P.LEAN)
        E = P.matmul_block(A, B)
        assert Cm.data.shape == E.data.shape
        if m and n:
            assert np.array_equal(Cm.data, E.data), (W, m, k, n)
            assert not np.signbit(Cm.data[:, :, n:]).any()
