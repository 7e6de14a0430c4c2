"""MPFK_FAST ("flags selects BIT_EXACT (default) or FAST
(reordered, tolerance-checked)").  FAST splits K only when the output is too
small to fill the GPU; it must then stay within the north star's normwise
4*k*u_p of the exact product (dyadic oracle, the restatement of
oracle.cpp:176-193), be deterministic, and everywhere else be the bit-exact
path itself."""
import numpy as np
import pytest

import oracle as O
from oracle import dyadic
from tests.helpers import mismatches

pytestmark = pytest.mark.gpu

U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}  # north star


def test_plan(gpu_lib):
    P = gpu_lib
    assert P.splitk_segments(2, 4096, 4096, 4096) == 1  # fills the GPU: bit-exact
    assert P.splitk_segments(3, 64, 64, 400) == 1       # k < 512
    for W in (2, 3, 4):
        s = P.splitk_segments(W, 8, 8, 1 << 16)
        assert 1 < s <= 4096
    with pytest.raises(ValueError, match="width"):
        P.splitk_segments(5, 8, 8, 8)


def normwise_err(Cm, exact, rows, cols):
    num = 0.0
    den = 0.0
    for i in range(rows):
        for j in range(cols):
            ex = exact[i][j]
            d = dyadic.from_components(Cm[:, i, j]) - ex
            num = max(num, abs(float(d)))
            den = max(den, abs(float(ex)))
    return num / den


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("signed", [False, True])
def test_fast_within_tolerance(gpu_lib, W, signed):
    P = gpu_lib
    m, n, k = 6, 5, 3000
    if signed:
        A = P.MPMatrix.from_planes(O.orc_fill_baseline(W, m, k, 11, wide=True)[:, :, :k])
        B = P.MPMatrix.from_planes(O.orc_fill_baseline(W, k, n, 12, wide=True)[:, :, :n])
    else:
        A = P.fill_random(W, m, k, 11)
        B = P.fill_random(W, k, n, 12)
    assert P.splitk_segments(W, m, n, k) > 1
    Cf = P.gemm(A, B, flags=P.FAST)
    Ce = P.gemm(A, B, flags=P.BIT_EXACT)
    assert mismatches(Ce.data, O.ref_gemm(A.data, B.data, k, n)) == 0  # BIT_EXACT is the reference
    exact = dyadic.matmul_exact(A.data, B.data, k, n)
    err = normwise_err(Cf.data, exact, m, n)
    assert err <= 4 * k * U_P[W], err  # tolerance of the north star
    if not signed:  # positive inputs: componentwise, like test_linalg.cpp:250-268
        worst = dyadic.max_rel_err(Cf.data, exact)
        assert worst <= 4 * k * U_P[W], worst
    Cf2 = P.gemm(A, B, flags=P.FAST)
    assert P.bits_equal(Cf, Cf2)  # deterministic
    assert np.all(Cf.data[:, :, n:] == 0)  # pads +0


@pytest.mark.parametrize("W", [2, 3, 4])
def test_fast_device_ragged_segments(gpu_lib, W):
    """device entry point, k not a multiple of the segment length (the
    ragged last segment through GemmArgs::klast), submatrix strides."""
    import torch
    P = gpu_lib
    m, n, k = 40, 33, 5001
    A = O.orc_fill_baseline(W, m, k, 21, wide=True)
    B = O.orc_fill_baseline(W, k, n, 22, wide=True)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ldc = 40
    dC = torch.full((W, m, ldc), 5.0, dtype=torch.float64, device="cuda")
    segs = P.splitk_segments(W, m, n, k)
    assert segs > 1
    launches = P.gemm_device_ex(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), B.shape[2],
                                k * B.shape[2], dC.data_ptr(), ldc, m * ldc, P.FAST)
    torch.cuda.synchronize()
    assert launches == 2
    got = dC.cpu().numpy()
    assert np.all(got[:, :, n:] == 5.0)  # only the m x n cells are written
    rows = [0, 17, 39]
    exact = [dyadic.matmul_exact(A, B, k, n, rows=(i, i + 1))[0] for i in rows]
    sub = np.ascontiguousarray(got[:, rows, :])
    err = normwise_err(sub, exact, len(rows), n)
    assert err <= 4 * k * U_P[W], err
    # the fold order is fixed: equal to folding the segment products of the
    # bit-exact kernel in order on the host
    ks = ((k + segs - 1) // segs + 15) // 16 * 16
    parts = []
    for s0 in range(0, k, ks):
        s1 = min(k, s0 + ks)
        parts.append(O.ref_gemm(np.ascontiguousarray(A[:, :, s0:s1]), np.ascontiguousarray(B[:, s0:s1]),
                                s1 - s0, n))
    assert len(parts) == segs
    acc = parts[0]
    for p in parts[1:]:
        acc = O.ref_ew(W, "add", acc, p, n)
    assert mismatches(got[:, :, :n], acc[:, :, :n]) == 0


@pytest.mark.parametrize("W", [2, 3, 4])
def test_fast_is_bit_exact_when_not_split(gpu_lib, W):
    P = gpu_lib
    m, n, k = 300, 260, 200
    A = P.fill_baseline(W, m, k, 1, wide=True)
    B = P.fill_baseline(W, k, n, 2, wide=True)
    assert P.splitk_segments(W, m, n, k) == 1
    assert P.bits_equal(P.gemm(A, B, flags=P.FAST), P.matmul_block(A, B))


def test_gemm_validation(gpu_lib):
    P = gpu_lib
    A = P.MPMatrix(2, 4, 5)
    with pytest.raises(ValueError, match="inner dimensions differ"):
        P.gemm(A, P.MPMatrix(2, 6, 3))
    with pytest.raises(ValueError, match="unknown flags"):
        P.gemm(A, P.MPMatrix(2, 5, 3), flags=4)
    C = P.MPMatrix(2, 4, 4)
    with pytest.raises(ValueError, match="result shape mismatch"):
        P.gemm_into(C, A, P.MPMatrix(2, 5, 3))
