"""GPU parity: libmpfk's sm_100a GEMM vs the reference GEMM (oracle/_ref, the
unmodified mpfkit compiled here) and the C restatement (oracle/_build), bit
for bit, through the product's public API (the C ABI via ctypes).

Mirrors the reference's hot-path tests:
  test_linalg.cpp:194-218 identity passthrough, ones x ones = twos
  test_linalg.cpp:220-248 block == naive bitwise incl. rectangular 7x12 . 12x9
  test_linalg.cpp:308-330 parallel == serial, _into clears stale C
  test_linalg.cpp:347-363 op counters
  acceptance.cpp:240-282  criterion 4 (n in {4,8,16,33}, all widths)
  acceptance.cpp:286-337  criterion 5 paper matrices n = 64, 256
  acceptance.cpp:363-395  criterion 7 n = 256, workers {1,2,4,8}
plus the BASELINE.json configurations (full compare at n = 1024, sampled rows
at the sharded sizes).
"""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed, special_matrix, to_mp

pytestmark = pytest.mark.gpu

WIDTHS = (2, 3, 4)


def gpu_gemm(P, A, B, K, n, workers=1):
    Am, Bm = to_mp(A, K), to_mp(B, n)
    Cm = P.matmul_block_parallel(Am, Bm, 32, P.KernelVariant.SIMD_LOADSTORE, workers)
    return Cm.data


def check_vs_reference(P, A, B, K, n, workers=1):
    got = gpu_gemm(P, A, B, K, n, workers)
    want = O.ref_gemm(A, B, K, n)
    assert mismatches(got, want) == 0
    # padding cells are +0 (linalg.hpp:98-106)
    assert not got[:, :, n:].view(np.uint64).any()
    return got


@pytest.mark.parametrize("W", WIDTHS)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 16, 31, 32, 33, 63, 64, 65, 100])
def test_square_random_bitwise(gpu_lib, W, n):
    A = random_signed(W, n, n, 430 + n)
    B = random_signed(W, n, n, 431 + n)
    got = check_vs_reference(gpu_lib, A, B, n, n)
    assert mismatches(got, O.orc_gemm(A, B, n, n)) == 0


@pytest.mark.parametrize("W", WIDTHS)
@pytest.mark.parametrize("m,k,n", [(7, 12, 9), (1, 1000, 1), (130, 3, 70), (65, 129, 33), (200, 1, 200),
                                   (3, 517, 250)])
def test_rectangular_bitwise(gpu_lib, W, m, k, n):
    A = random_signed(W, m, k, 460 + m)
    B = random_signed(W, k, n, 461 + n)
    check_vs_reference(gpu_lib, A, B, k, n)


@pytest.mark.parametrize("W", WIDTHS)
def test_special_values_bitwise(gpu_lib, W):
    """signed zeros, exact integers, powers of two: the zero-residual corners
    of renorm5 (eft.hpp:261-286) and vseb (eft.hpp:216-224)."""
    for seed, (m, k, n) in enumerate([(40, 40, 40), (17, 64, 23), (64, 7, 64)]):
        A = special_matrix(W, m, k, 900 + seed)
        B = special_matrix(W, k, n, 950 + seed)
        check_vs_reference(gpu_lib, A, B, k, n)


@pytest.mark.parametrize("W", WIDTHS)
def test_identity_and_ones(gpu_lib, W):
    P = gpu_lib
    b = random_signed(W, 4, 5, 420 + W)
    eye = O.planes(W, 4, 4)
    for i in range(4):
        eye[0, i, i] = 1.0
    got = gpu_gemm(P, eye, b, 4, 5)
    assert mismatches(got, b) == 0
    ones = O.planes(W, 2, 2)
    ones[0, :, :2] = 1.0
    twos = gpu_gemm(P, ones, ones, 2, 2)
    assert (twos[0, :, :2] == 2.0).all() and not twos[1:, :, :2].view(np.uint64).any()


@pytest.mark.parametrize("W", WIDTHS)
@pytest.mark.parametrize("n", [4, 8, 16, 33])
def test_criterion4_fill_random(gpu_lib, W, n):
    """acceptance.cpp:240-282: bench::fill_random inputs, bitwise vs reference
    and within n*4*format_eps of the exact product."""
    from oracle import dyadic
    A = O.ref_fill_random(W, n, n, 4000 + 10 * W + n)
    B = O.ref_fill_random(W, n, n, 4001 + 10 * W + n)
    got = check_vs_reference(gpu_lib, A, B, n, n)
    rows = (0, n) if n <= 16 else (0, 6)
    exact = dyadic.matmul_exact(A, B, n, n, rows=rows)
    err = dyadic.max_rel_err(got, exact, rows=rows)
    assert err <= n * 4.0 * gpu_lib.format_eps(W)


@pytest.mark.parametrize("W", WIDTHS)
@pytest.mark.parametrize("n", [64, 256])
def test_criterion5_paper_matrices(gpu_lib, W, n):
    """acceptance.cpp:286-337: the paper's generators (renorm5 paths B/C/D)."""
    A, B = O.ref_gen_paper(W, n)
    Ao, Bo = O.orc_gen_paper(W, n)
    assert mismatches(A, Ao) == 0 and mismatches(B, Bo) == 0
    got = check_vs_reference(gpu_lib, A, B, n, n)
    if n == 64:
        from oracle import dyadic
        exact = dyadic.matmul_exact(A, B, n, n, rows=(0, 8))
        loss = dyadic.digit_loss(dyadic.max_rel_err(got, exact, rows=(0, 8)), gpu_lib.format_eps(W))
        assert loss <= 2.5


@pytest.mark.parametrize("W", WIDTHS)
def test_criterion7_workers(gpu_lib, W):
    """acceptance.cpp:363-395 / test_linalg.cpp:308-330: any worker (GPU)
    count is bit-identical; _into clears stale C."""
    P = gpu_lib
    n = 256
    A = O.ref_fill_random(W, n, n, 7000 + W)
    B = O.ref_fill_random(W, n, n, 7001 + W)
    want = O.ref_gemm(A, B, n, n)
    for w in (1, 2, 4, 8):
        assert mismatches(gpu_gemm(P, A, B, n, n, workers=w), want) == 0
    Am, Bm = to_mp(A, n), to_mp(B, n)
    Cm = P.MPMatrix(W, n, n)
    Cm.data[...] = 7.0
    P.matmul_block_into(Cm, Am, Bm, 8, P.KernelVariant.SIMD_SET)
    assert mismatches(Cm.data, want) == 0
    P.matmul_naive_into(Cm, Am, Bm)
    assert mismatches(Cm.data, want) == 0


def test_op_counters(gpu_lib):
    """test_linalg.cpp:347-363: 4x4 -> muls 64, adds 48."""
    P = gpu_lib
    A = random_signed(2, 4, 4, 530)
    B = random_signed(2, 4, 4, 531)
    P.op_counters_reset()
    P.matmul_naive(to_mp(A, 4), to_mp(B, 4))
    c = P.op_counters_read()
    assert (c.muls, c.adds, c.leaf_multiplies) == (64, 48, 0)


@pytest.mark.parametrize("W", WIDTHS)
def test_degenerate_shapes(gpu_lib, W):
    P = gpu_lib
    # K == 0: C is all +0 (fill_zero, no products)
    A, B = P.MPMatrix(W, 5, 0), P.MPMatrix(W, 0, 6)
    C = P.MPMatrix(W, 5, 6)
    C.data[...] = 3.0
    P.matmul_block_into(C, A, B)
    assert not C.data.view(np.uint64).any()
    # empty results
    for (m, k, n) in [(0, 3, 4), (3, 4, 0), (0, 0, 0)]:
        A, B = P.MPMatrix(W, m, k), P.MPMatrix(W, k, n)
        C = P.matmul_block(A, B)
        assert (C.rows(), C.cols()) == (m, n)


@pytest.mark.parametrize("W", WIDTHS)
def test_baseline_config_n1024_full(gpu_lib, W):
    """BASELINE.json configs 0-2: n = 1024, full bitwise compare against the
    reference's multithreaded CPU GEMM on identical inputs."""
    P = gpu_lib
    n = 1024
    A = P.fill_baseline(W, n, n, 1, wide=False)
    B = P.fill_baseline(W, n, n, 2, wide=False)
    C = P.matmul_block_parallel(A, B, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
    want = O.ref_gemm(A.data, B.data, n, n)
    assert mismatches(C.data, want) == 0


@pytest.mark.parametrize("W,n,wide", [(2, 8192, False), (3, 4096, True), (4, 4096, True)])
def test_baseline_config_sharded_sampled_rows(gpu_lib, W, n, wide):
    """BASELINE.json configs 3-4 at full size: rows of C are independent
    (linalg.hpp:399-401), so a bitwise check of sampled rows against the
    reference's GEMM on those rows of A is exact evidence for them."""
    P = gpu_lib
    A = P.fill_baseline(W, n, n, 11, wide=wide)
    B = P.fill_baseline(W, n, n, 12, wide=wide)
    C = P.matmul_block_parallel(A, B, 32, P.KernelVariant.SIMD_LOADSTORE, 8)
    rows = [0, 1, n // 2 + 3, n - 1]
    sub = np.ascontiguousarray(A.data[:, rows, :])
    want = O.ref_gemm(sub, B.data, n, n)
    assert mismatches(C.data[:, rows, :], want) == 0


@pytest.mark.parametrize("W,n,wide,nrows", [(2, 8192, False, 64), (3, 4096, True, 24), (4, 4096, True, 16)])
def test_baseline_config_device_path_sampled_rows(gpu_lib, W, n, wide, nrows):
    """The bench's device-resident path (mpfk_gemm_device, the kernel timed
    for `value`) at the BASELINE full sizes: rows at tile edges (31/32, 63/64),
    in the first and last tile bands and seeded random ones, bitwise against
    the reference GEMM on those rows of A."""
    import torch
    P = gpu_lib
    A = P.fill_baseline(W, n, n, 21, wide=wide).data
    B = P.fill_baseline(W, n, n, 22, wide=wide).data
    ld = A.shape[2]
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros_like(dA)
    P.gemm_device(W, n, n, n, dA.data_ptr(), ld, n * ld, dB.data_ptr(), ld, n * ld, dC.data_ptr(), ld, n * ld)
    torch.cuda.synchronize()
    rng = np.random.default_rng(n + W)
    fixed = [0, 31, 32, 63, 64, n // 2 - 1, n // 2, n - 65, n - 64, n - 33, n - 32, n - 1]
    rows = sorted(set(fixed[:nrows // 2] + fixed[-(nrows // 4):] +
                      rng.integers(0, n, nrows - nrows // 2 - nrows // 4).tolist()))
    sub = np.ascontiguousarray(A[:, rows, :])
    want = O.ref_gemm(sub, B, n, n)
    got = dC[:, rows, :].cpu().numpy()
    assert mismatches(got, want) == 0, rows


@pytest.mark.parametrize("W", WIDTHS)
def test_elementwise_kernels_bitwise(gpu_lib, W):
    """acceptance.cpp criterion 2 analog: device mpf::add/mul<W> lanewise
    bit-identical to the reference scalar kernels on 2e5 signed pairs."""
    P = gpu_lib
    import ctypes as C
    count = 200_000
    st = (C.c_uint64 * 1)(3000 + W)
    x = np.zeros((count, W))
    y = np.zeros((count, W))
    for arr in (x, y):
        for i in range(count):
            O.ref().ref_random_normalized(W, C.cast(st, C.c_void_p), 1, arr[i].ctypes.data)
    rng = np.random.default_rng(W)
    y *= np.ldexp(1.0, rng.integers(-60, 60, size=(count, 1)))
    for op in ("add", "mul"):
        assert mismatches(P.binop_batch(W, op, x, y).T[:, :, None], O.ref_binop_batch(W, op, x, y).T[:, :, None]) == 0


def test_device_api_with_torch_stream(gpu_lib):
    """mpfk_gemm_device on torch-owned device memory and torch's stream."""
    import torch
    P = gpu_lib
    W, m, k, n = 3, 70, 45, 38
    A = random_signed(W, m, k, 77)
    B = random_signed(W, k, n, 78)
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.zeros((W, m, B.shape[2]), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    launches = P.gemm_device(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), B.shape[2],
                             k * B.shape[2], dC.data_ptr(), B.shape[2], m * B.shape[2], s.cuda_stream)
    s.synchronize()
    assert launches == 1
    assert mismatches(dC.cpu().numpy(), O.ref_gemm(A, B, k, n)) == 0


@pytest.mark.parametrize("W", WIDTHS)
def test_k_panel_continuation_bitwise(gpu_lib, W):
    """C from mpfk_gemm_device over panel 0 then mpfk_gemm_device_acc over
    the remaining K panels (uneven, even-aligned splits) == one-shot C ==
    reference: the chain state between k steps is exactly C (linalg.hpp:261)."""
    import torch
    P = gpu_lib
    m, k, n = 45, 203, 37
    A = random_signed(W, m, k, 880 + W)
    B = random_signed(W, k, n, 890 + W)
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    lda, ldb = A.shape[2], B.shape[2]
    dC = torch.zeros((W, m, ldb), dtype=torch.float64, device="cuda")
    cuts = [0, 16, 18, 100, 150, k]
    for p, (k0, k1) in enumerate(zip(cuts, cuts[1:])):
        f = P.gemm_device if p == 0 else P.gemm_device_acc
        f(W, m, n, k1 - k0, dA.data_ptr() + 8 * k0, lda, m * lda, dB.data_ptr() + 8 * k0 * ldb, ldb, k * ldb,
          dC.data_ptr(), ldb, m * ldb)
    torch.cuda.synchronize()
    assert mismatches(dC.cpu().numpy(), O.ref_gemm(A, B, k, n)) == 0


@pytest.mark.parametrize("W", WIDTHS)
@pytest.mark.parametrize("scale", [-520, -560, 480])
def test_extreme_magnitudes_bitwise(gpu_lib, W, scale):
    """Products in the subnormal range (two_prod's error term underflows,
    eft.hpp:61-62) and near the top of the exponent range: both sides follow
    IEEE binary64 without flush-to-zero, so the bits must still agree."""
    n = 24
    A = random_signed(W, n, n, 700 + W) * np.ldexp(1.0, scale)
    B = random_signed(W, n, n, 710 + W) * np.ldexp(1.0, scale if scale < 0 else 20)
    check_vs_reference(gpu_lib, A, B, n, n)
