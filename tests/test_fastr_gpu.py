"""TD/QD GEMM with the branch-free renormalisation (TileCfg::FASTR,
gemm_kernel.cuh): every k-tile runs renorm5's paths A/B only
(eft.hpp:255-260) and a warp whose inputs needed paths C/D (eft.hpp:261-286,
a zero residual) restores its chains from the snapshot taken at the k-tile
start and recomputes the k-tile with the exact form.  The recomputation must
actually happen on such inputs (mpfk_gemm_redo_count) and the result must
stay bit-identical to the reference GEMM (linalg.hpp:338-344), including
when only some warps of a tile redo."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed, special_matrix

pytestmark = pytest.mark.gpu


def device_gemm(P, A, B, m, k, n):
    import torch
    W = A.shape[0]
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    lda, ldb = A.shape[2], B.shape[2]
    dC = torch.full((W, m, ldb), float("nan"), dtype=torch.float64, device="cuda")
    P.gemm_device(W, m, n, k, dA.data_ptr(), lda, m * lda, dB.data_ptr(), ldb, k * ldb, dC.data_ptr(), ldb,
                  m * ldb)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


@pytest.mark.parametrize("W", (3, 4))
def test_redo_on_zero_residual_inputs(gpu_lib, W):
    P = gpu_lib
    m, k, n = 96, 200, 70  # several k-tiles, ragged edges
    A = special_matrix(W, m, k, 9100 + W)
    B = special_matrix(W, k, n, 9200 + W)
    P.gemm_redo_count(reset=True)
    got = device_gemm(P, A, B, m, k, n)
    redo = P.gemm_redo_count(reset=True)
    assert redo > 0, "structured inputs should need renorm5 paths C/D"
    assert mismatches(got[:, :, :n], O.ref_gemm(A, B, k, n)[:, :, :n]) == 0


@pytest.mark.parametrize("W", (3, 4))
def test_redo_in_some_warps_only(gpu_lib, W):
    """Rows 40-47 of A and columns 10-19 of B are integer-valued (their
    products and sums have zero residuals), the rest full-width random: the
    warps holding those cells redo, their neighbours in the same tile keep
    the branch-free results."""
    P = gpu_lib
    m, k, n = 128, 160, 96
    A = random_signed(W, m, k, 9300 + W)
    B = random_signed(W, k, n, 9400 + W)
    rng = np.random.default_rng(W)
    A[:, 40:48, :k] = 0.0
    A[0, 40:48, :k] = rng.integers(-4, 5, size=(8, k)).astype(np.float64)
    B[:, :, 10:20] = 0.0
    B[0, :, 10:20] = rng.integers(-4, 5, size=(k, 10)).astype(np.float64)
    P.gemm_redo_count(reset=True)
    got = device_gemm(P, A, B, m, k, n)
    redo = P.gemm_redo_count(reset=True)
    assert redo > 0
    assert mismatches(got[:, :, :n], O.ref_gemm(A, B, k, n)[:, :, :n]) == 0


@pytest.mark.parametrize("W", (3, 4))
def test_random_inputs_bitwise_and_redo_rate(gpu_lib, W):
    """Full-width random inputs: bit-exact, and the exact recomputation is
    (nearly) never needed -- the branch-free form is the common path."""
    P = gpu_lib
    m, k, n = 256, 256, 256
    A = random_signed(W, m, k, 9500 + W)
    B = random_signed(W, k, n, 9600 + W)
    P.gemm_redo_count(reset=True)
    got = device_gemm(P, A, B, m, k, n)
    redo = P.gemm_redo_count(reset=True)
    warp_ktiles = (m * n // 32) * ((k + 15) // 16)
    assert redo <= warp_ktiles // 100, (redo, warp_ktiles)
    assert mismatches(got[:, :, :n], O.ref_gemm(A, B, k, n)[:, :, :n]) == 0


@pytest.mark.parametrize("W", (3, 4))
@pytest.mark.parametrize("which", ("A", "B", "both"))
def test_redo_when_two_sum_order_fails(gpu_lib, W, which):
    """The fast pass's ordered two-sums (two_sum_ordered, three_sum_c_small)
    assume a leading product at least in the binade of its lower-order
    terms.  Operands whose components are NOT in decreasing order (here:
    reversed, every value nonzero so no zero-residual path is involved) break
    that; the warps must notice (mag_ge), recompute exactly, and the result
    stays bit-identical to the reference, which accepts any operands."""
    P = gpu_lib
    m, k, n = 64, 96, 64
    A = random_signed(W, m, k, 9700 + W)
    B = random_signed(W, k, n, 9800 + W)
    if which in ("A", "both"):
        A = np.ascontiguousarray(A[::-1])
    if which in ("B", "both"):
        B = np.ascontiguousarray(B[::-1])
    P.gemm_redo_count(reset=True)
    got = device_gemm(P, A, B, m, k, n)
    redo = P.gemm_redo_count(reset=True)
    assert redo > 0, "reversed components should fail the order test"
    assert mismatches(got[:, :, :n], O.ref_gemm(A, B, k, n)[:, :, :n]) == 0
