"""The fused all-gather -> GEMM kernel (mpfk_gemm_device_pull) on one GPU,
with the "ranks" emulated as one kernel over all ranks' data (the B200
profiling guide's prescription): B's row slices live in separate device
buffers standing in for peer GPUs; the kernel pulls every K panel on demand
into the local B while computing.  Must be bit-identical to the one-shot
GEMM and leave the whole B in the local buffer, for uneven slices, short
last panels, tiny chunks (many CTAs racing for tickets) and all widths."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed

pytestmark = pytest.mark.gpu


def run_pull(P, W, m, k, n, cuts, panel_rows, chunk_rows, seed=0):
    import torch
    A = random_signed(W, m, k, 300 + seed)
    B = random_signed(W, k, n, 400 + seed)
    ld = B.shape[2]
    dA = torch.from_numpy(A).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    dB = torch.full((W, k, ld), float("nan"), dtype=torch.float64, device="cuda")  # must be overwritten
    dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    launches = P.gemm_device_pull(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld, k * ld,
                                  dC.data_ptr(), ld, m * ld, [t.data_ptr() for t in slices], cuts, panel_rows,
                                  chunk_rows)
    torch.cuda.synchronize()
    return A, B, dB.cpu().numpy(), dC.cpu().numpy(), launches


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,k,n,cuts,panel_rows,chunk_rows", [
    (37, 45, 29, [0, 45], 16, 16),
    (64, 100, 70, [0, 13, 60, 100], 32, 5),
    (130, 257, 66, [0, 1, 2, 100, 200, 230, 250, 257], 48, 3),
    (300, 128, 300, [0, 64, 128], 64, 64),
])
def test_pull_bitwise(gpu_lib, W, m, k, n, cuts, panel_rows, chunk_rows):
    A, B, gotB, gotC, launches = run_pull(gpu_lib, W, m, k, n, cuts, panel_rows, chunk_rows, seed=m + W)
    assert launches == 1
    assert mismatches(gotC, O.ref_gemm(A, B, k, n)) == 0
    assert np.array_equal(gotB.view(np.uint64), B.view(np.uint64))  # every row, pads included


def test_pull_many_ctas_racing(gpu_lib):
    """thousands of CTAs, 8 slices, 4-row chunks: every panel is claimed by
    many CTAs at once."""
    import torch
    P = gpu_lib
    W, m, k, n = 2, 2048, 1024, 256
    cuts = [0, 128, 256, 384, 512, 640, 768, 896, 1024]
    A = P.fill_baseline(W, m, k, 1).data
    B = P.fill_baseline(W, k, n, 2).data
    ld = B.shape[2]
    dA = torch.from_numpy(A).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    dB = torch.zeros((W, k, ld), dtype=torch.float64, device="cuda")
    dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    ref = torch.zeros_like(dC)
    dBfull = torch.from_numpy(B).cuda()
    P.gemm_device(W, m, n, k, dA.data_ptr(), k, m * k, dBfull.data_ptr(), ld, k * ld, ref.data_ptr(), ld, m * ld)
    for _ in range(3):
        dB.zero_()
        P.gemm_device_pull(W, m, n, k, dA.data_ptr(), k, m * k, dB.data_ptr(), ld, k * ld, dC.data_ptr(), ld, m * ld,
                           [t.data_ptr() for t in slices], cuts, 64, 4)
        torch.cuda.synchronize()
        assert torch.equal(dC.view(torch.int64), ref.view(torch.int64))
        assert torch.equal(dB.view(torch.int64), dBfull.view(torch.int64))


def test_pull_validation(gpu_lib):
    P = gpu_lib
    with pytest.raises(ValueError, match="cover rows"):
        P.gemm_device_pull(2, 4, 4, 8, 16, 8, 32, 16, 4, 32, 16, 4, 16, [16], [0, 7], 16, 4)
    with pytest.raises(ValueError, match="multiple of 16"):
        P.gemm_device_pull(2, 4, 4, 8, 16, 8, 32, 16, 4, 32, 16, 4, 16, [16], [0, 8], 10, 4)


def run_gathered(P, W, m, k, n, cuts, panel_rows, seed=0):
    import torch
    A = random_signed(W, m, k, 500 + seed)
    B = random_signed(W, k, n, 600 + seed)
    ld = B.shape[2]
    dA = torch.from_numpy(A).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    dB = torch.full((W, k, ld), float("nan"), dtype=torch.float64, device="cuda")
    dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    launches = P.gemm_device_gathered(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld,
                                      k * ld, dC.data_ptr(), ld, m * ld, [t.data_ptr() for t in slices], cuts,
                                      panel_rows)
    torch.cuda.synchronize()
    return A, B, dB.cpu().numpy(), dC.cpu().numpy(), launches


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,k,n,cuts,panel_rows", [
    (37, 45, 29, [0, 45], 16),
    (64, 100, 70, [0, 13, 60, 100], 32),
    (130, 257, 66, [0, 1, 2, 100, 200, 230, 250, 257], 48),
    (300, 1000, 300, [0, 500, 1000], 64),
])
def test_gathered_bitwise(gpu_lib, W, m, k, n, cuts, panel_rows):
    """copy-engine gather (stream-memory flags per K panel, one gated GEMM
    launch): bit-identical to the one-shot GEMM, the whole B gathered."""
    A, B, gotB, gotC, launches = run_gathered(gpu_lib, W, m, k, n, cuts, panel_rows, seed=m + W)
    assert launches == 1
    assert mismatches(gotC, O.ref_gemm(A, B, k, n)) == 0
    assert np.array_equal(gotB.view(np.uint64), B.view(np.uint64))


def test_gathered_repeated_and_validation(gpu_lib):
    """back-to-back calls reuse the device's gather stream and events; the
    panel height is validated"""
    import torch
    P = gpu_lib
    W, m, k, n = 2, 512, 2048, 256
    A = P.fill_baseline(W, m, k, 1).data
    B = P.fill_baseline(W, k, n, 2).data
    ld = B.shape[2]
    cuts = [0, 512, 1024, 1536, 2048]
    dA = torch.from_numpy(A).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    ref = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    dBfull = torch.from_numpy(B).cuda()
    P.gemm_device(W, m, n, k, dA.data_ptr(), k, m * k, dBfull.data_ptr(), ld, k * ld, ref.data_ptr(), ld, m * ld)
    for _ in range(4):
        dB = torch.zeros((W, k, ld), dtype=torch.float64, device="cuda")
        dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
        P.gemm_device_gathered(W, m, n, k, dA.data_ptr(), k, m * k, dB.data_ptr(), ld, k * ld, dC.data_ptr(), ld,
                               m * ld, [t.data_ptr() for t in slices], cuts, 128)
        torch.cuda.synchronize()
        assert torch.equal(dC.view(torch.int64), ref.view(torch.int64))
    with pytest.raises(ValueError, match="multiple of 16"):
        P.gemm_device_gathered(2, 4, 4, 8, 16, 8, 32, 16, 4, 32, 16, 4, 16, [16], [0, 8], 10)
