"""The staged all-gather -> GEMM (mpfk_gemm_device_staged, bench.py's
default multi-GPU transport) on one GPU: B's row slices live in separate
device buffers standing in for the peer GPUs' slices; the copy engines
gather them in growing K panels and one GEMM launch per panel continues the
chains kept in C.  Must be bit-identical to the reference GEMM and leave the
whole B in the local buffer, for uneven slices, panel cuts that fall inside
slices, short k and all widths."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed

pytestmark = pytest.mark.gpu


def expected_panels(k, head=0):
    """Mirror of staged_panels (capi.cu): first panel head (64), then x4,
    at most 8 panels, no panel shorter than the rest it would leave."""
    cut, h = [0], max(16, ((head or 64) + 15) // 16 * 16)
    while len(cut) < 8 and cut[-1] + h < k and h * 2 <= k - cut[-1]:
        cut.append(cut[-1] + h)
        h *= 4
    return cut + [k]


def run_staged(P, W, m, k, n, cuts, head=0, seed=0):
    import torch
    A = random_signed(W, m, k, 500 + seed)
    B = random_signed(W, k, n, 600 + seed)
    ld = B.shape[2]
    dA = torch.from_numpy(A).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    dB = torch.full((W, k, ld), float("nan"), dtype=torch.float64, device="cuda")  # must be overwritten
    dC = torch.full((W, m, ld), 7.0, dtype=torch.float64, device="cuda")  # cleared by the first panel
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        launches = P.gemm_device_staged(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld,
                                        k * ld, dC.data_ptr(), ld, m * ld, [t.data_ptr() for t in slices], cuts,
                                        head, s.cuda_stream)
    s.synchronize()
    return A, B, dB.cpu().numpy(), dC.cpu().numpy(), launches


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,k,n,cuts,head", [
    (37, 45, 29, [0, 45], 0),
    (64, 300, 70, [0, 13, 160, 300], 0),
    (130, 1000, 66, [0, 1, 2, 100, 500, 930, 999, 1000], 16),
    (300, 2048, 96, [0, 256, 512, 768, 1024, 1280, 1536, 1792, 2048], 32),
])
def test_staged_bitwise(gpu_lib, W, m, k, n, cuts, head):
    A, B, gotB, gotC, launches = run_staged(gpu_lib, W, m, k, n, cuts, head, seed=m + W)
    assert launches == len(expected_panels(k, head)) - 1
    assert mismatches(gotC[:, :, :n], O.ref_gemm(A, B, k, n)[:, :, :n]) == 0
    assert (gotC[:, :, n:] == 7.0).all()  # device GEMMs write only the m x n cells
    assert np.array_equal(gotB.view(np.uint64), B.view(np.uint64))  # every row, pads included


def test_staged_panel_plan():
    assert expected_panels(8192) == [0, 64, 320, 1344, 8192]
    assert expected_panels(1024) == [0, 64, 320, 1024]
    assert expected_panels(100) == [0, 100]


def test_staged_baseline_shape_repeated(gpu_lib):
    """a BASELINE-shaped shard (1024 rows of DD n=4096, 8 slices) three
    times in a row on one stream: each call reuses the gather stream and
    the panel events."""
    import torch
    P = gpu_lib
    W, m, k, n = 2, 1024, 4096, 4096
    cuts = [i * 512 for i in range(9)]
    A = P.fill_baseline(W, m, k, 1).data
    B = P.fill_baseline(W, k, n, 2).data
    ld = B.shape[2]
    dA = torch.from_numpy(A).cuda()
    slices = [torch.from_numpy(np.ascontiguousarray(B[:, r0:r1])).cuda() for r0, r1 in zip(cuts, cuts[1:])]
    dBfull = torch.from_numpy(B).cuda()
    ref = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    P.gemm_device(W, m, n, k, dA.data_ptr(), k, m * k, dBfull.data_ptr(), ld, k * ld, ref.data_ptr(), ld, m * ld)
    dB = torch.zeros((W, k, ld), dtype=torch.float64, device="cuda")
    dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
    for _ in range(3):
        dB.zero_()
        P.gemm_device_staged(W, m, n, k, dA.data_ptr(), k, m * k, dB.data_ptr(), ld, k * ld, dC.data_ptr(), ld,
                             m * ld, [t.data_ptr() for t in slices], cuts)
        torch.cuda.synchronize()
        assert torch.equal(dC.view(torch.int64), ref.view(torch.int64))
        assert torch.equal(dB.view(torch.int64), dBfull.view(torch.int64))


def test_staged_validation(gpu_lib):
    P = gpu_lib
    with pytest.raises(ValueError, match="cover rows"):
        P.gemm_device_staged(2, 4, 4, 8, 16, 8, 32, 16, 4, 32, 16, 4, 16, [16], [0, 7])
    with pytest.raises(ValueError, match="head_rows"):
        P.gemm_device_staged(2, 4, 4, 8, 16, 8, 32, 16, 4, 32, 16, 4, 16, [16], [0, 8], 10)
    with pytest.raises(ValueError, match="source slices"):
        P.gemm_device_staged(2, 4, 4, 8, 16, 8, 32, 16, 4, 32, 16, 4, 16, [], [0])
