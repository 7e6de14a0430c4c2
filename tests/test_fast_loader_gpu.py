"""The interior fast loader (gemm_kernel.cuh: FastLoad, round 2): interior
tiles load full k-tiles through precomputed per-thread addresses, edge tiles
and the last partial k-tile through the general loader.  Shapes here mix
all three in one launch -- interior tiles, a ragged column edge, a ragged
row edge, K not a multiple of BK -- for every width and both DD tile
configurations (64x64 at this size; 32x32 when the grid is small), on
unpadded leading dimensions and on the reference's pad4 ones; rows at tile
edges are compared bitwise with the reference GEMM."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,n,k,extra_ld", [
    (2048, 1540, 1000, 0),   # 64x64 DD tiles: ragged n, partial last k-tile
    (1000, 1030, 777, 6),    # ragged m and n, odd k, padded leading dimensions
    (256, 256, 16 * 37, 0),  # small grid (DD 32x32 tiles), k a multiple of BK
])
def test_interior_and_edge_tiles_bitwise(gpu_lib, W, m, n, k, extra_ld):
    import torch
    P = gpu_lib
    A = P.fill_baseline(W, m, k, 31 + W, wide=W > 2).data
    B = P.fill_baseline(W, k, n, 41 + W, wide=W > 2).data
    lda, ldb = A.shape[2] + extra_ld, B.shape[2] + extra_ld
    ldc = P.pad_columns(n) + extra_ld
    dA = torch.zeros((W, m, lda), dtype=torch.float64, device="cuda")
    dB = torch.zeros((W, k, ldb), dtype=torch.float64, device="cuda")
    dA[:, :, :A.shape[2]] = torch.from_numpy(A).cuda()
    dB[:, :, :B.shape[2]] = torch.from_numpy(B).cuda()
    dC = torch.full((W, m, ldc), 5.0, dtype=torch.float64, device="cuda")
    P.gemm_device(W, m, n, k, dA.data_ptr(), lda, m * lda, dB.data_ptr(), ldb, k * ldb, dC.data_ptr(), ldc,
                  m * ldc)
    torch.cuda.synchronize()
    rows = sorted({0, 31, 32, 63, 64, 127, m // 2, m - 65, m - 64, m - 33, m - 32, m - 1})
    want = O.ref_gemm(np.ascontiguousarray(A[:, rows, :]), B, k, n)
    got = dC[:, rows, :n].cpu().numpy()
    assert mismatches(got, want[:, :, :n]) == 0
    assert bool((dC[:, :, n:] == 5.0).all())  # nothing written past n
