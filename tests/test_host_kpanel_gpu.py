"""The single-GPU host-buffer pipeline with page-locked operands (host_gemm.inl):
chunk 0's A columns go up in the same growing K panels as B and chunk 0's
GEMM runs panel by panel, continuing the chains kept in C; later chunks use
the whole B.  Shapes here take that path (>= 3 row chunks, K >= 1024) and
the plain chunked / pageable paths for contrast; every C must equal the
device-resident product bit for bit, with rows at chunk and panel edges
also checked against the reference build."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("m,n,k,pinned", [
    (2048, 4096, 1024, True),    # K-panelled chunk 0: panels [0, 64, 320, 1024)
    (2048, 4096, 1500, True),    # ragged K
    (2048, 4096, 1024, False),   # pageable: the staging ring, uniform panels
])
def test_host_pipeline_bitwise(gpu_lib, W, m, n, k, pinned):
    import torch
    P = gpu_lib
    A = P.fill_baseline(W, m, k, 70 + W, wide=W > 2, pinned=pinned)
    B = P.fill_baseline(W, k, n, 80 + W, wide=W > 2, pinned=pinned)
    C = P.MPMatrix(W, m, n, pinned=pinned)
    C.data[...] = 9.0  # stale contents must go
    P.matmul_block_parallel_into(C, A, B, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
    ld = A.stride()
    dA, dB = torch.from_numpy(np.ascontiguousarray(A.data)).cuda(), torch.from_numpy(np.ascontiguousarray(B.data)).cuda()
    dC = torch.zeros((W, m, B.stride()), dtype=torch.float64, device="cuda")
    P.gemm_device(W, m, n, k, dA.data_ptr(), ld, m * ld, dB.data_ptr(), B.stride(), k * B.stride(), dC.data_ptr(),
                  B.stride(), m * B.stride())
    torch.cuda.synchronize()
    want_dev = dC.cpu().numpy()
    assert mismatches(C.data[:, :, :n], want_dev[:, :, :n]) == 0
    assert (C.data[:, :, n:] == 0.0).all()  # pads +0 (zero_pads)
    rows = [0, 63, 351, 352, 1055, 1056, 1759, 1760, m - 1]
    want = O.ref_gemm(np.ascontiguousarray(A.data[:, rows, :]), np.ascontiguousarray(B.data), k, n)
    assert mismatches(C.data[:, rows, :n], want[:, :, :n]) == 0
