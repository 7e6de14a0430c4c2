"""Small GEMMs on zero-residual inputs through the device path (the TD/QD
FASTR redo path) and the host-buffer gated (page-locked) and chunked
(pageable) paths, bitwise against the reference; prints the redo count.
(compute-sanitizer is closed on the GPU pool, so this is the small-case
check instead.)  python scripts/smallcheck.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2101_06584_b200 as P  # noqa: E402
from tests.helpers import mismatches, special_matrix  # noqa: E402

bad = 0
for W in (2, 3, 4):
    m, k, n = 70, 100, 66
    A = special_matrix(W, m, k, 5 + W)
    B = special_matrix(W, k, n, 6 + W)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros((W, m, B.shape[2]), dtype=torch.float64, device="cuda")
    P.gemm_device(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), B.shape[2],
                  k * B.shape[2], dC.data_ptr(), B.shape[2], m * B.shape[2])
    torch.cuda.synchronize()
    want = O.ref_gemm(A, B, k, n)
    bad += mismatches(dC.cpu().numpy(), want)
    # host-buffer path (page-locked: gated single launch; pageable: chunked)
    for pinned in (True, False):
        Am = P.MPMatrix(W, m, k, pinned=pinned)
        Bm = P.MPMatrix(W, k, n, pinned=pinned)
        Am.data[...] = A
        Bm.data[...] = B
        Cm = P.matmul_block_parallel(Am, Bm, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
        bad += mismatches(Cm.data, want)
print("redo count", P.gemm_redo_count(reset=True), "mismatches", bad)
sys.exit(1 if bad else 0)
