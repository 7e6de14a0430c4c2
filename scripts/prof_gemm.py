"""Minimal driver for ncu: the GEMM kernel on device-resident BASELINE inputs.
  python scripts/prof_gemm.py --workload dd8192 --launches 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402
from bench import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="dd8192")
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--n", type=int, default=0, help="override the workload's size")
ap.add_argument("--lean", action="store_true", help="flags = MPFK_LEAN (tolerance mode)")
a = ap.parse_args()
W, n, wide = WORKLOADS[a.workload]
n = a.n or n
ld = P.pad_columns(n)
A = torch.from_numpy(P.fill_baseline(W, n, n, 1, wide=wide).data).cuda()
B = torch.from_numpy(P.fill_baseline(W, n, n, 2, wide=wide).data).cuda()
C = torch.zeros_like(A)
s = torch.cuda.current_stream()
for _ in range(a.launches):
    P.gemm_device_ex(W, n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, C.data_ptr(), ld, n * ld,
                     P.LEAN if a.lean else P.BIT_EXACT, s.cuda_stream)
torch.cuda.synchronize()
print("ok", a.workload, float(C[0, 0, 0]))
