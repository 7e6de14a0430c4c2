"""Time device-resident Strassen vs the block GEMM (scripts/prof_strassen.py W n cutoff)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402

W, n, cutoff = (int(x) for x in sys.argv[1:4])
ld = P.pad_columns(n)
A = torch.from_numpy(P.fill_baseline(W, n, n, 1).data).cuda()
B = torch.from_numpy(P.fill_baseline(W, n, n, 2).data).cuda()
C = torch.zeros_like(A)
s = torch.cuda.current_stream().cuda_stream
args = (W, n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, C.data_ptr(), ld, n * ld)
for name, f in (("block", lambda: P.gemm_device(*args, s)), ("strassen", lambda: P.strassen_device(*args, cutoff, s))):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = f()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    print(f"W={W} n={n} cutoff={cutoff} {name:8s} {t:9.2f} ms  classic-op Gflops {2*n**3/(t*1e-3)/1e9:8.1f}"
          f"  launches {launches}", flush=True)
