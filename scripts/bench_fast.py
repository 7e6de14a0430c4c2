"""MPFK_FAST vs BIT_EXACT on products whose output cannot fill the GPU
(device-resident operands, CUDA events, median of 5 after 2 warm-ups).
  python scripts/bench_fast.py > gpurun_out/fast.log"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402

OPS = P.OPS_PER_MAC
peak, _ = P.fp64_peak()
s = torch.cuda.current_stream()
print(f"fp64 peak {peak / 1e9:.0f} Gop/s")
print("W   m     n     k        segs  exact_ms   fast_ms   speedup  exact_frac  fast_frac")
for W in (2, 3, 4):
    for m, n, k in ((32, 32, 1 << 20), (64, 64, 1 << 18), (128, 128, 1 << 16), (256, 256, 1 << 15),
                    (512, 512, 8192)):
        if W > 2:
            k //= 4
        lda, ldb = P.pad_columns(k), P.pad_columns(n)
        A = torch.from_numpy(P.fill_baseline(W, m, k, 1, wide=True).data).cuda()
        B = torch.from_numpy(P.fill_baseline(W, k, n, 2, wide=True).data).cuda()
        C = torch.zeros((W, m, ldb), dtype=torch.float64, device="cuda")
        segs = P.splitk_segments(W, m, n, k)
        times = {}
        for flags in (P.BIT_EXACT, P.FAST):
            ts = []
            for it in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                P.gemm_device_ex(W, m, n, k, A.data_ptr(), lda, m * lda, B.data_ptr(), ldb, k * ldb, C.data_ptr(),
                                 ldb, m * ldb, flags, s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                if it >= 2:
                    ts.append(e0.elapsed_time(e1))
            times[flags] = statistics.median(ts)
        te, tf = times[P.BIT_EXACT], times[P.FAST]
        work = m * n * k * OPS[W]
        print(f"{W}  {m:5d} {n:5d} {k:8d}  {segs:4d}  {te:9.3f} {tf:9.3f}  {te / tf:7.2f}  "
              f"{work / (te * 1e-3) / peak:10.4f}  {work / (tf * 1e-3) / peak:9.4f}", flush=True)
        del A, B, C
