"""Kernel time of the DD tile configurations on the shapes the host-buffer
pipeline launches (row chunks x K panels), to check the per-launch tile
choice (capi.cu: dd_small_tiles / predicted_eff) against measurement.
  python scripts/shape_probe.py > gpurun_out/shape_probe.log"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402

T = C.CDLL(os.path.join(ROOT, "paper_2101_06584_b200", "libmpfk_tune.so"))
T.tune_name.restype = C.c_char_p
T.tune_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p,
                       C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p]
names = {T.tune_name(i).decode(): i for i in range(T.tune_count())}
cfgs = {"64x64": names["pb1/2/64x64/product"], "32x32": names["pb1/2/32x32/product"]}
peak, _ = P.fp64_peak()
W, n = 2, 8192
A = torch.from_numpy(P.fill_baseline(W, 2048, n, 1).data).cuda()
B = torch.from_numpy(P.fill_baseline(W, n, n, 2).data).cuda()
Cm = torch.zeros((W, 2048, n), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for m, k in [(512, 512), (512, 1024), (512, 8192), (1024, 512), (1024, 8192), (2048, 8192), (256, 8192),
             (768, 8192), (1536, 8192)]:
    row = []
    for name, i in cfgs.items():
        args = (m, n, k, A.data_ptr(), n, 2048 * n, B.data_ptr(), n, n * n, Cm.data_ptr(), n, 2048 * n,
                s.cuda_stream)
        T.tune_run(i, *args)
        best = 1e30
        for _ in range(3):
            e0.record(s)
            T.tune_run(i, *args)
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        row.append(f"{name} {best:8.3f} ms frac {m * n * k * 20 / (best * 1e-3) / peak:.4f}")
    print(f"m={m:5d} k={k:5d}  " + "   ".join(row), flush=True)
