"""Per-CTA durations of the persistent round-robin and dynamic-counter
schedules (tune.cu persist_kernel with g_trace): is per-SM throughput
uniform?  python scripts/persist_trace.py > gpurun_out/persist_trace.log"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_06584_b200 as P  # noqa: E402

T = C.CDLL(os.path.join(ROOT, "paper_2101_06584_b200", "libmpfk_tune.so"))
T.tune_name.restype = C.c_char_p
T.tune_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p,
                       C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p]
T.persist_trace.argtypes = [C.c_void_p]
s = torch.cuda.current_stream()
for W, n in ((3, 2048), (2, 4096)):
    ld = P.pad_columns(n)
    A = torch.from_numpy(P.fill_baseline(W, n, n, 1).data).cuda()
    B = torch.from_numpy(P.fill_baseline(W, n, n, 2).data).cuda()
    Cm = torch.zeros_like(A)
    for i in range(T.tune_count()):
        name = T.tune_name(i).decode()
        if not (name.startswith("rr/") or name.startswith("dyn/")) or int(name.split("/")[1]) != W:
            continue
        if W == 2 and "64x64" not in name:
            continue
        buf = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
        T.persist_trace(buf.data_ptr())
        rc = T.tune_run(i, n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, Cm.data_ptr(), ld, n * ld,
                        s.cuda_stream)
        torch.cuda.synchronize()
        T.persist_trace(None)
        r = buf.view(-1, 4).cpu().numpy()
        r = r[r[:, 2] > 0]
        t0 = r[:, 1].min()
        dur = (r[:, 2] - r[:, 1]) / 1e6
        end = (r[:, 2] - t0) / 1e6
        per_tile = dur / np.maximum(r[:, 3], 1)
        sm = r[:, 0]
        sm_tile = np.array([per_tile[sm == k].mean() for k in np.unique(sm)])
        print(f"W={W} n={n} {name:34s} rc={rc} CTAs {len(r)} makespan {end.max():8.3f} ms; "
              f"CTA end min/med/max {end.min():.3f}/{np.median(end):.3f}/{end.max():.3f} ms; tiles/CTA "
              f"{r[:, 3].min()}-{r[:, 3].max()}; per-tile ms by SM min/med/max {sm_tile.min():.4f}/"
              f"{np.median(sm_tile):.4f}/{sm_tile.max():.4f}", flush=True)
