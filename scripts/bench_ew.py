"""Elementwise DD/TD/QD add / mul / TD merge-add on the GPU (SURVEY.md 8(f)
row 1; the paper's vector benchmarks, bench.cpp:77-127).

One JSON line per (width, op): MPF Mops = n / s (the paper's DD/TD/QD MFLOPS
unit, scaled), the kernel's HBM roofline (3*W*8 algorithmic bytes per
element / kernel time vs MEASURED_PEAKS.json hbm_gbs), and the reference's
ew_apply_into (SIMD_LOADSTORE, single thread as in the reference) on a
bounded sample on this host.

  python scripts/bench_ew.py [--n 67108864] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 26)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cpu-n", type=int, default=1 << 21)
a = ap.parse_args()

try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    peak_src = "MEASURED_PEAKS.json hbm_gbs"
except Exception:
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"

s = torch.cuda.current_stream()
n = a.n
ld = P.pad_columns(n)
for W in (2, 3, 4):
    A = torch.from_numpy(P.fill_baseline(W, 1, n, 5, wide=True).data).cuda()
    B = torch.from_numpy(P.fill_baseline(W, 1, n, 6, wide=True).data).cuda()
    O_ = torch.empty_like(A)
    for op in (["add", "mul"] + (["add_merge"] if W == 3 else [])):
        code = int(P.EwOp[op])

        def run():
            return P.ew_device(W, code, 1, n, O_.data_ptr(), ld, ld, A.data_ptr(), ld, ld, B.data_ptr(), ld, ld,
                               s.cuda_stream)

        for _ in range(3):
            run()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            run()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        gbs = 3 * W * 8 * n / (t * 1e-3) / 1e9
        cpu = None
        try:
            import oracle as Orc
            m = a.cpu_n
            x = P.fill_baseline(W, 1, m, 5, wide=True)
            y = P.fill_baseline(W, 1, m, 6, wide=True)
            t0 = time.perf_counter()
            Orc.ref_ew(W, op, x.data, y.data, m, variant=2)
            tc = time.perf_counter() - t0
            cpu = {"value": round(m / tc / 1e6, 2), "unit": "MPF Mops/s", "cores": 1, "kind": "reference",
                   "sample": f"{m} elements, ew_apply_into SIMD_LOADSTORE (includes MPMatrix copies in the shim)"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)[:120]}
        print(json.dumps({"metric": f"ew_{op} MPF Mops/s", "precision": {2: "DD", 3: "TD", 4: "QD"}[W],
                          "n": n, "value": round(n / (t * 1e-3) / 1e6, 1), "unit": "MPF Mops/s",
                          "kernel_ms": round(t, 4),
                          "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                                       "frac": round(gbs / peak, 4), "bytes_per_elem": 3 * W * 8,
                                       "peak_source": peak_src},
                          "cpu_baseline": cpu}), flush=True)
