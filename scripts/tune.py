"""Time every tile configuration of libmpfk_tune.so on device-resident
BASELINE inputs; each result must be bit-identical to the product kernel's.
  python scripts/tune.py [--sizes 1024,4096] [--reps 2] > gpurun_out/tune.log"""
import argparse
import ctypes as C
import json
import re
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402

OPS = {2: 20, 3: 132, 4: 218}
ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="1024,4096")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--widths", default="2,3,4")
ap.add_argument("--match", default="", help="regex: only entries whose name matches")
ap.add_argument("--lean", action="store_true",
                help="MPFK_LEAN entries (TUNE_LIB=libmpfk_tune_lean.so): compared with the bit-exact product within "
                     "4*k*u_p (normwise), fractions in executed FP64 instructions")
a = ap.parse_args()
LEAN_OPS = {2: 10 + 6 / 16, 3: 42 + 18 / 16, 4: 107 + 30 / 16}  # mpf_lean.cuh, renorm_loose per 16-step k-tile
U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}


def lean_diff(Cm, ref, W, n):
    """max |lean - bitexact| / max |bitexact| over the matrix, summing the
    component differences from the smallest up in binary64 (the leading
    components cancel exactly where the results agree)."""
    d = (Cm[W - 1] - ref[W - 1])
    for w in range(W - 2, -1, -1):
        d = d + (Cm[w] - ref[w])
    return float(d[:, :n].abs().max() / ref[0][:, :n].abs().max())


T = C.CDLL(os.path.join(ROOT, "paper_2101_06584_b200", os.environ.get("TUNE_LIB", "libmpfk_tune.so")))
T.tune_name.restype = C.c_char_p
T.tune_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p,
                       C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p]
peak, _ = P.fp64_peak()
print(f"fp64 peak {peak/1e9:.0f} Gop/s", flush=True)
s = torch.cuda.current_stream()
results = []
for W in [int(x) for x in a.widths.split(",")]:
    for n in [int(x) for x in a.sizes.split(",")]:
        ld = P.pad_columns(n)
        wide = W > 2 and n >= 4096
        A = torch.from_numpy(P.fill_baseline(W, n, n, 1, wide=wide).data).cuda()
        B = torch.from_numpy(P.fill_baseline(W, n, n, 2, wide=wide).data).cuda()
        ref = torch.zeros_like(A)
        P.gemm_device(W, n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, ref.data_ptr(), ld, n * ld,
                      s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        P.gemm_device(W, n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, ref.data_ptr(), ld, n * ld,
                      s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        base = e0.elapsed_time(e1)
        print(f"W={W} n={n} product kernel {base:.3f} ms frac {n**3*OPS[W]/(base*1e-3)/peak:.4f}", flush=True)
        for i in range(T.tune_count()):
            if T.tune_width(i) != W:
                continue
            name = T.tune_name(i).decode()
            if a.match and not re.search(a.match, name):
                continue
            regs, smem, thr = C.c_int(), C.c_int(), C.c_int()
            T.tune_info(i, C.byref(regs), C.byref(smem), C.byref(thr))
            Cm = torch.zeros_like(A)
            args = (n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, Cm.data_ptr(), ld, n * ld,
                    s.cuda_stream)
            rc = T.tune_run(i, *args)
            if rc:
                print(f"  {name:40s} launch error {rc}", flush=True)
                continue
            ts = []
            for _ in range(a.reps):
                e0.record(s)
                T.tune_run(i, *args)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = min(ts)
            if a.lean:
                diff = lean_diff(Cm, ref, W, n) / (4 * n * U_P[W])
                ok = diff <= 1.0
                frac = n ** 3 * LEAN_OPS[W] / (t * 1e-3) / peak
                print(f"  {name:52s} regs {regs.value:3d} smem {smem.value:6d} thr {thr.value} {t:9.3f} ms "
                      f"{2 * n ** 3 / (t * 1e-3) / 1e9:8.1f} MPF Gflops frac_executed {frac:.4f} speedup {base/t:.3f} "
                      f"diff_vs_bitexact {diff:.2e} of 4ku_p", flush=True)
                results.append(dict(W=W, n=n, cfg=name, ms=t, frac=frac, regs=regs.value, ok=ok))
                continue
            ok = bool(torch.equal(Cm.view(torch.int64), ref.view(torch.int64)))
            frac = n ** 3 * OPS[W] / (t * 1e-3) / peak
            print(f"  {name:40s} regs {regs.value:3d} smem {smem.value:6d} thr {thr.value} {t:9.3f} ms "
                  f"frac {frac:.4f} speedup {base/t:.3f} bitexact {ok}", flush=True)
            results.append(dict(W=W, n=n, cfg=name, ms=t, frac=frac, regs=regs.value, ok=ok))
json.dump(results, open(os.path.join(ROOT, "gpurun_out", "tune.json"), "w"), indent=1)
