"""Compute-only ceilings next to the product GEMM (libmpfk_tune.so).

* pipe peaks: 8 independent DFMA / DADD / DMUL chains per thread;
* ceiling/<cfg>: the product tile configuration's mac_step loop on one
  shared-memory stage filled once (no global loads, no barriers), at the
  product's occupancy, grid = SMs x MINB x waves.
  python scripts/ceiling.py > gpurun_out/ceiling.log"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

OPS = {2: 20, 3: 132, 4: 218}
MINB = {"mb1": 1, "mb2": 2, "mb3": 3, "mb4": 4, "mb6": 6, "mb8": 8}
T = C.CDLL(os.path.join(ROOT, "paper_2101_06584_b200", os.environ.get("TUNE_LIB", "libmpfk_tune.so")))
T.ceil_name.restype = C.c_char_p
T.ceil_macs.restype = C.c_longlong
T.ceil_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
T.pipe_peak_run.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]

sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=3):
    fn()
    best = 1e30
    for _ in range(reps):
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = torch.zeros(1 << 22, dtype=torch.float64, device="cuda")
peaks = {}
for kind, name in ((0, "DFMA"), (1, "DADD"), (2, "DMUL")):
    blocks, threads, iters = sms * 8, 256, 1 << 15
    t = timed(lambda: T.pipe_peak_run(kind, out.data_ptr(), blocks, threads, iters, s.cuda_stream))
    peaks[name] = blocks * threads * iters * 8 / (t * 1e-3)
    print(f"pipe peak {name}: {peaks[name]/1e9:.0f} Gop/s ({t:.3f} ms)", flush=True)
peak = peaks["DFMA"]

src = torch.rand(4096, dtype=torch.float64, device="cuda") * 2 - 1
for i in range(T.ceil_count()):
    name = T.ceil_name(i).decode()
    W = T.ceil_width(i)
    mb = MINB[name.rsplit("/", 1)[1]]
    for waves in (1, 4):
        blocks = sms * mb * waves
        ktiles = {2: 256, 3: 48, 4: 32}[W]
        t = timed(lambda: T.ceil_run(i, src.data_ptr(), out.data_ptr(), blocks, ktiles, s.cuda_stream))
        ops = blocks * T.ceil_macs(i) * ktiles * OPS[W]
        print(f"  {name:36s} blocks {blocks:5d} {t:8.3f} ms  {ops/(t*1e-3)/1e9:8.0f} Gop/s  "
              f"frac of DFMA peak {ops/(t*1e-3)/peak:.4f}", flush=True)
