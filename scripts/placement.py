"""Where does the hardware put the CTAs of a grid?  smid_probe_kernel
(csrc/tune.cu) records each CTA's SM and start time; CTAs spin long enough
to overlap.  Prints, per (grid, CTA size, dynamic smem), how many SMs got
how many CTAs in the first wave and the start-time spread.
  python scripts/placement.py > gpurun_out/placement.log"""
import collections
import ctypes as C
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T = C.CDLL(os.path.join(ROOT, "paper_2101_06584_b200", "libmpfk_tune.so"))
T.smid_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.current_stream()
for blocks, threads, smem in [(1024, 64, 0), (1024, 64, 19 * 1024), (1024, 64, 30 * 1024), (1024, 256, 0),
                              (1024, 256, 36 * 1024), (256, 256, 70 * 1024), (444, 256, 54 * 1024),
                              (592, 256, 36 * 1024), (1000, 256, 36 * 1024), (2048, 256, 53 * 1024)]:
    smid = torch.zeros(blocks, dtype=torch.int32, device="cuda")
    start = torch.zeros(blocks, dtype=torch.int64, device="cuda")
    rc = T.smid_probe(blocks, threads, smem, 2_000_000, smid.data_ptr(), start.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    if rc:
        print(blocks, threads, smem, "error", rc)
        continue
    sm = smid.cpu().numpy()
    st = start.cpu().numpy()
    st = (st - st.min()) / 1e3  # us
    first = st < 1000  # started within 1 ms: the first wave
    per_sm = collections.Counter(sm[first].tolist())
    hist = collections.Counter(per_sm.values())
    print(f"grid {blocks:5d} x {threads:3d} thr, smem {smem // 1024:3d} KB: first wave {first.sum():5d} CTAs on "
          f"{len(per_sm):3d}/{sms} SMs, CTAs-per-SM histogram {dict(sorted(hist.items()))}, "
          f"waves {int(np.ceil(st.max() / 2000 + 1e-9))}", flush=True)
