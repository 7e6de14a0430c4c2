import ctypes as C, os, sys
ROOT='/root/repo'; sys.path.insert(0, ROOT)
import torch
import paper_2101_06584_b200 as P
T = C.CDLL(os.path.join(ROOT, "paper_2101_06584_b200", "libmpfk_tune.so"))
T.tune_name.restype = C.c_char_p
T.tune_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p,
                       C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p]
idx = [i for i in range(T.tune_count()) if T.tune_name(i).decode() == "2/64x64x16/4x4/st2/ku2/g16/mb2"][0]
n = 4096; W = 2; ld = n
A = torch.from_numpy(P.fill_baseline(W, n, n, 1).data).cuda()
B = torch.from_numpy(P.fill_baseline(W, n, n, 2).data).cuda()
Cm = torch.zeros_like(A)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
peak, _ = P.fp64_peak()
for name, lda, ldb in (("normal", ld, ld), ("A rows aliased", 0, ld), ("B rows aliased", ld, 0), ("both aliased", 0, 0)):
    args = (n, n, n, A.data_ptr(), lda, n * ld, B.data_ptr(), ldb, n * ld, Cm.data_ptr(), ld, n * ld, s.cuda_stream)
    T.tune_run(idx, *args)
    best = 1e9
    for _ in range(3):
        e0.record(s); T.tune_run(idx, *args); e1.record(s); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"{name:16s} {best:8.3f} ms frac {n**3*20/(best*1e-3)/peak:.4f}", flush=True)
