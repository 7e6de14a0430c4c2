"""Why the cpu_baseline leg inside the GPU process reads lower than the
reference arm on the same box: the reference's CPU GEMM (bench.CpuReference,
DD n=8192, 2 waves) timed in a fresh process after progressively more of
the GPU arm's state is set up.
  python scripts/cpu_probe.py <plain|cuda|mpfk|mpfk+e2e>"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
mode = sys.argv[1]
info = {}
if mode != "plain":
    import torch
    x = torch.zeros(1 << 20, device="cuda")
    torch.cuda.synchronize()
if mode.startswith("mpfk"):
    import paper_2101_06584_b200 as P
    A = P.fill_baseline(2, 1024, 1024, 1)
    C = P.matmul_block(A, A)
    if mode == "mpfk+e2e":
        Ap = P.fill_baseline(2, 2048, 2048, 1)
        for _ in range(3):
            P.matmul_block_parallel_into(P.MPMatrix(2, 2048, 2048), Ap, Ap, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
import bench  # noqa: E402
info["affinity"] = len(os.sched_getaffinity(0))
info["threads_before"] = threading.active_count()
info["os_threads"] = len(os.listdir("/proc/self/task"))
ref = bench.CpuReference("dd8192", waves=2)
ref.step()
rates = [round(ref.step()[0], 2) for _ in range(2)]
print(mode, rates, info, flush=True)
