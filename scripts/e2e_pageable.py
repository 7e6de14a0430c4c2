"""Host-buffer GEMM with pageable (plain numpy / aligned_alloc-like) vs
pinned operands: what a reference caller passing its own MPMatrix buffers
gets.  python scripts/e2e_pageable.py [workload]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2101_06584_b200 as P  # noqa: E402
from bench import WORKLOADS  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "dd8192"
W, n, wide = WORKLOADS[w]
for pinned in (True, False):
    A = P.fill_baseline(W, n, n, 1, wide=wide, pinned=pinned)
    B = P.fill_baseline(W, n, n, 2, wide=wide, pinned=pinned)
    C = P.MPMatrix(W, n, n, pinned=pinned)
    P.matmul_block_parallel_into(C, A, B)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        P.matmul_block_parallel_into(C, A, B)
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[1]
    st = P.last_stats()
    print(f"{w} pinned={pinned}: {2.0 * n**3 / t / 1e9:.1f} MPF Gflops e2e, {t * 1e3:.1f} ms, "
          f"h2d {st['h2d_ms']:.1f} ms kernel {st['kernel_ms']:.1f} ms d2h {st['d2h_ms']:.1f} ms", flush=True)
    del A, B, C
