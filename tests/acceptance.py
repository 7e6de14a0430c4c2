#!/usr/bin/env python
"""Release acceptance gate of the GPU path, mirroring the reference's
proj/tests/acceptance.cpp criteria 1-9 (TEST INFRASTRUCTURE: compares the
product against the reference build in oracle/_ref and the exact oracle).

One line per criterion, the reference's format:
  PASS/FAIL criterion N: <what was checked> (<measurements>)
  INFO criterion N: ...
Exit code = number of asserted failures.  Differences from the C++ gate are
stated in each line (sample sizes where exact rational arithmetic in Python
is slower than Boost's cpp_int; the GPU replaces the AVX2 backends).

  python tests/acceptance.py
"""
from __future__ import annotations

import math
import os
import sys
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2101_06584_b200 as P  # noqa: E402
from oracle import dyadic  # noqa: E402

FAILS = 0
GOLD = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def verdict(idx, ok, what, detail):
    global FAILS
    print(f"{'PASS' if ok else 'FAIL'} criterion {idx}: {what} ({detail})", flush=True)
    if not ok:
        FAILS += 1


def info(idx, detail):
    print(f"INFO criterion {idx}: {detail}", flush=True)


def sm64_stream(seed, count):
    """SplitMix64 outputs 1..count from `seed` (random.hpp:17-27), vectorised:
    output i mixes seed + i * golden."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + np.arange(1, count + 1, dtype=np.uint64) * np.uint64(GOLD))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def random_finite(seed, count, lo, hi):
    """rng::random_finite (random.hpp:44-49): 3 draws per value."""
    d = sm64_stream(seed, 3 * count).reshape(count, 3)
    e = lo + (d[:, 0] % np.uint64(hi - lo + 1)).astype(np.int64)
    m = 1.0 + (d[:, 1] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    s = np.where((d[:, 2] & np.uint64(1)) != 0, -1.0, 1.0)
    return s * np.ldexp(m, e)


def normalized_pairs(W, count, seed, signed=True):
    st = (C.c_uint64 * 1)(seed)
    x = np.zeros((count, W))
    for i in range(count):
        O.ref().ref_random_normalized(W, C.cast(st, C.c_void_p), int(signed), x[i].ctypes.data)
    return x


def criterion1():
    t0 = time.time()
    n = 1_000_000
    a = random_finite(1001, n, -400, 400)
    b = random_finite(1002, n, -400, 400)
    hi = np.where(np.abs(a) >= np.abs(b), a, b)
    lo = np.where(np.abs(a) >= np.abs(b), b, a)
    bad = {}
    for name, x, y, op in (("two_sum", a, b, 0), ("quick_two_sum", hi, lo, 1), ("two_prod", a, b, 2)):
        s, e = P.eft_batch(name, x, y)
        rs, re_ = np.empty_like(x), np.empty_like(x)
        O.ref().ref_eft_batch(op, n, x.ctypes.data, y.ctypes.data, rs.ctypes.data, re_.ctypes.data)
        mism = int(((s.view(np.uint64) != rs.view(np.uint64)) | (e.view(np.uint64) != re_.view(np.uint64))).sum())
        # exactness on a 2e4 subsample with exact rationals
        inexact = 0
        for i in range(0, n, n // 20000):
            want = Fraction(float(x[i])) * Fraction(float(y[i])) if op == 2 else Fraction(float(x[i])) + Fraction(
                float(y[i]))
            inexact += Fraction(float(s[i])) + Fraction(float(e[i])) != want
        bad[name] = (mism, inexact)
    ok = all(m == 0 and i == 0 for m, i in bad.values())
    verdict(1, ok, "EFT exactness on the GPU, 1e6 seeded pairs per op",
            ", ".join(f"{k} {m} mismatches vs reference, {i} inexact of 2e4 exact checks" for k, (m, i) in bad.items())
            + f"; {time.time() - t0:.1f} s")


def criterion2():
    ops = [(2, "add"), (2, "mul"), (3, "td_add_merge"), (3, "add"), (3, "mul"), (3, "td_mul_q"), (4, "add"),
           (4, "mul")]
    bad = 0
    for idx, (W, op) in enumerate(ops):
        x = normalized_pairs(W, 100_000, 2001 + 2 * idx)
        y = normalized_pairs(W, 100_000, 2002 + 2 * idx)
        got = P.binop_batch(W, op, x, y)
        if op in ("add", "mul"):
            want = O.ref_binop_batch(W, op, x, y)
        else:
            want = np.empty_like(x)
            f = O.ref().ref_td_add_merge_batch if op == "td_add_merge" else O.ref().ref_td_mul_q_batch
            f(x.shape[0], x.ctypes.data, y.ctypes.data, want.ctypes.data)
        bad += int((got.view(np.uint64) != want.view(np.uint64)).sum())
    verdict(2, bad == 0, "lanewise bit-identity, GPU kernels vs reference scalar kernels",
            f"{len(ops)} ops (dd_add dd_mul td_add_merge td_add_q td_mul td_mul_q qd_add qd_mul) x 1e5 inputs: "
            f"{bad} component mismatches")


def criterion3():
    bounds = [(2, "add", 2.0 ** -102), (2, "mul", 2.0 ** -100), (3, "add", 2.0 ** -144), (3, "td_add_merge", 2.0 ** -144),
              (3, "mul", 2.0 ** -140), (4, "add", 2.0 ** -200), (4, "mul", 2.0 ** -195)]
    names = {(2, "add"): "dd_add", (2, "mul"): "dd_mul", (3, "add"): "td_add_q", (3, "td_add_merge"): "td_add_merge",
             (3, "mul"): "td_mul", (4, "add"): "qd_add", (4, "mul"): "qd_mul"}
    ok, parts = True, []
    for i, (W, op, bound) in enumerate(bounds):
        n = 10_000
        x = normalized_pairs(W, n, 3001 + 2 * i, signed=False)
        y = normalized_pairs(W, n, 3002 + 2 * i, signed=False)
        r = P.binop_batch(W, op, x, y)
        worst = 0.0
        for j in range(n):
            ex = dyadic.from_components(x[j]) * dyadic.from_components(y[j]) if op == "mul" else \
                dyadic.from_components(x[j]) + dyadic.from_components(y[j])
            worst = max(worst, dyadic.rel_err(r[j], ex))
        ok &= worst <= bound
        parts.append(f"{names[(W, op)]} 2^{math.log2(worst) if worst > 0 else -1074:.1f} vs 2^{math.log2(bound):.0f}"
                     + (" VIOLATED" if worst > bound else ""))
    verdict(3, ok, "kernel error bounds, 1e4 same-sign normalized pairs per op (GPU results, exact rationals)",
            ", ".join(parts))


def criterion4():
    ok, combos, worst = True, 0, 0.0
    for W in (2, 3, 4):
        for n in (4, 8, 16, 33):
            A = O.ref_fill_random(W, n, n, 4000 + 10 * W + n)
            B = O.ref_fill_random(W, n, n, 4001 + 10 * W + n)
            exact = dyadic.matmul_exact(A, B, n, n)
            bound = n * 4.0 * P.format_eps(W)
            Am, Bm = P.MPMatrix.from_planes(A[:, :, :n]), P.MPMatrix.from_planes(B[:, :, :n])
            naive = P.matmul_naive(Am, Bm)
            for algo in ("naive", "block", "strassen"):
                ref_v = None
                for v in (P.KernelVariant.NORMAL, P.KernelVariant.SIMD_SET, P.KernelVariant.SIMD_LOADSTORE):
                    if algo == "naive":
                        Cm = P.matmul_naive(Am, Bm, v)
                    elif algo == "block":
                        Cm = P.matmul_block(Am, Bm, 32, v)
                    else:
                        Cm = P.matmul_strassen(Am, Bm, 64, 32, v)
                    combos += 1
                    e = dyadic.max_rel_err(Cm.data, exact)
                    worst = max(worst, e / bound)
                    ok &= e <= bound
                    if ref_v is None:
                        ref_v = Cm
                    else:
                        ok &= P.bits_equal(Cm, ref_v)
                    if algo == "block":
                        ok &= P.bits_equal(Cm, naive)
            ok &= np.array_equal(naive.data.view(np.uint64), O.ref_gemm(A, B, n, n).view(np.uint64))
    verdict(4, ok, "matmul within n*4*eps of oracle; block==naive; variants bit-identical; == reference bits",
            f"{combos} algo x variant x precision x size combos; worst rel err at {100 * worst:.2f}% of bound")


def criterion5():
    ok, worst, cells = True, 0.0, ""
    for n in (64, 256):
        rows = (0, 8) if n == 256 else (0, n)
        A2, B2 = P.gen_paper_matrices(2, n)
        exact = dyadic.matmul_exact(A2.data, B2.data, n, n, rows=rows)
        for W in (2, 3, 4):
            A, B = P.gen_paper_matrices(W, n)
            ok &= all(dyadic.from_components(A.data[:, i, j]) == dyadic.from_components(A2.data[:, i, j])
                      for i in range(0, n, 17) for j in range(0, n, 13))
            for algo in ("naive", "block", "strassen"):
                Cm = P.matmul_naive(A, B) if algo == "naive" else (P.matmul_block(A, B) if algo == "block" else
                                                                    P.matmul_strassen(A, B, 64, 32))
                dl = dyadic.digit_loss(dyadic.max_rel_err(Cm.data, exact, rows=rows), P.format_eps(W))
                worst = max(worst, dl)
                if dl > 2.5:
                    ok = False
                    cells += f" [{W} n={n} {algo} loss {dl:.2f}]"
    verdict(5, ok, "paper generators at n=64,256: digit loss <= 2.5 everywhere (n=256: rows 0-7 vs exact)",
            f"worst {worst:.3f} digits{cells}")


def criterion6():
    counts = {}
    for n in (32, 128, 256):
        A = P.fill_random(2, n, n, 6000 + n)
        B = P.fill_random(2, n, n, 6001 + n)
        P.op_counters_reset()
        P.matmul_strassen(A, B, 32, 32)
        counts[n] = P.op_counters_read().leaf_multiplies
    ok = counts[32] > 0 and counts[128] == 49 * counts[32] and counts[256] == 343 * counts[32]
    verdict(6, ok, "strassen leaf multiplies follow the 7^k recursion law",
            f"n=32: {counts[32]}, n=128: {counts[128]} (want {49 * counts[32]}), "
            f"n=256: {counts[256]} (want {343 * counts[32]})")


def criterion7():
    ok, cells = True, 0
    for W in (2, 3, 4):
        n = 256
        A = P.fill_random(W, n, n, 7000 + W)
        B = P.fill_random(W, n, n, 7001 + W)
        sb = P.matmul_block(A, B, 32, P.KernelVariant.SIMD_LOADSTORE)
        ss = P.matmul_strassen(A, B, 64, 32, P.KernelVariant.SIMD_LOADSTORE)
        ok &= np.array_equal(sb.data.view(np.uint64), O.ref_gemm(A.data, B.data, n, n).view(np.uint64))
        ok &= np.array_equal(ss.data.view(np.uint64), O.ref_strassen(A.data, B.data, n, n, 64, 32, 2).view(np.uint64))
        for w in (1, 2, 4, 8):
            cells += 2
            ok &= P.bits_equal(P.matmul_block_parallel(A, B, 32, P.KernelVariant.SIMD_LOADSTORE, w), sb)
            ok &= P.bits_equal(P.matmul_strassen_parallel(A, B, 64, 32, P.KernelVariant.SIMD_LOADSTORE, w), ss)
    verdict(7, ok, "parallel block and strassen bit-identical to serial and to the reference at n=256",
            f"{cells} worker (GPU-count) cells across dd/td/qd, workers {{1,2,4,8}}")


def criterion8():
    for W, name in ((2, "dd"), (4, "qd")):
        n = 1024
        A = P.fill_random(W, n, n, 8000 + W)
        B = P.fill_random(W, n, n, 8001 + W)
        P.matmul_block(A, B)
        t0 = time.perf_counter()
        P.matmul_block(A, B)
        tg = time.perf_counter() - t0
        rows = min(n, 32 * (os.cpu_count() or 1))  # one 32-row block per reference thread
        t0 = time.perf_counter()
        O.ref_gemm(np.ascontiguousarray(A.data[:, :rows]), B.data, n, n, workers=os.cpu_count())
        tc = (time.perf_counter() - t0) * n / rows
        info(8, f"{name} blocked matmul n={n}: GPU (host buffers) {tg:.4f} s vs reference CPU "
                f"({os.cpu_count()} threads, extrapolated from {rows} rows) {tc:.2f} s -> {tc / tg:.0f}x")
    info(8, "performance is recorded, not asserted (bench.py carries the measured numbers)")


def criterion9():
    import io
    from contextlib import redirect_stdout, redirect_stderr
    from paper_2101_06584_b200 import mpfbench
    buf = io.StringIO()
    with redirect_stdout(buf), redirect_stderr(io.StringIO()):
        rc = mpfbench.main(["ewise", "--precision", "td", "--variant", "normal,loadstore", "--sizes", "16384",
                            "--reps", "3", "--seed", "9", "--oracle-max", "0"])
    rows = [l.split(",") for l in buf.getvalue().splitlines()[1:]]
    q = [float(r[7]) for r in rows if r[2] == "add_q"]
    m = [float(r[7]) for r in rows if r[2] == "add_merge"]
    verdict(9, rc == 0 and q and m, "bench report carries both triple-double addition kinds",
            f"{len(q)} add_q rows, {len(m)} add_merge rows")
    if q and m:
        info(9, f"best add_q {max(q):.1f} MFLOPS vs best add_merge {max(m):.1f} MFLOPS (host-buffer calls)")


def main():
    t0 = time.time()
    for idx, fn in enumerate((criterion1, criterion2, criterion3, criterion4, criterion5, criterion6, criterion7,
                              criterion8, criterion9), 1):
        try:
            fn()
        except Exception as e:  # noqa: BLE001 -- the gate's contract: an exception is a FAIL
            verdict(idx, False, fn.__name__, f"exception: {e!r}")
    print(f"acceptance: {FAILS} asserted failure(s), {time.time() - t0:.1f} s total", flush=True)
    return FAILS


if __name__ == "__main__":
    sys.exit(main())
