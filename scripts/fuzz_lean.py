"""Randomised sweep of MPFK_LEAN (one-off evidence, not a unit test): random
widths, shapes and inputs (signed random, structured values with zero tails,
BASELINE wide) through the device entry point (offset windows) and the host
API (pageable / page-locked) -- every result compared BIT FOR BIT with the
chain the same source computes on the host (tests/csrc/arith_host.cpp:
hst_lean_gemm) and, in units of 4*k*u_p, with the reference build's product.
  python scripts/fuzz_lean.py [cases] [seed]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2101_06584_b200 as P  # noqa: E402
from scripts.fuzz_parity import structured  # noqa: E402
from tests.helpers import mismatches, random_signed  # noqa: E402

U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}
H = C.CDLL(os.path.join(ROOT, "tests", "_build", "libarith_host.so"))
H.hst_lean_gemm.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                            C.c_size_t, C.c_void_p, C.c_size_t]


def host_chain(W, A, B, m, n, k):
    Cm = np.zeros((W, m, n))
    assert H.hst_lean_gemm(W, m, k, n, A.ctypes.data, A.shape[2], B.ctypes.data, B.shape[2], Cm.ctypes.data, n) == 0
    return Cm


def diff_over_tol(got, ref, W, n, k):
    d = got[W - 1] - ref[W - 1]
    for w in range(W - 2, -1, -1):
        d = d + (got[w] - ref[w])
    den = np.abs(ref[0][:, :n]).max()
    if den == 0:
        return 0.0 if np.abs(d[:, :n]).max() == 0 else float("inf")
    return float(np.abs(d[:, :n]).max() / den / (4 * max(k, 1) * U_P[W]))


def main(cases, seed):
    rng = np.random.default_rng(seed)
    bad = 0
    worst = 0.0
    for t in range(cases):
        def dim():
            return int(rng.choice([rng.integers(1, 20), rng.integers(20, 120), rng.integers(120, 330)]))
        W = int(rng.integers(2, 5))
        m, n, k = dim(), dim(), dim()
        r = rng.random()
        if r < 0.25:
            A, B = structured(W, m, k, rng), structured(W, k, n, rng)
        elif r < 0.5:
            A = O.orc_fill_baseline(W, m, k, 500 + t, wide=True)
            B = O.orc_fill_baseline(W, k, n, 700 + t, wide=True)
        else:
            A, B = random_signed(W, m, k, 1000 + t), random_signed(W, k, n, 2000 + t)
        want = host_chain(W, A, B, m, n, k)
        if t % 2 == 0:
            dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
            ldc = n + 2 * int(rng.integers(0, 3)) + (n & 1)
            dC = torch.full((W, m, ldc), 2.5, dtype=torch.float64, device="cuda")
            P.gemm_device_ex(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), B.shape[2],
                             k * B.shape[2], dC.data_ptr(), ldc, m * ldc, P.LEAN)
            torch.cuda.synchronize()
            got = dC.cpu().numpy()[:, :, :n]
            what = "device"
        else:
            pinned = bool(rng.integers(0, 2))
            Am = P.MPMatrix.from_planes(A[:, :, :k], pinned=pinned)
            Bm = P.MPMatrix.from_planes(B[:, :, :n], pinned=pinned)
            got = np.ascontiguousarray(P.gemm(Am, Bm, flags=P.LEAN, pinned=pinned).data[:, :, :n])
            what = f"host pinned={pinned}"
        mm = mismatches(got, want)
        ref = O.ref_gemm(A, B, k, n)[:, :, :n]
        d = diff_over_tol(got, ref, W, n, k)
        worst = max(worst, d)
        if mm or not d <= 1.0:
            bad += 1
            print(f"FAIL case {t}: W={W} m={m} n={n} k={k} {what}: {mm} cells off the host chain, "
                  f"{d:.3e} of 4ku_p from the reference", flush=True)
    print(f"{cases} cases, {bad} failures; worst distance from the reference product {worst:.3e} of 4*k*u_p")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 200, int(sys.argv[2]) if len(sys.argv) > 2 else 1))
