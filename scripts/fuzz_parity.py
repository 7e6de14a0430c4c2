"""Randomised parity sweep (one-off evidence, not a unit test): random widths,
shapes, host-buffer kinds, device counts (MPFK_EMULATED_DEVICES), device
entry points with offset windows, K-panel continuation, fused all-gather
(pull, copy-engine flag-gated and staged variants) -- every result compared bit for bit with
the reference build.  python scripts/fuzz_parity.py [cases] [seed] [host threads]"""
import os
import sys

os.environ.setdefault("MPFK_EMULATED_DEVICES", "3")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2101_06584_b200 as P  # noqa: E402
from tests.helpers import mismatches, random_signed  # noqa: E402

def structured(W, rows, cols, rng):
    """planes of exactly representable values with many zero components:
    leading components from {0, +-1, +-2^-j, +-(1 + 2^-52)}, the next
    component 0 or a power of two far below, the rest 0 (normalized)"""
    ld = (cols + 3) & ~3
    a = np.zeros((W, rows, ld))
    lead = rng.choice([0.0, 1.0, -1.0, 0.5, -0.25, 2.0 ** -20, 1.0 + 2.0 ** -52, -(1.0 + 2.0 ** -52)],
                      size=(rows, cols))
    a[0, :, :cols] = lead
    tail = rng.choice([0.0, 2.0 ** -60, -(2.0 ** -70)], size=(rows, cols))
    a[1, :, :cols] = np.where(lead != 0.0, tail, 0.0)
    return a


def one_case(t, rng):
    """case t with its own generator; returns the number of mismatching cases (0/1)"""
    bad_here = 0

    def dim():
        return int(rng.choice([rng.integers(1, 20), rng.integers(20, 200), rng.integers(200, 900)]))

    W = int(rng.integers(2, 5))
    m, n, k = dim(), dim(), dim()
    if t % 9 == 0 and rng.random() < 0.4:  # wide host problems: multi-chunk, half-size end chunks, staging pieces
        m, n, k = int(rng.integers(1500, 3200)), int(rng.integers(1500, 3200)), int(rng.integers(1, 64))
    if rng.random() < 0.25:  # structured: exact small values, zero tails -> renorm5 / vseb zero-residual paths
        A, B = structured(W, m, k, rng), structured(W, k, n, rng)
    else:
        A = random_signed(W, m, k, 1000 + t)
        B = random_signed(W, k, n, 2000 + t)
    want = O.ref_gemm(A, B, k, n)
    kind = t % 9
    if os.environ.get("FUZZ_VERBOSE"):
        print(f"start {t} W={W} m={m} n={n} k={k} kind={kind}", flush=True)
    if kind == 0:  # host API, pageable or pinned, 1..3 (emulated) devices
        pinned = bool(rng.integers(0, 2))
        Am = P.MPMatrix.from_planes(A[:, :, :k], pinned=pinned)
        Bm = P.MPMatrix.from_planes(B[:, :, :n], pinned=pinned)
        Cm = P.MPMatrix(W, m, n, pinned=pinned)
        Cm.data[...] = 1.5
        workers = int(rng.integers(1, 4))
        if os.environ.get("FUZZ_VERBOSE"):
            print(f"  host pinned={pinned} workers={workers}", flush=True)
        P.matmul_block_parallel_into(Cm, Am, Bm, 32, P.KernelVariant.SIMD_LOADSTORE, workers)
        got = Cm.data
        what = f"host pinned={pinned}"
    elif kind == 1:  # device API on offset windows
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        ldc = n + 2 * int(rng.integers(0, 3)) + (n & 1)
        dC = torch.full((W, m, ldc), 2.5, dtype=torch.float64, device="cuda")
        P.gemm_device(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), B.shape[2],
                      k * B.shape[2], dC.data_ptr(), ldc, m * ldc)
        got = dC.cpu().numpy()[:, :, :n]
        want = want[:, :, :n]
        what = "device"
    elif kind == 2:  # K-panel continuation at a random even split
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        ld = B.shape[2]
        dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
        h = int(rng.integers(0, k // 2 + 1)) * 2 if k > 1 else 0
        P.gemm_device(W, m, n, h, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld, k * ld,
                      dC.data_ptr(), ld, m * ld)
        P.gemm_device_acc(W, m, n, k - h, dA.data_ptr() + 8 * h, A.shape[2], m * A.shape[2],
                          dB.data_ptr() + 8 * h * ld, ld, k * ld, dC.data_ptr(), ld, m * ld)
        got = dC.cpu().numpy()
        what = f"continuation h={h}"
        if h == 0:  # a 0-length first panel leaves C = +0; the continuation then is not the product
            return 0
    elif kind == 5:  # Strassen (host API) at a random cutoff
        cut = int(rng.choice([8, 16, 32, 64, 128]))
        Am = P.MPMatrix.from_planes(A[:, :, :k])
        Bm = P.MPMatrix.from_planes(B[:, :, :n])
        got = P.matmul_strassen(Am, Bm, cutoff=cut).data
        want = O.ref_strassen(A, B, k, n, cutoff=cut)
        what = f"strassen cutoff={cut}"
    elif kind == 6:  # elementwise on an m x n pair
        op = ["add", "mul", "add_merge"][int(rng.integers(0, 3 if W == 3 else 2))]
        X = random_signed(W, m, n, 3000 + t)
        Y = random_signed(W, m, n, 4000 + t)
        Xm, Ym = P.MPMatrix.from_planes(X[:, :, :n]), P.MPMatrix.from_planes(Y[:, :, :n])
        out = P.MPMatrix(W, m, n)
        P.ew_apply_into(out, Xm, Ym, {"add": P.EwOp.add, "mul": P.EwOp.mul, "add_merge": P.EwOp.add_merge}[op],
                        P.KernelVariant.SIMD_LOADSTORE)
        got = out.data
        want = O.ref_ew(W, op, X, Y, n, variant=2)
        what = f"ew {op}"
    elif kind == 8:  # dist.matmul_sharded_into without a process group (host panels, gated continuation)
        from paper_2101_06584_b200.dist import matmul_sharded_into
        pinned = bool(rng.integers(0, 2))
        Am = P.MPMatrix.from_planes(A[:, :, :k], pinned=pinned)
        Bm = P.MPMatrix.from_planes(B[:, :, :n], pinned=pinned)
        Cm = P.MPMatrix(W, m, n, pinned=pinned)
        Cm.data[...] = 4.5
        matmul_sharded_into(Cm, Am, Bm, panels=int(rng.integers(1, 9)), device=torch.device("cuda", 0))
        got = Cm.data
        what = f"sharded_into pinned={pinned}"
    elif kind == 7:  # MPFK_FAST: the bit-exact path where no split is planned, deterministic where it is
        Am = P.MPMatrix.from_planes(A[:, :, :k], pinned=bool(rng.integers(0, 2)))
        Bm = P.MPMatrix.from_planes(B[:, :, :n])
        F1 = P.gemm(Am, Bm, flags=P.FAST)
        if P.splitk_segments(W, m, n, k) > 1:
            F2 = P.gemm(Am, Bm, flags=P.FAST)
            if not P.bits_equal(F1, F2):
                bad_here += 1
                print(f"NONDETERMINISTIC FAST case {t}: W={W} m={m} n={n} k={k}", flush=True)
            return bad_here
        got = F1.data
        what = "fast (not split)"
    else:  # fused all-gather, random slice cuts
        kind = 3 if kind == 3 else 4
        ns = int(rng.integers(1, min(8, k) + 1))
        cuts = sorted(set([0, k] + [int(x) for x in rng.integers(0, k + 1, size=ns - 1)]))
        ld = B.shape[2]
        dA = torch.from_numpy(A).cuda()
        sl = [torch.from_numpy(np.ascontiguousarray(B[:, a:b])).cuda() for a, b in zip(cuts, cuts[1:])]
        dB = torch.full((W, k, ld), float("nan"), dtype=torch.float64, device="cuda")
        dC = torch.zeros((W, m, ld), dtype=torch.float64, device="cuda")
        pr = 16 * int(rng.integers(1, 9))
        ptrs = [t_.data_ptr() if t_.numel() else dA.data_ptr() for t_ in sl]
        if kind == 3:
            P.gemm_device_pull(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld, k * ld,
                               dC.data_ptr(), ld, m * ld, ptrs, cuts, pr, int(rng.integers(1, 9)))
            what = f"pull cuts={cuts} panel={pr}"
        elif rng.integers(0, 2) == 0:
            P.gemm_device_gathered(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld,
                                   k * ld, dC.data_ptr(), ld, m * ld, ptrs, cuts, pr)
            what = f"gathered cuts={cuts} panel={pr}"
        else:  # staged: copy-engine gather in growing K panels, one launch per panel
            head = 16 * int(rng.integers(0, 5))
            P.gemm_device_staged(W, m, n, k, dA.data_ptr(), A.shape[2], m * A.shape[2], dB.data_ptr(), ld,
                                 k * ld, dC.data_ptr(), ld, m * ld, ptrs, cuts, head)
            what = f"staged cuts={cuts} head={head}"
        torch.cuda.synchronize()
        got = dC.cpu().numpy()
    torch.cuda.synchronize()
    if os.environ.get("FUZZ_VERBOSE"):
        print(f"case {t} W={W} m={m} n={n} k={k} {what}", flush=True)
    mm = mismatches(got, want)
    if mm:
        bad_here += 1
        print(f"MISMATCH case {t}: W={W} m={m} n={n} k={k} {what}: {mm} cells", flush=True)
    return bad_here


def run(cases, seed, threads=1):
    """cases split over `threads` host threads calling the library at once"""
    import threading
    total = [0]
    lock = threading.Lock()

    def worker(i):
        rng = np.random.default_rng([seed, i])
        for t in range(i, cases, threads):
            b = one_case(t, rng)
            with lock:
                total[0] += b

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return total[0]


if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    threads = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    bad = run(cases, seed, threads)
    print(f"{cases} cases, {bad} with mismatches")
    sys.exit(1 if bad else 0)
