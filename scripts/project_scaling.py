"""Per-rank time of the row-sharded GEMM at N = 1, 2, 4, 8 ranks, measured on
ONE B200: rank 0's shard (rows shard_rows(m, N, 0) of C, full B) through

  * plain: mpfk_gemm_device on a resident B (the compute alone), and
  * pull:  mpfk_gemm_device_pull with B split into N row slices that live in
           this GPU's own memory (the fused all-gather kernel's bookkeeping and
           copies, HBM-to-HBM instead of over NVLink),
  * staged: mpfk_gemm_device_staged (bench.py's default transport) on the same
           slices: copy-engine gather in growing K panels, one GEMM launch per
           panel gated on its event (HBM-to-HBM copies here),

and the projected strong-scaling efficiency T(1) / (N * T(N)).  Projection
only: the NVLink leg is not exercised (each rank pulls (N-1)/N of B, DD n=8192
7/8 GiB at N = 8: ~1.3 ms at 700 GB/s against ~80 ms of compute, overlapped
tile by tile), and the driver computes real scaling from its own multi-GPU
runs.  python scripts/project_scaling.py [--workload dd8192] > gpurun_out/scaling.log"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_06584_b200 as P  # noqa: E402
from bench import WORKLOADS, OPS_PER_MAC  # noqa: E402
from paper_2101_06584_b200.dist import shard_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="dd8192")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--lean", action="store_true",
                help="flags = MPFK_LEAN (tolerance mode): the plain and staged legs only; each shard is compared "
                     "with the one-shot lean product's rows (plain: bitwise; staged: within 4*k*u_p)")
a = ap.parse_args()
W, n, wide = WORKLOADS[a.workload]
ld = P.pad_columns(n)
A = torch.from_numpy(P.fill_baseline(W, n, n, 1, wide=wide).data).cuda()
B = torch.from_numpy(P.fill_baseline(W, n, n, 2, wide=wide).data).cuda()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn):
    fn()
    best = 1e30
    for _ in range(a.reps):
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


ref = torch.zeros_like(A)
P.gemm_device_ex(W, n, n, n, A.data_ptr(), ld, n * ld, B.data_ptr(), ld, n * ld, ref.data_ptr(), ld, n * ld,
                 P.LEAN if a.lean else P.BIT_EXACT, s.cuda_stream)
U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}


def lean_leg(N, r0, r1, rows, Ash, slices, cuts, t1):
    """plain and staged with MPFK_LEAN"""
    Csh = torch.zeros((W, rows, ld), dtype=torch.float64, device="cuda")
    plain = timed(lambda: P.gemm_device_ex(W, rows, n, n, Ash.data_ptr(), ld, rows * ld, B.data_ptr(), ld, n * ld,
                                           Csh.data_ptr(), ld, rows * ld, P.LEAN, s.cuda_stream))
    same = bool(torch.equal(Csh.view(torch.int64), ref[:, r0:r1].view(torch.int64)))  # shard-independent
    Cs, Bst = torch.zeros_like(Csh), torch.zeros_like(B)
    ts = timed(lambda: P.gemm_device_staged(W, rows, n, n, Ash.data_ptr(), ld, rows * ld, Bst.data_ptr(), ld, n * ld,
                                            Cs.data_ptr(), ld, rows * ld, [x.data_ptr() for x in slices], cuts, 0,
                                            s.cuda_stream, flags=P.LEAN))
    d = Cs[W - 1] - ref[W - 1, r0:r1]
    for w in range(W - 2, -1, -1):
        d = d + (Cs[w] - ref[w, r0:r1])
    diff = float(d[:, :n].abs().max() / ref[0, r0:r1, :n].abs().max()) / (4 * n * U_P[W])
    t1 = plain if N == 1 else t1
    print(json.dumps({"workload": a.workload, "flags": "MPFK_LEAN", "ranks": N, "rows_per_rank": rows,
                      "plain_ms": round(plain, 3), "staged_ms": round(ts, 3), "plain_equals_one_shot_rows": same,
                      "staged_diff_over_tolerance": round(diff, 6),
                      "projected_efficiency_plain": round(t1 / (N * plain), 4),
                      "projected_efficiency_staged": round(t1 / (N * ts), 4)}), flush=True)
    return t1


t1 = None
for N in (1, 2, 4, 8):
    r0, r1 = shard_rows(n, N, 0)
    rows = r1 - r0
    Ash = A[:, r0:r1].contiguous()
    if a.lean:
        cuts = [shard_rows(n, N, r, 16)[0] for r in range(N)] + [n]
        t1 = lean_leg(N, r0, r1, rows, Ash, [B[:, cuts[r]:cuts[r + 1]].contiguous() for r in range(N)], cuts, t1)
        continue
    Csh = torch.zeros((W, rows, ld), dtype=torch.float64, device="cuda")
    plain = timed(lambda: P.gemm_device(W, rows, n, n, Ash.data_ptr(), ld, rows * ld, B.data_ptr(), ld, n * ld,
                                        Csh.data_ptr(), ld, rows * ld, s.cuda_stream))
    ok_plain = bool(torch.equal(Csh.view(torch.int64), ref[:, r0:r1].view(torch.int64)))
    # B in N row slices (the ranks' own uploads), gathered by the GEMM kernel
    cuts = [shard_rows(n, N, r, 16)[0] for r in range(N)] + [n]
    slices = [B[:, cuts[r]:cuts[r + 1]].contiguous() for r in range(N)]
    Bfull = torch.zeros_like(B)
    Cp = torch.zeros_like(Csh)

    def pull():
        P.gemm_device_pull(W, rows, n, n, Ash.data_ptr(), ld, rows * ld, Bfull.data_ptr(), ld, n * ld,
                           Cp.data_ptr(), ld, rows * ld, [x.data_ptr() for x in slices], cuts, 256, 2, s.cuda_stream)

    tp = timed(pull)
    ok_pull = bool(torch.equal(Cp.view(torch.int64), ref[:, r0:r1].view(torch.int64)))
    Cs = torch.zeros_like(Csh)
    Bst = torch.zeros_like(B)

    def staged():
        P.gemm_device_staged(W, rows, n, n, Ash.data_ptr(), ld, rows * ld, Bst.data_ptr(), ld, n * ld,
                             Cs.data_ptr(), ld, rows * ld, [x.data_ptr() for x in slices], cuts, 0, s.cuda_stream)

    ts = timed(staged)
    ok_staged = bool(torch.equal(Cs.view(torch.int64), ref[:, r0:r1].view(torch.int64)))
    if N == 1:
        t1 = plain
    macs = rows * n * n
    line = {"workload": a.workload, "ranks": N, "rows_per_rank": rows, "plain_ms": round(plain, 3),
            "pull_ms": round(tp, 3), "staged_ms": round(ts, 3), "bit_exact": ok_plain and ok_pull and ok_staged,
            "per_rank_frac_of_fp64_peak": round(macs * OPS_PER_MAC[W] / (plain * 1e-3) / P.fp64_peak()[0], 4),
            "projected_efficiency_plain": round(t1 / (N * plain), 4),
            "projected_efficiency_pull": round(t1 / (N * tp), 4),
            "projected_efficiency_staged": round(t1 / (N * ts), 4)}
    print(json.dumps(line), flush=True)
