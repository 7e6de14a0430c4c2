#!/usr/bin/env python
"""bench.py -- DD/TD/QD GEMM throughput on B200 (the BASELINE.json metric).

One "step" is one C = A*B over the workload (BASELINE.json configs), C sharded
by contiguous row blocks across ranks (one process per GPU).  Inside the
timed step: for N > 1 the B replication from rank 0 over NVLink (NCCL
broadcast), then the sm_100a GEMM on the rank's row shard.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload dd8192]
  python bench.py --impl reference ...   the reference's own CPU GEMM

Prints ONE JSON line on rank 0.  `value` is MPF Gflops = 2*m*n*k / t over the
whole job (max over ranks of the device-timed step), `e2e` the same metric
through the public host-buffer API (the C ABI; H2D + kernel + D2H every
step), `roofline` the GEMM kernel's FP64 lane-op rate against the FP64 pipe
peak measured on this GPU, `cpu_baseline` the reference's CPU GEMM timed on a
bounded sample on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs -> (width, n, wide inputs)
WORKLOADS = {
    "dd1024": (2, 1024, False),   # configs[0]
    "td1024": (3, 1024, False),   # configs[1]
    "qd1024": (4, 1024, False),   # configs[2]
    "dd8192": (2, 8192, False),   # configs[3]
    "td4096": (3, 4096, True),    # configs[4]
    "qd4096": (4, 4096, True),    # configs[4]
}
DEFAULT_WORKLOAD = "dd8192"
OPS_PER_MAC = {2: 20, 3: 132, 4: 218}
# FP64 instructions the kernels execute per MAC (ncu sass op counts /
# (m n k), profiles/r01b/metrics_*.csv): TD folds 11 operations on the
# zero-extended fourth lane of td_add_q (DESIGN 4.1) and, in the fast pass,
# skips the two operations of vseb's residual that only its rare path reads
EXEC_OPS_PER_MAC = {2: 20, 3: 119, 4: 218}
NAMES = {2: "DD", 3: "TD", 4: "QD"}
L2_BYTES = 126 * 2 ** 20
METRIC = "MPF Gflops (2mnk/s), DD/TD/QD GEMM"
NOMINAL_FP64_LANE_OPS = 148 * 64 * 1.965e9  # 18.61e12 lane-ops/s


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mpfk", "reference"], default="mpfk")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample time")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N > 1: broadcast all of B before the GEMM instead of K-panel overlap")
    ap.add_argument("--panels", type=int, default=4, help="N > 1: K panels for the overlapped broadcast")
    ap.add_argument("--dist", action="store_true",
                    help="initialise the NCCL process group and run the collective path even at N == 1")
    ap.add_argument("--fused-allgather", action="store_true",
                    help="B row-sliced across ranks and pulled over NVLink inside the GEMM kernel "
                         "(mpfk_gemm_device_pull) instead of an NCCL broadcast (the default at N > 1; "
                         "this flag forces it at N == 1 with --dist)")
    ap.add_argument("--nccl-bcast", action="store_true",
                    help="N > 1: replicate B with NCCL broadcasts in K panels instead of the fused kernel")
    ap.add_argument("--gather-mode", choices=["copy", "pull"], default="pull",
                    help="fused all-gather: the GEMM's CTAs pull B's panels over peer memory (pull; progress "
                         "guaranteed by construction) or the copy engines gather and flag them (copy; needs the "
                         "peer copies to run on copy engines)")
    ap.add_argument("--pull-panel", type=int, default=256, help="fused all-gather: K rows per panel")
    ap.add_argument("--pull-chunk", type=int, default=2,
                    help="fused all-gather: rows per copy chunk (small chunks spread each panel over many CTAs)")
    ap.add_argument("--check", action="store_true",
                    help="after timing, check the sharded step's C bitwise against a plain one-shot GEMM")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "reasons": reasons}


def load_traffic(workload):
    """dram bytes per launch of the GEMM kernel from the committed ncu
    summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(workload)
    except Exception:
        return None


class CpuReference:
    """The reference's own matmul_block_parallel_into (oracle/_ref, compiled
    from the unmodified mpfkit sources with its own flags) on a bounded row
    sample of the same workload.  Rows of C are independent and the
    reference hands whole 32-row blocks to its threads (linalg.hpp:413-421),
    so a sample of 32*threads rows keeps every thread busy and its rate is
    the full GEMM's rate."""

    def __init__(self, W, n, wide, threads=None):
        import paper_2101_06584_b200 as P  # input generator only
        self.P, self.W, self.n, self.wide = P, W, n, wide
        self.threads = threads or os.cpu_count() or 1
        self.B = P.fill_baseline(W, n, n, 2, wide=wide)

    def run(self, rows):
        import oracle as O
        A = self.P.fill_baseline(self.W, rows, self.n, 1, wide=self.wide)
        t0 = time.perf_counter()
        O.ref_gemm(A.data, self.B.data, self.n, self.n, workers=self.threads, n_min=32, variant=2)
        return time.perf_counter() - t0

    def measure(self, target_s):
        """(gflops, seconds, rows): grow the sample in whole waves of
        32-row blocks until it takes >= target_s / 2."""
        wave = 32 * self.threads
        rows = min(self.n, wave)
        while True:
            t = self.run(rows)
            if t >= target_s / 2 or rows >= self.n:
                break
            waves = max(1, int(target_s / max(t, 1e-3)))
            rows = min(self.n, rows * waves)
        return 2.0 * rows * self.n * self.n / t / 1e9, t, rows


def cpu_model():
    """The host CPU model (report the core count and CPU model)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or None


def run_reference(args, ws, rank):
    W, n, wide = WORKLOADS[args.workload]
    if rank != 0:
        return
    ref = CpuReference(W, n, wide)
    vals, secs = [], []
    rows = None
    for i in range(args.warmup + args.steps):
        g, s, rows = ref.measure(max(2.0, args.cpu_seconds / max(1, args.steps)))
        if i >= args.warmup:
            vals.append(g)
            secs.append(s)
    v = statistics.median(vals)
    threads = ref.threads
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 4),
        "unit": "Gflop/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(secs), 2),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE.json seeded distributions, SplitMix64)",
        "config": {"workload": args.workload, "precision": NAMES[W], "m": n, "n": n, "k": n,
                   "inputs": "wide 2^[-30,30]" if wide else "U[-1,1)"},
        "cpu_baseline": {"value": round(v, 4), "unit": "Gflop/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{rows} of {n} rows of C per step (rows are independent), "
                                   "mpfkit matmul_block_parallel_into(n_min=32, SIMD_LOADSTORE, "
                                   f"workers={threads}), AVX2 build of /root/reference/proj"},
        "e2e": {"value": round(v, 4), "unit": "Gflop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


def run_mpfk(args, ws, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2101_06584_b200 as P
    from paper_2101_06584_b200.dist import shard_rows, sharded_gemm_step, sharded_gemm_step_overlapped

    W, n, wide = WORKLOADS[args.workload]
    m = k = n
    torch.cuda.set_device(local)
    P.set_device(local)  # libmpfk has its own CUDA runtime: mirror the choice
    dev = torch.device("cuda", local)
    use_dist = ws > 1 or args.dist
    if use_dist and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)

    r0, r1 = shard_rows(m, ws, rank)
    rows = r1 - r0
    ld = P.pad_columns(n)
    stream = torch.cuda.current_stream(dev)

    # ---- inputs resident in HBM: A row shard, B on rank 0 (replicated per step)
    A = P.fill_baseline(W, rows, k, 1, wide=wide, row0=r0)
    dA = torch.from_numpy(A.data).to(dev)
    dB = torch.empty((W, k, ld), dtype=torch.float64, device=dev)
    if rank == 0:
        Bh = P.fill_baseline(W, k, n, 2, wide=wide)
        dB.copy_(torch.from_numpy(Bh.data))
    dC = torch.zeros((W, max(rows, 1), ld), dtype=torch.float64, device=dev)
    flush = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device=dev) if \
        (W * 8 * (m * k + k * n) < 2 * L2_BYTES) else None

    launches = [0]

    overlap = use_dist and not args.no_overlap
    slices = None
    fused_note = None
    # N > 1: the fused all-gather -> GEMM kernel (B pulled over NVLink peer
    # memory inside the GEMM) unless --nccl-bcast; if the CUDA IPC mapping
    # is unavailable on any rank, every rank falls back to the NCCL K-panel
    # broadcast together
    if args.fused_allgather or (ws > 1 and not args.nccl_bcast and not args.no_overlap):
        from paper_2101_06584_b200.dist import PeerBSlices
        ok = 1
        try:
            slices = PeerBSlices(W, k, ld)
            c0, c1 = slices.cuts[slices.rank], slices.cuts[slices.rank + 1]
            slices.upload(P.fill_baseline(W, c1 - c0, n, 2, wide=wide, row0=c0).data)
        except Exception as e:  # e.g. CUDA IPC not permitted in this container
            ok = 0
            fused_note = f"fused all-gather unavailable ({type(e).__name__}: {str(e)[:120]})"
            print(f"bench: {fused_note}; using the NCCL K-panel broadcast", file=sys.stderr)
        if use_dist:
            t = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = int(t.item())
            dist.barrier()
        if not ok and slices is not None:
            slices.close()
            slices = None

    def step():
        ev_mid = torch.cuda.Event(enable_timing=True)
        if slices is not None:
            # one kernel: pull B's panels from the ranks' slices while computing
            ev_mid.record(stream)
            launches[0] += slices.step(W, dA, dB, dC, rows, n, k, args.pull_panel, args.pull_chunk, stream,
                                       mode=args.gather_mode)
            return ev_mid
        if overlap:
            # B broadcast in K panels, each panel's GEMM gated on its own panel
            ev_mid.record(stream)
            launches[0] += sharded_gemm_step_overlapped(W, dA, dB, dC, rows, n, k, ld, panels=args.panels,
                                                        stream=stream)
            return ev_mid

        def gemm(W_, dA_, dB_, dC_, rows_, n_, k_, ld_):
            ev_mid.record(stream)  # after the B broadcast
            return P.gemm_device(W_, rows_, n_, k_, dA_.data_ptr(), ld_, rows_ * ld_, dB_.data_ptr(), ld_,
                                 k_ * ld_, dC_.data_ptr(), ld_, rows_ * ld_, stream.cuda_stream)

        launches[0] += sharded_gemm_step(W, dA, dB, dC, rows, n, k, ld, gemm=gemm)
        if not rows:
            ev_mid.record(stream)
        return ev_mid

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # FP64 pipe peak on this GPU (the roofline denominator)
    peak_ops, _ = P.fp64_peak()

    clocks = ClockSampler(local)
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    P.gemm_redo_count(reset=True)  # TD/QD fast-pass redo counter (synchronises; outside the timed region)
    clocks.start()
    time.sleep(0.3)
    launches[0] = 0
    evs = []
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()  # L2 flush between timed iterations, outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mid = step()
        e1.record(stream)
        evs.append((e0, mid, e1))
    torch.cuda.synchronize(dev)
    if use_dist:
        dist.barrier()
    clk = clocks.stop()
    redo = P.gemm_redo_count(reset=True)
    check = None
    if args.check and rows:
        ref = torch.zeros_like(dC)
        P.gemm_device(W, rows, n, k, dA.data_ptr(), ld, rows * ld, dB.data_ptr(), ld, k * ld, ref.data_ptr(), ld,
                      rows * ld, stream.cuda_stream)
        torch.cuda.synchronize(dev)
        check = bool(torch.equal(ref.view(torch.int64), dC.view(torch.int64)))
    step_ms = [a.elapsed_time(c) for a, _, c in evs]
    kern_ms = [b.elapsed_time(c) for _, b, c in evs]
    bc_ms = [a.elapsed_time(b) for a, b, _ in evs]
    t_step = sum(step_ms) / len(step_ms)
    t_kern = sum(kern_ms) / len(kern_ms)
    if use_dist:
        t = torch.tensor([t_step, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step, t_kern = t.tolist()
    flops = 2.0 * m * n * k
    value = flops / (t_step * 1e-3) / 1e9

    # ---- e2e through the public host-buffer API (C ABI), pinned host buffers
    e2e = None
    if not args.no_e2e:
        Ah = P.fill_baseline(W, rows, k, 1, wide=wide, row0=r0, pinned=True)
        Bh2 = P.fill_baseline(W, k, n, 2, wide=wide, pinned=True)
        Ch = P.MPMatrix(W, rows, n, pinned=True)
        if use_dist:
            # one rank per GPU: each rank copies its A shard and 1/ws of B
            # from the host; B's panels are all-gathered over NVLink
            from paper_2101_06584_b200.dist import matmul_sharded_into

            def e2e_call():
                matmul_sharded_into(Ch, Ah, Bh2, panels=args.panels, device=dev)
        else:
            def e2e_call():
                P.matmul_block_parallel_into(Ch, Ah, Bh2, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
        e2e_call()  # warm
        e2e_steps = max(1, min(args.steps, 3))
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_call()
            _ = float(Ch.data[0, 0, 0]) if rows else 0.0  # result read on the host
        if use_dist:
            dist.barrier()
        t_e2e = (time.perf_counter() - t0) / e2e_steps
        st = None if use_dist else P.last_stats()
        if use_dist:
            t = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = t.item()
        h2d = 8 * W * (m * k + k * n)  # (ws > 1: each rank copies 1/ws of B)
        d2h = 8 * W * m * n
        e2e = {"value": round(flops / t_e2e / 1e9, 3), "unit": "Gflop/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e2e_steps,
               "api": "dist.matmul_sharded_into (per rank)" if use_dist else
                      "matmul_block_parallel_into (C ABI, host buffers)"}
        if st is not None:
            e2e["ms_breakdown"] = {k_: round(st[k_], 3) for k_ in ("h2d_ms", "kernel_ms", "d2h_ms", "total_ms")}
        # spot-check the e2e result against the device-resident run (same inputs)
        if rows:
            same = bool((torch.from_numpy(np.ascontiguousarray(Ch.data)).view(torch.int64) ==
                         dC[:, :rows, :].cpu().view(torch.int64)).all())
            e2e["matches_device_run"] = same

    # ---- CPU baseline: the reference's own GEMM on this host (rank 0, N == 1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            ref = CpuReference(W, n, wide)
            g, s, srows = ref.measure(args.cpu_seconds)
            thr = ref.threads
            cpu = {"value": round(g, 4), "unit": "Gflop/s", "cores": thr, "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"{srows} of {n} rows of C ({s:.1f} s), mpfkit matmul_block_parallel_into"
                             f"(n_min=32, SIMD_LOADSTORE, workers={thr}), AVX2 build of the reference"}
        except Exception as e:  # the checker is optional; the GPU number stands alone
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        ops = OPS_PER_MAC[W]
        # dominant kernel (the GEMM) of rank 0's shard: algorithmic FP64 ops / launch time
        achieved = rows * n * k * ops / (t_kern * 1e-3) / 1e9  # Gop/s
        traffic = load_traffic(args.workload) if ws == 1 else None  # captured on the 1-GPU launch
        parallelism = f"row-shard x{ws}"
        if fused_note:
            parallelism += f" [{fused_note}]"
        if slices is not None and args.gather_mode == "copy":
            parallelism += (" + fused all-gather->GEMM (copy engines gather B's K panels from the peers' slices, "
                            "one GEMM launch waits per panel on stream-memory flags)")
        elif slices is not None:
            parallelism += " + fused all-gather->GEMM (B pulled over peer memory inside the GEMM kernel)"
        elif overlap:
            parallelism += f" + NCCL broadcast of B in {args.panels} K panels overlapped with the GEMM"
        elif use_dist:
            parallelism += " + NCCL broadcast of B"
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "Gflop/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(t_step, 3),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE.json seeded distributions, SplitMix64), generated on the host",
            "config": {"workload": args.workload, "precision": NAMES[W], "m": m, "n": n, "k": k,
                       "inputs": "wide 2^[-30,30]" if wide else "U[-1,1)", "rows_per_rank": rows,
                       "parallelism": parallelism,
                       "l2": "flushed between timed steps" if flush is not None else
                             "inputs larger than L2 (126 MB)",
                       "bit_exact": True},
            "roofline": {"bound": "fp64", "achieved": round(achieved, 1),
                         "peak": round(peak_ops / 1e9, 1), "unit": "Gop/s (FP64 lane ops)",
                         "frac": round(achieved / (peak_ops / 1e9), 4),
                         "frac_of_nominal": round(achieved / (NOMINAL_FP64_LANE_OPS / 1e9), 4),
                         "ops_per_mac": ops, "kernel_ms": round(t_kern, 3),
                         "ops_per_mac_executed": EXEC_OPS_PER_MAC[W],
                         # TD/QD: warp k-tiles per step that left the branch-free fast
                         # pass and were recomputed exactly (DESIGN 4.2)
                         "redo_warp_ktiles_per_step": round(redo / max(args.steps, 1), 1),
                         "frac_executed": round(achieved * EXEC_OPS_PER_MAC[W] / ops / (peak_ops / 1e9), 4),
                         "peak_source": "measured on this GPU by mpfk_fp64_peak (DFMA chains); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "traffic": traffic,
                         # the bound is the FP64 pipe: DRAM traffic (L2 re-reads of B across
                         # tile bands) vs the compulsory bytes, and the HBM rate it implies
                         "compulsory_bytes": 8 * W * (rows * k + k * n + rows * n),
                         "traffic_gbs": round(traffic / (t_kern * 1e-3) / 1e9, 1) if traffic else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches[0],
            "clocks": clk,
            "bcast_ms": round(sum(bc_ms) / len(bc_ms), 3) if (ws > 1 and not overlap) else 0.0,
        }
        if check is not None:
            line["check_sharded_equals_one_shot"] = check
        emit(line, args)
    if use_dist:
        dist.barrier()
    if slices is not None:
        slices.close()
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_mpfk(args, ws, rank, local)


if __name__ == "__main__":
    main()
