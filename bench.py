#!/usr/bin/env python
"""bench.py -- DD/TD/QD GEMM throughput on B200 (the BASELINE.json metric).

One "step" is one C = A*B over the workload (BASELINE.json configs), C sharded
by contiguous row spans across ranks (one process per GPU), the reference's
worker partition (linalg.hpp:402-433, spans :413-421) lifted to GPUs.
Inside the timed step at N > 1: B's replication -- by default the copy
engines gather it over NVLink from the ranks' 1/N slices in growing K panels
while per-panel GEMM launches compute (mpfk_gemm_device_staged) -- and the
sm_100a GEMM on the rank's row shard.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload dd8192]
  python bench.py --impl reference ...   the reference's own CPU GEMM

`--gpus N` outside torchrun spawns N local ranks itself (launch.py) and fails
loudly when fewer than N B200s are visible; under torchrun it must equal
WORLD_SIZE.

Prints ONE JSON line on rank 0.  `value` is MPF Gflops = 2*m*n*k / t over the
whole job (max over ranks of the device-timed step) for the headline
workload (DD 8192, BASELINE configs[3]); `workloads` carries the same record
for TD/QD 4096 (configs[4]) and the three n=1024 configs (configs[0-2]).
`e2e` is the same metric through the public host-buffer API (the C ABI;
H2D + kernel + D2H every step) from page-locked buffers, `e2e_pageable` from
ordinary (pageable) host memory like a reference MPMatrix; `roofline` the
GEMM kernel's FP64 lane-op rate against the FP64 pipe peak measured on this
GPU; `cpu_baseline` the reference's CPU GEMM timed on a bounded sample on
this host.
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
DEFAULT_EXTRA = "td4096,qd4096,dd1024,td1024,qd1024"
OPS_PER_MAC = {2: 20, 3: 132, 4: 218}
# FP64 instructions the kernels execute per MAC (ncu sass op counts /
# (m n k), profiles/r01b/metrics_*.csv): TD folds 11 operations on the
# zero-extended fourth lane of td_add_q (DESIGN 4.1) and, in the fast pass,
# skips the two operations of vseb's residual that only its rare path reads
EXEC_OPS_PER_MAC = {2: 20, 3: 110, 4: 212}
NAMES = {2: "DD", 3: "TD", 4: "QD"}
L2_BYTES = 126 * 2 ** 20
METRIC = "MPF Gflops (2mnk/s), DD/TD/QD GEMM"
NOMINAL_FP64_LANE_OPS = 148 * 64 * 1.965e9  # 18.61e12 lane-ops/s
SEED_A, SEED_B = 1, 2
TRANSPORTS = ("staged", "nccl", "bcast", "pull", "copy")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks) of this node; outside torchrun N > 1 spawns N local ranks")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mpfk", "reference"], default="mpfk")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD,
                    help="the headline workload (value, e2e, roofline, cpu_baseline)")
    ap.add_argument("--extra", default=DEFAULT_EXTRA,
                    help="comma-separated further workloads reported under 'workloads' ('none': skip)")
    ap.add_argument("--extra-steps", type=int, default=0, help="timed steps per extra workload (0: min(steps, 5))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pageable", action="store_true", help="skip the pageable-buffer e2e leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-waves", type=int, default=2,
                    help="CPU samples: waves of 32-row blocks per reference worker")
    ap.add_argument("--cpu-steps", type=int, default=3, help="cpu_baseline: timed reference calls (median)")
    ap.add_argument("--no-lean", action="store_true",
                    help="skip the MPFK_LEAN (tolerance mode) leg reported next to each bit-exact workload")
    ap.add_argument("--lean-dist", action="store_true",
                    help="N > 1: also run the MPFK_LEAN leg over the staged transport (off by default: the "
                         "multi-rank line is about the bit-exact headline; always on with --emulate-on-one-gpu)")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    ap.add_argument("--transport", choices=TRANSPORTS, default=None,
                    help="N > 1 replication of B: staged (copy engines gather B's growing K panels from the "
                         "ranks' slices over NVLink, one GEMM launch per panel gated on its event; default), "
                         "nccl (NCCL broadcast in K panels overlapped with per-panel GEMMs), bcast (NCCL "
                         "broadcast of all of B, then the GEMM), pull (the GEMM's CTAs pull B over peer "
                         "memory), copy (copy engines + in-kernel panel flags)")
    ap.add_argument("--panels", type=int, default=4, help="nccl transport: K panels")
    ap.add_argument("--dist", action="store_true",
                    help="initialise the process group and run the collective path even at N == 1")
    ap.add_argument("--pull-panel", type=int, default=256, help="pull/copy transports: K rows per panel")
    ap.add_argument("--pull-chunk", type=int, default=2, help="pull transport: rows per copy chunk")
    ap.add_argument("--check", dest="check", action="store_true", default=None,
                    help="check the sharded step's C bitwise against a one-shot GEMM (default at N > 1)")
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--emulate-on-one-gpu", action="store_true",
                    help="TEST ONLY: run the N ranks on GPU 0 with a gloo group (the full N > 1 code path -- "
                         "launcher, IPC slices, staged gather, sharded check -- on a one-GPU box; timings "
                         "are meaningless, no e2e leg)")
    # round-1 spellings of --transport
    ap.add_argument("--no-overlap", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--nccl-bcast", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--fused-allgather", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--gather-mode", choices=["copy", "pull", "staged"], default=None, help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.transport is None:
        if args.fused_allgather:
            args.transport = args.gather_mode or "pull"
        elif args.nccl_bcast:
            args.transport = "nccl"
        elif args.no_overlap:
            args.transport = "bcast"
    return args


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def extra_workloads(args):
    if not args.extra or args.extra.strip().lower() == "none":
        return []
    out = []
    for w in args.extra.split(","):
        w = w.strip()
        if not w or w == args.workload:
            continue
        if w not in WORKLOADS:
            raise SystemExit(f"bench: unknown workload {w!r} in --extra")
        out.append(w)
    return out


def flush_needed(W, n):
    """Inputs smaller than twice the L2 get an L2 flush between timed steps."""
    return W * 8 * 2 * n * n < 2 * L2_BYTES


def config_for(workload, ws):
    """The workload's config dict, identical in both arms (the driver
    compares them)."""
    W, n, wide = WORKLOADS[workload]
    return {"workload": workload, "precision": NAMES[W], "m": n, "n": n, "k": n,
            "inputs": "wide 2^[-30,30]" if wide else "U[-1,1)",
            "parallelism": f"C row-sharded over {ws} GPU(s) (reference worker partition, linalg.hpp:413-421)",
            "l2": "flushed between timed steps" if flush_needed(W, n) else "inputs larger than L2 (126 MB)",
            "bit_exact": True}


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


# ---------------------------------------------------------------------------
# the reference's CPU GEMM (test infrastructure: oracle/ only)
# ---------------------------------------------------------------------------

class CpuReference:
    """The reference's own matmul_block_parallel_into (oracle/_ref: the
    unmodified mpfkit sources compiled with its own flags) on a bounded row
    sample of the workload.  Inputs come from the oracle's restatement of
    the BASELINE generator (bit-identical to the library's,
    tests/test_capi.py), the reference MPMatrix operands are built ONCE
    (oracle.RefPrepared), and only the matmul_block_parallel_into call is
    timed, inside C++ (steady_clock), like bench::time_matmul
    (bench.cpp:33-38).  Rows of C are independent and the reference hands
    each worker a contiguous span of whole 32-row blocks (linalg.hpp:413-421),
    so a sample of `waves` blocks per worker keeps every worker busy for the
    whole call and its rate is the full GEMM's rate."""

    def __init__(self, workload, waves=3):
        import oracle as O
        W, n, wide = WORKLOADS[workload]
        self.O, self.W, self.n = O, W, n
        info = O.host_cpu_info()
        # the reference's default worker count for its threads (bench.cpp:196-200)
        self.threads = int(O.ref().ref_hardware_concurrency()) or info["threads"]
        self.physical_cores = info["physical_cores"]
        self.cpu_model = info["cpu_model"]
        self.rows = min(n, 32 * self.threads * max(1, waves))
        self.warm_rows = min(n, 32 * self.threads)
        A = O.orc_fill_baseline(W, self.rows, n, SEED_A, wide=wide)
        B = O.orc_fill_baseline(W, n, n, SEED_B, wide=wide)
        self.prep = O.RefPrepared(A, B, n, n)
        del A, B
        self.warm = self.prep.with_a(O.orc_fill_baseline(W, self.warm_rows, n, SEED_A, wide=wide))

    def warmup(self):
        return self.warm.run(self.threads, n_min=32, variant=2)

    def step(self):
        """(Gflop/s, seconds) of one timed reference call on the sample."""
        s = self.prep.run(self.threads, n_min=32, variant=2)
        return 2.0 * self.rows * self.n * self.n / s / 1e9, s

    def describe(self, value):
        return {"value": round(value, 4), "unit": "Gflop/s", "cores": self.threads,
                "physical_cores": self.physical_cores, "kind": "reference", "cpu_model": self.cpu_model,
                "sample": f"{self.rows} of {self.n} rows of C per step ({self.rows // (32 * self.threads)} waves of "
                          f"32-row blocks per worker); mpfkit matmul_block_parallel_into(n_min=32, "
                          f"SIMD_LOADSTORE, workers={self.threads}) on operands built once, only that call "
                          f"timed (C++ steady_clock); AVX2 build of the reference's own sources"}

    def close(self):
        self.prep.close()
        self.warm.close()


def run_reference(args, n_gpus):
    """The reference arm: the reference's CPU GEMM, nothing of this repo's
    library on the path (only oracle/)."""
    ref = CpuReference(args.workload, waves=args.cpu_waves)
    for i in range(args.warmup):
        # the first warm-up is the timed handle's own first call (its pages,
        # its threads); the rest run the one-wave sample
        if i == 0:
            ref.step()
        else:
            ref.warmup()
    vals, secs = [], []
    for _ in range(args.steps):
        g, s = ref.step()
        vals.append(g)
        secs.append(s)
    ref.close()
    v = statistics.median(vals)
    spread = [round(min(secs), 3), round(max(secs), 3)]
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 4),
        "unit": "Gflop/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(secs), 2),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE.json seeded distributions, SplitMix64)",
        "config": config_for(args.workload, n_gpus),
        "cpu_baseline": ref.describe(v),
        "e2e": {"value": round(v, 4), "unit": "Gflop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line["cpu_baseline"]["warmup_sample"] = (f"the timed sample once, then {ref.warm_rows} rows (one wave) per "
                                             "further warm-up step")
    line["cpu_baseline"]["step_seconds_min_max"] = spread
    # the other configs, each on a one-wave sample (one untimed call, then
    # the median of two), next to the product arm's `workloads`
    extras = {}
    for w in extra_workloads(args):
        r = CpuReference(w, waves=1)
        r.step()
        runs = [r.step() for _ in range(2)]
        g = statistics.median(x for x, _ in runs)
        extras[w] = {"value": round(g, 4), "ms_per_step": round(1e3 * statistics.median(t for _, t in runs), 2),
                     "config": config_for(w, n_gpus), "cpu_baseline": r.describe(g)}
        r.close()
    if extras:
        line["workloads"] = extras
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


# ---------------------------------------------------------------------------
# the product arm
# ---------------------------------------------------------------------------

class Ctx:
    """Per-process state shared by the workloads of one run."""

    def __init__(self, args, ws, rank, local):
        import torch
        import torch.distributed as dist

        import paper_2101_06584_b200 as P
        self.args, self.ws, self.rank, self.local = args, ws, rank, local
        self.torch, self.dist, self.P = torch, dist, P
        self.emulate = bool(args.emulate_on_one_gpu)
        dev_index = 0 if self.emulate else local
        torch.cuda.set_device(dev_index)
        P.set_device(dev_index)  # libmpfk has its own CUDA runtime: mirror the choice
        self.dev = torch.device("cuda", dev_index)
        self.use_dist = ws > 1 or args.dist
        if self.use_dist and not dist.is_initialized():
            if self.emulate:  # NCCL refuses two ranks on one device
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
        # collectives of the bench's own bookkeeping (timings, flags): host
        # tensors under gloo
        self.coll_dev = torch.device("cpu") if self.emulate else self.dev
        self.transport = args.transport or ("staged" if ws > 1 else ("nccl" if self.use_dist else None))
        if self.transport == "pull" and ws > 8:
            raise SystemExit("bench: the pull transport maps at most 8 peer slices; use --transport staged")
        if self.emulate and self.transport not in ("staged", "pull", "copy"):
            raise SystemExit("bench: --emulate-on-one-gpu runs the peer-slice transports only")
        if not self.use_dist:
            self.transport = None
        self.stream = torch.cuda.current_stream(self.dev)
        self.peak_ops = None
        self.comm = None
        if self.use_dist:
            self.comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size()}
            if rank == 0:
                print(f"bench: {'NCCL' if self.comm['backend'] == 'nccl' else 'process-group'} communicator "
                      f"nranks={self.comm['nranks']} backend={self.comm['backend']} transport={self.transport}",
                      file=sys.stderr, flush=True)

    def barrier(self):
        if self.use_dist:
            self.dist.barrier()

    def max_over_ranks(self, vals):
        if not self.use_dist:
            return list(vals)
        t = self.torch.tensor(list(vals), dtype=self.torch.float64, device=self.coll_dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def min_int(self, v):
        if not self.use_dist:
            return v
        t = self.torch.tensor([v], dtype=self.torch.int32, device=self.coll_dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return int(t.item())

    def gather_float(self, v):
        if not self.use_dist:
            return [v]
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.coll_dev)
        out = [self.torch.zeros_like(t) for _ in range(self.ws)]
        self.dist.all_gather(out, t)
        return [x.item() for x in out]


def measure_workload(ctx, workload, steps, warmup, with_cpu):
    """Device-resident timing, the sharded check, e2e (pinned and pageable)
    and the roofline of one workload.  Returns rank 0's record (None on the
    other ranks)."""
    import numpy as np
    torch, dist, P, args = ctx.torch, ctx.dist, ctx.P, ctx.args
    from paper_2101_06584_b200.dist import shard_rows, sharded_gemm_step, sharded_gemm_step_overlapped

    W, n, wide = WORKLOADS[workload]
    m = k = n
    ws, rank, dev, stream = ctx.ws, ctx.rank, ctx.dev, ctx.stream
    r0, r1 = shard_rows(m, ws, rank)
    rows = r1 - r0
    ld = P.pad_columns(n)

    # ---- inputs resident in HBM: A row shard; B on rank 0 or as 1/N slices
    A = P.fill_baseline(W, rows, k, SEED_A, wide=wide, row0=r0)
    dA = torch.from_numpy(A.data).to(dev)
    del A
    dB = torch.empty((W, k, ld), dtype=torch.float64, device=dev)
    dC = torch.zeros((W, max(rows, 1), ld), dtype=torch.float64, device=dev)
    flush = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device=dev) if flush_needed(W, n) else None

    transport = ctx.transport
    slices = None
    note = None
    if transport in ("staged", "pull", "copy"):
        from paper_2101_06584_b200.dist import PeerBSlices
        ok = 1
        try:
            slices = PeerBSlices(W, k, ld)
            c0, c1 = slices.cuts[slices.rank], slices.cuts[slices.rank + 1]
            slices.upload(P.fill_baseline(W, c1 - c0, n, SEED_B, wide=wide, row0=c0).data)
        except Exception as e:  # e.g. CUDA IPC not permitted in this container
            ok = 0
            note = f"peer slices unavailable ({type(e).__name__}: {str(e)[:120]})"
            print(f"bench: {note}; using the NCCL K-panel broadcast", file=sys.stderr)
        if not ctx.min_int(ok):
            if slices is not None:
                slices.close()
            slices = None
            transport = "nccl"
        dist.barrier()
    if slices is None and rank == 0:
        Bh = P.fill_baseline(W, k, n, SEED_B, wide=wide)
        dB.copy_(torch.from_numpy(Bh.data))
        del Bh
    peer_bytes = 0
    if slices is not None:
        own = slices.cuts[rank + 1] - slices.cuts[rank]
        peer_bytes = 8 * W * (k - own) * ld
    elif transport in ("nccl", "bcast") and rank != 0:
        peer_bytes = 8 * W * k * ld

    launches = [0]

    def step():
        ev_mid = torch.cuda.Event(enable_timing=True)
        if slices is not None:
            ev_mid.record(stream)
            launches[0] += slices.step(W, dA, dB, dC, rows, n, k, args.pull_panel, args.pull_chunk, stream,
                                       mode=transport)
            return ev_mid
        if transport == "nccl":
            ev_mid.record(stream)
            launches[0] += sharded_gemm_step_overlapped(W, dA, dB, dC, rows, n, k, ld, panels=args.panels,
                                                        stream=stream)
            return ev_mid

        def gemm(W_, dA_, dB_, dC_, rows_, n_, k_, ld_):
            ev_mid.record(stream)  # after the B broadcast (if any)
            return P.gemm_device(W_, rows_, n_, k_, dA_.data_ptr(), ld_, rows_ * ld_, dB_.data_ptr(), ld_,
                                 k_ * ld_, dC_.data_ptr(), ld_, rows_ * ld_, stream.cuda_stream)

        if transport == "bcast":
            launches[0] += sharded_gemm_step(W, dA, dB, dC, rows, n, k, ld, gemm=gemm)
        elif rows:
            launches[0] += gemm(W, dA, dB, dC, rows, n, k, ld)
        if not rows:
            ev_mid.record(stream)
        return ev_mid

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    if ctx.peak_ops is None:
        ctx.peak_ops, _ = P.fp64_peak()  # FP64 pipe peak on this GPU (the roofline denominator)

    clocks = ClockSampler(ctx.dev.index)
    ctx.barrier()
    torch.cuda.synchronize(dev)
    P.gemm_redo_count(reset=True)  # TD/QD fast-pass redo counter (synchronises; outside the timed region)
    clocks.start()
    time.sleep(0.3)
    launches[0] = 0
    evs = []
    for _ in range(steps):
        if flush is not None:
            flush.zero_()  # L2 flush between timed iterations, outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mid = step()
        e1.record(stream)
        evs.append((e0, mid, e1))
    torch.cuda.synchronize(dev)
    ctx.barrier()
    clk = clocks.stop()
    redo = P.gemm_redo_count(reset=True)
    n_launch = launches[0]

    check_default = ctx.use_dist
    check = None
    if args.check if args.check is not None else check_default:
        # the sharded step's C vs a one-shot GEMM of the shard on the now
        # complete B (every transport leaves all of B in dB)
        ok = True
        if rows:
            ref = torch.zeros_like(dC)
            P.gemm_device(W, rows, n, k, dA.data_ptr(), ld, rows * ld, dB.data_ptr(), ld, k * ld, ref.data_ptr(),
                          ld, rows * ld, stream.cuda_stream)
            torch.cuda.synchronize(dev)
            ok = bool(torch.equal(ref.view(torch.int64), dC.view(torch.int64)))
            del ref
        check = min(ctx.gather_float(1.0 if ok else 0.0)) == 1.0

    lean = None
    if not args.no_lean and ((ws == 1 and rows and slices is None and transport not in ("nccl", "bcast")) or
                             (slices is not None and transport == "staged" and (args.lean_dist or ctx.emulate))):
        try:
            lean = measure_lean(ctx, W, dA, dB, dC, rows, n, k, ld, steps, flush, stream, slices=slices)
        except Exception as e:  # an optional leg must not cost the bit-exact line
            if ctx.use_dist:
                raise  # (ranks would desynchronise)
            lean = None
            print(f"bench: MPFK_LEAN leg failed ({type(e).__name__}: {str(e)[:160]})", file=sys.stderr)

    step_ms = [a.elapsed_time(c) for a, _, c in evs]
    kern_ms = [b.elapsed_time(c) for _, b, c in evs]
    t_step_local = sum(step_ms) / len(step_ms)
    t_kern_local = sum(kern_ms) / len(kern_ms)
    per_rank_kern = ctx.gather_float(t_kern_local)
    t_step, t_kern = ctx.max_over_ranks([t_step_local, t_kern_local])
    flops = 2.0 * m * n * k
    value = flops / (t_step * 1e-3) / 1e9
    dC_host = dC[:, :rows, :].cpu() if rows and not args.no_e2e else None
    del dA, dB, dC, flush
    if slices is not None:
        ctx.barrier()
        slices.close()
    torch.cuda.empty_cache()

    # ---- e2e through the public host-buffer API (C ABI)
    e2e = e2e_pg = None
    if not args.no_e2e and not ctx.emulate:
        e2e = measure_e2e(ctx, W, n, wide, r0, rows, flops, steps, pinned=True, dC_host=dC_host)
        if not ctx.use_dist and not args.no_pageable:
            e2e_pg = measure_e2e(ctx, W, n, wide, r0, rows, flops, steps, pinned=False, dC_host=dC_host)
            e2e_pg["registered"] = measure_e2e(ctx, W, n, wide, r0, rows, flops, steps, pinned=False,
                                               dC_host=dC_host, register=True)
        if lean is not None and not ctx.use_dist:
            try:
                lean["e2e"] = measure_e2e(ctx, W, n, wide, r0, rows, flops, steps, pinned=True, dC_host=None,
                                          lean=True)
            except Exception as e:
                print(f"bench: MPFK_LEAN e2e leg failed ({type(e).__name__}: {str(e)[:160]})", file=sys.stderr)

    # ---- CPU baseline: the reference's own GEMM on this host (rank 0, N == 1)
    cpu = None
    if with_cpu and rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            ref = CpuReference(workload, waves=args.cpu_waves)
            ref.warmup()
            ref.step()  # the timed handle's own first call, untimed
            runs = [ref.step() for _ in range(max(1, args.cpu_steps))]
            cpu = ref.describe(statistics.median(g for g, _ in runs))
            cpu["step_seconds"] = [round(t, 3) for _, t in runs]
            ref.close()
        except Exception as e:  # the checker is optional; the GPU number stands alone
            cpu = {"value": None, "error": str(e)[:200]}

    if rank != 0:
        return None
    ops = OPS_PER_MAC[W]
    # dominant kernel (the GEMM) of the slowest rank's shard: algorithmic FP64
    # ops / launch time (shards differ by at most one 64-row block)
    achieved = rows * n * k * ops / (t_kern * 1e-3) / 1e9  # Gop/s
    peak = ctx.peak_ops / 1e9
    traffic = load_traffic(workload) if ws == 1 else None  # captured on the 1-GPU launch
    rec = {
        "value": round(value, 3),
        "ms_per_step": round(t_step, 3),
        "steps": steps,
        "warmup": warmup,
        "config": config_for(workload, ws),
        "rows_per_rank": rows,
        "transport": describe_transport(transport, ws, args, note),
        "roofline": {"bound": "fp64", "achieved": round(achieved, 1), "peak": round(peak, 1),
                     "unit": "Gop/s (FP64 lane ops)",
                     "frac": round(achieved / peak, 4),
                     "frac_of_nominal": round(achieved / (NOMINAL_FP64_LANE_OPS / 1e9), 4),
                     "ops_per_mac": ops, "kernel_ms": round(t_kern, 3),
                     "ops_per_mac_executed": EXEC_OPS_PER_MAC[W],
                     # executed FP64 instructions / launch time: the FP64 pipe's
                     # busy fraction (TD: frac counts 13 algorithmic ops per MAC
                     # the kernel folds away, so quote frac_executed)
                     "frac_executed": round(achieved * EXEC_OPS_PER_MAC[W] / ops / peak, 4),
                     # TD/QD: warp k-tiles per step that left the branch-free fast
                     # pass and were recomputed exactly (DESIGN 4.2)
                     "redo_warp_ktiles_per_step": round(redo / max(steps, 1), 1),
                     "peak_source": "measured on this GPU by mpfk_fp64_peak (DFMA chains); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "traffic": traffic,
                     # the bound is the FP64 pipe: DRAM traffic (L2 re-reads of B across
                     # tile bands) vs the compulsory bytes, and the HBM rate it implies
                     "compulsory_bytes": 8 * W * (rows * k + k * n + rows * n),
                     "traffic_gbs": round(traffic / (t_kern * 1e-3) / 1e9, 1) if traffic else None},
        "e2e": e2e,
        "gpu_launches": n_launch,
        "clocks": clk,
    }
    if lean is not None:
        lean["frac_executed"] = round(rows * n * k * lean["ops_per_mac_executed"] /
                                      (lean["ms_per_step"] * 1e-3) / 1e9 / peak, 4)
        lean["speedup_vs_bit_exact"] = round((t_step if ctx.use_dist else t_kern) / lean["ms_per_step"], 3)
        rec["lean"] = lean
    if e2e_pg is not None:
        rec["e2e_pageable"] = e2e_pg
    if cpu is not None:
        rec["cpu_baseline"] = cpu
    if ctx.use_dist:
        rec["per_rank_kernel_ms"] = [round(x, 3) for x in per_rank_kern]
        rec["peer_bytes_per_step"] = peer_bytes
        rec["check_sharded_equals_one_shot"] = check
    elif check is not None:
        rec["check_sharded_equals_one_shot"] = check
    return rec


def describe_transport(transport, ws, args, note):
    if transport is None:
        return "single GPU, operands resident"
    s = {
        "staged": "copy engines gather B over NVLink from the ranks' 1/N slices in growing K panels; one GEMM "
                  "launch per panel waits on its panel's event (mpfk_gemm_device_staged)",
        "pull": "fused all-gather->GEMM: the GEMM's CTAs pull B over peer memory (mpfk_gemm_device_pull)",
        "copy": "copy engines gather B's K panels; one GEMM launch waits per panel on stream-memory flags "
                "(mpfk_gemm_device_gathered)",
        "nccl": f"NCCL broadcast of B in {args.panels} K panels overlapped with per-panel GEMMs",
        "bcast": "NCCL broadcast of B, then the GEMM",
    }[transport]
    return s + (f" [{note}]" if note else "")


LEAN_OPS_PER_MAC = {2: 10 + 6 / 16, 3: 42 + 18 / 16, 4: 107 + 30 / 16}  # csrc/mpf_lean.cuh (+ renorm per 16-step k-tile)
U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}  # north star


def measure_lean(ctx, W, dA, dB, dC, rows, n, k, ld, steps, flush, stream, slices=None):
    """The same device-resident GEMM with flags = MPFK_LEAN (the north star's
    tolerance mode: 10 / 42 / 107 FP64 instructions per multiply-add instead
    of the bit-exact kernels' 20 / 110 / 212; NOT bit-identical to the reference).  Timed like the
    bit-exact steps (N > 1: the staged all-gather -> GEMM of every rank's
    shard, max over ranks); its result is compared with theirs (dC,
    bit-identical to the reference) as a normwise difference in units of
    4*k*u_p."""
    torch, P, args = ctx.torch, ctx.P, ctx.args
    dL = torch.zeros_like(dC)

    def step():
        if slices is not None:
            return slices.step(W, dA, dB, dL, rows, n, k, args.pull_panel, args.pull_chunk, stream, mode="staged",
                               flags=P.LEAN)
        return P.gemm_device_ex(W, rows, n, k, dA.data_ptr(), ld, rows * ld, dB.data_ptr(), ld, k * ld,
                                dL.data_ptr(), ld, rows * ld, P.LEAN, stream.cuda_stream)
    for _ in range(2):
        step()
    torch.cuda.synchronize(ctx.dev)
    ctx.barrier()
    n_steps = max(2, min(steps, 5))
    evs = []
    for _ in range(n_steps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize(ctx.dev)
    ctx.barrier()
    t_local = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    # sum the component differences from the smallest up: the leading
    # components cancel exactly where the two results agree
    num = den = 0.0
    if rows:
        d = dL[W - 1] - dC[W - 1]
        for w in range(W - 2, -1, -1):
            d = d + (dL[w] - dC[w])
        num, den = float(d[:rows, :n].abs().max()), float(dC[0][:rows, :n].abs().max())
        del d
    del dL
    t, num, den = ctx.max_over_ranks([t_local, num, den])
    diff = num / den if den else 0.0
    m_total = n  # square workloads: all ranks' rows
    return {"flags": "MPFK_LEAN (tolerance mode; not bit-identical to the reference)",
            "value": round(2.0 * m_total * n * k / (t * 1e-3) / 1e9, 3), "unit": "Gflop/s",
            "ms_per_step": round(t, 3), "steps": n_steps,
            "ops_per_mac_executed": LEAN_OPS_PER_MAC[W],
            "normwise_diff_vs_bit_exact": diff,
            "tolerance_4ku_p": 4 * k * U_P[W],
            "diff_over_tolerance": round(diff / (4 * k * U_P[W]), 6)}


def measure_e2e(ctx, W, n, wide, r0, rows, flops, steps, pinned, dC_host, register=False, lean=False):
    """The metric through the public host-buffer API: every step copies the
    step's operands from host memory, computes and reads C back.
    register: pageable operands with the library's opt-in registration
    cache on (mpfk_host_register_cache): the first (warm-up) call page-locks
    them, the timed calls reuse them."""
    import numpy as np
    torch, dist, P, args = ctx.torch, ctx.dist, ctx.P, ctx.args
    m = k = n
    Ah = P.fill_baseline(W, rows, k, SEED_A, wide=wide, row0=r0, pinned=pinned)
    Bh = P.fill_baseline(W, k, n, SEED_B, wide=wide, pinned=pinned)
    Ch = P.MPMatrix(W, rows, n, pinned=pinned)
    if register:
        P.host_register_cache(8 * W * (rows * k + k * n + rows * n) + (64 << 20))
    if ctx.use_dist:
        # one rank per GPU: each rank copies its A shard and 1/ws of B from
        # the host; B's panels are all-gathered over NVLink
        from paper_2101_06584_b200.dist import matmul_sharded_into

        def call():
            matmul_sharded_into(Ch, Ah, Bh, panels=args.panels, device=ctx.dev)
    elif lean:
        def call():
            P.gemm_into(Ch, Ah, Bh, 1, P.LEAN)
    else:
        def call():
            P.matmul_block_parallel_into(Ch, Ah, Bh, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
    call()  # warm
    n_steps = max(1, min(steps, 3))
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        call()
        _ = float(Ch.data[0, 0, 0]) if rows else 0.0  # result read on the host
    ctx.barrier()
    t = (time.perf_counter() - t0) / n_steps
    st = None if ctx.use_dist else P.last_stats()
    (t,) = ctx.max_over_ranks([t])
    h2d = 8 * W * (m * k + k * n)  # (ws > 1: each rank copies 1/ws of B)
    d2h = 8 * W * m * n
    out = {"value": round(flops / t / 1e9, 3), "unit": "Gflop/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": n_steps,
           "host_memory": "page-locked" if pinned else "pageable (like a reference MPMatrix)",
           "api": "dist.matmul_sharded_into (per rank)" if ctx.use_dist else
                  "mpfk_gemm(flags = MPFK_LEAN) (C ABI, host buffers)" if lean else
                  "matmul_block_parallel_into (C ABI, host buffers)"}
    if st is not None:
        out["ms_breakdown"] = {k_: round(st[k_], 3) for k_ in ("h2d_ms", "kernel_ms", "d2h_ms", "total_ms")}
    if register:
        out["host_memory"] = "pageable, page-locked on first use by the registration cache (opt-in)"
        out["registered_entries"] = P.host_register_cache_stats()["entries"]
    if rows and dC_host is not None and not lean:
        # the e2e result equals the device-resident run (same inputs)
        out["matches_device_run"] = bool(
            (torch.from_numpy(np.ascontiguousarray(Ch.data)).view(torch.int64) == dC_host.view(torch.int64)).all())
    if register:  # drop the registrations before the buffers are freed
        P.host_register_cache(0)
    del Ah, Bh, Ch
    return out


def run_mpfk(args, ws, rank, local):
    ctx = Ctx(args, ws, rank, local)
    head = measure_workload(ctx, args.workload, args.steps, args.warmup, with_cpu=True)
    extras = {}
    xsteps = args.extra_steps or min(args.steps, 5)
    for w in extra_workloads(args):
        r = measure_workload(ctx, w, xsteps, args.warmup, with_cpu=False)
        if rank == 0:
            extras[w] = r
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": head["value"],
            "unit": "Gflop/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE.json seeded distributions, SplitMix64), generated on the host",
            "config": head["config"],
            "rows_per_rank": head["rows_per_rank"],
            "transport": head["transport"],
            "roofline": head["roofline"],
            "cpu_baseline": head.get("cpu_baseline"),
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
        }
        for key in ("lean", "e2e_pageable", "per_rank_kernel_ms", "peer_bytes_per_step",
                    "check_sharded_equals_one_shot"):
            if key in head:
                line[key] = head[key]
        if ctx.comm is not None:
            line["comm"] = ctx.comm
        if ctx.emulate:
            line["emulated_on_one_gpu"] = True  # a test of the N > 1 path, not a measurement
        if extras:
            line["workloads"] = extras
        emit(line, args)
    if ctx.use_dist:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        ws, rank, _ = dist_env()
        n = args.gpus or ws
        if rank == 0:  # the CPU reference runs once, on rank 0; other ranks exit 0
            run_reference(args, n)
        return 0
    from paper_2101_06584_b200 import launch
    if args.gpus is not None and args.gpus > 1 and not launch.under_launcher():
        try:
            launch.require_devices(1 if args.emulate_on_one_gpu else args.gpus)
        except RuntimeError as e:
            print(f"bench: {e}", file=sys.stderr)
            return 2
        return launch.spawn_local_ranks(args.gpus, os.path.abspath(__file__), sys.argv[1:] if argv is None else argv)
    ws, rank, local = dist_env()
    if args.gpus is not None and args.gpus != ws:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    if ws > 1:
        try:
            launch.require_devices(1 if args.emulate_on_one_gpu else ws)
        except RuntimeError as e:
            print(f"bench: {e}", file=sys.stderr)
            return 2
    run_mpfk(args, ws, rank, local)
    return 0


if __name__ == "__main__":
    sys.exit(main())
