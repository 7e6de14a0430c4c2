"""mpfbench-compatible benchmark driver with a GPU variant (SURVEY.md 8(f)
row 3).

Same subcommands, flags, defaults, data, timing convention and CSV columns
as the reference's CLI (tools/mpfbench.cpp:62-156, src/bench.cpp), so the
reference's report tooling reads both:

  python -m paper_2101_06584_b200.mpfbench matmul [--precision dd,td,qd|all]
      [--algo naive,block,strassen|all] [--variant gpu|gpu-lean|normal|set|loadstore|all]
      [--sizes 64,128,...] [--nmin 32] [--cutoff 64] [--workers 1,2]
      [--reps 5] [--seed 1] [--oracle-max 64] [--out path]
      [--paper-matrices | --random]
  python -m paper_2101_06584_b200.mpfbench ewise [...common flags...]

CSV: case,precision,op,variant,n,workers,seconds,mflops,max_rel_err,
digits_lost,fastest (bench.cpp:320-336).  `seconds` is the median wall time
of the public host-buffer call (H2D + GPU + D2H, like the reference's
wall-clock of run_matmul, bench.cpp:196-200); `mflops` uses the reference's
classic op count n^3 + n^2(n-1) (bench.cpp:169-170), the measured
adds+muls for Strassen, and n per vector op for ewise.  `workers` counts
GPUs.  Every variant of one algorithm is checked bit-identical before it is
timed (bench.cpp:187-195, :97-101).  "all" variants = "gpu" (the CPU
variant names are accepted and run the same GPU kernel).
"""
from __future__ import annotations

import argparse
import sys
import time

from . import linalg as L
from . import verify

PRECISIONS = {"dd": 2, "td": 3, "qd": 4}
NAMES = {2: "dd", 3: "td", 4: "qd"}
VARIANTS = {"normal": L.KernelVariant.NORMAL, "set": L.KernelVariant.SIMD_SET,
            "loadstore": L.KernelVariant.SIMD_LOADSTORE, "gpu": L.KernelVariant.SIMD_LOADSTORE,
            # the tolerance mode (MPFK_LEAN, DESIGN 9.2): block algorithm only, not
            # bit-identical to the other variants by design -- its rows carry their own
            # max_rel_err / digits_lost against the exact oracle instead
            "gpu-lean": L.KernelVariant.SIMD_LOADSTORE}
ALGOS = ("naive", "block", "strassen")
MASK = (1 << 64) - 1


def _sm64_next(state: int):
    state = (state + 0x9E3779B97F4A7C15) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return state, z ^ (z >> 31)


def sub_seed(seed: int, purpose: int, width: int, n: int) -> int:
    """bench.cpp:42-47: per-case data seed."""
    state = (seed ^ ((purpose * 0x9E3779B97F4A7C15) & MASK)) & MASK
    state = (state + width * 0x100000001B3 + n) & MASK
    return _sm64_next(state)[1]


def _list(s, conv=str):
    return [conv(x) for x in s.split(",") if x != ""]


def parse(argv=None):
    ap = argparse.ArgumentParser(prog="mpfbench", description="multi-component extended-precision benchmark driver")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("ewise", "matmul"):
        p = sub.add_parser(name)
        p.add_argument("--precision", default="all")
        p.add_argument("--variant", default="all")
        p.add_argument("--sizes", default="")
        p.add_argument("--reps", type=int, default=5)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--oracle-max", type=int, default=64)
        p.add_argument("--out", default="")
        if name == "matmul":
            p.add_argument("--algo", default="all")
            p.add_argument("--nmin", type=int, default=32)
            p.add_argument("--cutoff", type=int, default=64)
            p.add_argument("--workers", default="1")
            g = p.add_mutually_exclusive_group()
            g.add_argument("--paper-matrices", action="store_true")
            g.add_argument("--random", action="store_true")
    return ap.parse_args(argv)


def _config(a):
    """BenchConfig + bench::validate (bench.cpp:259-275)."""
    precs = [2, 3, 4] if a.precision == "all" else [PRECISIONS.get(p, -1) for p in _list(a.precision)]
    if not precs:
        raise ValueError("bench: no precisions")
    if any(p not in (2, 3, 4) for p in precs):
        raise ValueError("bench: precision width must be 2, 3, or 4")
    variants = ["gpu"] if a.variant == "all" else _list(a.variant)
    if not variants:
        raise ValueError("bench: no variants")
    for v in variants:
        if v not in VARIANTS:
            raise ValueError(f"bench: unknown variant {v}")
    if a.reps < 1:
        raise ValueError("bench: reps must be at least 1")
    cfg = dict(precisions=precs, variants=variants, reps=a.reps, seed=a.seed, oracle_max=a.oracle_max)
    if a.cmd == "matmul":
        sizes = _list(a.sizes, int) or [64, 128, 256, 512, 1024]
        algos = list(ALGOS) if a.algo == "all" else _list(a.algo)
        if not algos:
            raise ValueError("bench: no algorithms")
        for x in algos:
            if x not in ALGOS:
                raise ValueError(f"bench: unknown algorithm {x}")
        workers = _list(a.workers, int)
        if not workers:
            raise ValueError("bench: no worker counts")
        if any(w < 1 for w in workers):
            raise ValueError("bench: workers must be at least 1")
        if a.nmin < 1:
            raise ValueError("bench: n_min must be at least 1")
        if a.cutoff < 1:
            raise ValueError("bench: cutoff must be at least 1")
        cfg.update(algos=algos, workers=workers, n_min=a.nmin, cutoff=a.cutoff, paper=a.paper_matrices)
    else:
        sizes = _list(a.sizes, int) or [1024, 16384, 262144]
    if not sizes:
        raise ValueError("bench: no sizes")
    if any(n < 1 for n in sizes):
        raise ValueError("bench: sizes must be at least 1")
    cfg["sizes"] = sizes
    return cfg


def _median_seconds(reps, f):
    """bench.cpp:33-38"""
    t = sorted(f() for _ in range(reps))
    return t[len(t) // 2]


def _run_matmul(cfg, algo, v, workers, A, B):
    var = VARIANTS[v]
    if v == "gpu-lean":
        return L.gemm(A, B, n_gpus=workers, flags=L.LEAN)
    if algo == "strassen":
        return L.matmul_strassen_parallel(A, B, cfg["cutoff"], cfg["n_min"], var, workers)
    if algo == "naive":
        return L.matmul_naive(A, B, var)
    return L.matmul_block_parallel(A, B, cfg["n_min"], var, workers)


def matmul_records(cfg):
    """bench.cpp:148-228"""
    recs = []
    for W in cfg["precisions"]:
        prec = NAMES[W]
        for n in cfg["sizes"]:
            if cfg["paper"]:
                A, B = L.gen_paper_matrices(W, n)
            else:
                A = L.fill_random(W, n, n, sub_seed(cfg["seed"], 3, W, n))
                B = L.fill_random(W, n, n, sub_seed(cfg["seed"], 4, W, n))
            exact = verify.exact_matmul(A.data, B.data, n, n) if n <= cfg["oracle_max"] else None
            group = len(recs)
            classic = float(n) * n * n + float(n) * n * (n - 1)
            strassen_ops = None
            for algo in cfg["algos"]:
                ref = None
                for v in cfg["variants"]:
                    if v == "gpu-lean" and algo != "block":
                        continue
                    measure = algo == "strassen" and strassen_ops is None
                    if measure:
                        L.op_counters_reset()
                    serial = _run_matmul(cfg, algo, v, 1, A, B)  # warm-up + bit-identity reference
                    if measure:
                        c = L.op_counters_read()
                        strassen_ops = float(c.adds + c.muls)
                    if v == "gpu-lean":
                        pass  # tolerance mode: judged by its error columns
                    elif ref is None:
                        ref = serial
                    elif not L.bits_equal(serial, ref):
                        raise RuntimeError(f"{algo} variant {v} diverged from {cfg['variants'][0]}")
                    ops = strassen_ops if algo == "strassen" else classic
                    for w in cfg["workers"]:
                        if w > 1 and algo == "naive":
                            continue
                        if w > 1 and not L.bits_equal(_run_matmul(cfg, algo, v, w, A, B), serial):
                            raise RuntimeError(f"parallel {algo} with {w} workers diverged from serial")

                        def once():
                            t0 = time.perf_counter()
                            _run_matmul(cfg, algo, v, w, A, B)
                            return time.perf_counter() - t0

                        sec = _median_seconds(cfg["reps"], once)
                        r = dict(case=f"matmul/{prec}/{algo}/{v}/n{n}/w{w}", precision=prec, op=algo, variant=v, n=n,
                                 workers=w, seconds=sec, mflops=ops / (1e6 * sec), max_rel_err=None,
                                 digits_lost=None, fastest=False)
                        if exact is not None:
                            e = verify.max_rel_err(serial.data, exact, n)
                            r["max_rel_err"] = e
                            r["digits_lost"] = verify.digit_loss(e, L.format_eps(W))
                        recs.append(r)
            if len(recs) > group:  # fastest cell per (precision, n), bench.cpp:219-226
                best = min(range(group, len(recs)), key=lambda i: recs[i]["seconds"])
                recs[best]["fastest"] = True
    return recs


def ewise_records(cfg):
    """bench.cpp:77-127"""
    from fractions import Fraction
    recs = []
    for W in cfg["precisions"]:
        prec = NAMES[W]
        ops = [("add_q", L.EwOp.add), ("add_merge", L.EwOp.add_merge), ("mul", L.EwOp.mul)] if W == 3 else \
            [("add", L.EwOp.add), ("mul", L.EwOp.mul)]
        for n in cfg["sizes"]:
            a = L.fill_random(W, 1, n, sub_seed(cfg["seed"], 1, W, n))
            b = L.fill_random(W, 1, n, sub_seed(cfg["seed"], 2, W, n))
            out = L.MPMatrix(W, 1, n)
            for name, op in ops:
                L.ew_apply_into(out, a, b, op, L.KernelVariant.NORMAL)
                ref = out.copy()
                exact = None
                if n <= cfg["oracle_max"]:
                    exact = []
                    for j in range(n):
                        x = verify._value(a.data[:, 0, j])
                        y = verify._value(b.data[:, 0, j])
                        exact.append(x * y if op == L.EwOp.mul else x + y)
                for v in cfg["variants"]:
                    L.ew_apply_into(out, a, b, op, VARIANTS[v])
                    if not L.bits_equal(out, ref):
                        raise RuntimeError(f"ewise variant {v} diverged from the scalar kernel")
                    batch = max(1, 262144 // max(n, 1))

                    def once():
                        t0 = time.perf_counter()
                        for _ in range(batch):
                            L.ew_apply_into(out, a, b, op, VARIANTS[v])
                        return (time.perf_counter() - t0) / batch

                    sec = _median_seconds(cfg["reps"], once)
                    r = dict(case=f"ewise/{prec}/{name}/{v}/n{n}/w1", precision=prec, op=name, variant=v, n=n,
                             workers=1, seconds=sec, mflops=n / (1e6 * sec), max_rel_err=None, digits_lost=None,
                             fastest=False)
                    if exact is not None:
                        e = max((verify.rel_err(ref.data[:, 0, j], exact[j]) if exact[j] != Fraction(0) else 0.0)
                                for j in range(n))
                        r["max_rel_err"] = e
                        r["digits_lost"] = verify.digit_loss(e, L.format_eps(W))
                    recs.append(r)
    return recs


def to_csv(recs) -> str:
    """bench.cpp:320-336 (round-trip %.17g formatting)."""
    out = ["case,precision,op,variant,n,workers,seconds,mflops,max_rel_err,digits_lost,fastest"]
    for r in recs:
        cells = [r["case"], r["precision"], r["op"], r["variant"], str(r["n"]), str(r["workers"]),
                 f"{r['seconds']:.17g}", f"{r['mflops']:.17g}",
                 "" if r["max_rel_err"] is None else f"{r['max_rel_err']:.17g}",
                 "" if r["digits_lost"] is None else f"{r['digits_lost']:.17g}", "1" if r["fastest"] else "0"]
        out.append(",".join(cells))
    return "\n".join(out) + "\n"


def main(argv=None) -> int:
    a = parse(argv)
    try:
        cfg = _config(a)
        recs = matmul_records(cfg) if a.cmd == "matmul" else ewise_records(cfg)
        body = to_csv(recs)
        if a.out:
            try:
                with open(a.out, "w") as f:
                    f.write(body)
            except OSError:
                raise RuntimeError(f"{a.out}: cannot open for writing")
        else:
            sys.stdout.write(body)
        sys.stderr.write(f"{len(recs)} records written to {a.out or 'stdout'}\n")
        return 0
    except Exception as e:  # noqa: BLE001 -- the CLI's contract: message + exit 1
        sys.stderr.write(f"mpfbench: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
