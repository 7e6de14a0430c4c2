"""the mpfbench-compatible CSV driver
(tools/mpfbench.cpp, src/bench.cpp).  Argument validation and the seed
derivation run on the CPU; the timed runs are @gpu."""
import csv
import io

import pytest

from paper_2101_06584_b200 import mpfbench as MB

HEADER = "case,precision,op,variant,n,workers,seconds,mflops,max_rel_err,digits_lost,fastest"


def test_sub_seed_matches_bench_cpp():
    """bench.cpp:42-47 restated with the oracle's SplitMix64."""
    import ctypes as C

    import oracle as O
    for seed, purpose, width, n in [(1, 3, 2, 64), (7, 4, 4, 1024), (2 ** 63 + 5, 1, 3, 262144)]:
        st = C.c_uint64((seed ^ (purpose * 0x9E3779B97F4A7C15)) % 2 ** 64)
        st.value = (st.value + width * 0x100000001B3 + n) % 2 ** 64
        want = O.orc().orc_sm64_next(C.addressof(st))
        assert MB.sub_seed(seed, purpose, width, n) == want


@pytest.mark.parametrize("argv,msg", [
    (["matmul", "--precision", "xd"], "bench: precision width must be 2, 3, or 4"),
    (["matmul", "--reps", "0"], "bench: reps must be at least 1"),
    (["matmul", "--workers", "0"], "bench: workers must be at least 1"),
    (["matmul", "--nmin", "0"], "bench: n_min must be at least 1"),
    (["matmul", "--cutoff", "0"], "bench: cutoff must be at least 1"),
    (["matmul", "--sizes", "0"], "bench: sizes must be at least 1"),
    (["ewise", "--variant", "avx"], "bench: unknown variant avx"),
])
def test_validation_messages(argv, msg, capsys):
    assert MB.main(argv) == 1
    assert capsys.readouterr().err.strip() == f"mpfbench: {msg}"


def test_csv_format():
    recs = [dict(case="matmul/dd/block/gpu/n4/w1", precision="dd", op="block", variant="gpu", n=4, workers=1,
                 seconds=0.5, mflops=0.25, max_rel_err=None, digits_lost=None, fastest=True)]
    body = MB.to_csv(recs)
    assert body.splitlines()[0] == HEADER
    assert body.splitlines()[1] == "matmul/dd/block/gpu/n4/w1,dd,block,gpu,4,1,0.5,0.25,,,1"


@pytest.mark.gpu
def test_matmul_and_ewise_runs(gpu_lib, tmp_path):
    out = tmp_path / "mm.csv"
    assert MB.main(["matmul", "--sizes", "16,33", "--reps", "1", "--oracle-max", "16", "--cutoff", "8",
                    "--nmin", "8", "--workers", "1,2", "--out", str(out)]) == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    # 3 widths x 2 sizes x (naive w1 + block w1,w2 + strassen w1,w2)
    assert len(rows) == 3 * 2 * 5
    for (prec, n) in {(r["precision"], r["n"]) for r in rows}:
        grp = [r for r in rows if (r["precision"], r["n"]) == (prec, n)]
        assert sum(r["fastest"] == "1" for r in grp) == 1
    eps = {"dd": 2.0 ** -104, "td": 2.0 ** -157, "qd": 2.0 ** -209}
    for r in rows:
        if r["n"] == "16" and r["op"] != "strassen":
            assert float(r["max_rel_err"]) <= 16 * 4 * eps[r["precision"]]
            assert float(r["digits_lost"]) < 2.5
    # the tolerance-mode variant: block rows only, its own error columns
    out3 = tmp_path / "lean.csv"
    assert MB.main(["matmul", "--sizes", "16,40", "--reps", "1", "--oracle-max", "40", "--algo", "block",
                    "--variant", "gpu,gpu-lean", "--workers", "1,2", "--out", str(out3)]) == 0
    rows3 = list(csv.DictReader(io.StringIO(out3.read_text())))
    assert len(rows3) == 3 * 2 * 2 * 2
    for r in rows3:
        n3 = int(r["n"])
        assert float(r["max_rel_err"]) <= n3 * 4 * eps[r["precision"]] * 8
    assert {r["variant"] for r in rows3} == {"gpu", "gpu-lean"}
    out2 = tmp_path / "ew.csv"
    assert MB.main(["ewise", "--sizes", "64,4096", "--reps", "1", "--out", str(out2)]) == 0
    rows = list(csv.DictReader(io.StringIO(out2.read_text())))
    assert {r["op"] for r in rows if r["precision"] == "td"} == {"add_q", "add_merge", "mul"}
    assert len(rows) == (2 + 3 + 2) * 2
