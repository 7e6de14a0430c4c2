"""The node launcher behind `bench.py --gpus N` (paper_2101_06584_b200.launch)
on the CPU: N ranks spawned with the torchrun environment, gloo for the
group, the oracle as the per-rank compute; and bench.py's refusal to run
N > 1 on fewer visible B200s (this container has none)."""
import json
import os
import subprocess
import sys

import pytest

from paper_2101_06584_b200 import launch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "launch_worker.py")


def _run(n, args, timeout=180):
    r = subprocess.run([sys.executable, "-c",
                        "import sys; from paper_2101_06584_b200 import launch; "
                        f"sys.exit(launch.spawn_local_ranks({n}, {WORKER!r}, {list(map(str, args))!r}, "
                        "quiet_ranks=True))"],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    return r


@pytest.mark.parametrize("n,W,m,k,n_", [(2, 2, 37, 21, 19), (2, 4, 20, 7, 6), (3, 3, 40, 9, 10)])
def test_spawned_gloo_ranks_row_shards_bit_identical(n, W, m, k, n_):
    r = _run(n, [W, m, k, n_])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone reports
    assert lines[0]["nranks"] == n and lines[0]["backend"] == "gloo"
    assert lines[0]["check_sharded_equals_one_shot"] is True


def test_failed_rank_stops_the_group():
    r = _run(2, [2, 16, 8, 8, 1], timeout=120)
    assert r.returncode == 3
    assert "rank 1 exited with 3" in r.stderr


def test_spawn_rejects_bad_count():
    with pytest.raises(ValueError):
        launch.spawn_local_ranks(0, WORKER, [])


def test_bench_gpus_n_fails_loudly_without_enough_gpus():
    """--gpus 2 on a box with fewer than two B200s must not quietly run one."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    if launch.visible_sm100_devices() >= 2:
        pytest.skip("this box has two B200s")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0
    assert "--gpus 2 needs 2 visible sm_100" in r.stderr
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_bench_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2
    assert "--gpus 4 but WORLD_SIZE=2" in r.stderr


def test_bench_config_identical_in_both_arms():
    """The driver compares the two arms' config dicts."""
    sys.path.insert(0, ROOT)
    import bench
    for w in bench.WORKLOADS:
        for ws in (1, 2, 8):
            c = bench.config_for(w, ws)
            assert c == bench.config_for(w, ws) and c["workload"] == w
            assert "rows_per_rank" not in c


def test_bench_reference_arm_loads_no_product_library():
    """--impl reference runs the reference's CPU GEMM through oracle/ only:
    nothing of paper_2101_06584_b200 (or libmpfk.so) is imported or mapped."""
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','1',"
            "'--workload','dd1024','--cpu-waves','1','--extra','td1024']; import bench; bench.main(sys.argv[1:]); "
            "maps=[l.split()[-1] for l in open('/proc/self/maps') if '.so' in l]; "
            "print(json.dumps({'mods':[m for m in sys.modules if m.startswith('paper_2101')], "
            "'libmpfk':[m for m in maps if 'libmpfk.so' in m], 'ref':[m for m in maps if 'libmpfkref' in m]}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    out = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    line, probe = out[0], out[-1]
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"] == __import__("bench").config_for("dd1024", 1)
    assert line["workloads"]["td1024"]["value"] > 0  # the other configs, each with its own sample
    assert line["workloads"]["td1024"]["config"] == __import__("bench").config_for("td1024", 1)
    assert probe["mods"] == [] and probe["libmpfk"] == [] and probe["ref"]
