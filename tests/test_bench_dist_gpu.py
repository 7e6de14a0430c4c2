"""bench.py's collective path on the GPU box (one GPU): torchrun with one
rank and a forced NCCL process group runs the K-panel overlapped broadcast +
continuation GEMMs exactly as N > 1 ranks would, and the sharded result must
equal a one-shot GEMM bit for bit."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["dd1024", "qd1024"])
def test_torchrun_collective_path(gpu_lib, workload):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--workload", workload,
           "--steps", "2", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--dist", "--check", "--panels", "3",
           "--extra", "none"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["check_sharded_equals_one_shot"] is True
    assert line["gpu_launches"] == 2 * 3  # 3 K panels per step
    assert "K panels overlapped" in line["transport"]
    assert line["comm"] == {"backend": "nccl", "nranks": 1}
    assert len(line["per_rank_kernel_ms"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode,launches", [("copy", 1), ("pull", 1), ("staged", 3)])
def test_torchrun_fused_allgather_path(gpu_lib, mode, launches):
    """B gathered from the rank's slice while the GEMM computes: copy
    engines + in-kernel flags (copy), in-kernel pulls (pull), or copy
    engines + one launch per growing K panel (staged: k=1024 -> panels
    [0,64), [64,320), [320,1024)); the result equals the one-shot GEMM."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--workload", "td1024",
           "--steps", "2", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--dist",
           "--transport", mode, "--pull-panel", "64", "--pull-chunk", "8", "--extra", "none", "--lean-dist"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["check_sharded_equals_one_shot"] is True  # the default with a process group
    assert line["gpu_launches"] == 2 * launches
    assert {"copy": "gathered", "pull": "device_pull", "staged": "device_staged"}[mode] in line["transport"]
    if mode == "staged":  # the tolerance-mode leg rides the same transport (mpfk_gemm_device_staged_ex)
        assert line["lean"]["value"] > line["value"]
        assert 0 < line["lean"]["diff_over_tolerance"] <= 0.05
    else:
        assert "lean" not in line


@pytest.mark.gpu
def test_bench_line_carries_every_workload(gpu_lib):
    """The default line's `workloads`: every BASELINE config besides the
    headline, each with value, roofline (frac and frac_executed), pinned and
    pageable e2e (bit-identical to the device run) and clocks."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--workload", "dd1024", "--extra",
           "td1024,qd1024", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["config"]["workload"] == "dd1024"
    assert set(line["workloads"]) == {"td1024", "qd1024"}
    for rec in [line] + list(line["workloads"].values()):
        assert rec["value"] > 0
        assert 0 < rec["roofline"]["frac_executed"] <= 1.02
        assert rec["e2e"]["matches_device_run"] is True
        assert rec["e2e_pageable"]["matches_device_run"] is True
        assert rec["gpu_launches"] >= 2


@pytest.mark.gpu
def test_torchrun_e2e_host_operands(gpu_lib):
    """the e2e leg under torchrun: every rank copies its A shard and 1/ws of
    B from pinned host memory (dist.matmul_sharded_into); its C shard must
    equal the device-resident run bit for bit."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--workload", "td1024",
           "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--dist", "--panels", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    e2e = line["e2e"]
    assert e2e["matches_device_run"] is True
    assert e2e["api"].startswith("dist.matmul_sharded_into")
    assert e2e["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("W,m,k,n,panels", [(2, 100, 300, 70, 3), (3, 64, 1000, 33, 8), (4, 17, 31, 9, 2)])
def test_matmul_sharded_into_single_rank(gpu_lib, W, m, k, n, panels):
    """without a process group: panels copied from the host, continuation
    GEMMs; bit-identical to matmul_block_into, pads +0."""
    import torch

    import oracle as O
    from paper_2101_06584_b200.dist import gather_panels, matmul_sharded_into
    P = gpu_lib
    A = P.MPMatrix.from_planes(O.orc_fill_baseline(W, m, k, 5, wide=True)[:, :, :k], pinned=True)
    B = P.MPMatrix.from_planes(O.orc_fill_baseline(W, k, n, 6, wide=True)[:, :, :n], pinned=True)
    C1 = P.MPMatrix(W, m, n, pinned=True)
    C1.data[...] = 3.0
    launches = matmul_sharded_into(C1, A, B, panels=panels, device=torch.device("cuda", 0))
    C2 = P.MPMatrix(W, m, n)
    P.matmul_block_into(C2, A, B)
    assert P.bits_equal(C1, C2)
    assert launches == len(gather_panels(k, panels, 1)[1])
    with pytest.raises(ValueError, match="inner dimensions differ"):
        matmul_sharded_into(C1, A, P.MPMatrix(W, k + 1, n))


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["staged", "pull"])
def test_bench_gpus2_emulated_on_one_gpu(gpu_lib, transport):
    """`bench.py --gpus 2` end to end on the one-GPU box: the launcher spawns
    two ranks (gloo group, both on GPU 0), each uploads its half of B into a
    CUDA-IPC-exported slice, gathers the other rank's half and computes its
    row shard; the line must report two ranks and every rank's shard must
    equal a one-shot GEMM of it bit for bit.  No cross-rank kernel waits:
    the slices are resident before a barrier, then only read."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--emulate-on-one-gpu",
           "--workload", "dd1024", "--extra", "qd1024", "--steps", "2", "--warmup", "1", "--no-cpu-baseline",
           "--transport", transport]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["emulated_on_one_gpu"] is True
    assert line["comm"] == {"backend": "gloo", "nranks": 2}
    assert line["check_sharded_equals_one_shot"] is True
    assert line["workloads"]["qd1024"]["check_sharded_equals_one_shot"] is True
    assert len(line["per_rank_kernel_ms"]) == 2 and line["rows_per_rank"] == 512
    assert line["peer_bytes_per_step"] == 8 * 2 * 512 * 1024
    assert ("device_staged" if transport == "staged" else "device_pull") in line["transport"]
