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
           "--steps", "2", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--dist", "--check", "--panels", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["check_sharded_equals_one_shot"] is True
    assert line["gpu_launches"] == 2 * 3  # 3 K panels per step
    assert "K panels overlapped" in line["config"]["parallelism"] or line["n_gpus"] == 1


@pytest.mark.gpu
def test_torchrun_fused_allgather_path(gpu_lib):
    """--fused-allgather with one rank: the GEMM pulls B from the rank's slice
    inside the kernel; the result equals the one-shot GEMM."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--workload", "td1024",
           "--steps", "2", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--dist", "--check",
           "--fused-allgather", "--pull-panel", "64", "--pull-chunk", "8"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["check_sharded_equals_one_shot"] is True
    assert line["gpu_launches"] == 2
    assert "fused all-gather" in line["config"]["parallelism"]
