"""One process per GPU on one node, without torchrun.

`bench.py --gpus N` (and any script) uses spawn_local_ranks() when it is not
already running under torchrun: it starts N copies of the script with
RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT set -- the same
environment torch.distributed.run would give them -- waits for all of them,
and stops the rest as soon as one fails.  Each rank then initialises its own
process group (NCCL over NVLink on the GPU box, gloo in the CPU tests).

This replaces the reference's in-process worker fan-out (run_on_threads,
linalg.hpp:314-334) at the node level: the workers own disjoint contiguous
row spans (linalg.hpp:413-421) and never exchange partial results.
"""
from __future__ import annotations

import os
import signal
import socket
import subprocess
import sys
import time
from typing import Dict, List, Optional, Sequence


def free_port(host: str = "127.0.0.1") -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind((host, 0))
        return s.getsockname()[1]


def under_launcher() -> bool:
    """True when this process is one rank of a launched group."""
    return "WORLD_SIZE" in os.environ and "RANK" in os.environ


def visible_sm100_devices() -> int:
    """Number of visible CUDA devices of compute capability 10.x (B200)."""
    import torch
    if not torch.cuda.is_available():
        return 0
    return sum(1 for i in range(torch.cuda.device_count())
               if torch.cuda.get_device_capability(i)[0] == 10)


def require_devices(n: int) -> None:
    """Raise unless n sm_100 devices are visible: a --gpus N run must never
    quietly run on fewer GPUs."""
    have = visible_sm100_devices()
    if have < n:
        raise RuntimeError(f"--gpus {n} needs {n} visible sm_100 (B200) devices, found {have}")


def spawn_local_ranks(n: int, script: str, argv: Sequence[str], *, env: Optional[Dict[str, str]] = None,
                      timeout: Optional[float] = None, quiet_ranks: bool = False) -> int:
    """Run `python script argv...` as ranks 0..n-1 of one group on this node.

    Rank 0 inherits stdout (it prints the result line); with quiet_ranks the
    other ranks' stdout is discarded.  stderr of every rank is inherited.
    Returns 0 when every rank exits 0, else the first nonzero exit code
    (the remaining ranks are terminated)."""
    if n < 1:
        raise ValueError("spawn_local_ranks: n must be at least 1")
    base = dict(os.environ)
    if env:
        base.update(env)
    base["MASTER_ADDR"] = "127.0.0.1"
    base["MASTER_PORT"] = str(free_port())
    base["WORLD_SIZE"] = str(n)
    base["LOCAL_WORLD_SIZE"] = str(n)
    procs: List[subprocess.Popen] = []
    for r in range(n):
        e = dict(base, RANK=str(r), LOCAL_RANK=str(r), GROUP_RANK="0")
        out = subprocess.DEVNULL if (quiet_ranks and r) else None
        procs.append(subprocess.Popen([sys.executable, script, *argv], env=e, stdout=out,
                                      start_new_session=True))
    deadline = None if timeout is None else time.monotonic() + timeout
    rc = 0
    try:
        live = set(range(n))
        while live:
            for r in sorted(live):
                c = procs[r].poll()
                if c is None:
                    continue
                live.discard(r)
                if c != 0 and rc == 0:
                    rc = c
                    print(f"launch: rank {r} exited with {c}; stopping the other ranks", file=sys.stderr)
            if rc:
                break
            if deadline is not None and time.monotonic() > deadline:
                print(f"launch: timeout after {timeout} s; stopping the ranks", file=sys.stderr)
                rc = 124
                break
            time.sleep(0.05)
    finally:
        for p in procs:
            if p.poll() is None:
                try:
                    os.killpg(p.pid, signal.SIGTERM)
                except ProcessLookupError:
                    pass
        for p in procs:
            try:
                p.wait(timeout=10)
            except subprocess.TimeoutExpired:
                os.killpg(p.pid, signal.SIGKILL)
                p.wait()
    return rc
