"""The in-process multi-GPU host path (workers > 1: row shards, each device
uploading a 1/G slice of B and gathering the rest with peer copies, one host
thread per device) on the one-GPU box: MPFK_EMULATED_DEVICES=G presents G
logical devices on physical device 0 (a testing hook of libmpfk; the peer
copies become device-local copies ordered by the same events, and no kernel
waits on another).  The result must be bit-identical to the reference for
every G, exactly as the reference's worker count is (linalg.hpp:399-401)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import oracle as O
import paper_2101_06584_b200 as P
out = {"devices": P.device_count(), "cases": []}
# (3, 194, ...) with 3 devices: 128-row spans leave the third shard empty
for W, m, n, k, workers in [(2, 300, 129, 77, 3), (3, 200, 64, 300, 2), (4, 130, 33, 47, 3), (2, 700, 260, 1030, 3),
                            (3, 5, 9, 11, 3), (3, 194, 463, 367, 3)]:
    A = P.fill_baseline(W, m, k, 1, wide=True)
    B = P.fill_baseline(W, k, n, 2, wide=True)
    C = P.MPMatrix(W, m, n)
    C.data[...] = 3.0
    P.matmul_block_parallel_into(C, A, B, 32, P.KernelVariant.NORMAL, workers)
    st = P.last_stats()
    want = O.ref_gemm(A.data, B.data, k, n)
    same = bool(np.array_equal(C.data.view(np.uint64), want.view(np.uint64)))
    out["cases"].append({"W": W, "m": m, "workers": workers, "same": same, "n_gpus": st["n_gpus"],
                         "peer_bytes": st["peer_bytes"], "launches": st["kernel_launches"]})
A = P.fill_baseline(2, 520, 300, 3, wide=True)
B = P.fill_baseline(2, 300, 70, 4, wide=True)
G = P.gemm(A, B, n_gpus=0)
out["gemm_all_devices"] = P.last_stats()["n_gpus"]
out["gemm_same"] = P.bits_equal(G, P.matmul_block(A, B))
# FAST across devices: shards too small to fill a GPU split K; the result is
# deterministic and its leading components agree with the bit-exact product
# within the north star's tolerance
A = P.fill_baseline(3, 130, 4000, 5, wide=True)
B = P.fill_baseline(3, 4000, 20, 6, wide=True)
F1 = P.gemm(A, B, n_gpus=0, flags=P.FAST)
F2 = P.gemm(A, B, n_gpus=0, flags=P.FAST)
out["fast_deterministic"] = P.bits_equal(F1, F2)
E = P.matmul_block(A, B)
d = np.abs(F1.data[0] - E.data[0]).max()
out["fast_close"] = bool(d <= 4 * 4000 * 2.0 ** -156 * np.abs(E.data[0]).max() + 1e-300)
# LEAN across devices: every element is the same chain whatever the row
# shard, so G devices give the one-device lean result bit for bit
A = P.fill_baseline(4, 390, 500, 7, wide=True)
B = P.fill_baseline(4, 500, 130, 8, wide=True)
L1 = P.gemm(A, B, n_gpus=1, flags=P.LEAN)
LG = P.gemm(A, B, n_gpus=0, flags=P.LEAN)
out["lean_devices"] = P.last_stats()["n_gpus"]
out["lean_same_on_all_devices"] = P.bits_equal(L1, LG)
out["lean_is_not_the_reference_bits"] = not P.bits_equal(L1, P.matmul_block(A, B))
print(json.dumps(out))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("emulated", [2, 3])
def test_multi_device_host_path_emulated(gpu_lib, emulated):
    env = dict(os.environ, MPFK_EMULATED_DEVICES=str(emulated))
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], capture_output=True, text=True, timeout=600, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["devices"] == emulated
    for c in out["cases"]:
        assert c["same"], c
        g = min(c["workers"], emulated, (c["m"] + 63) // 64)
        assert c["n_gpus"] == g, c
        assert (c["peer_bytes"] > 0) == (g > 1), c
    assert any(c["m"] == 194 and c["n_gpus"] == emulated for c in out["cases"]) or emulated < 3
    assert out["gemm_all_devices"] == emulated
    assert out["gemm_same"]
    assert out["fast_deterministic"] and out["fast_close"]
    assert out["lean_devices"] == emulated and out["lean_same_on_all_devices"]
    assert out["lean_is_not_the_reference_bits"]
