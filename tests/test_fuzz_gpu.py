"""A short run of the randomised parity sweep (scripts/fuzz_parity.py) in a
subprocess with three emulated devices: random widths and shapes through the
host API (pageable / page-locked, 1-3 devices), the device API on windows,
K-panel continuation, both fused all-gather variants, Strassen, elementwise,
MPFK_FAST and dist.matmul_sharded_into -- all bit-compared with the
reference build.  Longer sweeps: profiles/r01_fuzz.log."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [101, 202])
def test_randomised_parity_sweep(gpu_lib, seed):
    env = dict(os.environ, MPFK_EMULATED_DEVICES="3")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_parity.py"), "72", str(seed)],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "72 cases, 0 with mismatches" in r.stdout
