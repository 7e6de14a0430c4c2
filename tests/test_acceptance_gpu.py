"""The acceptance gate (tests/acceptance.py, the GPU twin of the reference's
proj/tests/acceptance.cpp) must report 0 asserted failures."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_acceptance_gate(gpu_lib):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "acceptance.py")], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert "acceptance: 0 asserted failure(s)" in r.stdout
