"""The C++ drop-in on the GPU: tests/_build/shim_parity multiplies the
reference's own mpfkit::linalg::MPMatrix<W> with the reference CPU GEMM and
with libmpfk through include/mpfk/linalg.hpp and requires bits_equal, plus
the reference's exception types/messages through the shim."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_build", "shim_parity")


@pytest.mark.gpu
def test_cpp_shim_drop_in(gpu_lib):
    assert os.path.exists(BIN), "shim_parity not built (needs the reference headers at build time)"
    r = subprocess.run([BIN, "97"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
