"""The device twin of runtime::verify_fp_environment (runtime.cpp:19-38,
72-81): mpfk_selftest passes on a B200, and a failing probe surfaces with
the reference's messages as MPFK_ERUNTIME -> RuntimeError (Python) /
std::runtime_error (C++ shim).  The failure is injected with the library's
MPFK_SELFTEST_INJECT testing hook in a fresh process (the probe runs once
per device context)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_selftest_passes(gpu_lib):
    from paper_2101_06584_b200 import _native as N
    assert N.lib().mpfk_selftest() == N.MPFK_OK


@pytest.mark.parametrize("probe,text", [("rn", "not rounding to nearest-even"),
                                        ("fma", "not a correctly rounded fused multiply-add")])
def test_selftest_failure_maps_to_runtime_error(gpu_lib, probe, text):
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2101_06584_b200 as P\n"
            "from paper_2101_06584_b200 import _native as N\n"
            "rc = N.lib().mpfk_selftest()\n"
            "assert rc == N.MPFK_ERUNTIME, rc\n"
            "try:\n"
            "    P.matmul_block(P.fill_baseline(2, 8, 8, 1), P.fill_baseline(2, 8, 8, 2))\n"
            "except RuntimeError as e:\n"
            "    print('RuntimeError:', e)\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, MPFK_SELFTEST_INJECT=probe))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "RuntimeError:" in r.stdout and text in r.stdout
    assert "unusable in this environment" in r.stdout


def test_selftest_failure_through_cpp_shim(gpu_lib):
    binp = os.path.join(ROOT, "tests", "_build", "shim_parity")
    assert os.path.exists(binp)
    r = subprocess.run([binp, "--selftest-error"], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, MPFK_SELFTEST_INJECT="fma"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS std::runtime_error" in r.stdout
