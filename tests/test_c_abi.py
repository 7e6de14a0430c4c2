"""The C ABI from plain C: tests/csrc/c_abi_demo.c compiled with gcc -std=c11
-Wall -Werror against include/mpfk.h and linked to libmpfk.so."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2101_06584_b200")


def _build(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    exe = str(tmp_path / "c_abi_demo")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-pedantic", "-I",
                           os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "csrc", "c_abi_demo.c"),
                           "-L", PKG, "-lmpfk", f"-Wl,-rpath,{PKG}", "-o", exe])
    return exe


def test_header_is_c11_and_links(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "matmul: result shape mismatch" in r.stdout


@pytest.mark.gpu
def test_c_consumer_on_gpu(gpu_lib, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "gemm rc=0" in r.stdout, r.stdout + r.stderr
