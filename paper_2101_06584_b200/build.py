"""Build every native artefact in-tree (no JIT cache: the .so files travel to
the GPU box with the repo snapshot).

  paper_2101_06584_b200/libmpfk.so   the product: sm_100a kernels + C ABI
  tests/_build/libarith_host.so      test shim: csrc/mpf_arith.cuh compiled for
                                     the host, checked bit-for-bit against the
                                     reference on the CPU
  tests/_build/shim_parity           C++ drop-in demo/test: the reference's own
                                     MPMatrix<W> fed to include/mpfk/linalg.hpp
                                     (only when /root/reference is present)
  oracle/_build, oracle/_ref         the checkers (oracle/Makefile)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2101_06584_b200")
CSRC = os.path.join(PKG, "csrc")
REF = "/root/reference/proj"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"]


def _run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, **kw)


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _csrc_deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "mpfk.h")]


def build_lib(force=False):
    out = os.path.join(PKG, "libmpfk.so")
    if force or _stale(out, _csrc_deps()):
        _run([NVCC, *NVCC_FLAGS, "-shared", "-o", out, os.path.join(CSRC, "capi.cu")])
    return out


def build_tune(force=False):
    """The tile-configuration sweep library (scripts/tune.py); not the product."""
    out = os.path.join(PKG, "libmpfk_tune.so")
    if force or _stale(out, _csrc_deps()):
        _run([NVCC, *NVCC_FLAGS, "-shared", "-o", out, os.path.join(CSRC, "tune.cu")])
    return out


def build_tune_lean(force=False):
    """The MPFK_LEAN tile sweep library (scripts/tune.py --lean, TUNE_LIB); not the product."""
    out = os.path.join(PKG, "libmpfk_tune_lean.so")
    if force or _stale(out, _csrc_deps()):
        _run([NVCC, *NVCC_FLAGS, "-shared", "-o", out, os.path.join(CSRC, "tune_lean.cu")])
    return out


def build_host_arith(force=False):
    outdir = os.path.join(ROOT, "tests", "_build")
    os.makedirs(outdir, exist_ok=True)
    out = os.path.join(outdir, "libarith_host.so")
    src = os.path.join(ROOT, "tests", "csrc", "arith_host.cpp")
    if force or _stale(out, [src, os.path.join(CSRC, "mpf_arith.cuh"), os.path.join(CSRC, "mpf_lean.cuh")]):
        _run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
              "-I", CSRC, "-o", out, src])
    return out


def build_shim_parity(force=False):
    """C++ drop-in test binary; needs the reference headers (this container only)."""
    outdir = os.path.join(ROOT, "tests", "_build")
    os.makedirs(outdir, exist_ok=True)
    out = os.path.join(outdir, "shim_parity")
    src = os.path.join(ROOT, "tests", "csrc", "shim_parity.cpp")
    if not os.path.isdir(os.path.join(REF, "include")):
        return out if os.path.exists(out) else None
    deps = [src, os.path.join(ROOT, "include", "mpfk", "linalg.hpp"), os.path.join(PKG, "libmpfk.so")]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O3", "-mavx2", "-mfma", "-ffp-contract=off", "-DMPFKIT_HAVE_AVX2=1",
              "-DNDEBUG", "-pthread", "-I", os.path.join(REF, "include"), "-I", os.path.join(ROOT, "include"),
              "-o", out, src, os.path.join(REF, "src", "runtime.cpp"), os.path.join(REF, "src", "linalg.cpp"),
              "-L", PKG, "-lmpfk", "-Wl,-rpath,$ORIGIN/../../paper_2101_06584_b200"])
    return out


def build_oracle():
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


def build_all(force=False):
    build_lib(force)
    build_oracle()
    build_host_arith(force)
    build_shim_parity(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
