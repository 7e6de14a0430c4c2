"""Test-infrastructure checkers (never the product path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package.

  orc   -- ctypes binding of _build/libmpfk_oracle.so, the C restatement of the
           reference's GEMM path (mpfk_oracle.c)
  ref   -- ctypes binding of _ref/libmpfkref.so, the UNMODIFIED reference
           (mpfkit) compiled here from /root/reference/proj by oracle/Makefile
  dyadic -- exact dyadic-rational arithmetic (the reference's DyadicReal
           semantics, proj/src/oracle.cpp) for error-bound checks
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmpfk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmpfkref.so")

_D = C.c_void_p
_S = C.c_size_t
_U64 = C.c_uint64

_orc = None
_ref = None


def _p(a):
    return a.ctypes.data


def orc():
    global _orc
    if _orc is None:
        L = C.CDLL(ORACLE_SO)
        L.orc_gemm.argtypes = [C.c_int, _S, _S, _S, _D, _S, _D, _S, _D, _S]
        L.orc_gemm_rows.argtypes = [C.c_int, _S, _S, _S, _D, _S, _D, _S, _D, _S, _S, _S]
        L.orc_add.argtypes = [C.c_int, _D, _D, _D]
        L.orc_gemm_acc.argtypes = [C.c_int, _S, _S, _S, _D, _S, _S, _D, _S, _S, _D, _S, _S]
        L.orc_mul.argtypes = [C.c_int, _D, _D, _D]
        L.orc_renorm5.argtypes = [_D, _D]
        L.orc_vseb.argtypes = [_D, _S, _D, _S]
        L.orc_vec_sum.argtypes = [_D, _S, _D]
        L.orc_two_sum.argtypes = [C.c_double, C.c_double, _D, _D]
        L.orc_quick_two_sum.argtypes = [C.c_double, C.c_double, _D, _D]
        L.orc_two_prod.argtypes = [C.c_double, C.c_double, _D, _D]
        L.orc_fill_random.argtypes = [C.c_int, _S, _S, _S, _U64, _D]
        L.orc_fill_baseline.argtypes = [C.c_int, C.c_int, _S, _S, _S, _S, _U64, _D]
        L.orc_gen_paper.argtypes = [C.c_int, _S, _S, _D, _D]
        L.orc_random_normalized.argtypes = [C.c_int, _D, _D]
        L.orc_sm64_next.argtypes = [_D]
        L.orc_sm64_next.restype = _U64
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gemm.argtypes = [C.c_int, _S, _S, _S, _D, _S, _D, _S, _D, _S, _S, C.c_int, C.c_uint, C.c_int,
                               C.c_int, C.c_int]
        L.ref_gemm_shapes.argtypes = [C.c_int, _S, _S, _S, _S, _S, _S, _S, C.c_int, C.c_uint]
        L.ref_fill_random.argtypes = [C.c_int, _S, _S, _U64, _D, _S]
        L.ref_gen_paper.argtypes = [C.c_int, _S, _D, _D, _S]
        L.ref_binop.argtypes = [C.c_int, C.c_int, _D, _D, _D]
        L.ref_binop_batch.argtypes = [C.c_int, C.c_int, _S, _D, _D, _D]
        L.ref_renorm5.argtypes = [_D, _D]
        L.ref_vseb.argtypes = [_D, _S, _D, _S]
        L.ref_two_sum.argtypes = [C.c_double, C.c_double, _D, _D]
        L.ref_quick_two_sum.argtypes = [C.c_double, C.c_double, _D, _D]
        L.ref_two_prod.argtypes = [C.c_double, C.c_double, _D, _D]
        L.ref_op_counts.argtypes = [_D, _D]
        L.ref_random_normalized.argtypes = [C.c_int, _D, C.c_int, _D]
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_strassen.argtypes = [C.c_int, _S, _S, _S, _D, _S, _D, _S, _D, _S, _S, _S, C.c_int, C.c_uint]
        L.ref_leaf_multiplies.restype = _U64
        L.ref_ew.argtypes = [C.c_int, C.c_int, C.c_int, _S, _S, _D, _S, _D, _S, _D, _S]
        L.ref_td_add_merge_batch.argtypes = [_S, _D, _D, _D]
        L.ref_td_mul_q_batch.argtypes = [_S, _D, _D, _D]
        L.ref_eft_batch.argtypes = [C.c_int, _S, _D, _D, _D, _D]
        L.ref_prep_new.argtypes = [C.c_int, _S, _S, _S, _D, _S, _D, _S]
        L.ref_prep_new.restype = C.c_void_p
        L.ref_prep_run.argtypes = [C.c_void_p, _S, C.c_int, C.c_uint, C.POINTER(C.c_double)]
        L.ref_prep_result.argtypes = [C.c_void_p, _D, _S]
        L.ref_prep_free.argtypes = [C.c_void_p]
        L.ref_prep_with_a.argtypes = [C.c_void_p, _S, _D, _S]
        L.ref_prep_with_a.restype = C.c_void_p
        _ref = L
    return _ref


# ---- convenience wrappers over (W, rows, ld) float64 plane arrays ------------

def planes(W, rows, cols, ld=None):
    ld = ld if ld is not None else (cols + 3) & ~3
    return np.zeros((W, rows, ld), dtype=np.float64)


def orc_gemm(A: np.ndarray, B: np.ndarray, K: int, n: int, rows=None) -> np.ndarray:
    """Oracle C = A*B over padded plane arrays (W, m, lda), (W, K, ldb)."""
    W, m, lda = A.shape
    ldb = B.shape[2]
    ldc = (n + 3) & ~3
    Cm = np.zeros((W, m, ldc), dtype=np.float64)
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    r0, r1 = (0, m) if rows is None else rows
    orc().orc_gemm_rows(W, m, K, n, _p(A), lda, _p(B), ldb, _p(Cm), ldc, r0, r1)
    return Cm


def ref_gemm(A: np.ndarray, B: np.ndarray, K: int, n: int, workers=None, n_min=32, variant=2,
             naive=False) -> np.ndarray:
    """The reference's matmul_block_parallel_into on plane arrays."""
    W, m, lda = A.shape
    ldb = B.shape[2]
    ldc = (n + 3) & ~3
    Cm = np.zeros((W, m, ldc), dtype=np.float64)
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    if workers is None:
        workers = max(1, os.cpu_count() or 1)
    rc = ref().ref_gemm(W, m, K, n, _p(A), lda, _p(B), ldb, _p(Cm), ldc, n_min, variant, workers,
                        int(naive), -1, -1)
    if rc:
        raise ValueError(ref().ref_last_error().decode())
    return Cm


def ref_fill_random(W, rows, cols, seed):
    a = planes(W, rows, cols)
    ref().ref_fill_random(W, rows, cols, seed, _p(a), a.shape[2])
    return a


def orc_fill_random(W, rows, cols, seed):
    a = planes(W, rows, cols)
    orc().orc_fill_random(W, rows, cols, a.shape[2], seed, _p(a))
    return a


def orc_fill_baseline(W, rows, cols, seed, wide=False, row0=0):
    a = planes(W, rows, cols)
    orc().orc_fill_baseline(W, int(wide), row0, rows, cols, a.shape[2], seed, _p(a))
    return a


def ref_gen_paper(W, n):
    A = planes(W, n, n)
    B = planes(W, n, n)
    ref().ref_gen_paper(W, n, _p(A), _p(B), A.shape[2])
    return A, B


def orc_gen_paper(W, n):
    A = planes(W, n, n)
    B = planes(W, n, n)
    orc().orc_gen_paper(W, n, A.shape[2], _p(A), _p(B))
    return A, B


def ref_binop_batch(W, op, x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = np.empty_like(x)
    ref().ref_binop_batch(W, {"add": 0, "mul": 1}[op], x.shape[0], _p(x), _p(y), _p(r))
    return r


def orc_binop_batch(W, op, x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    r = np.empty_like(x)
    f = orc().orc_add if op == "add" else orc().orc_mul
    for i in range(x.shape[0]):
        f(W, x[i].ctypes.data, y[i].ctypes.data, r[i].ctypes.data)
    return r


def ref_ew(W, op, a, b, cols, variant=0):
    """linalg::ew_apply_into on plane arrays (W, rows, ld); op 'add'|'mul'|'add_merge'."""
    _, rows, lda = a.shape
    out = np.zeros_like(a)
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    rc = ref().ref_ew(W, {"add": 0, "mul": 1, "add_merge": 2}[op], variant, rows, cols, _p(a), lda, _p(b),
                      b.shape[2], _p(out), out.shape[2])
    if rc:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_strassen(A, B, K, n, cutoff=64, n_min=32, variant=0, workers=1):
    """The reference's matmul_strassen / matmul_strassen_parallel."""
    W, m, lda = A.shape
    ldb = B.shape[2]
    ldc = (n + 3) & ~3
    Cm = np.zeros((W, m, ldc), dtype=np.float64)
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    rc = ref().ref_strassen(W, m, K, n, _p(A), lda, _p(B), ldb, _p(Cm), ldc, cutoff, n_min, variant, workers)
    if rc:
        raise ValueError(ref().ref_last_error().decode())
    return Cm


class RefPrepared:
    """The reference's matmul_block_parallel_into on operands converted to
    mpfkit MPMatrix objects ONCE; run() returns the seconds of one call,
    timed inside C++ (ref_prep_run).  The CPU baseline of bench.py."""

    def __init__(self, A: np.ndarray, B: np.ndarray, K: int, n: int):
        W, m, lda = A.shape
        self.W, self.m, self.n = W, m, n
        self.h = None
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B)
        self.h = ref().ref_prep_new(W, m, K, n, _p(A), lda, _p(B), B.shape[2])
        if not self.h:
            raise ValueError(ref().ref_last_error().decode())

    def with_a(self, A: np.ndarray) -> "RefPrepared":
        """A second problem over the same reference B (shared, not copied)."""
        W, m, lda = A.shape
        A = np.ascontiguousarray(A)
        o = RefPrepared.__new__(RefPrepared)
        o.W, o.m, o.n = W, m, self.n
        o.h = ref().ref_prep_with_a(self.h, m, _p(A), lda)
        if not o.h:
            raise ValueError(ref().ref_last_error().decode())
        return o

    def run(self, workers, n_min=32, variant=2) -> float:
        s = C.c_double(0.0)
        if ref().ref_prep_run(self.h, n_min, variant, workers, C.byref(s)):
            raise ValueError(ref().ref_last_error().decode())
        return s.value

    def result(self) -> np.ndarray:
        out = np.zeros((self.W, self.m, (self.n + 3) & ~3), dtype=np.float64)
        ref().ref_prep_result(self.h, _p(out), out.shape[2])
        return out

    def close(self):
        if self.h:
            ref().ref_prep_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_cpu_info() -> dict:
    """Physical cores, hardware threads usable by this process and the CPU
    model of this host (from /proc/cpuinfo and the affinity mask)."""
    cores, model = set(), None
    phys = None
    try:
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                continue
            key, val = (s.strip() for s in line.split(":", 1))
            if key == "model name" and model is None:
                model = val
            elif key == "physical id":
                phys = val
            elif key == "core id":
                cores.add((phys, val))
    except OSError:
        pass
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1
    return {"physical_cores": len(cores) or None, "threads": threads, "cpu_model": model}
