"""Python mirror of the reference's matrix API (mpfkit::linalg,
/root/reference/proj/include/mpfkit/linalg.hpp) over libmpfk.

Same names, argument meaning and error behaviour as the reference:
  MPMatrix(W, rows, cols)                 MPMatrix<W> (linalg.hpp:36-129)
  pad_columns(cols)                       linalg.hpp:32-34
  bits_equal(a, b)                        linalg.hpp:132-140
  KernelVariant.{NORMAL,SIMD_SET,SIMD_LOADSTORE}   linalg.hpp:149
  matmul_naive[_into], matmul_block[_into], matmul_block_parallel[_into]
                                          linalg.hpp:346-443
  op_counters_reset / op_counters_read    linalg.hpp:160-170, linalg.cpp:13-25
std::invalid_argument surfaces as ValueError with the reference's message.
The `workers` argument of the parallel form is the number of GPUs (capped by
the visible devices); C is sharded by contiguous row spans exactly like the
reference's worker partition, and the result is bit-identical for any count.
"""
from __future__ import annotations

import ctypes as C
import enum
from collections import namedtuple

import numpy as np

from . import _native as N


class KernelVariant(enum.IntEnum):
    NORMAL = 0
    SIMD_SET = 1
    SIMD_LOADSTORE = 2


OpCounts = namedtuple("OpCounts", "adds muls leaf_multiplies")


def pad_columns(cols: int) -> int:
    return (cols + 3) & ~3


def format_eps(W: int) -> float:
    """mpf::format_eps<W>, mpf.hpp:48-53."""
    return {2: 2.0 ** -104, 3: 2.0 ** -157, 4: 2.0 ** -209}[W]


class _Pinned:
    """Owner of a page-locked host allocation (mpfk_host_alloc)."""

    def __init__(self, nbytes):
        self.ptr = N.lib().mpfk_host_alloc(nbytes)
        if not self.ptr:
            raise MemoryError(N.last_error())

    def __del__(self):
        try:
            if self.ptr:
                N.lib().mpfk_host_free(self.ptr)
        except Exception:
            pass


class MPMatrix:
    """Component-planar width-W matrix: W planes of rows x stride binary64,
    stride = pad_columns(cols), padding cells +0 (linalg.hpp:25-34).

    ``data`` is a (W, rows, stride) float64 numpy array.  ``pinned=True``
    places it in page-locked memory so host<->device copies run at full
    PCIe speed (the e2e path of bench.py)."""

    def __init__(self, W: int, rows: int = 0, cols: int = 0, pinned: bool = False):
        if W not in (2, 3, 4):
            raise ValueError("MPMatrix: width must be 2, 3 or 4")
        self.W = W
        self._rows, self._cols = int(rows), int(cols)
        self._stride = pad_columns(self._cols)
        shape = (W, self._rows, self._stride)
        self._owner = None
        if pinned and self._rows * self._stride > 0:
            nbytes = 8 * W * self._rows * self._stride
            self._owner = _Pinned(nbytes)
            buf = (C.c_double * (nbytes // 8)).from_address(self._owner.ptr)
            # numpy's base chain (data -> buf) keeps the page-locked block alive
            # for views that outlive this MPMatrix
            buf._owner = self._owner
            self.data = np.frombuffer(buf, dtype=np.float64).reshape(shape)
            self.data[...] = 0.0
        else:
            self.data = np.zeros(shape, dtype=np.float64)

    # --- reference accessors -------------------------------------------------
    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def stride(self):
        return self._stride

    def plane_size(self):
        return self._rows * self._stride

    def plane(self, w: int):
        if not 0 <= w < self.W:
            raise ValueError("MPMatrix::plane: component out of range")
        return self.data[w]

    def at(self, i: int, j: int):
        if not (0 <= i < self._rows and 0 <= j < self._cols):
            raise ValueError("MPMatrix::at: index out of range")
        return tuple(float(self.data[w, i, j]) for w in range(self.W))

    def set(self, i: int, j: int, v):
        if not (0 <= i < self._rows and 0 <= j < self._cols):
            raise ValueError("MPMatrix::set: index out of range")
        for w in range(self.W):
            self.data[w, i, j] = v[w]

    def same_shape(self, o: "MPMatrix") -> bool:
        return self._rows == o._rows and self._cols == o._cols

    def fill_zero(self):
        self.data[...] = 0.0

    def zero_pads(self):
        self.data[:, :, self._cols:] = 0.0

    def copy(self, pinned: bool = False) -> "MPMatrix":
        m = MPMatrix(self.W, self._rows, self._cols, pinned=pinned)
        m.data[...] = self.data
        return m

    # --- numpy interop -------------------------------------------------------
    @classmethod
    def from_planes(cls, planes, pinned: bool = False) -> "MPMatrix":
        """planes: (W, rows, cols) float64 array-like."""
        p = np.asarray(planes, dtype=np.float64)
        W, r, c = p.shape
        m = cls(W, r, c, pinned=pinned)
        m.data[:, :, :c] = p
        return m

    def planes(self):
        """(W, rows, cols) view without padding."""
        return self.data[:, :, : self._cols]

    def _c(self) -> N.MpfkMat:
        return N.MpfkMat(self.data.ctypes.data if self.data.size else None, self._rows, self._cols,
                         self._stride, self._rows * self._stride)


def bits_equal(a: MPMatrix, b: MPMatrix) -> bool:
    """Full-representation equality, padding included (linalg.hpp:132-140)."""
    if a.W != b.W or not a.same_shape(b):
        return False
    return a.data.view(np.uint64).tobytes() == b.data.view(np.uint64).tobytes()


def _check_same_width(*ms):
    W = ms[0].W
    for m in ms:
        if m.W != W:
            raise ValueError("matmul: operands must share one width")
    return W


def matmul_block_parallel_into(C_: MPMatrix, A: MPMatrix, B: MPMatrix, n_min: int = 32,
                               variant: KernelVariant = KernelVariant.NORMAL, workers: int = 1):
    """linalg.hpp:402-433 on min(workers, GPUs) devices."""
    W = _check_same_width(C_, A, B)
    c, a, b = C_._c(), A._c(), B._c()
    # negative counts reach the C ABI as 0, which it rejects in the reference's order
    N.check(N.lib().mpfk_matmul_block_parallel_into(W, C.byref(c), C.byref(a), C.byref(b), max(int(n_min), 0),
                                                    int(variant), max(int(workers), 0)))


def matmul_block_into(C_: MPMatrix, A: MPMatrix, B: MPMatrix, n_min: int = 32,
                      variant: KernelVariant = KernelVariant.NORMAL):
    """linalg.hpp:368-388."""
    W = _check_same_width(C_, A, B)
    c, a, b = C_._c(), A._c(), B._c()
    N.check(N.lib().mpfk_matmul_block_into(W, C.byref(c), C.byref(a), C.byref(b), max(int(n_min), 0), int(variant)))


def matmul_naive_into(C_: MPMatrix, A: MPMatrix, B: MPMatrix,
                      variant: KernelVariant = KernelVariant.NORMAL):
    """linalg.hpp:346-358."""
    W = _check_same_width(C_, A, B)
    c, a, b = C_._c(), A._c(), B._c()
    N.check(N.lib().mpfk_matmul_naive_into(W, C.byref(c), C.byref(a), C.byref(b), int(variant)))


BIT_EXACT, FAST, LEAN = N.MPFK_BIT_EXACT, N.MPFK_FAST, N.MPFK_LEAN


def gemm_into(C_: MPMatrix, A: MPMatrix, B: MPMatrix, n_gpus: int = 1, flags: int = BIT_EXACT):
    """mpfk_gemm: C = A*B on n_gpus GPUs (<= 0: all).  flags=BIT_EXACT is
    matmul_block_parallel_into; flags=FAST may split K for outputs too small
    to fill the GPU (deterministic, tolerance-checked: normwise 4*k*u_p);
    flags=LEAN runs the tolerance-mode arithmetic (csrc/mpf_lean.cuh: 12 / 46 /
    113 FP64 instructions per multiply-add, 1.75-2.6x the bit-exact rate, NOT
    the reference's bits).  FAST | LEAN combines them."""
    W = _check_same_width(C_, A, B)
    c, a, b = C_._c(), A._c(), B._c()
    N.check(N.lib().mpfk_gemm(W, C.byref(a), C.byref(b), C.byref(c), int(n_gpus), int(flags)))


def gemm(A: MPMatrix, B: MPMatrix, n_gpus: int = 1, flags: int = BIT_EXACT, pinned: bool = False) -> MPMatrix:
    C_ = MPMatrix(A.W, A.rows(), B.cols(), pinned=pinned)
    gemm_into(C_, A, B, n_gpus, flags)
    return C_


def splitk_segments(W: int, m: int, n: int, k: int) -> int:
    """K segments FAST uses for an m x n x k product here (1 = bit-exact)."""
    r = N.lib().mpfk_splitk_segments(W, m, n, k)
    if r < 0:
        N.check(-r)
    return r


def gemm_redo_count(reset: bool = False) -> int:
    """Warp k-tiles the TD/QD GEMM recomputed with the exact renorm5 paths
    C/D on the current device since the last reset (mpfk_gemm_redo_count)."""
    v = C.c_uint64(0)
    N.check(N.lib().mpfk_gemm_redo_count(C.byref(v), 1 if reset else 0))
    return v.value


def matmul_block_parallel(A: MPMatrix, B: MPMatrix, n_min: int = 32,
                          variant: KernelVariant = KernelVariant.NORMAL, workers: int = 1,
                          pinned: bool = False) -> MPMatrix:
    C_ = MPMatrix(A.W, A.rows(), B.cols(), pinned=pinned)
    matmul_block_parallel_into(C_, A, B, n_min, variant, workers)
    return C_


def matmul_block(A: MPMatrix, B: MPMatrix, n_min: int = 32,
                 variant: KernelVariant = KernelVariant.NORMAL) -> MPMatrix:
    C_ = MPMatrix(A.W, A.rows(), B.cols())
    matmul_block_into(C_, A, B, n_min, variant)
    return C_


def matmul_naive(A: MPMatrix, B: MPMatrix, variant: KernelVariant = KernelVariant.NORMAL) -> MPMatrix:
    C_ = MPMatrix(A.W, A.rows(), B.cols())
    matmul_naive_into(C_, A, B, variant)
    return C_


class EwOp(enum.IntEnum):
    """linalg.hpp:623"""
    add = 0
    mul = 1
    add_merge = 2


def ew_apply_into(out: MPMatrix, a: MPMatrix, b: MPMatrix, op: EwOp,
                  variant: KernelVariant = KernelVariant.NORMAL):
    """linalg::ew_apply_into (linalg.hpp:647-684) on the GPU."""
    W = _check_same_width(out, a, b)
    o, x, y = out._c(), a._c(), b._c()
    N.check(N.lib().mpfk_ew_apply_into(W, int(op), C.byref(o), C.byref(x), C.byref(y), int(variant)))


def ew_add(a: MPMatrix, b: MPMatrix, variant: KernelVariant = KernelVariant.NORMAL) -> MPMatrix:
    """linalg.hpp:686-692"""
    r = MPMatrix(a.W, a.rows(), a.cols())
    ew_apply_into(r, a, b, EwOp.add, variant)
    return r


def ew_mul(a: MPMatrix, b: MPMatrix, variant: KernelVariant = KernelVariant.NORMAL) -> MPMatrix:
    """linalg.hpp:694-700"""
    r = MPMatrix(a.W, a.rows(), a.cols())
    ew_apply_into(r, a, b, EwOp.mul, variant)
    return r


def ew_add_merge(a: MPMatrix, b: MPMatrix, variant: KernelVariant = KernelVariant.NORMAL) -> MPMatrix:
    """linalg.hpp:702-707 (triple width only)"""
    r = MPMatrix(a.W, a.rows(), a.cols())
    ew_apply_into(r, a, b, EwOp.add_merge, variant)
    return r


def ew_device(W: int, op: int, rows: int, cols: int, out_ptr: int, ldo: int, o_plane: int, a_ptr: int, lda: int,
              a_plane: int, b_ptr: int, ldb: int, b_plane: int, stream: int = 0) -> int:
    launches = C.c_int(0)
    N.check(N.lib().mpfk_ew_device(W, int(op), rows, cols, out_ptr, ldo, o_plane, a_ptr, lda, a_plane, b_ptr, ldb,
                                   b_plane, stream or None, C.byref(launches)))
    return launches.value


# --- MPFM matrix files (linalg_io.cpp:66-111) ----------------------------------

def mpfm_info(path: str):
    """(width, rows, cols) from an MPFM header (validated)."""
    w, r, c = C.c_int(), C.c_uint64(), C.c_uint64()
    N.check(N.lib().mpfk_mpfm_info(path.encode(), C.byref(w), C.byref(r), C.byref(c)))
    return w.value, r.value, c.value


def save_matrix_binary(m: MPMatrix, path: str):
    """linalg::save_matrix_binary (linalg_io.cpp:66-83)."""
    x = m._c()
    N.check(N.lib().mpfk_mpfm_save_host(path.encode(), m.W, C.byref(x)))


def load_matrix_binary(W: int, path: str, pinned: bool = False) -> MPMatrix:
    """linalg::load_matrix_binary<W> (linalg_io.cpp:85-111)."""
    w, r, c = C.c_int(), C.c_uint64(), C.c_uint64()
    N.check(N.lib().mpfk_mpfm_info(path.encode(), C.byref(w), C.byref(r), C.byref(c)))
    if w.value != W:
        raise RuntimeError(f"{path}: component width mismatch")
    m = MPMatrix(W, r.value, c.value, pinned=pinned)
    x = m._c()
    N.check(N.lib().mpfk_mpfm_load_host(path.encode(), W, C.byref(x)))
    return m


def mpfm_load_device(path: str, W: int, dev_ptr: int, ld: int, plane: int, stream: int = 0):
    """Stream an MPFM file into device memory (current device)."""
    N.check(N.lib().mpfk_mpfm_load_device(path.encode(), W, dev_ptr, ld, plane, stream or None))


def mpfm_save_device(path: str, W: int, dev_ptr: int, rows: int, cols: int, ld: int, plane: int,
                     stream: int = 0):
    """Write device-resident planes as an MPFM file."""
    N.check(N.lib().mpfk_mpfm_save_device(path.encode(), W, dev_ptr, rows, cols, ld, plane, stream or None))


def op_counters_reset():
    N.lib().mpfk_op_counters_reset()


def op_counters_read() -> OpCounts:
    a, m, l_ = C.c_uint64(), C.c_uint64(), C.c_uint64()
    N.lib().mpfk_op_counters_read(C.byref(a), C.byref(m), C.byref(l_))
    return OpCounts(a.value, m.value, l_.value)


def host_register_cache(capacity_bytes: int):
    """Opt-in page-locking of long-lived pageable operands
    (mpfk_host_register_cache): a bounded LRU set of registered MPMatrix
    buffers; 0 disables and empties it.  Drop a buffer with
    host_unregister() before freeing it."""
    N.check(N.lib().mpfk_host_register_cache(int(capacity_bytes)))


def host_register_cache_stats() -> dict:
    cap, used, ents = C.c_uint64(), C.c_uint64(), C.c_uint64()
    N.check(N.lib().mpfk_host_register_cache_stats(C.byref(cap), C.byref(used), C.byref(ents)))
    return {"capacity": cap.value, "used": used.value, "entries": ents.value}


def host_unregister(m):
    """Remove an MPMatrix (or a raw base address) from the registration cache."""
    base = m.data.ctypes.data if isinstance(m, MPMatrix) else int(m)
    N.check(N.lib().mpfk_host_unregister(base))


def last_stats() -> dict:
    s = N.MpfkStats()
    N.check(N.lib().mpfk_last_stats(C.byref(s)))
    return s.as_dict()


# --- device-resident operands ---------------------------------------------------

def gemm_device(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int, ldb: int,
                b_plane: int, C_ptr: int, ldc: int, c_plane: int, stream: int = 0) -> int:
    """Enqueue C = A*B on the current device/stream (mpfk_gemm_device).
    Returns the number of kernel launches."""
    launches = C.c_int(0)
    N.check(N.lib().mpfk_gemm_device(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc,
                                     c_plane, stream or None, C.byref(launches)))
    return launches.value


def gemm_device_ex(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int, ldb: int,
                   b_plane: int, C_ptr: int, ldc: int, c_plane: int, flags: int = BIT_EXACT, stream: int = 0) -> int:
    """mpfk_gemm_device_ex: gemm_device with flags (FAST may split K, LEAN
    selects the tolerance-mode arithmetic)."""
    launches = C.c_int(0)
    N.check(N.lib().mpfk_gemm_device_ex(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc,
                                        c_plane, int(flags), stream or None, C.byref(launches)))
    return launches.value


def gemm_device_acc(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int, ldb: int,
                    b_plane: int, C_ptr: int, ldc: int, c_plane: int, stream: int = 0,
                    flags: int = BIT_EXACT) -> int:
    """Continue the chains in C over one K panel (mpfk_gemm_device_acc[_ex];
    flags: BIT_EXACT or LEAN)."""
    launches = C.c_int(0)
    N.check(N.lib().mpfk_gemm_device_acc_ex(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc,
                                            c_plane, int(flags), stream or None, C.byref(launches)))
    return launches.value


def binop_batch(W: int, op: str, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Elementwise mpf::add/mul<W> on the GPU over (count, W) arrays."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 2 or x.shape[1] != W:
        raise ValueError("binop_batch: x and y must be (count, W)")
    r = np.empty_like(x)
    N.check(N.lib().mpfk_binop_batch(W, {"add": 0, "mul": 1, "td_mul_q": 2, "td_add_merge": 3}[op], x.shape[0],
                                     x.ctypes.data, y.ctypes.data,
                                     r.ctypes.data))
    return r


def eft_batch(op: str, a: np.ndarray, b: np.ndarray):
    """two_sum / quick_two_sum / two_prod of float64 arrays on the GPU -> (s, e)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    s, e = np.empty_like(a), np.empty_like(a)
    code = {"two_sum": 0, "quick_two_sum": 1, "two_prod": 2}[op]
    N.check(N.lib().mpfk_eft_batch(code, a.size, a.ctypes.data, b.ctypes.data, s.ctypes.data, e.ctypes.data))
    return s, e


def fill_baseline(W: int, rows: int, cols: int, seed: int, wide: bool = False, pinned: bool = False,
                  threads: int = 0, row0: int = 0) -> MPMatrix:
    """BASELINE.json inputs (include/mpfk.h: mpfk_fill_baseline): rows
    [row0, row0 + rows) of the seeded matrix."""
    m = MPMatrix(W, rows, cols, pinned=pinned)
    if rows and cols:
        N.check(N.lib().mpfk_fill_baseline(W, int(bool(wide)), row0, rows, cols, m.stride(),
                                           seed & (2 ** 64 - 1), m.data.ctypes.data, threads))
    return m


def fp64_peak() -> tuple:
    """(FP64 lane-ops/s, ms) measured on the current device."""
    ops, ms = C.c_double(), C.c_double()
    N.check(N.lib().mpfk_fp64_peak(C.byref(ops), C.byref(ms)))
    return ops.value, ms.value


def set_device(dev: int):
    """Make `dev` libmpfk's current device (mirror torch.cuda.set_device)."""
    N.check(N.lib().mpfk_set_device(int(dev)))


def get_device() -> int:
    return N.lib().mpfk_get_device()


def device_count() -> int:
    return N.lib().mpfk_device_count()


def fill_random(W: int, rows: int, cols: int, seed: int, pinned: bool = False) -> MPMatrix:
    """bench::fill_random (bench.cpp:295-302): sequential SplitMix64 stream of
    rng::random_normalized<W> values (lead in [1, 2))."""
    m = MPMatrix(W, rows, cols, pinned=pinned)
    if rows and cols:
        N.check(N.lib().mpfk_fill_random(W, rows, cols, m.stride(), seed & (2 ** 64 - 1), m.data.ctypes.data))
    return m


def gen_paper_matrices(W: int, n: int):
    """bench::gen_paper_matrices (bench.cpp:278-292) -> (A, B)."""
    if n < 1:
        raise ValueError("gen_paper_matrices: n must be at least 1")
    A, B = MPMatrix(W, n, n), MPMatrix(W, n, n)
    N.check(N.lib().mpfk_gen_paper(W, n, A.stride(), A.data.ctypes.data, B.data.ctypes.data))
    return A, B


def matmul_strassen(A: MPMatrix, B: MPMatrix, cutoff: int = 64, n_min: int = 32,
                    variant: KernelVariant = KernelVariant.NORMAL) -> MPMatrix:
    """linalg::matmul_strassen (linalg.hpp:582-591) with GPU block leaves."""
    return matmul_strassen_parallel(A, B, cutoff, n_min, variant, 1)


def matmul_strassen_parallel(A: MPMatrix, B: MPMatrix, cutoff: int = 64, n_min: int = 32,
                             variant: KernelVariant = KernelVariant.NORMAL, workers: int = 1) -> MPMatrix:
    """linalg::matmul_strassen_parallel (linalg.hpp:596-617); bit-identical to
    the serial form, as in the reference."""
    W = _check_same_width(A, B)
    C_ = MPMatrix(W, A.rows(), B.cols())
    c, a, b = C_._c(), A._c(), B._c()
    N.check(N.lib().mpfk_matmul_strassen(W, C.byref(c), C.byref(a), C.byref(b), max(int(cutoff), 0),
                                         max(int(n_min), 0), int(variant), max(int(workers), 0)))
    return C_


def strassen_device(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int, ldb: int,
                    b_plane: int, C_ptr: int, ldc: int, c_plane: int, cutoff: int = 64, stream: int = 0) -> int:
    """Device-resident Strassen (mpfk_strassen_device); returns kernel launches."""
    launches = C.c_int(0)
    N.check(N.lib().mpfk_strassen_device(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc, c_plane,
                                         cutoff, stream or None, C.byref(launches)))
    return launches.value


def gemm_device_pull(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int, ldb: int,
                     b_plane: int, C_ptr: int, ldc: int, c_plane: int, src_ptrs, src_row0, panel_rows: int = 64,
                     chunk_rows: int = 8, stream: int = 0) -> int:
    """Fused all-gather -> GEMM (mpfk_gemm_device_pull): B's rows come from the
    source slices (peer-mapped device pointers); B_ptr receives the whole B."""
    ns = len(src_ptrs)
    srcs = (C.c_void_p * ns)(*src_ptrs)
    rows = (C.c_uint64 * (ns + 1))(*src_row0)
    launches = C.c_int(0)
    N.check(N.lib().mpfk_gemm_device_pull(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc, c_plane,
                                          ns, srcs, rows, panel_rows, chunk_rows, stream or None,
                                          C.byref(launches)))
    return launches.value


def gemm_device_gathered(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int,
                         ldb: int, b_plane: int, C_ptr: int, ldc: int, c_plane: int, src_ptrs, src_row0,
                         panel_rows: int = 256, stream: int = 0) -> int:
    """All-gather -> GEMM with the copy engines gathering B's panels from the
    source slices while ONE gated GEMM launch computes
    (mpfk_gemm_device_gathered); B_ptr receives the whole B."""
    ns = len(src_ptrs)
    srcs = (C.c_void_p * ns)(*src_ptrs)
    rows = (C.c_uint64 * (ns + 1))(*src_row0)
    launches = C.c_int(0)
    N.check(N.lib().mpfk_gemm_device_gathered(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc,
                                              c_plane, ns, srcs, rows, panel_rows, stream or None,
                                              C.byref(launches)))
    return launches.value


def gemm_device_staged(W: int, m: int, n: int, k: int, A_ptr: int, lda: int, a_plane: int, B_ptr: int,
                       ldb: int, b_plane: int, C_ptr: int, ldc: int, c_plane: int, src_ptrs, src_row0,
                       head_rows: int = 0, stream: int = 0, flags: int = BIT_EXACT) -> int:
    """All-gather -> GEMM with the copy engines gathering B's K panels from
    the source slices and one GEMM launch per panel gated on that panel's
    event (mpfk_gemm_device_staged[_ex]; flags: BIT_EXACT or LEAN); B_ptr
    receives the whole B."""
    ns = len(src_ptrs)
    srcs = (C.c_void_p * ns)(*src_ptrs)
    rows = (C.c_uint64 * (ns + 1))(*src_row0)
    launches = C.c_int(0)
    N.check(N.lib().mpfk_gemm_device_staged_ex(W, m, n, k, A_ptr, lda, a_plane, B_ptr, ldb, b_plane, C_ptr, ldc,
                                               c_plane, ns, srcs, rows, head_rows, int(flags), stream or None,
                                               C.byref(launches)))
    return launches.value


def ipc_handle(dev_ptr: int) -> bytes:
    """The 64-byte CUDA IPC handle of a libmpfk device allocation."""
    buf = (C.c_char * 64)()
    N.check(N.lib().mpfk_ipc_get_handle(dev_ptr, buf))
    return bytes(buf)


def ipc_open(handle: bytes) -> int:
    p = C.c_void_p()
    buf = (C.c_char * 64).from_buffer_copy(handle)
    N.check(N.lib().mpfk_ipc_open(buf, C.byref(p)))
    return p.value


def ipc_close(dev_ptr: int):
    N.check(N.lib().mpfk_ipc_close(dev_ptr))


def device_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    N.check(N.lib().mpfk_device_alloc(nbytes, C.byref(p)))
    return p.value


def device_free(dev_ptr: int):
    N.check(N.lib().mpfk_device_free(dev_ptr))


def memcpy(dst: int, src: int, nbytes: int):
    """cudaMemcpy with cudaMemcpyDefault (host or device pointers)."""
    N.check(N.lib().mpfk_memcpy(dst, src, nbytes))
