"""ctypes binding of libmpfk.so (the C ABI in include/mpfk.h).

The library is the product: there is no Python or CPU fallback.  If it is
missing the import of any compute entry point raises, loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpfk.so")

MPFK_OK, MPFK_EINVAL, MPFK_ERUNTIME, MPFK_ECUDA, MPFK_ENOMEM, MPFK_ENODEV = range(6)
MPFK_BIT_EXACT, MPFK_FAST, MPFK_LEAN = 0, 1, 2  # mpfk_flags


class MpfkMat(C.Structure):
    _fields_ = [
        ("base", C.c_void_p),
        ("rows", C.c_uint64),
        ("cols", C.c_uint64),
        ("stride", C.c_uint64),
        ("plane_stride", C.c_uint64),
    ]


class MpfkStats(C.Structure):
    _fields_ = [
        ("h2d_ms", C.c_double),
        ("bcast_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("total_ms", C.c_double),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("peer_bytes", C.c_uint64),
        ("n_gpus", C.c_int),
        ("kernel_launches", C.c_int),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class MpfkError(RuntimeError):
    """CUDA / device failure inside libmpfk (MPFK_ECUDA, MPFK_ENODEV)."""


_lib = None

_U64 = C.c_uint64
_P = C.c_void_p
_SIGS = {
    "mpfk_abi_version": (C.c_int, []),
    "mpfk_last_error": (C.c_char_p, []),
    "mpfk_device_count": (C.c_int, []),
    "mpfk_init": (C.c_int, [C.c_int]),
    "mpfk_shutdown": (None, []),
    "mpfk_selftest": (C.c_int, []),
    "mpfk_set_device": (C.c_int, [C.c_int]),
    "mpfk_get_device": (C.c_int, []),
    "mpfk_matmul_block_parallel_into": (C.c_int, [C.c_int, C.POINTER(MpfkMat), C.POINTER(MpfkMat),
                                                  C.POINTER(MpfkMat), _U64, C.c_int, C.c_uint]),
    "mpfk_matmul_block_into": (C.c_int, [C.c_int, C.POINTER(MpfkMat), C.POINTER(MpfkMat),
                                         C.POINTER(MpfkMat), _U64, C.c_int]),
    "mpfk_matmul_naive_into": (C.c_int, [C.c_int, C.POINTER(MpfkMat), C.POINTER(MpfkMat),
                                         C.POINTER(MpfkMat), C.c_int]),
    "mpfk_matmul_strassen": (C.c_int, [C.c_int, C.POINTER(MpfkMat), C.POINTER(MpfkMat), C.POINTER(MpfkMat), _U64,
                                       _U64, C.c_int, C.c_uint]),
    "mpfk_strassen_device": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                       _U64, _U64, _P, C.POINTER(C.c_int)]),
    "mpfk_last_stats": (C.c_int, [C.POINTER(MpfkStats)]),
    "mpfk_gemm_device": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                   _U64, _P, C.POINTER(C.c_int)]),
    "mpfk_gemm": (C.c_int, [C.c_int, C.POINTER(MpfkMat), C.POINTER(MpfkMat), C.POINTER(MpfkMat), C.c_int,
                            C.c_uint]),
    "mpfk_gemm_device_ex": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                      _U64, C.c_uint, _P, C.POINTER(C.c_int)]),
    "mpfk_splitk_segments": (C.c_int, [C.c_int, _U64, _U64, _U64]),
    "mpfk_gemm_redo_count": (C.c_int, [C.POINTER(_U64), C.c_int]),
    "mpfk_ew_apply_into": (C.c_int, [C.c_int, C.c_int, C.POINTER(MpfkMat), C.POINTER(MpfkMat),
                                     C.POINTER(MpfkMat), C.c_int]),
    "mpfk_ew_device": (C.c_int, [C.c_int, C.c_int, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64,
                                 _P, C.POINTER(C.c_int)]),
    "mpfk_mpfm_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(_U64), C.POINTER(_U64)]),
    "mpfk_mpfm_load_device": (C.c_int, [C.c_char_p, C.c_int, _P, _U64, _U64, _P]),
    "mpfk_mpfm_save_device": (C.c_int, [C.c_char_p, C.c_int, _P, _U64, _U64, _U64, _U64, _P]),
    "mpfk_mpfm_load_host": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(MpfkMat)]),
    "mpfk_mpfm_save_host": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(MpfkMat)]),
    "mpfk_gemm_device_acc": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                       _U64, _P, C.POINTER(C.c_int)]),
    "mpfk_gemm_device_acc_ex": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                          _U64, C.c_uint, _P, C.POINTER(C.c_int)]),
    "mpfk_gemm_device_staged_ex": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                             _U64, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_U64), _U64, C.c_uint,
                                             _P, C.POINTER(C.c_int)]),
    "mpfk_gemm_device_pull": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                        _U64, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_U64), _U64, _U64, _P,
                                        C.POINTER(C.c_int)]),
    "mpfk_gemm_device_gathered": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                            _U64, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_U64), _U64, _P,
                                            C.POINTER(C.c_int)]),
    "mpfk_gemm_device_staged": (C.c_int, [C.c_int, _U64, _U64, _U64, _P, _U64, _U64, _P, _U64, _U64, _P, _U64,
                                          _U64, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_U64), _U64, _P,
                                          C.POINTER(C.c_int)]),
    "mpfk_device_alloc": (C.c_int, [_U64, C.POINTER(C.c_void_p)]),
    "mpfk_device_free": (C.c_int, [_P]),
    "mpfk_memcpy": (C.c_int, [_P, _P, _U64]),
    "mpfk_ipc_get_handle": (C.c_int, [_P, _P]),
    "mpfk_ipc_open": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "mpfk_ipc_close": (C.c_int, [_P]),
    "mpfk_eft_batch": (C.c_int, [C.c_int, _U64, _P, _P, _P, _P]),
    "mpfk_binop_batch": (C.c_int, [C.c_int, C.c_int, _U64, _P, _P, _P]),
    "mpfk_op_counters_reset": (None, []),
    "mpfk_op_counters_read": (None, [C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_U64)]),
    "mpfk_host_register_cache": (C.c_int, [_U64]),
    "mpfk_host_register_cache_stats": (C.c_int, [C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_U64)]),
    "mpfk_host_unregister": (C.c_int, [_P]),
    "mpfk_last_op_counts": (None, [C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_U64)]),
    "mpfk_host_alloc": (_P, [_U64]),
    "mpfk_host_free": (None, [_P]),
    "mpfk_fill_baseline": (C.c_int, [C.c_int, C.c_int, _U64, _U64, _U64, _U64, _U64, _P, C.c_int]),
    "mpfk_fill_random": (C.c_int, [C.c_int, _U64, _U64, _U64, _U64, _P]),
    "mpfk_gen_paper": (C.c_int, [C.c_int, _U64, _U64, _P, _P]),
    "mpfk_fp64_peak": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libmpfk.so once; raise if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA library was not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().mpfk_last_error().decode(errors="replace")


def check(rc: int):
    """Map a status code to the Python twin of the reference's exception."""
    if rc == MPFK_OK:
        return
    msg = last_error()
    if rc == MPFK_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == MPFK_ENOMEM:
        raise MemoryError(msg)  # std::bad_alloc
    if rc == MPFK_ERUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    raise MpfkError(msg)
