"""The drop-in boundary without a GPU: libmpfk loads, exports every symbol
include/mpfk.h declares, validates arguments before any device work with the
reference's exception types and messages (linalg.hpp:279-294, :409), and
fails loudly (no CPU fallback) when no device is visible.  Also the host
input generator against the oracle's restatement."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2101_06584_b200 as P
from paper_2101_06584_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "mpfk.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(mpfk_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 18
    L = C.CDLL(N.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(N.EXPORTED)
    assert N.lib().mpfk_abi_version() == 1


def test_no_fallback_without_device():
    if P.device_count() > 0:
        pytest.skip("a device is visible")
    A, B, Cm = P.MPMatrix(2, 4, 4), P.MPMatrix(2, 4, 4), P.MPMatrix(2, 4, 4)
    with pytest.raises(N.MpfkError, match="no CUDA sm_100 device"):
        P.matmul_block_into(Cm, A, B)


@pytest.mark.parametrize("call,msg", [
    (lambda: P.matmul_block_into(P.MPMatrix(2, 3, 2), P.MPMatrix(2, 3, 4), P.MPMatrix(2, 5, 2)),
     "matmul: inner dimensions differ"),
    (lambda: P.matmul_block_into(P.MPMatrix(2, 3, 3), P.MPMatrix(2, 3, 4), P.MPMatrix(2, 4, 2)),
     "matmul: result shape mismatch"),
    (lambda: P.matmul_block_into(P.MPMatrix(3, 3, 2), P.MPMatrix(3, 3, 4), P.MPMatrix(3, 4, 2), 0),
     "matmul: n_min must be at least 1"),
    (lambda: P.matmul_block_into(P.MPMatrix(4, 3, 2), P.MPMatrix(4, 3, 4), P.MPMatrix(4, 4, 2), 5,
                                 P.KernelVariant.SIMD_SET), "matmul: SIMD variants need n_min divisible by 4"),
    (lambda: P.matmul_block_parallel_into(P.MPMatrix(2, 3, 2), P.MPMatrix(2, 3, 4), P.MPMatrix(2, 4, 2), 32,
                                          P.KernelVariant.NORMAL, 0), "matmul: workers must be at least 1"),
    (lambda: P.matmul_naive_into(P.MPMatrix(2, 3, 2), P.MPMatrix(2, 3, 5), P.MPMatrix(2, 4, 2)),
     "matmul: inner dimensions differ"),
])
def test_validation_messages_match_reference(call, msg):
    with pytest.raises(ValueError) as e:
        call()
    assert str(e.value) == msg


def test_width_and_device_api_validation():
    L = N.lib()
    m = N.MpfkMat(None, 0, 0, 0, 0)
    assert L.mpfk_matmul_block_into(5, C.byref(m), C.byref(m), C.byref(m), 32, 0) == N.MPFK_EINVAL
    assert "width" in N.last_error()
    # odd device strides are rejected before any device call
    rc = L.mpfk_gemm_device(2, 4, 4, 4, 16, 5, 20, 16, 4, 16, 16, 4, 16, None, None)
    assert rc == N.MPFK_EINVAL and "even" in N.last_error()


def test_mpmatrix_layout_mirrors_reference():
    """linalg.hpp:32-34, 36-129; test_linalg.cpp:111-147."""
    assert [P.pad_columns(c) for c in (0, 1, 4, 5, 9)] == [0, 4, 4, 8, 12]
    m = P.MPMatrix(3, 3, 5)
    assert (m.rows(), m.cols(), m.stride()) == (3, 5, 8)
    v = (1.5, 2.0 ** -60, -2.0 ** -120)
    m.set(2, 4, v)
    assert m.at(2, 4) == v
    with pytest.raises(ValueError):
        m.at(3, 0)
    with pytest.raises(ValueError):
        m.plane(3)
    c = m.copy()
    assert P.bits_equal(c, m)
    c.set(0, 0, (7.0, 0.0, 0.0))
    assert not P.bits_equal(c, m)


@pytest.mark.parametrize("W,wide", [(2, False), (3, False), (4, False), (3, True), (4, True)])
def test_host_generator_matches_oracle_restatement(W, wide):
    a = P.fill_baseline(W, 13, 11, 99, wide=wide)
    b = O.orc_fill_baseline(W, 13, 11, 99, wide)
    assert np.array_equal(a.data.view(np.uint64), b.view(np.uint64))
    # row shards reproduce the full matrix's rows
    s = P.fill_baseline(W, 5, 11, 99, wide=wide, row0=4)
    assert np.array_equal(s.data.view(np.uint64), a.data[:, 4:9].view(np.uint64))
    # normalized: |c[i+1]| <= ulp(c[i]) (mpf.hpp:60-65)
    d = a.data[:, :, :11]
    for w in range(W - 1):
        ulp = np.where(d[w] == 0, 0, np.ldexp(1.0, np.frexp(d[w])[1] - 53))
        assert (np.abs(d[w + 1]) <= ulp).all()


def test_op_counters_interface():
    P.op_counters_reset()
    c = P.op_counters_read()
    assert (c.adds, c.muls, c.leaf_multiplies) == (0, 0, 0)
