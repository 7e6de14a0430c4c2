"""MPFM matrix files (linalg_io.cpp:20-111).  Host
forms and header validation run on the CPU; the device streaming forms are
@gpu.  Bytes must equal the reference format's (restated in oracle/mpfm.py);
every reference error text must come through."""
import os
import struct

import numpy as np
import pytest

import paper_2101_06584_b200 as P
from oracle import mpfm
from tests.helpers import random_signed


def _mat(W, rows, cols, seed):
    a = random_signed(W, rows, cols, seed)
    if rows and cols:
        a[0, 0, 0] *= 2.0 ** -300
        a[0, rows - 1, cols - 1] *= 2.0 ** 300
    return a


@pytest.mark.parametrize("W,rows,cols", [(2, 3, 5), (3, 4, 8), (4, 1, 1), (2, 0, 0), (3, 17, 33)])
def test_host_roundtrip_and_bytes(tmp_path, W, rows, cols):
    a = _mat(W, rows, cols, 540 + W)
    m = P.MPMatrix.from_planes(a[:, :, :cols]) if rows and cols else P.MPMatrix(W, rows, cols)
    p = str(tmp_path / "m.mpfm")
    P.save_matrix_binary(m, p)
    q = str(tmp_path / "ref.mpfm")
    mpfm.write(q, m.data, cols)
    assert open(p, "rb").read() == open(q, "rb").read()
    back = P.load_matrix_binary(W, q)
    assert P.bits_equal(back, m)
    assert P.mpfm_info(p) == (W, rows, cols)


def _write_raw(path, magic=b"MPFM", version=1, W=2, rows=2, cols=3, stride=None, payload=None):
    stride = (cols + 3) & ~3 if stride is None else stride
    if payload is None:
        payload = np.zeros(W * rows * stride).tobytes()
    with open(path, "wb") as f:
        f.write(magic + struct.pack("<IB", version, W) + struct.pack("<QQQ", rows, cols, stride) + payload)


@pytest.mark.parametrize("kw,msg", [
    (dict(magic=b"MPFX"), "not an MPFM file"),
    (dict(version=2), "unsupported version"),
    (dict(W=3), "component width mismatch"),
    (dict(rows=2 ** 33, payload=b""), "implausible dimensions"),
    # 8 W rows stride wraps 2^64 to 0: must not pass as a 33-byte file + payload
    (dict(rows=2 ** 32, cols=2 ** 32, payload=b"\0" * 64), "implausible dimensions"),
    (dict(stride=5), "bad stride"),
    (dict(payload=b"\0" * 8), "truncated"),
    (dict(payload=b"\0" * (2 * 2 * 4 * 8 + 8)), "trailing data"),
    (dict(payload=struct.pack("<8d", 1, 2, 3, 7.0, 4, 5, 6, 0) + b"\0" * 64), "nonzero padding"),
])
def test_reference_error_texts(tmp_path, kw, msg):
    p = str(tmp_path / "bad.mpfm")
    _write_raw(p, **kw)
    with pytest.raises(RuntimeError) as e:
        P.load_matrix_binary(2, p)
    assert str(e.value) == f"{p}: {msg}"


def test_missing_and_short_files(tmp_path):
    p = str(tmp_path / "nope.mpfm")
    with pytest.raises(RuntimeError, match=": cannot open$"):
        P.mpfm_info(p)
    open(p, "wb").write(b"MPFM\1\0")
    with pytest.raises(RuntimeError, match=": truncated$"):
        P.mpfm_info(p)
    with pytest.raises(RuntimeError, match="cannot open for writing"):
        P.save_matrix_binary(P.MPMatrix(2, 1, 1), str(tmp_path / "no_dir" / "x.mpfm"))


@pytest.mark.gpu
@pytest.mark.parametrize("W,rows,cols", [(2, 300, 1001), (3, 5, 7), (4, 64, 64)])
def test_device_streaming_roundtrip(gpu_lib, tmp_path, W, rows, cols):
    import torch
    a = _mat(W, rows, cols, 560 + W)
    q = str(tmp_path / "in.mpfm")
    mpfm.write(q, a, cols)
    ld = (cols + 3) & ~3
    d = torch.zeros((W, rows, ld), dtype=torch.float64, device="cuda")
    P.mpfm_load_device(q, W, d.data_ptr(), ld, rows * ld)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), a.view(np.uint64))
    p = str(tmp_path / "out.mpfm")
    P.mpfm_save_device(p, W, d.data_ptr(), rows, cols, ld, rows * ld)
    assert open(p, "rb").read() == open(q, "rb").read()
