"""Restatement of the reference's MPFM writer/reader (TEST INFRASTRUCTURE
ONLY): /root/reference/proj/src/linalg_io.cpp:20-111 (the reference's own
linalg_io.cpp cannot be compiled here: its translation unit includes the
Boost-based decimal converter).  Header: b"MPFM", u32 version 1, u8 width,
u64 rows, cols, stride = pad4(cols), little-endian; then W planes of
rows*stride little-endian binary64, padding included."""
import struct

import numpy as np


def write(path, planes, cols):
    """planes: (W, rows, stride) float64 with stride = pad4(cols)."""
    W, rows, stride = planes.shape
    assert stride == (cols + 3) & ~3
    with open(path, "wb") as f:
        f.write(b"MPFM" + struct.pack("<IB", 1, W) + struct.pack("<QQQ", rows, cols, stride))
        f.write(np.ascontiguousarray(planes, dtype="<f8").tobytes())


def read(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"MPFM"
    version, W = struct.unpack("<IB", raw[4:9])
    rows, cols, stride = struct.unpack("<QQQ", raw[9:33])
    data = np.frombuffer(raw[33:], dtype="<f8").reshape(W, rows, stride)
    return W, rows, cols, data
