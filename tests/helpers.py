"""Shared test helpers: seeded inputs as (W, rows, stride) plane arrays in the
reference layout, conversion to the product's MPMatrix, bit comparisons."""
from __future__ import annotations

import numpy as np

import oracle as O


def to_mp(planes, cols=None, pinned=False):
    import paper_2101_06584_b200 as P
    W, r, ld = planes.shape
    cols = ld if cols is None else cols
    m = P.MPMatrix(W, r, cols, pinned=pinned)
    m.data[:, :, :cols] = planes[:, :, :cols]
    return m


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def mismatches(a, b):
    """number of (row, col) cells whose W components are not all bit-identical"""
    a, b = bits(a), bits(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    return int((a != b).any(axis=0).sum())


def random_signed(W, rows, cols, seed, scale_lo=-3, scale_hi=3):
    """test_linalg.cpp:60-69 analog: reference random_normalized_signed values
    times 2^[lo, hi]."""
    a = O.ref_fill_random(W, rows, cols, seed) if O.ref_available() else O.orc_fill_random(W, rows, cols, seed)
    rng = np.random.default_rng(seed)
    sign = np.where(rng.integers(0, 2, size=(rows, cols)) == 1, -1.0, 1.0)
    scale = np.ldexp(1.0, rng.integers(scale_lo, scale_hi + 1, size=(rows, cols)))
    a[:, :, :cols] *= (sign * scale)[None]
    return a


def special_matrix(W, rows, cols, seed):
    """Inputs that drive the zero-residual corners of renorm5/vseb: exact
    zeros of both signs, small integers, powers of two, single-component
    values and full-width normalized values, mixed."""
    rng = np.random.default_rng(seed)
    a = O.planes(W, rows, cols)
    base = random_signed(W, rows, cols, seed + 7)
    kind = rng.integers(0, 7, size=(rows, cols))
    for i in range(rows):
        for j in range(cols):
            k = kind[i, j]
            if k == 0:
                v = [0.0] * W
            elif k == 1:
                v = [-0.0] + [0.0] * (W - 1)
            elif k == 2:
                v = [float(rng.integers(-8, 9))] + [0.0] * (W - 1)
            elif k == 3:
                v = [float(np.ldexp(1.0, int(rng.integers(-5, 6))))] + [-0.0] * (W - 1)
            elif k == 4:
                v = [1.0] + [float(np.ldexp(1.0, -53 * (w + 1))) for w in range(W - 1)]
            else:
                v = list(base[:, i, j])
            a[:, i, j] = v
    return a
