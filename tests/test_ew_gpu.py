"""elementwise kernels (linalg::ew_apply_into,
linalg.hpp:623-707) on the GPU vs the reference build, bit for bit; mirrors
test_linalg.cpp:149-192 (ragged widths, every variant, pads, add_merge
width check, shape mismatch) and the op counters."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import mismatches, random_signed, special_matrix, to_mp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("shape", [(3, 5), (1, 1), (1, 1001), (7, 4), (33, 17)])
def test_ew_matches_reference(gpu_lib, W, shape):
    P = gpu_lib
    rows, cols = shape
    for gen, seed in ((random_signed, 401), (special_matrix, 403)):
        a = gen(W, rows, cols, seed)
        b = gen(W, rows, cols, seed + 1)
        ops = ["add", "mul"] + (["add_merge"] if W == 3 else [])
        for op in ops:
            want = O.ref_ew(W, op, a, b, cols)
            for v in (P.KernelVariant.NORMAL, P.KernelVariant.SIMD_SET, P.KernelVariant.SIMD_LOADSTORE):
                out = P.MPMatrix(W, rows, cols)
                P.ew_apply_into(out, to_mp(a, cols), to_mp(b, cols), P.EwOp[op], v)
                assert mismatches(out.data, want) == 0
                assert not out.data[:, :, cols:].view(np.uint64).any()


def test_ew_pads_and_errors(gpu_lib):
    P = gpu_lib
    a = to_mp(random_signed(2, 3, 5, 405), 5)
    b = to_mp(random_signed(2, 3, 5, 406), 5)
    out = P.MPMatrix(2, 3, 5)
    out.data[:, :, 5:] = 9.0  # stale pads: NORMAL leaves them, SIMD zeroes them
    P.ew_apply_into(out, a, b, P.EwOp.add, P.KernelVariant.NORMAL)
    assert (out.data[:, :, 5:] == 9.0).all()
    P.ew_apply_into(out, a, b, P.EwOp.add, P.KernelVariant.SIMD_LOADSTORE)
    assert not out.data[:, :, 5:].view(np.uint64).any()
    with pytest.raises(ValueError, match="ew: add_merge is a triple-width operation"):
        P.ew_apply_into(out, a, b, P.EwOp.add_merge)
    with pytest.raises(ValueError, match="ew: shape mismatch"):
        P.ew_add(a, P.MPMatrix(2, 3, 4))
    P.op_counters_reset()
    P.ew_mul(a, b)
    P.ew_add(a, b)
    c = P.op_counters_read()
    assert (c.adds, c.muls) == (15, 15)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_ew_large_vectors(gpu_lib, W):
    """1 x n vectors as in the paper's benchmarks (bench.cpp:77-127)."""
    P = gpu_lib
    n = 1 << 20
    a = P.fill_baseline(W, 1, n, 5, wide=True)
    b = P.fill_baseline(W, 1, n, 6, wide=True)
    for op in (["add", "mul"] + (["add_merge"] if W == 3 else [])):
        out = P.MPMatrix(W, 1, n)
        P.ew_apply_into(out, a, b, P.EwOp[op], P.KernelVariant.SIMD_LOADSTORE)
        want = O.ref_ew(W, op, a.data, b.data, n)
        assert mismatches(out.data, want) == 0


def test_ew_add_merge_ranked_and_fallback_paths(gpu_lib):
    """The device merge-add (mpf_arith.cuh:td_add_merge_ranked) on operands
    that take every branch: magnitude-sorted (ranked merge through the
    per-thread shared-memory slots), ties across the operands with either
    sign, unsorted components (the greedy merge6 fallback), and exactly
    cancelling pairs (zero residuals: the vseb_3_6 fallback) -- bit for bit
    against the reference's td_add_merge (mpf.hpp:125-131)."""
    P = gpu_lib
    rng = np.random.default_rng(125)
    rows, cols = 64, 257
    pool = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, 0.75, 3.0, 2.0 ** -53, -2.0 ** -53, 2.0 ** -106, 2.0 ** -60])
    a = O.planes(3, rows, cols)
    b = O.planes(3, rows, cols)
    a[:, :, :cols] = rng.choice(pool, size=(3, rows, cols))
    b[:, :, :cols] = rng.choice(pool, size=(3, rows, cols))
    srt = np.argsort(-np.abs(a[:, :16, :cols]), axis=0, kind="stable")
    a[:, :16, :cols] = np.take_along_axis(a[:, :16, :cols], srt, axis=0)
    srt = np.argsort(-np.abs(b[:, :16, :cols]), axis=0, kind="stable")
    b[:, :16, :cols] = np.take_along_axis(b[:, :16, :cols], srt, axis=0)
    b[:, 16:32, :cols] = -a[:, 16:32, :cols]          # exact cancellation
    b[:, 32:40, :cols] = a[:, 32:40, :cols]           # ties with the same sign
    want = O.ref_ew(3, "add_merge", a, b, cols)
    out = P.MPMatrix(3, rows, cols)
    P.ew_apply_into(out, to_mp(a, cols), to_mp(b, cols), P.EwOp.add_merge, P.KernelVariant.SIMD_LOADSTORE)
    assert mismatches(out.data, want) == 0
