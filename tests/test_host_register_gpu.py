"""Opt-in page-locking of long-lived pageable operands
(mpfk_host_register_cache): pageable MPMatrix buffers -- what a reference
caller passes (aligned_alloc, linalg.hpp:115) -- are cudaHostRegister'ed on
first use and take the page-locked paths afterwards.  Results stay
bit-identical to the staging path; the set is bounded (LRU) and empties on
request."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,n", [(2, 1024), (3, 300), (4, 257)])
def test_registered_operands_bit_identical(gpu_lib, W, n):
    P = gpu_lib
    A = P.fill_baseline(W, n, n, 1)
    B = P.fill_baseline(W, n, n, 2)
    want = P.matmul_block(A, B)  # staging path (cache off)
    P.host_register_cache(1 << 30)
    try:
        for _ in range(3):  # first call registers, later calls reuse
            C = P.MPMatrix(W, n, n)
            P.matmul_block_parallel_into(C, A, B, 32, P.KernelVariant.SIMD_LOADSTORE, 1)
            assert P.bits_equal(C, want)
            P.host_unregister(C)
        st = P.host_register_cache_stats()
        # A and B stay registered: each exactly its span, first cell to the
        # last cell of its last plane
        span = 8 * ((W * n - 1) * P.pad_columns(n) + n)
        assert st["entries"] >= 2 and st["used"] >= 2 * span
    finally:
        P.host_register_cache(0)
    assert P.host_register_cache_stats()["entries"] == 0


def test_cache_is_bounded_lru(gpu_lib):
    P = gpu_lib
    W, n = 2, 512
    bytes_one = 8 * ((W * n - 1) * P.pad_columns(n) + n)  # the registered span of one operand
    mats = [P.fill_baseline(W, n, n, s) for s in range(4)]
    C = P.MPMatrix(W, n, n)
    P.host_register_cache(3 * bytes_one)
    try:
        P.matmul_block_into(C, mats[0], mats[1])  # registers A, B, C: full
        assert P.host_register_cache_stats()["entries"] == 3
        P.matmul_block_into(C, mats[2], mats[3])  # evicts the two oldest
        st = P.host_register_cache_stats()
        assert st["entries"] == 3 and st["used"] <= 3 * bytes_one
        want = P.MPMatrix(W, n, n)
        P.host_register_cache(0)
        P.matmul_block_into(want, mats[2], mats[3])
        assert P.bits_equal(C, want)
    finally:
        P.host_register_cache(0)


def test_small_operands_stay_on_the_staging_path(gpu_lib):
    P = gpu_lib
    P.host_register_cache(1 << 30)
    try:
        A = P.fill_baseline(2, 64, 64, 1)
        C = P.matmul_block(A, A)
        assert P.host_register_cache_stats()["entries"] == 0  # < 1 MiB each
        assert C.rows() == 64
    finally:
        P.host_register_cache(0)
