"""Generate the golden GEMM fixtures from the REFERENCE build (oracle/_ref:
the unmodified mpfkit compiled from /root/reference/proj).  Run here, where
the reference exists; the .npz files are committed so the tests can check the
oracle and the GPU kernel against reference outputs on any box.

  python tests/golden/make_golden.py

Each fixture: A (W, m, lda), B (W, k, ldb), C = reference
matmul_block_parallel_into(A, B, n_min=32, SIMD_LOADSTORE) (W, m, ldc),
with W, m, k, n scalars and a description.  Inputs follow the reference's
own test generators (bench::fill_random, random_signed of test_linalg.cpp,
gen_paper_matrices) and the BASELINE.json distributions.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from tests.helpers import random_signed, special_matrix  # noqa: E402


def save(name, W, A, B, k, n, desc):
    C = O.ref_gemm(A, B, k, n, workers=4)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), A=A, B=B, C=C, W=W, m=A.shape[1], k=k, n=n,
                        desc=desc)
    print(name, A.shape, B.shape, desc)


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle)"
    for W in (2, 3, 4):
        p = {2: "dd", 3: "td", 4: "qd"}[W]
        save(f"{p}_fill_random_n8", W, O.ref_fill_random(W, 8, 8, 4000 + 10 * W + 8),
             O.ref_fill_random(W, 8, 8, 4001 + 10 * W + 8), 8, 8,
             "acceptance.cpp criterion 4 inputs (bench::fill_random), n=8")
        save(f"{p}_signed_rect_7x12x9", W, random_signed(W, 7, 12, 460), random_signed(W, 12, 9, 461), 12, 9,
             "test_linalg.cpp:242-247 rectangular shape, random_signed-style inputs")
        A, B = O.ref_gen_paper(W, 16)
        save(f"{p}_paper_n16", W, A, B, 16, 16, "bench::gen_paper_matrices n=16 (renorm5 paths B/C/D)")
        save(f"{p}_special_13x11x10", W, special_matrix(W, 13, 11, 31), special_matrix(W, 11, 10, 32), 11, 10,
             "signed zeros, integers, powers of two: zero-residual corners")
        wide = W > 2
        save(f"{p}_baseline_{'wide' if wide else 'narrow'}_n12", W, O.orc_fill_baseline(W, 12, 12, 1, wide),
             O.orc_fill_baseline(W, 12, 12, 2, wide), 12, 12, "BASELINE.json distribution, n=12")


if __name__ == "__main__":
    main()
