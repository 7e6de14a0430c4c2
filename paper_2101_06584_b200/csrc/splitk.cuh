// splitk.cuh -- MPFK_FAST: split-K combine for products whose output is too
// small to fill the GPU ("flags selects BIT_EXACT (default)
// or FAST (reordered, tolerance-checked)").
//
// The bit-exact GEMM keeps the reference's per-element order (one chain
// over ascending k, linalg.hpp:338-344), so an m x n output has only
// ceil(m/BM)*ceil(n/BN) independent tiles.  FAST cuts K into S segments, runs
// each segment as its own reference-order chain (one batched launch of the
// same GEMM kernel, the ragged last segment through GemmArgs::klast), and
// folds the S partial products here in a fixed order:
//   C = ((P_0 + P_1) + P_2) + ... + P_{S-1}     (mpf::add<W>, mpf.hpp:242-260)
// Deterministic for a given (m, n, k, S); not bit-identical to the reference
// (a different summation order), so it is tolerance-checked instead: the
// normwise relative error stays within the north star's 4*k*u_p.
#pragma once

#include <cuda_runtime.h>

#include "mpf_arith.cuh"

namespace mpfk {
namespace kern {

// part: S partial products, partial s at part + s*sw, W planes of pw doubles,
// row stride ldw.  One thread per output element, consecutive threads on
// consecutive columns (coalesced across every partial and plane).
template <int W>
__global__ void __launch_bounds__(256)
    splitk_reduce_kernel(const double* __restrict__ part, long long ldw, long long pw, long long sw, int S,
                         double* __restrict__ C, long long ldc, long long pc, int M, int N) {
  const long long total = (long long)M * N;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / N), j = (int)(t % N);
    const double* p = part + (long long)i * ldw + j;
    double acc[W], x[W], r[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = __ldcs(p + w * pw);
#pragma unroll 4
    for (int s = 1; s < S; ++s) {
#pragma unroll
      for (int w = 0; w < W; ++w) x[w] = __ldcs(p + s * sw + w * pw);
      arith::mp_add<W>(acc, x, r);
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] = r[w];
    }
#pragma unroll
    for (int w = 0; w < W; ++w) C[w * pc + (long long)i * ldc + j] = acc[w];
  }
}

}  // namespace kern
}  // namespace mpfk
