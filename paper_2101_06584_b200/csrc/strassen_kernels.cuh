// strassen_kernels.cuh -- fused, batched kernels for level-synchronous
// Strassen (see strassen.inl).
//
// Every node at one depth of the reference's recursion (linalg.hpp:565-578)
// has the same padded shape, so a whole level is processed by one launch:
//  * strassen_operands<SIDE>: from each parent operand, the 7 child operands
//    (linalg.hpp:522-540) -- quadrant windows with the +0 fill of copy_block
//    (:483-498) and the width's exact add / sub (mat_add/mat_sub, :450-470);
//  * strassen_combine: each parent's C from its 7 children's products
//    (linalg.hpp:543-563), quadrant by quadrant with clipping (:501-514).
// Element by element these are the reference's operations on the same
// values in the same order, so results are bit-identical.
#pragma once

#include <cuda_runtime.h>

#include "mpf_arith.cuh"

namespace mpfk {
namespace kern {

// W component planes per matrix; matrix b of a batch at p + b * bstride.
struct BatchRef {
  const double* p;
  long long ld, plane, bstride;
};
struct BatchOut {
  double* p;
  long long ld, plane, bstride;
};

template <int W>
__device__ __forceinline__ void load_w(const BatchRef& s, long long b, int i, int j, int rows, int cols,
                                       double* v) {
  const bool ok = i < rows && j < cols;  // outside the source: +0 (copy_block's zero fill)
#pragma unroll
  for (int w = 0; w < W; ++w) v[w] = ok ? s.p[b * s.bstride + w * s.plane + (long long)i * s.ld + j] : 0.0;
}

template <int W>
__device__ __forceinline__ void store_w(const BatchOut& d, long long b, int i, int j, const double* v) {
#pragma unroll
  for (int w = 0; w < W; ++w) d.p[b * d.bstride + w * d.plane + (long long)i * d.ld + j] = v[w];
}

template <int W>
__device__ __forceinline__ void sub_w(const double* x, const double* y, double* r) {
  double ny[W];
#pragma unroll
  for (int w = 0; w < W; ++w) ny[w] = -y[w];  // mpf::sub = add(x, neg(y)), mpf.hpp:267-272
  arith::mp_add<W>(x, ny, r);
}

// SIDE 0: A-side operands L0..L6; SIDE 1: B-side R0..R6 (linalg.hpp:532-538).
// Parent matrices rows x cols, children h0 x h1; child t of parent b is
// written to matrix b * (t1 - t0) + (t - t0) of dst.
template <int W, int SIDE>
__global__ void __launch_bounds__(256) strassen_operands(BatchRef src, BatchOut dst, int batch, int rows,
                                                         int cols, int h0, int h1, int t0, int t1) {
  const long long per = (long long)h0 * h1, total = per * batch;
  const int nt = t1 - t0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / per;
    const int i = (int)((e % per) / h1), j = (int)(e % h1);
    double q11[W], q12[W], q21[W], q22[W], r[W];
    load_w<W>(src, b, i, j, rows, cols, q11);
    load_w<W>(src, b, i, h1 + j, rows, cols, q12);
    load_w<W>(src, b, h0 + i, j, rows, cols, q21);
    load_w<W>(src, b, h0 + i, h1 + j, rows, cols, q22);
    for (int t = t0; t < t1; ++t) {
      if (SIDE == 0) {
        switch (t) {
          case 0: arith::mp_add<W>(q11, q22, r); break;  // A11 + A22
          case 1: arith::mp_add<W>(q21, q22, r); break;  // A21 + A22
          case 2: for (int w = 0; w < W; ++w) r[w] = q11[w]; break;
          case 3: for (int w = 0; w < W; ++w) r[w] = q22[w]; break;
          case 4: arith::mp_add<W>(q11, q12, r); break;  // A11 + A12
          case 5: sub_w<W>(q21, q11, r); break;          // A21 - A11
          default: sub_w<W>(q12, q22, r); break;         // A12 - A22
        }
      } else {
        switch (t) {
          case 0: arith::mp_add<W>(q11, q22, r); break;  // B11 + B22
          case 1: for (int w = 0; w < W; ++w) r[w] = q11[w]; break;
          case 2: sub_w<W>(q12, q22, r); break;          // B12 - B22
          case 3: sub_w<W>(q21, q11, r); break;          // B21 - B11
          case 4: for (int w = 0; w < W; ++w) r[w] = q22[w]; break;
          case 5: arith::mp_add<W>(q11, q12, r); break;  // B11 + B12
          default: arith::mp_add<W>(q21, q22, r); break; // B21 + B22
        }
      }
      store_w<W>(dst, b * nt + (t - t0), i, j, r);
    }
  }
}

// C (m x n) of parent b from the products M_t = child b*7+t (hm x hn).
template <int W>
__global__ void __launch_bounds__(256) strassen_combine(BatchRef M, BatchOut C, int batch, int m, int n, int hm,
                                                        int hn) {
  const long long per = (long long)m * n, total = per * batch;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / per;
    const int i = (int)((e % per) / n), j = (int)(e % n);
    const bool bot = i >= hm, right = j >= hn;
    const int li = bot ? i - hm : i, lj = right ? j - hn : j;
    const long long c0 = b * 7;
    double x[W], y[W], t1[W], t2[W], r[W];
    auto ld = [&](int t, double* v) { load_w<W>(M, c0 + t, li, lj, hm, hn, v); };
    if (!bot && !right) {  // C11 = ((M1 + M4) - M5) + M7
      ld(0, x), ld(3, y);
      arith::mp_add<W>(x, y, t1);
      ld(4, y);
      sub_w<W>(t1, y, t2);
      ld(6, y);
      arith::mp_add<W>(t2, y, r);
    } else if (!bot) {  // C12 = M3 + M5
      ld(2, x), ld(4, y);
      arith::mp_add<W>(x, y, r);
    } else if (!right) {  // C21 = M2 + M4
      ld(1, x), ld(3, y);
      arith::mp_add<W>(x, y, r);
    } else {  // C22 = ((M1 - M2) + M3) + M6
      ld(0, x), ld(1, y);
      sub_w<W>(x, y, t1);
      ld(2, y);
      arith::mp_add<W>(t1, y, t2);
      ld(5, y);
      arith::mp_add<W>(t2, y, r);
    }
    store_w<W>(C, b, i, j, r);
  }
}

}  // namespace kern
}  // namespace mpfk
