// ew_kernel.cuh -- elementwise DD/TD/QD add / mul / TD merge-add over SoA
// planes (the paper's vector benchmarks, Figs. 2-4).
//
// Replaces linalg::ew_apply_into (linalg.hpp:623-684): out(i,j) =
// op(a(i,j), b(i,j)) with op = mpf::add<W> / mpf::mul<W> (mpf.hpp:242-260) or
// td_add_merge (mpf.hpp:125-131).  HBM-bound: 3*W*8 bytes per element against
// 20-133 FP64 operations, so the kernel streams all W planes with 16-byte
// loads (two adjacent elements per thread; the reference layout's pad4
// strides keep pairs inside a row) and a grid-stride loop sized to the SM
// count.
#pragma once

#include <cuda_runtime.h>

#include "mpf_arith.cuh"

namespace mpfk {

namespace kern {

// linalg.hpp:623; EW_SUB is internal (mat_sub of the Strassen plumbing,
// linalg.hpp:461-470: mpf::sub = add(x, neg(y)), mpf.hpp:267-272)
enum EwOp { EW_ADD = 0, EW_MUL = 1, EW_ADD_MERGE = 2, EW_SUB = 3 };

struct EwArgs {
  double* out;
  const double* a;
  const double* b;
  long long ldo, lda, ldb;  // row strides (even)
  long long po, pa, pb;     // plane strides
  int rows, cols;  // only the rows x cols cells of `out` are written
};

template <int W, int OP>
__device__ __forceinline__ void ew_one(const double* x, const double* y, double* r, double* zb) {
  if constexpr (OP == EW_SUB) {
    double ny[W];
#pragma unroll
    for (int w = 0; w < W; ++w) ny[w] = -y[w];  // exact sign flip (Ops::neg, eft.hpp:126)
    arith::mp_add<W>(x, ny, r);
  } else if constexpr (OP == EW_MUL) arith::mp_mul<W>(x, y, r);
  else if constexpr (OP == EW_ADD_MERGE && W == 3) arith::td_add_merge_ranked(x, y, r, zb, 256);
  else arith::mp_add<W>(x, y, r);
}

// one thread = two adjacent columns (j, j+1), j even
template <int W, int OP>
__global__ void __launch_bounds__(256) ew_kernel(const EwArgs g) {
  // merge-add: per-thread scatter slots for the ranked merge (slot k of
  // thread t at zbuf[k * 256 + t]: conflict-free for any slot pattern)
  __shared__ double zbuf[OP == EW_ADD_MERGE ? 6 * 256 : 1];
  double* zb = zbuf + (OP == EW_ADD_MERGE ? threadIdx.x : 0);
  const int half = (g.cols + 1) / 2;
  const long long total = (long long)g.rows * half;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / half);
    const int j = 2 * (int)(t % half);
    double x0[W], x1[W], y0[W], y1[W], r0[W], r1[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const double2 av = __ldcs(reinterpret_cast<const double2*>(g.a + w * g.pa + i * g.lda + j));
      const double2 bv = __ldcs(reinterpret_cast<const double2*>(g.b + w * g.pb + i * g.ldb + j));
      x0[w] = av.x, x1[w] = av.y, y0[w] = bv.x, y1[w] = bv.y;
    }
    ew_one<W, OP>(x0, y0, r0, zb);
    const bool second = j + 1 < g.cols;
    if (second) ew_one<W, OP>(x1, y1, r1, zb);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      double* o = g.out + w * g.po + i * g.ldo + j;
      if (second) {
        __stcs(reinterpret_cast<double2*>(o), make_double2(r0[w], r1[w]));
      } else {
        o[0] = r0[w];
      }
    }
  }
}

}  // namespace kern
}  // namespace mpfk
