// mpfk/linalg.hpp -- C++ drop-in for the reference's GEMM entry points.
//
// The reference's surface is the template API of mpfkit::linalg
// (/root/reference/proj/include/mpfkit/linalg.hpp:346-443).  This header
// re-exposes the same entry points -- same names, argument order, defaults,
// exception types and messages -- over libmpfk's C ABI (include/mpfk.h),
// for ANY matrix type with the MPMatrix<W> accessors rows(), cols(),
// stride(), plane(w) (so the reference's own mpfkit::linalg::MPMatrix<W>
// plugs in unchanged, see tests/csrc/shim_parity.cpp).
//
// Differences a caller can observe, by design:
//  * `workers` in matmul_block_parallel[_into] counts GPUs (capped by the
//    visible devices); results stay bit-identical for any count, exactly as
//    the reference's thread count (linalg.hpp:399-401).
//  * KernelVariant only selects validation (SIMD variants need n_min % 4 == 0,
//    linalg.hpp:290-294); all variants run the same GPU kernel and give the
//    same bits, as the reference guarantees for its variants.
//  * Op counters live in libmpfk (mpfk::linalg::op_counters_read).
#pragma once

#include <cstddef>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "mpfk.h"

namespace mpfk::linalg {

enum class KernelVariant { NORMAL, SIMD_SET, SIMD_LOADSTORE };  // linalg.hpp:149

struct OpCounts {  // linalg.hpp:162-166
  std::uint64_t adds = 0, muls = 0, leaf_multiplies = 0;
};

inline void op_counters_reset() { mpfk_op_counters_reset(); }
inline OpCounts op_counters_read() {
  OpCounts c;
  mpfk_op_counters_read(&c.adds, &c.muls, &c.leaf_multiplies);
  return c;
}

namespace detail {

// status -> the reference's exception types (config.hpp:25-28,
// runtime.cpp:73-80, linalg.hpp:116)
inline void throw_on(int rc) {
  if (rc == MPFK_OK) return;
  const std::string msg = mpfk_last_error();
  switch (rc) {
    case MPFK_EINVAL: throw std::invalid_argument(msg);
    case MPFK_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

template <class Mat>
mpfk_mat view(const Mat& m) {
  mpfk_mat v;
  v.base = m.rows() && m.cols() ? const_cast<double*>(m.plane(0)) : nullptr;
  v.rows = m.rows();
  v.cols = m.cols();
  v.stride = m.stride();
  v.plane_stride = m.rows() * m.stride();
  return v;
}

}  // namespace detail

// matmul_block_parallel_into, linalg.hpp:402-433
template <int W, class Mat>
void matmul_block_parallel_into(Mat& C, const Mat& A, const Mat& B, std::size_t n_min = 32,
                                KernelVariant variant = KernelVariant::NORMAL,
                                unsigned workers = 1) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::throw_on(mpfk_matmul_block_parallel_into(W, &c, &a, &b, n_min, static_cast<int>(variant),
                                                   workers));
}

// matmul_block_into, linalg.hpp:368-388
template <int W, class Mat>
void matmul_block_into(Mat& C, const Mat& A, const Mat& B, std::size_t n_min = 32,
                       KernelVariant variant = KernelVariant::NORMAL) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::throw_on(mpfk_matmul_block_into(W, &c, &a, &b, n_min, static_cast<int>(variant)));
}

// matmul_naive_into, linalg.hpp:346-358
template <int W, class Mat>
void matmul_naive_into(Mat& C, const Mat& A, const Mat& B,
                       KernelVariant variant = KernelVariant::NORMAL) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::throw_on(mpfk_matmul_naive_into(W, &c, &a, &b, static_cast<int>(variant)));
}

// mpfk_gemm: the SURVEY's proposed entry point with flags.  BIT_EXACT is
// matmul_block_parallel_into on n_gpus GPUs (<= 0: all); FAST may split K
// when the output cannot fill the GPU (deterministic, within 4*k*u_p).
enum class GemmFlags : unsigned { BIT_EXACT = MPFK_BIT_EXACT, FAST = MPFK_FAST };

template <int W, class Mat>
void gemm_into(Mat& C, const Mat& A, const Mat& B, int n_gpus = 1, GemmFlags flags = GemmFlags::BIT_EXACT) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::throw_on(mpfk_gemm(W, &a, &b, &c, n_gpus, static_cast<unsigned>(flags)));
}

// value forms, linalg.hpp:360-366, 390-397, 435-443
template <int W, class Mat>
Mat matmul_block_parallel(const Mat& A, const Mat& B, std::size_t n_min = 32,
                          KernelVariant variant = KernelVariant::NORMAL, unsigned workers = 1) {
  Mat C(A.rows(), B.cols());
  matmul_block_parallel_into<W>(C, A, B, n_min, variant, workers);
  return C;
}

template <int W, class Mat>
Mat matmul_block(const Mat& A, const Mat& B, std::size_t n_min = 32,
                 KernelVariant variant = KernelVariant::NORMAL) {
  Mat C(A.rows(), B.cols());
  matmul_block_into<W>(C, A, B, n_min, variant);
  return C;
}

template <int W, class Mat>
Mat matmul_naive(const Mat& A, const Mat& B, KernelVariant variant = KernelVariant::NORMAL) {
  Mat C(A.rows(), B.cols());
  matmul_naive_into<W>(C, A, B, variant);
  return C;
}

}  // namespace mpfk::linalg
