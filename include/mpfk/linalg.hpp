// mpfk/linalg.hpp -- C++ drop-in for the reference's matrix entry points.
//
// The reference's surface is the template API of mpfkit::linalg
// (/root/reference/proj/include/mpfkit/linalg.hpp).  This header re-exposes
// it -- same names, argument order, defaults, exception types and messages --
// over libmpfk's C ABI (include/mpfk.h), for ANY matrix class template M<W>
// with the MPMatrix<W> accessors rows(), cols(), stride(), plane(w) and an
// (rows, cols) constructor, so the reference's own
// mpfkit::linalg::MPMatrix<W> plugs in unchanged:
//
//   namespace la = mpfk::linalg;            // was: namespace la = mpfkit::linalg;
//   la::matmul_block_parallel_into(C, A, B, 32, la::KernelVariant::SIMD_LOADSTORE, 8);
//
// W is deduced from M<W> exactly as at the reference's call sites
// (linalg.hpp:368-371); the explicit form f<W>(...) is kept too.
//
//   matmul_naive[_into], matmul_block[_into],
//   matmul_block_parallel[_into]              linalg.hpp:346-443
//   matmul_strassen[_parallel]                linalg.hpp:582-617
//   ew_apply_into, ew_add, ew_mul, ew_add_merge   linalg.hpp:623-707
//   save_matrix_binary / load_matrix_binary   linalg.hpp:716-721 (linalg_io.cpp:66-111)
//   op_counters_reset / op_counters_read      linalg.hpp:160-170 (linalg.cpp:10-25)
//   gemm_into (flags BIT_EXACT / FAST / LEAN) SURVEY.md 8(b)
//
// Op counts: every call bumps libmpfk's counters (mpfk::linalg::
// op_counters_read) with the reference's semantics (count_matmul
// linalg.hpp:175-180, ew :682-683, Strassen :457/:468/:570).  When the
// matrix type is mpfkit::linalg::MPMatrix<W>, the same counts also go to the
// reference's own tally (mpfkit::linalg::detail::g_adds / g_muls /
// g_leaf_multiplies, linalg.cpp:10-11), so a switched caller reading
// mpfkit::linalg::op_counters_read() sees what the reference would have
// counted.  That needs mpfkit's linalg.cpp linked (as any use of its
// counters does); define MPFK_NO_MPFKIT_COUNTERS to opt out.
//
// Differences a caller can observe, by design:
//  * `workers` in the parallel forms counts GPUs (capped by the visible
//    devices); results stay bit-identical for any count, exactly as the
//    reference's thread count (linalg.hpp:399-401).
//  * KernelVariant only selects validation (SIMD variants need n_min % 4 == 0,
//    linalg.hpp:290-294) and, for ew_apply_into, whether out's padding is
//    rewritten (:654-680); all variants compute the same bits, as the
//    reference guarantees for its variants.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "mpfk.h"

// The reference's matrix template and op tally, declared exactly as
// mpfkit/linalg.hpp / linalg.cpp declare them (both orders of inclusion work).
namespace mpfkit::linalg {
template <int W>
class MPMatrix;
#ifndef MPFK_NO_MPFKIT_COUNTERS
namespace detail {
extern std::atomic<std::uint64_t> g_adds, g_muls, g_leaf_multiplies;
}  // namespace detail
#endif
}  // namespace mpfkit::linalg

namespace mpfk::linalg {

enum class KernelVariant { NORMAL, SIMD_SET, SIMD_LOADSTORE };  // linalg.hpp:149
enum class EwOp { add, mul, add_merge };                          // linalg.hpp:623

struct OpCounts {  // linalg.hpp:162-166
  std::uint64_t adds = 0, muls = 0, leaf_multiplies = 0;
};

inline void op_counters_reset() { mpfk_op_counters_reset(); }
inline OpCounts op_counters_read() {
  OpCounts c;
  mpfk_op_counters_read(&c.adds, &c.muls, &c.leaf_multiplies);
  return c;
}

// Page-locking of long-lived pageable operands for the lifetime of a scope
// (mpfk_host_register_cache): operands used inside are registered on first
// use and all registrations are dropped when the scope ends -- so destroy
// the matrices AFTER the scope, never inside it.
class HostRegisterScope {
 public:
  explicit HostRegisterScope(std::uint64_t capacity_bytes) { mpfk_host_register_cache(capacity_bytes); }
  ~HostRegisterScope() { mpfk_host_register_cache(0); }
  HostRegisterScope(const HostRegisterScope&) = delete;
  HostRegisterScope& operator=(const HostRegisterScope&) = delete;
};

namespace detail {

// status -> the reference's exception types (config.hpp:25-28,
// runtime.cpp:73-80, linalg.hpp:116, linalg_io.cpp's runtime_errors)
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

template <class Mat>
struct is_mpfkit_matrix : std::false_type {};
template <int W>
struct is_mpfkit_matrix<mpfkit::linalg::MPMatrix<W>> : std::true_type {};

// after a successful call: forward its op counts to the reference's own
// tally when the caller works on mpfkit matrices
template <class Mat>
void forward_counts() {
#ifndef MPFK_NO_MPFKIT_COUNTERS
  if constexpr (is_mpfkit_matrix<Mat>::value) {
    std::uint64_t a = 0, m = 0, l = 0;
    mpfk_last_op_counts(&a, &m, &l);
    mpfkit::linalg::detail::g_adds.fetch_add(a, std::memory_order_relaxed);
    mpfkit::linalg::detail::g_muls.fetch_add(m, std::memory_order_relaxed);
    mpfkit::linalg::detail::g_leaf_multiplies.fetch_add(l, std::memory_order_relaxed);
  }
#endif
}

template <class Mat>
void done(int rc) {
  throw_on(rc);
  forward_counts<Mat>();
}

template <class E>
int as_int(E e) {
  static_assert(std::is_enum_v<E>, "variant / op must be an enumeration");
  return static_cast<int>(e);
}

}  // namespace detail

// ---- GEMM: explicit-width forms f<W>(...) --------------------------------

// matmul_block_parallel_into, linalg.hpp:402-433
template <int W, class Mat, class V = KernelVariant>
void matmul_block_parallel_into(Mat& C, const Mat& A, const Mat& B, std::size_t n_min = 32,
                                V variant = V::NORMAL, unsigned workers = 1) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::done<Mat>(mpfk_matmul_block_parallel_into(W, &c, &a, &b, n_min, detail::as_int(variant), workers));
}

// matmul_block_into, linalg.hpp:368-388
template <int W, class Mat, class V = KernelVariant>
void matmul_block_into(Mat& C, const Mat& A, const Mat& B, std::size_t n_min = 32, V variant = V::NORMAL) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::done<Mat>(mpfk_matmul_block_into(W, &c, &a, &b, n_min, detail::as_int(variant)));
}

// matmul_naive_into, linalg.hpp:346-358
template <int W, class Mat, class V = KernelVariant>
void matmul_naive_into(Mat& C, const Mat& A, const Mat& B, V variant = V::NORMAL) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::done<Mat>(mpfk_matmul_naive_into(W, &c, &a, &b, detail::as_int(variant)));
}

// mpfk_gemm: the SURVEY's proposed entry point with flags.  BIT_EXACT is
// matmul_block_parallel_into on n_gpus GPUs (<= 0: all); FAST may split K
// when the output cannot fill the GPU (deterministic, within 4*k*u_p).
enum class GemmFlags : unsigned {
  BIT_EXACT = MPFK_BIT_EXACT,
  FAST = MPFK_FAST,
  LEAN = MPFK_LEAN,  // tolerance-mode arithmetic (mpfk.h); combine as GemmFlags(MPFK_FAST | MPFK_LEAN)
};

template <int W, class Mat>
void gemm_into(Mat& C, const Mat& A, const Mat& B, int n_gpus = 1, GemmFlags flags = GemmFlags::BIT_EXACT) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::done<Mat>(mpfk_gemm(W, &a, &b, &c, n_gpus, static_cast<unsigned>(flags)));
}

// value forms, linalg.hpp:360-366, 390-397, 435-443
template <int W, class Mat, class V = KernelVariant>
Mat matmul_block_parallel(const Mat& A, const Mat& B, std::size_t n_min = 32, V variant = V::NORMAL,
                          unsigned workers = 1) {
  Mat C(A.rows(), B.cols());
  matmul_block_parallel_into<W>(C, A, B, n_min, variant, workers);
  return C;
}

template <int W, class Mat, class V = KernelVariant>
Mat matmul_block(const Mat& A, const Mat& B, std::size_t n_min = 32, V variant = V::NORMAL) {
  Mat C(A.rows(), B.cols());
  matmul_block_into<W>(C, A, B, n_min, variant);
  return C;
}

template <int W, class Mat, class V = KernelVariant>
Mat matmul_naive(const Mat& A, const Mat& B, V variant = V::NORMAL) {
  Mat C(A.rows(), B.cols());
  matmul_naive_into<W>(C, A, B, variant);
  return C;
}

// matmul_strassen / matmul_strassen_parallel, linalg.hpp:582-617 (GPU top
// levels, block-GEMM leaves; bit-identical to the reference's Strassen)
template <int W, class Mat, class V = KernelVariant>
Mat matmul_strassen(const Mat& A, const Mat& B, std::size_t cutoff = 64, std::size_t n_min = 32,
                    V variant = V::NORMAL) {
  static_assert(W >= 2 && W <= 4);
  Mat C(A.rows(), B.cols());
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::done<Mat>(mpfk_matmul_strassen(W, &c, &a, &b, cutoff, n_min, detail::as_int(variant), 1));
  return C;
}

template <int W, class Mat, class V = KernelVariant>
Mat matmul_strassen_parallel(const Mat& A, const Mat& B, std::size_t cutoff = 64, std::size_t n_min = 32,
                             V variant = V::NORMAL, unsigned workers = 1) {
  static_assert(W >= 2 && W <= 4);
  Mat C(A.rows(), B.cols());
  mpfk_mat c = detail::view(C), a = detail::view(A), b = detail::view(B);
  detail::done<Mat>(mpfk_matmul_strassen(W, &c, &a, &b, cutoff, n_min, detail::as_int(variant), workers));
  return C;
}

// ---- elementwise, linalg.hpp:647-707 ---------------------------------------

template <int W, class Mat, class E, class V = KernelVariant>
void ew_apply_into(Mat& out, const Mat& a, const Mat& b, E op, V variant = V::NORMAL) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat o = detail::view(out), x = detail::view(a), y = detail::view(b);
  detail::done<Mat>(mpfk_ew_apply_into(W, detail::as_int(op), &o, &x, &y, detail::as_int(variant)));
}

template <int W, class Mat, class V = KernelVariant>
Mat ew_add(const Mat& a, const Mat& b, V variant = V::NORMAL) {
  Mat r(a.rows(), a.cols());
  ew_apply_into<W>(r, a, b, EwOp::add, variant);
  return r;
}

template <int W, class Mat, class V = KernelVariant>
Mat ew_mul(const Mat& a, const Mat& b, V variant = V::NORMAL) {
  Mat r(a.rows(), a.cols());
  ew_apply_into<W>(r, a, b, EwOp::mul, variant);
  return r;
}

// ---- MPFM binary files, linalg.hpp:716-721 ---------------------------------

template <int W, class Mat>
void save_matrix_binary(const Mat& m, const std::string& path) {
  static_assert(W >= 2 && W <= 4);
  mpfk_mat v = detail::view(m);
  detail::throw_on(mpfk_mpfm_save_host(path.c_str(), W, &v));
}

// load_matrix_binary<W>(path) returns the reference's MPMatrix<W> (the
// reference's signature); load_matrix_binary<W, M>(path) any M<W>.
template <int W, template <int> class M = mpfkit::linalg::MPMatrix>
M<W> load_matrix_binary(const std::string& path) {
  static_assert(W >= 2 && W <= 4);
  int width = 0;
  std::uint64_t rows = 0, cols = 0;
  detail::throw_on(mpfk_mpfm_info(path.c_str(), &width, &rows, &cols));
  M<W> m(rows, cols);
  mpfk_mat v = detail::view(m);
  detail::throw_on(mpfk_mpfm_load_host(path.c_str(), W, &v));
  return m;
}

// ---- the same entry points with W deduced from M<W> (reference call sites) ---

template <template <int> class M, int W, class V = KernelVariant>
void matmul_block_parallel_into(M<W>& C, const M<W>& A, const M<W>& B, std::size_t n_min = 32,
                                V variant = V::NORMAL, unsigned workers = 1) {
  matmul_block_parallel_into<W, M<W>>(C, A, B, n_min, variant, workers);
}

template <template <int> class M, int W, class V = KernelVariant>
void matmul_block_into(M<W>& C, const M<W>& A, const M<W>& B, std::size_t n_min = 32, V variant = V::NORMAL) {
  matmul_block_into<W, M<W>>(C, A, B, n_min, variant);
}

template <template <int> class M, int W, class V = KernelVariant>
void matmul_naive_into(M<W>& C, const M<W>& A, const M<W>& B, V variant = V::NORMAL) {
  matmul_naive_into<W, M<W>>(C, A, B, variant);
}

template <template <int> class M, int W>
void gemm_into(M<W>& C, const M<W>& A, const M<W>& B, int n_gpus = 1, GemmFlags flags = GemmFlags::BIT_EXACT) {
  gemm_into<W, M<W>>(C, A, B, n_gpus, flags);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> matmul_block_parallel(const M<W>& A, const M<W>& B, std::size_t n_min = 32, V variant = V::NORMAL,
                           unsigned workers = 1) {
  return matmul_block_parallel<W, M<W>>(A, B, n_min, variant, workers);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> matmul_block(const M<W>& A, const M<W>& B, std::size_t n_min = 32, V variant = V::NORMAL) {
  return matmul_block<W, M<W>>(A, B, n_min, variant);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> matmul_naive(const M<W>& A, const M<W>& B, V variant = V::NORMAL) {
  return matmul_naive<W, M<W>>(A, B, variant);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> matmul_strassen(const M<W>& A, const M<W>& B, std::size_t cutoff = 64, std::size_t n_min = 32,
                     V variant = V::NORMAL) {
  return matmul_strassen<W, M<W>>(A, B, cutoff, n_min, variant);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> matmul_strassen_parallel(const M<W>& A, const M<W>& B, std::size_t cutoff = 64, std::size_t n_min = 32,
                              V variant = V::NORMAL, unsigned workers = 1) {
  return matmul_strassen_parallel<W, M<W>>(A, B, cutoff, n_min, variant, workers);
}

template <template <int> class M, int W, class E, class V = KernelVariant>
void ew_apply_into(M<W>& out, const M<W>& a, const M<W>& b, E op, V variant = V::NORMAL) {
  ew_apply_into<W, M<W>>(out, a, b, op, variant);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> ew_add(const M<W>& a, const M<W>& b, V variant = V::NORMAL) {
  return ew_add<W, M<W>>(a, b, variant);
}

template <template <int> class M, int W, class V = KernelVariant>
M<W> ew_mul(const M<W>& a, const M<W>& b, V variant = V::NORMAL) {
  return ew_mul<W, M<W>>(a, b, variant);
}

// td_add_merge elementwise (linalg.hpp:701-707): triple width only
template <template <int> class M, class V = KernelVariant>
M<3> ew_add_merge(const M<3>& a, const M<3>& b, V variant = V::NORMAL) {
  M<3> r(a.rows(), a.cols());
  ew_apply_into<3, M<3>>(r, a, b, EwOp::add_merge, variant);
  return r;
}

template <template <int> class M, int W>
void save_matrix_binary(const M<W>& m, const std::string& path) {
  save_matrix_binary<W, M<W>>(m, path);
}

}  // namespace mpfk::linalg
