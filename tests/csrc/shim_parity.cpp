// shim_parity.cpp -- the drop-in demonstrated in C++: the reference's own
// mpfkit::linalg::MPMatrix<W> (unmodified headers from /root/reference) is
// multiplied by the reference CPU GEMM and by libmpfk through
// include/mpfk/linalg.hpp, and the results must be bits_equal
// (linalg.hpp:132-140).  Also checks the reference's exception types and
// messages come through the shim.  Exit code = number of failures.
// Usage: shim_parity [n]   (GPU required)
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <unistd.h>

#include "mpfk/linalg.hpp"
#include "mpfkit/linalg.hpp"
#include "mpfkit/random.hpp"

using namespace mpfkit;

namespace {
int failures = 0;

void verdict(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

template <int W>
linalg::MPMatrix<W> fill(std::size_t r, std::size_t c, std::uint64_t seed) {
  rng::SplitMix64 g(seed);
  linalg::MPMatrix<W> m(r, c);
  for (std::size_t i = 0; i < r; ++i)
    for (std::size_t j = 0; j < c; ++j) m.set(i, j, rng::random_normalized_signed<W>(g));
  return m;
}

template <int W>
void run(std::size_t m, std::size_t k, std::size_t n) {
  const auto A = fill<W>(m, k, 100 + W);
  const auto B = fill<W>(k, n, 200 + W);
  const auto ref = linalg::matmul_block_parallel(A, B, 32, linalg::KernelVariant::SIMD_LOADSTORE, 8);
  const auto gpu = mpfk::linalg::matmul_block<W>(A, B, 32, mpfk::linalg::KernelVariant::SIMD_LOADSTORE);
  verdict(linalg::bits_equal(ref, gpu), "W=" + std::to_string(W) + " " + std::to_string(m) + "x" +
                                            std::to_string(k) + "x" + std::to_string(n) + " bits_equal");
  linalg::MPMatrix<W> C(m, n);
  C.set(0, 0, mpf::from_f64<W>(42.0));  // stale contents must be cleared
  mpfk::linalg::matmul_block_parallel_into<W>(C, A, B, 32, mpfk::linalg::KernelVariant::NORMAL, 4);
  verdict(linalg::bits_equal(ref, C), "W=" + std::to_string(W) + " _into clears stale C, workers=4");
  linalg::MPMatrix<W> G(m, n);
  mpfk::linalg::gemm_into<W>(G, A, B, 1, mpfk::linalg::GemmFlags::BIT_EXACT);
  verdict(linalg::bits_equal(ref, G), "W=" + std::to_string(W) + " gemm_into BIT_EXACT");
  mpfk::linalg::gemm_into<W>(G, A, B, 1, mpfk::linalg::GemmFlags::FAST);
  verdict(G.rows() == m && G.cols() == n, "W=" + std::to_string(W) + " gemm_into FAST runs");
  // MPFK_LEAN, the tolerance mode: not the reference's bits, but within the
  // north star's normwise 4*k*u_p of them (the component differences summed
  // from the smallest up: the leading ones cancel exactly where both agree)
  mpfk::linalg::gemm_into<W>(G, A, B, 1, mpfk::linalg::GemmFlags::LEAN);
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      double d = 0.0;
      for (int w = W - 1; w >= 0; --w) d += G.plane(w)[i * G.stride() + j] - ref.plane(w)[i * ref.stride() + j];
      num = std::max(num, std::fabs(d));
      den = std::max(den, std::fabs(ref.plane(0)[i * ref.stride() + j]));
    }
  const double u_p = W == 2 ? 0x1p-104 : (W == 3 ? 0x1p-156 : 0x1p-208);
  verdict(num <= 4.0 * double(k) * u_p * den,
          "W=" + std::to_string(W) + " gemm_into LEAN within 4*k*u_p of the reference");
}

template <class F>
void expect_throw(F&& f, const std::string& msg) {
  try {
    f();
    verdict(false, "expected std::invalid_argument: " + msg);
  } catch (const std::invalid_argument& e) {
    verdict(std::string(e.what()) == msg, "invalid_argument \"" + std::string(e.what()) + "\"");
  }
}

// ---- the namespace switch: reference call sites compiled against the shim
// by swapping one alias (W deduced from MPMatrix<W>, linalg.hpp:368-371),
// each result bits_equal to the reference's and each call's op counts landing
// in the reference's own tally (mpfkit::linalg::op_counters_read,
// linalg.cpp:13-25) exactly as the reference counts them.
namespace ref = mpfkit::linalg;
namespace la = mpfk::linalg;

template <class F, class G>
void same_counts(F&& ref_call, G&& shim_call, const std::string& what) {
  ref::op_counters_reset();
  ref_call();
  const auto r = ref::op_counters_read();
  ref::op_counters_reset();
  shim_call();
  const auto s = ref::op_counters_read();
  verdict(r.adds == s.adds && r.muls == s.muls && r.leaf_multiplies == s.leaf_multiplies,
          what + " op counts (adds " + std::to_string(s.adds) + "/" + std::to_string(r.adds) + ", muls " +
              std::to_string(s.muls) + "/" + std::to_string(r.muls) + ", leaves " +
              std::to_string(s.leaf_multiplies) + "/" + std::to_string(r.leaf_multiplies) + ")");
}

template <int W>
void drop_in(std::size_t m, std::size_t k, std::size_t n) {
  const std::string tag = "switch W=" + std::to_string(W) + " ";
  const auto A = fill<W>(m, k, 300 + W);
  const auto B = fill<W>(k, n, 400 + W);
  // block GEMM, all forms, W deduced
  ref::MPMatrix<W> Cr(m, n), Cs(m, n);
  same_counts([&] { ref::matmul_block_parallel_into(Cr, A, B, 32, ref::KernelVariant::SIMD_LOADSTORE, 8); },
              [&] { la::matmul_block_parallel_into(Cs, A, B, 32, la::KernelVariant::SIMD_LOADSTORE, 8); },
              tag + "matmul_block_parallel_into");
  verdict(ref::bits_equal(Cr, Cs), tag + "matmul_block_parallel_into bits_equal");
  verdict(ref::bits_equal(Cr, la::matmul_block(A, B)), tag + "matmul_block bits_equal");
  verdict(ref::bits_equal(Cr, la::matmul_naive(A, B)), tag + "matmul_naive bits_equal");
  verdict(ref::bits_equal(Cr, la::matmul_block_parallel(A, B, 16, la::KernelVariant::NORMAL, 3)),
          tag + "matmul_block_parallel bits_equal");
  // the reference's own enum passes through too
  ref::MPMatrix<W> Ce(m, n);
  la::matmul_block_into(Ce, A, B, 32, ref::KernelVariant::SIMD_SET);
  verdict(ref::bits_equal(Cr, Ce), tag + "matmul_block_into(reference KernelVariant) bits_equal");
  // Strassen (a different algorithm: compared with the reference's Strassen)
  ref::MPMatrix<W> Sr, Ss;
  same_counts([&] { Sr = ref::matmul_strassen(A, B, 16, 8); }, [&] { Ss = la::matmul_strassen(A, B, 16, 8); },
              tag + "matmul_strassen");
  verdict(ref::bits_equal(Sr, Ss), tag + "matmul_strassen bits_equal");
  const auto Sp = la::matmul_strassen_parallel(A, B, 16, 8, la::KernelVariant::NORMAL, 4);
  verdict(ref::bits_equal(ref::matmul_strassen_parallel(A, B, 16, 8, ref::KernelVariant::NORMAL, 4), Sp),
          tag + "matmul_strassen_parallel bits_equal");
  // elementwise
  const auto X = fill<W>(m, n, 500 + W), Y = fill<W>(m, n, 600 + W);
  ref::MPMatrix<W> Er, Es;
  same_counts([&] { Er = ref::ew_add(X, Y); }, [&] { Es = la::ew_add(X, Y); }, tag + "ew_add");
  verdict(ref::bits_equal(Er, Es), tag + "ew_add bits_equal");
  same_counts([&] { Er = ref::ew_mul(X, Y, ref::KernelVariant::SIMD_LOADSTORE); },
              [&] { Es = la::ew_mul(X, Y, la::KernelVariant::SIMD_LOADSTORE); }, tag + "ew_mul");
  verdict(ref::bits_equal(Er, Es), tag + "ew_mul bits_equal");
  ref::MPMatrix<W> Or(m, n), Os(m, n);
  ref::ew_apply_into(Or, X, Y, ref::EwOp::add, ref::KernelVariant::SIMD_SET);
  la::ew_apply_into(Os, X, Y, la::EwOp::add, la::KernelVariant::SIMD_SET);
  verdict(ref::bits_equal(Or, Os), tag + "ew_apply_into bits_equal");
  if constexpr (W == 3) {
    verdict(ref::bits_equal(ref::ew_add_merge(X, Y), la::ew_add_merge(X, Y)), tag + "ew_add_merge bits_equal");
  }
  // the reference's own aligned_alloc'ed buffers page-locked for a scope
  // (exact operand spans, mpfk_host_register_cache): same bits, registered
  {
    la::HostRegisterScope pin(std::uint64_t(1) << 30);
    ref::MPMatrix<W> Cp(m, n);
    la::matmul_block_parallel_into(Cp, A, B, 32, la::KernelVariant::SIMD_LOADSTORE, 1);
    la::matmul_block_parallel_into(Cp, A, B, 32, la::KernelVariant::SIMD_LOADSTORE, 1);
    std::uint64_t cap = 0, used = 0, ents = 0;
    mpfk_host_register_cache_stats(&cap, &used, &ents);
    const bool big = sizeof(double) * W * m * A.stride() >= (std::size_t(1) << 20);
    verdict(ref::bits_equal(Cr, Cp) && (!big || ents >= 1),
            tag + "page-locked reference buffers (" + std::to_string(ents) + " registered) bits_equal");
    mpfk_host_unregister(Cp.plane(0));
  }
  // MPFM round trip through the shim (the reference's linalg_io.cpp needs Boost)
  const std::string path = "/tmp/shim_parity_" + std::to_string(getpid()) + "_" + std::to_string(W) + ".mpfm";
  la::save_matrix_binary(Cr, path);
  const auto L = la::load_matrix_binary<W>(path);
  verdict(ref::bits_equal(Cr, L), tag + "save/load_matrix_binary round trip");
  std::remove(path.c_str());
}

void drop_in_errors() {
  ref::MPMatrix<2> a(3, 4), b(5, 2), c(3, 2);
  expect_throw([&] { la::matmul_block_into(c, a, b); }, "matmul: inner dimensions differ");
  expect_throw([&] { (void)la::matmul_strassen(a, ref::MPMatrix<2>(4, 2), 0); }, "matmul: cutoff must be at least 1");
  expect_throw([&] { (void)la::ew_add(a, c); }, "ew: shape mismatch");
  try {
    (void)la::load_matrix_binary<2>("/nonexistent/shim.mpfm");
    verdict(false, "load_matrix_binary of a missing file throws");
  } catch (const std::runtime_error& e) {
    verdict(std::string(e.what()).find("cannot open") != std::string::npos,
            std::string("load_matrix_binary runtime_error \"") + e.what() + "\"");
  }
  verdict(mpfk_selftest() == MPFK_OK, "mpfk_selftest() == MPFK_OK on this GPU");
}
}  // namespace

// --selftest-error (run with MPFK_SELFTEST_INJECT=fma): the device self-test
// failure reaches a shim caller as std::runtime_error (runtime.cpp:73-80)
int selftest_error() {
  ref::MPMatrix<2> a(4, 4), b(4, 4);
  try {
    (void)la::matmul_block(a, b);
    verdict(false, "std::runtime_error expected from a failed device self-test");
  } catch (const std::runtime_error& e) {
    verdict(std::string(e.what()).find("fused multiply-add") != std::string::npos,
            std::string("std::runtime_error \"") + e.what() + "\"");
  } catch (...) {
    verdict(false, "wrong exception type from a failed device self-test");
  }
  return failures;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--selftest-error") return selftest_error();
  const std::size_t n = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 97;
  run<2>(n, n + 3, n - 5);
  run<3>(n, n, n);
  run<4>(33, 17, 9);
  linalg::MPMatrix<2> a(3, 4), b(5, 2), c(3, 2), ok_b(4, 2);
  expect_throw([&] { mpfk::linalg::matmul_block_into<2>(c, a, b); }, "matmul: inner dimensions differ");
  expect_throw([&] { mpfk::linalg::matmul_block_into<2>(a, a, ok_b); }, "matmul: result shape mismatch");
  expect_throw([&] { mpfk::linalg::matmul_block_into<2>(c, a, ok_b, 5, mpfk::linalg::KernelVariant::SIMD_SET); },
               "matmul: SIMD variants need n_min divisible by 4");
  expect_throw([&] { mpfk::linalg::matmul_block_into<2>(c, a, ok_b, 0); }, "matmul: n_min must be at least 1");
  expect_throw([&] { mpfk::linalg::matmul_block_parallel_into<2>(c, a, ok_b, 32, mpfk::linalg::KernelVariant::NORMAL, 0); },
               "matmul: workers must be at least 1");
  drop_in<2>(n, n + 3, n - 5);
  drop_in<2>(600, 512, 600);  // operands >= 1 MiB: the registration cache engages
  drop_in<3>(70, 45, 50);
  drop_in<4>(33, 40, 36);
  drop_in_errors();
  std::printf("%d failure(s)\n", failures);
  return failures;
}
