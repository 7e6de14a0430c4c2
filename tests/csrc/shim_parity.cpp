// shim_parity.cpp -- the drop-in demonstrated in C++: the reference's own
// mpfkit::linalg::MPMatrix<W> (unmodified headers from /root/reference) is
// multiplied by the reference CPU GEMM and by libmpfk through
// include/mpfk/linalg.hpp, and the results must be bits_equal
// (linalg.hpp:132-140).  Also checks the reference's exception types and
// messages come through the shim.  Exit code = number of failures.
// Usage: shim_parity [n]   (GPU required)
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

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
}  // namespace

int main(int argc, char** argv) {
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
  std::printf("%d failure(s)\n", failures);
  return failures;
}
