// ref_driver.cpp -- a C-ABI shim over the UNMODIFIED reference (mpfkit).
//
// TEST INFRASTRUCTURE ONLY (the checker and the reported CPU baseline; never
// the shipped path).  Compiled by oracle/Makefile together with the
// reference's own proj/src/runtime.cpp and proj/src/linalg.cpp, straight from
// where they lie under /root/reference, into oracle/_ref/libmpfkref.so.  No
// reference source is copied into this repository.
//
// Every entry point only marshals plain SoA arrays into mpfkit types and
// calls the reference's public API:
//   ref_gemm        -> mpfkit::linalg::matmul_block_parallel_into (linalg.hpp:402-433),
//                      or matmul_naive_into (linalg.hpp:346-358) with naive != 0
//   ref_strassen    -> matmul_strassen[_parallel]                  (linalg.hpp:582-617)
//   ref_ew          -> linalg::ew_apply_into                       (linalg.hpp:647-684)
//   ref_add/ref_mul -> mpfkit::mpf::add/mul<W>                    (mpf.hpp:341-353)
//   ref_fill_random -> the loop of bench::fill_random (bench.cpp:295-302) over
//                      rng::random_normalized<W> (random.hpp:54-67); bench.cpp
//                      itself needs Boost, which this image lacks
//   ref_gen_paper   -> the loop of bench::gen_paper_matrices (bench.cpp:278-292)
//   ref_renorm5 / ref_vseb / ref_two_* -> mpfkit::eft (eft.hpp)
//   ref_op_counts   -> linalg::op_counters_read (linalg.cpp:13-25)
//   ref_prep_*      -> matmul_block_parallel_into on operands built once,
//                      timed inside C++ (the reported CPU baseline)
// Errors: reference exceptions become a nonzero return and a message in
// ref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>

#include "mpfkit/linalg.hpp"
#include "mpfkit/random.hpp"
#include "mpfkit/runtime.hpp"

using namespace mpfkit;

namespace {
thread_local std::string g_err;

template <int W>
linalg::MPMatrix<W> load(const double* planes, std::size_t rows, std::size_t cols,
                         std::size_t ld) {
  linalg::MPMatrix<W> m(rows, cols);
  const std::size_t ps = rows * ld;
  for (int w = 0; w < W; ++w)
    for (std::size_t i = 0; i < rows; ++i)
      std::memcpy(m.plane(w) + i * m.stride(), planes + w * ps + i * ld,
                  cols * sizeof(double));
  return m;
}

template <int W>
void store(const linalg::MPMatrix<W>& m, double* planes, std::size_t ld) {
  const std::size_t ps = m.rows() * ld;
  for (int w = 0; w < W; ++w)
    for (std::size_t i = 0; i < m.rows(); ++i)
      std::memcpy(planes + w * ps + i * ld, m.plane(w) + i * m.stride(),
                  m.cols() * sizeof(double));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <int W>
int gemm_w(std::size_t m, std::size_t K, std::size_t n, const double* A, std::size_t lda,
           const double* B, std::size_t ldb, double* C, std::size_t ldc, std::size_t n_min,
           int variant, unsigned workers, int naive, int c_rows, int c_cols) {
  return guarded([&] {
    const auto a = load<W>(A, m, K, lda);
    const auto b = load<W>(B, K, n, ldb);
    linalg::MPMatrix<W> c(c_rows < 0 ? m : static_cast<std::size_t>(c_rows),
                          c_cols < 0 ? n : static_cast<std::size_t>(c_cols));
    const auto v = static_cast<linalg::KernelVariant>(variant);
    if (naive)
      linalg::matmul_naive_into(c, a, b, v);
    else
      linalg::matmul_block_parallel_into(c, a, b, n_min, v, workers);
    store<W>(c, C, ldc);
  });
}

template <int W>
void fill_random_w(std::size_t rows, std::size_t cols, std::uint64_t seed, double* planes,
                   std::size_t ld) {
  rng::SplitMix64 g(seed);
  std::memset(planes, 0, sizeof(double) * W * rows * ld);
  for (std::size_t i = 0; i < rows; ++i)
    for (std::size_t j = 0; j < cols; ++j) {
      const auto v = rng::random_normalized<W>(g);
      for (int w = 0; w < W; ++w) planes[w * rows * ld + i * ld + j] = v.c[w];
    }
}

template <int W>
void gen_paper_w(std::size_t n, double* A, double* B, std::size_t ld) {
  std::memset(A, 0, sizeof(double) * W * n * ld);
  std::memset(B, 0, sizeof(double) * W * n * ld);
  const auto r5 = mpf::from_f64<W>(std::sqrt(5.0));
  const auto r3 = mpf::from_f64<W>(std::sqrt(3.0));
  for (std::size_t i = 1; i <= n; ++i) {
    const auto brow = mpf::mul(r3, mpf::from_f64<W>(static_cast<double>(n - i)));
    for (std::size_t j = 1; j <= n; ++j) {
      const auto a = mpf::mul(r5, mpf::from_f64<W>(static_cast<double>(i + j - 1)));
      for (int w = 0; w < W; ++w) {
        A[w * n * ld + (i - 1) * ld + (j - 1)] = a.c[w];
        B[w * n * ld + (i - 1) * ld + (j - 1)] = brow.c[w];
      }
    }
  }
}

template <int W>
int ew_w(int op, int variant, std::size_t rows, std::size_t cols, const double* a, std::size_t lda,
         const double* b, std::size_t ldb, double* out, std::size_t ldo) {
  return guarded([&] {
    const auto x = load<W>(a, rows, cols, lda);
    const auto y = load<W>(b, rows, cols, ldb);
    linalg::MPMatrix<W> o(rows, cols);
    linalg::ew_apply_into(o, x, y, static_cast<linalg::EwOp>(op),
                          static_cast<linalg::KernelVariant>(variant));
    store<W>(o, out, ldo);
  });
}

template <int W>
void binop_w(int op, const double* x, const double* y, double* r) {
  mpf::MultiDouble<W> a, b;
  for (int w = 0; w < W; ++w) a.c[w] = x[w], b.c[w] = y[w];
  const auto c = op == 0 ? mpf::add(a, b) : mpf::mul(a, b);
  for (int w = 0; w < W; ++w) r[w] = c.c[w];
}


// ---- prepared operands for the timed CPU baseline (bench.py --impl reference)
// The reference MPMatrix objects are built ONCE (outside any timing); each
// ref_prep_run() then times exactly one mpfkit::linalg::
// matmul_block_parallel_into call (linalg.hpp:402-433) with steady_clock,
// the way bench::time_matmul times its repetitions (bench.cpp:33-38).
struct PrepBase {
  virtual ~PrepBase() = default;
  virtual void run(std::size_t n_min, int variant, unsigned workers) = 0;
  virtual void result(double* C, std::size_t ldc) const = 0;
  virtual PrepBase* with_a(std::size_t m, const double* A, std::size_t lda) const = 0;
};

template <int W>
struct Prep final : PrepBase {
  linalg::MPMatrix<W> a;
  std::shared_ptr<const linalg::MPMatrix<W>> b;  // shared by handles made with with_a()
  linalg::MPMatrix<W> c;
  Prep(std::size_t m, std::size_t K, const double* A, std::size_t lda,
       std::shared_ptr<const linalg::MPMatrix<W>> bm)
      : a(load<W>(A, m, K, lda)), b(std::move(bm)), c(m, b->cols()) {}
  void run(std::size_t n_min, int variant, unsigned workers) override {
    linalg::matmul_block_parallel_into(c, a, *b, n_min, static_cast<linalg::KernelVariant>(variant),
                                       workers);
  }
  void result(double* C, std::size_t ldc) const override { store<W>(c, C, ldc); }
  PrepBase* with_a(std::size_t m, const double* A, std::size_t lda) const override {
    return new Prep<W>(m, b->rows(), A, lda, b);
  }
};

template <int W>
PrepBase* new_prep(std::size_t m, std::size_t K, std::size_t n, const double* A, std::size_t lda,
                   const double* B, std::size_t ldb) {
  auto bm = std::make_shared<const linalg::MPMatrix<W>>(load<W>(B, K, n, ldb));
  return new Prep<W>(m, K, A, lda, std::move(bm));
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

unsigned ref_hardware_concurrency(void) { return std::thread::hardware_concurrency(); }

// 1 when the reference picked its AVX2 backend (runtime.cpp:48-57).
int ref_backend_is_hardware(void) {
  return runtime::active_backend() == runtime::Backend::hardware ? 1 : 0;
}

// variant: 0 NORMAL, 1 SIMD_SET, 2 SIMD_LOADSTORE (linalg.hpp:149).
// c_rows/c_cols < 0 -> C is m x n; otherwise a deliberately mis-shaped C
// (exercises "matmul: result shape mismatch").
int ref_gemm(int W, std::size_t m, std::size_t K, std::size_t n, const double* A,
             std::size_t lda, const double* B, std::size_t ldb, double* C, std::size_t ldc,
             std::size_t n_min, int variant, unsigned workers, int naive, int c_rows,
             int c_cols) {
  switch (W) {
    case 2: return gemm_w<2>(m, K, n, A, lda, B, ldb, C, ldc, n_min, variant, workers, naive, c_rows, c_cols);
    case 3: return gemm_w<3>(m, K, n, A, lda, B, ldb, C, ldc, n_min, variant, workers, naive, c_rows, c_cols);
    case 4: return gemm_w<4>(m, K, n, A, lda, B, ldb, C, ldc, n_min, variant, workers, naive, c_rows, c_cols);
  }
  g_err = "bad width";
  return 1;
}

// Shape-check probe with arbitrary (mismatched) A/B/C shapes; no data.
int ref_gemm_shapes(int W, std::size_t am, std::size_t ak, std::size_t bk, std::size_t bn,
                    std::size_t cm, std::size_t cn, std::size_t n_min, int variant,
                    unsigned workers) {
  return guarded([&] {
    if (W != 2) throw std::invalid_argument("probe is DD only");
    linalg::MPMatrix<2> a(am, ak), b(bk, bn), c(cm, cn);
    linalg::matmul_block_parallel_into(c, a, b, n_min,
                                       static_cast<linalg::KernelVariant>(variant), workers);
  });
}

void ref_op_counters_reset(void) { linalg::op_counters_reset(); }
void ref_op_counts(std::uint64_t* adds, std::uint64_t* muls) {
  const auto c = linalg::op_counters_read();
  *adds = c.adds, *muls = c.muls;
}

int ref_fill_random(int W, std::size_t rows, std::size_t cols, std::uint64_t seed,
                    double* planes, std::size_t ld) {
  if (W == 2) fill_random_w<2>(rows, cols, seed, planes, ld);
  else if (W == 3) fill_random_w<3>(rows, cols, seed, planes, ld);
  else if (W == 4) fill_random_w<4>(rows, cols, seed, planes, ld);
  else return 1;
  return 0;
}

int ref_gen_paper(int W, std::size_t n, double* A, double* B, std::size_t ld) {
  if (W == 2) gen_paper_w<2>(n, A, B, ld);
  else if (W == 3) gen_paper_w<3>(n, A, B, ld);
  else if (W == 4) gen_paper_w<4>(n, A, B, ld);
  else return 1;
  return 0;
}

// op: 0 add (library default for the width), 1 mul
int ref_binop(int W, int op, const double* x, const double* y, double* r) {
  if (W == 2) binop_w<2>(op, x, y, r);
  else if (W == 3) binop_w<3>(op, x, y, r);
  else if (W == 4) binop_w<4>(op, x, y, r);
  else return 1;
  return 0;
}

// linalg::matmul_strassen[_parallel] (linalg.hpp:582-617); leaf counter out.
int ref_strassen(int W, std::size_t m, std::size_t K, std::size_t n, const double* A,
                 std::size_t lda, const double* B, std::size_t ldb, double* C, std::size_t ldc,
                 std::size_t cutoff, std::size_t n_min, int variant, unsigned workers) {
  auto run = [&](auto wc) {
    constexpr int WW = decltype(wc)::value;
    return guarded([&] {
      const auto a = load<WW>(A, m, K, lda);
      const auto b = load<WW>(B, K, n, ldb);
      const auto v = static_cast<linalg::KernelVariant>(variant);
      const auto c = workers > 1 ? linalg::matmul_strassen_parallel(a, b, cutoff, n_min, v, workers)
                                 : linalg::matmul_strassen(a, b, cutoff, n_min, v);
      store<WW>(c, C, ldc);
    });
  };
  if (W == 2) return run(std::integral_constant<int, 2>{});
  if (W == 3) return run(std::integral_constant<int, 3>{});
  if (W == 4) return run(std::integral_constant<int, 4>{});
  return 1;
}

std::uint64_t ref_leaf_multiplies(void) { return linalg::op_counters_read().leaf_multiplies; }

// linalg::ew_apply_into (linalg.hpp:647-684); op: 0 add, 1 mul, 2 add_merge
int ref_ew(int W, int op, int variant, std::size_t rows, std::size_t cols, const double* a,
           std::size_t lda, const double* b, std::size_t ldb, double* out, std::size_t ldo) {
  if (W == 2) return ew_w<2>(op, variant, rows, cols, a, lda, b, ldb, out, ldo);
  if (W == 3) return ew_w<3>(op, variant, rows, cols, a, lda, b, ldb, out, ldo);
  if (W == 4) return ew_w<4>(op, variant, rows, cols, a, lda, b, ldb, out, ldo);
  return 1;
}

// EFT primitives over a batch: op 0 two_sum, 1 quick_two_sum, 2 two_prod
void ref_eft_batch(int op, std::size_t count, const double* a, const double* b, double* s,
                   double* e) {
  for (std::size_t i = 0; i < count; ++i) {
    const auto p = op == 0 ? eft::ScalarEft::two_sum(a[i], b[i])
                           : (op == 1 ? eft::ScalarEft::quick_two_sum(a[i], b[i])
                                      : eft::ScalarEft::two_prod(a[i], b[i]));
    s[i] = p.s, e[i] = p.e;
  }
}

// td_mul_q over a batch (mpf.hpp:323-327)
void ref_td_mul_q_batch(std::size_t count, const double* x, const double* y, double* r) {
  for (std::size_t i = 0; i < count; ++i) {
    const mpf::Double3 a{{x[3 * i], x[3 * i + 1], x[3 * i + 2]}};
    const mpf::Double3 b{{y[3 * i], y[3 * i + 1], y[3 * i + 2]}};
    const auto c = mpf::td_mul_q(a, b);
    for (int w = 0; w < 3; ++w) r[3 * i + w] = c.c[w];
  }
}

// td_add_merge over a batch (mpf.hpp:305-309)
void ref_td_add_merge_batch(std::size_t count, const double* x, const double* y, double* r) {
  for (std::size_t i = 0; i < count; ++i) {
    const mpf::Double3 a{{x[3 * i], x[3 * i + 1], x[3 * i + 2]}};
    const mpf::Double3 b{{y[3 * i], y[3 * i + 1], y[3 * i + 2]}};
    const auto c = mpf::td_add_merge(a, b);
    for (int w = 0; w < 3; ++w) r[3 * i + w] = c.c[w];
  }
}

// Batched forms for million-sample sweeps (one call, no per-call overhead).
int ref_binop_batch(int W, int op, std::size_t count, const double* x, const double* y,
                    double* r) {
  for (std::size_t i = 0; i < count; ++i)
    if (ref_binop(W, op, x + i * W, y + i * W, r + i * W)) return 1;
  return 0;
}

void ref_renorm5(const double* c, double* r) {
  const auto o = eft::renorm5(c[0], c[1], c[2], c[3], c[4]);
  for (int i = 0; i < 4; ++i) r[i] = o[i];
}

int ref_vseb(const double* e, std::size_t n, double* out, std::size_t k) {
  return guarded([&] { eft::vseb(std::span<const double>(e, n), std::span<double>(out, k)); });
}

void ref_two_sum(double a, double b, double* s, double* e) {
  const auto p = eft::two_sum(a, b);
  *s = p.s, *e = p.e;
}
void ref_quick_two_sum(double a, double b, double* s, double* e) {
  const auto p = eft::ScalarEft::quick_two_sum(a, b);
  *s = p.s, *e = p.e;
}
void ref_two_prod(double a, double b, double* s, double* e) {
  const auto p = eft::two_prod(a, b);
  *s = p.s, *e = p.e;
}

void ref_random_normalized(int W, std::uint64_t* state, int is_signed, double* out) {
  rng::SplitMix64 g(0);
  g.state = *state;
  if (W == 2) {
    const auto v = is_signed ? rng::random_normalized_signed<2>(g) : rng::random_normalized<2>(g);
    for (int w = 0; w < 2; ++w) out[w] = v.c[w];
  } else if (W == 3) {
    const auto v = is_signed ? rng::random_normalized_signed<3>(g) : rng::random_normalized<3>(g);
    for (int w = 0; w < 3; ++w) out[w] = v.c[w];
  } else {
    const auto v = is_signed ? rng::random_normalized_signed<4>(g) : rng::random_normalized<4>(g);
    for (int w = 0; w < 4; ++w) out[w] = v.c[w];
  }
  *state = g.state;
}


// Build the reference matrices for C(m x n) = A(m x K) * B(K x n) once.
// Returns an opaque handle (null on error, message in ref_last_error()).
void* ref_prep_new(int W, std::size_t m, std::size_t K, std::size_t n, const double* A,
                   std::size_t lda, const double* B, std::size_t ldb) {
  PrepBase* p = nullptr;
  const int rc = guarded([&] {
    if (W == 2) p = new_prep<2>(m, K, n, A, lda, B, ldb);
    else if (W == 3) p = new_prep<3>(m, K, n, A, lda, B, ldb);
    else if (W == 4) p = new_prep<4>(m, K, n, A, lda, B, ldb);
    else throw std::invalid_argument("bad width");
  });
  return rc ? nullptr : p;
}

// Another handle over the same (shared, not copied) B with a new m-row A.
void* ref_prep_with_a(void* h, std::size_t m, const double* A, std::size_t lda) {
  PrepBase* p = nullptr;
  const int rc = guarded([&] { p = static_cast<PrepBase*>(h)->with_a(m, A, lda); });
  return rc ? nullptr : p;
}

// One timed matmul_block_parallel_into on the prepared operands; the wall
// seconds of that call alone go to *seconds.
int ref_prep_run(void* h, std::size_t n_min, int variant, unsigned workers, double* seconds) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    static_cast<PrepBase*>(h)->run(n_min, variant, workers);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

void ref_prep_result(void* h, double* C, std::size_t ldc) {
  static_cast<PrepBase*>(h)->result(C, ldc);
}

void ref_prep_free(void* h) { delete static_cast<PrepBase*>(h); }

}  // extern "C"
