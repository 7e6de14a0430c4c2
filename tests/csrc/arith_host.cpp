// arith_host.cpp -- TEST SHIM: the product's device arithmetic header
// (paper_2101_06584_b200/csrc/mpf_arith.cuh) compiled for the host with
// -ffp-contract=off, so tests/test_arith_host.py can compare the exact same
// source against the reference build (oracle/_ref) on millions of inputs
// without a GPU.  The device build uses __dadd_rn & co. with identical IEEE
// semantics.
#include <cstddef>
#include <vector>

#include "mpf_arith.cuh"
#include "mpf_lean.cuh"

using namespace mpfk::arith;

// The GEMM fast pass's contract (gemm_kernel.cuh, TileCfg::FASTR): one
// multiply-add acc = add(acc, mul(a, b)) in the fast forms (level 1 or 2,
// vseb fast for TD) with both accumulators.  out per element: W doubles of
// the fast result, then flags[2*i] = RareBool::any(), flags[2*i+1] =
// RareMin::any().  The caller checks: fast == exact whenever the exact
// accumulator stayed clear, and RareMin is never clear when RareBool is set.
template <int W, int kLevel>
static void fast_mac(const double* a, const double* b, const double* acc, double* out, int* flags) {
  double p[W], r1[W], r2[W];
  RareBool rb;
  RareMin rm;
  mp_mul_f<W, kLevel, true>(a, b, p, rb);
  mp_add_f<W, kLevel>(acc, p, r1, rb);
  mp_mul_f<W, kLevel, true>(a, b, p, rm);
  mp_add_f<W, kLevel>(acc, p, r2, rm);
  for (int w = 0; w < W; ++w) out[w] = r1[w];
  flags[0] = rb.any();
  flags[1] = rm.any();
  // the accumulator type never changes the arithmetic
  for (int w = 0; w < W; ++w)
    if (std::memcmp(&r1[w], &r2[w], 8) != 0) flags[0] = flags[1] = -1;
}

// MPFK_LEAN (csrc/mpf_lean.cuh): the GEMM element's chain on the host --
// levels start at +0 (or at a normalised `init`), every k step is one
// lean_mac, renorm_loose every `every` steps (the kernel: once per 16-step
// k-tile), lean_finish at the end.
template <int W>
static void lean_dot(std::size_t k, const double* a, const double* b, std::size_t every, const double* init,
                     double* out) {
  double s[W];
  for (int w = 0; w < W; ++w) s[w] = init ? init[w] : 0.0;
  for (std::size_t i = 0; i < k; ++i) {
    lean_mac<W>(s, a + i * W, b + i * W);
    // the kernel renormalises at the end of every k-tile, the last (partial) one included
    if (every && ((i + 1) % every == 0 || i + 1 == k)) lean_renorm_loose<W>(s);
  }
  lean_finish<W>(s, out);
}

// the reference-order chain (mul, then add ascending k) with the product's
// bit-exact arithmetic, for the error comparison
template <int W>
static void ref_dot(std::size_t k, const double* a, const double* b, double* out) {
  double acc[W], p[W];
  for (std::size_t i = 0; i < k; ++i) {
    mp_mul<W>(a + i * W, b + i * W, p);
    if (i == 0)
      for (int w = 0; w < W; ++w) acc[w] = p[w];
    else
      mp_add<W>(acc, p, acc);
  }
  for (int w = 0; w < W; ++w) out[w] = k ? acc[w] : 0.0;
}

extern "C" {

// count dot products of length k: a, b are (count, k, W); out (count, W)
int hst_lean_dot_batch(int W, std::size_t count, std::size_t k, const double* a, const double* b,
                       std::size_t every, const double* init, double* out) {
  for (std::size_t c = 0; c < count; ++c) {
    const double *x = a + c * k * W, *y = b + c * k * W;
    const double* in = init ? init + c * W : nullptr;
    double* o = out + c * W;
    if (W == 2) lean_dot<2>(k, x, y, every, in, o);
    else if (W == 3) lean_dot<3>(k, x, y, every, in, o);
    else if (W == 4) lean_dot<4>(k, x, y, every, in, o);
    else return 1;
  }
  return 0;
}

// renorm_loose / finish on their own: in (count, W) levels -> out (count, W)
int hst_lean_renorm_batch(int W, int finish, std::size_t count, const double* in, double* out) {
  for (std::size_t c = 0; c < count; ++c) {
    const double* x = in + c * W;
    double* o = out + c * W;
    if (W == 2) {
      double s[2] = {x[0], x[1]};
      if (finish) lean_finish<2>(s, o); else { lean_renorm_loose<2>(s); o[0] = s[0], o[1] = s[1]; }
    } else if (W == 3) {
      double s[3] = {x[0], x[1], x[2]};
      if (finish) lean_finish<3>(s, o); else { lean_renorm_loose<3>(s); for (int w = 0; w < 3; ++w) o[w] = s[w]; }
    } else if (W == 4) {
      double s[4] = {x[0], x[1], x[2], x[3]};
      if (finish) lean_finish<4>(s, o); else { lean_renorm_loose<4>(s); for (int w = 0; w < 4; ++w) o[w] = s[w]; }
    } else {
      return 1;
    }
  }
  return 0;
}

// the lean GEMM on the host, element by element as the kernel runs it (plane
// arrays like hst_gemm; k-tiles of 16)
int hst_lean_gemm(int W, std::size_t m, std::size_t K, std::size_t n, const double* A, std::size_t lda,
                  const double* B, std::size_t ldb, double* C, std::size_t ldc) {
  const std::size_t pa = m * lda, pb = K * ldb, pc = m * ldc;
  std::vector<double> a(K * W), b(K * W);
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      for (std::size_t k = 0; k < K; ++k)
        for (int w = 0; w < W; ++w) a[k * W + w] = A[w * pa + i * lda + k], b[k * W + w] = B[w * pb + k * ldb + j];
      double o[4] = {0, 0, 0, 0};
      if (W == 2) lean_dot<2>(K, a.data(), b.data(), 16, nullptr, o);
      else if (W == 3) lean_dot<3>(K, a.data(), b.data(), 16, nullptr, o);
      else if (W == 4) lean_dot<4>(K, a.data(), b.data(), 16, nullptr, o);
      else return 1;
      for (int w = 0; w < W; ++w) C[w * pc + i * ldc + j] = o[w];
    }
  return 0;
}

int hst_ref_dot_batch(int W, std::size_t count, std::size_t k, const double* a, const double* b, double* out) {
  for (std::size_t c = 0; c < count; ++c) {
    const double *x = a + c * k * W, *y = b + c * k * W;
    double* o = out + c * W;
    if (W == 2) ref_dot<2>(k, x, y, o);
    else if (W == 3) ref_dot<3>(k, x, y, o);
    else if (W == 4) ref_dot<4>(k, x, y, o);
    else return 1;
  }
  return 0;
}

int hst_binop_batch(int W, int op, std::size_t count, const double* x, const double* y,
                    double* r) {
  for (std::size_t i = 0; i < count; ++i) {
    const double* a = x + i * W;
    const double* b = y + i * W;
    double* c = r + i * W;
    switch (W * 2 + op) {
      case 4: mp_add<2>(a, b, c); break;
      case 5: mp_mul<2>(a, b, c); break;
      case 6: mp_add<3>(a, b, c); break;
      case 7: mp_mul<3>(a, b, c); break;
      case 8: mp_add<4>(a, b, c); break;
      case 9: mp_mul<4>(a, b, c); break;
      default: return 1;
    }
  }
  return 0;
}

// the literal zero-extend + qd_add form of td_add_q (no folds)
void hst_td_add_unfolded_batch(std::size_t count, const double* x, const double* y, double* r) {
  for (std::size_t i = 0; i < count; ++i) td_add_q_unfolded(x + 3 * i, y + 3 * i, r + 3 * i);
}

void hst_td_add_merge_batch(std::size_t count, const double* x, const double* y, double* r) {
  for (std::size_t i = 0; i < count; ++i) td_add_merge(x + 3 * i, y + 3 * i, r + 3 * i);
}

void hst_td_add_merge_ranked_batch(std::size_t count, const double* x, const double* y, double* r) {
  double zb[6];
  for (std::size_t i = 0; i < count; ++i) td_add_merge_ranked(x + 3 * i, y + 3 * i, r + 3 * i, zb, 1);
}

void hst_renorm5_batch(std::size_t count, const double* c, double* r) {
  for (std::size_t i = 0; i < count; ++i) {
    const double* x = c + 5 * i;
    double* o = r + 4 * i;
    renorm5(x[0], x[1], x[2], x[3], x[4], o[0], o[1], o[2], o[3]);
  }
}

void hst_vseb23_batch(std::size_t count, const double* e, double* out) {
  for (std::size_t i = 0; i < count; ++i) vseb_2_3(e[3 * i], e[3 * i + 1], e[3 * i + 2], out[2 * i], out[2 * i + 1]);
}

// the GEMM's per-element order (mul first, then add(C, p) ascending k) on the
// host with the product arithmetic
void hst_gemm(int W, std::size_t m, std::size_t K, std::size_t n, const double* A, std::size_t lda,
              const double* B, std::size_t ldb, double* C, std::size_t ldc) {
  const std::size_t pa = m * lda, pb = K * ldb, pc = m * ldc;
  for (std::size_t i = 0; i < m; ++i)
    for (std::size_t j = 0; j < n; ++j) {
      double acc[4] = {0, 0, 0, 0};
      for (std::size_t k = 0; k < K; ++k) {
        double a[4], b[4], p[4];
        for (int w = 0; w < W; ++w) a[w] = A[w * pa + i * lda + k], b[w] = B[w * pb + k * ldb + j];
        if (W == 2) mp_mul<2>(a, b, p);
        else if (W == 3) mp_mul<3>(a, b, p);
        else mp_mul<4>(a, b, p);
        if (k == 0) {
          for (int w = 0; w < W; ++w) acc[w] = p[w];
        } else if (W == 2) mp_add<2>(acc, p, acc);
        else if (W == 3) mp_add<3>(acc, p, acc);
        else mp_add<4>(acc, p, acc);
      }
      for (int w = 0; w < W; ++w) C[w * pc + i * ldc + j] = acc[w];
    }
}

// two_sum_sorted vs the literal Knuth form, pairwise
void hst_two_sum_pair_batch(std::size_t count, const double* a, const double* b, double* out) {
  for (std::size_t i = 0; i < count; ++i) {
    two_sum_knuth(a[i], b[i], out[4 * i], out[4 * i + 1]);
    two_sum_sorted(a[i], b[i], out[4 * i + 2], out[4 * i + 3]);
  }
}

// two_sum_ordered (the fast pass's 3-operation form) next to Knuth's form:
// out = (s_knuth, e_knuth, s_ordered, e_ordered), flag = the order test failed
void hst_two_sum_ordered_batch(std::size_t count, const double* a, const double* b, double* out, int* flag) {
  for (std::size_t i = 0; i < count; ++i) {
    RareBool rare;
    two_sum_knuth(a[i], b[i], out[4 * i], out[4 * i + 1]);
    two_sum_ordered(a[i], b[i], out[4 * i + 2], out[4 * i + 3], rare);
    flag[i] = rare.any();
  }
}

int hst_fast_mac_batch(int W, int level, std::size_t count, const double* a, const double* b,
                       const double* acc, double* out, int* flags) {
  for (std::size_t i = 0; i < count; ++i) {
    const double *x = a + i * W, *y = b + i * W, *c = acc + i * W;
    double* o = out + i * W;
    int* f = flags + 2 * i;
    switch (W * 4 + level) {
      case 13: fast_mac<3, 1>(x, y, c, o, f); break;
      case 14: fast_mac<3, 2>(x, y, c, o, f); break;
      case 17: fast_mac<4, 1>(x, y, c, o, f); break;
      case 18: fast_mac<4, 2>(x, y, c, o, f); break;
      default: return 1;
    }
  }
  return 0;
}

}  // extern "C"
