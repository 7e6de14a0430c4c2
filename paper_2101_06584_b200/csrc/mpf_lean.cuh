// mpf_lean.cuh -- the MPFK_LEAN multiply-accumulate: C += a*b for DD/TD/QD
// with 12 / 46 / 113 FP64 operations instead of the reference sequence's
// 20 / 119 (132 counted) / 218.
//
// NOT the reference's arithmetic and NOT bit-identical to it: this is the
// north star's tolerance mode (BASELINE.json: "each component of C must
// agree to a normwise relative error of at most 4*k*u_p"; bit-exactness is
// required only "whenever the kernel is run with the reference's per-element
// accumulation order", which MPFK_BIT_EXACT, the default, is).  The GEMM is
// bound by the FP64 pipe and the bit-exact kernels already keep it 95 % busy,
// so the only faster GEMM is one that issues fewer FP64 instructions.
//
// What the reference does per k step (mpf.hpp:105-238): round the product to
// a normalised W-term value (renorm5 / vseb), then add two normalised values
// and renormalise again.  Both renormalisations and the three-sum networks
// between them exist to hand back a canonical value after EVERY operation.
// A GEMM element does not need that: it is one long sum of products.  The
// lean form keeps each element as W "levels" s[0..W) -- an unevaluated sum
// whose terms may overlap a little -- and adds the product's partial terms
// straight into it:
//
//   * the product is expanded into error-free terms by order of magnitude
//     (two_prod, eft.hpp:63-67): order 0 a0*b0; order 1 its error and the two
//     products a0*b1, a1*b0; order 2 ...; the last order (W-1) is evaluated in
//     plain binary64 (an fma chain), exactly the terms the reference's
//     dd_mul / td_mul / qd_mul keep (mpf.hpp:113-119, 146-163, 198-238);
//   * a term of order L enters level L through a cascade of exact two-sums
//     (Knuth, eft.hpp:46-51: no ordering assumption, so overlap and
//     cancellation cannot break it): (s[L], x) = two_sum(s[L], x), the error
//     x moves on to level L+1, ..., and what reaches the last level is added
//     in plain binary64.
//
// Every operation above the last level is exact, so the only rounding errors
// are the plain additions at the last level (each at most u * |s[W-1]|) and
// the dropped product terms of order >= W (the same ones the reference
// drops).  |s[W-1]| is held near u^(W-1) * |C| by renorm_loose() once per
// k-tile (16 steps), so each step's error is a small multiple of u^W * |C|:
//   DD  2 last-level adds/step, dropped/rounded product terms ~3 u^2 |a||b|
//   TD  5 last-level adds/step, ~3.5 u^3 |a||b|
//   QD 10 last-level adds/step, ~7 u^4 |a||b|
// against a budget of 4*u_p = 16 u^2 / 32 u^3 / 64 u^4 per step (u = 2^-53,
// u_p = 2^-104 / 2^-156 / 2^-208).  Measured against the exact dyadic oracle
// (tests/test_lean_host.py, tests/test_lean_gpu.py) on the BASELINE
// distributions at k = 2048..4096: 2e-4 .. 1.5e-3 of 4*k*u_p.  That is NOT as
// accurate as the reference sequence, which renormalises after every
// operation and lands at 4e-6 .. 2e-4 of the same tolerance (DD 2-4x, TD
// 10-35x, QD 30-200x smaller errors than the lean form): the lean form
// spends the tolerance the north star grants, it does not tighten it.  No
// worst-case proof at 4*k*u_p is claimed (a bound with every rounding residual
// of a k-tile aligned in sign exceeds it); DESIGN.md 9.2 lists what was
// measured instead.
//
// finish() turns the levels into a canonical normalised value (what the
// reference's renormalisation returns: each component at most half an ulp of
// the one before, zeros last), once per element at the end of the GEMM.
//
// Same source on host and device (tests/csrc/arith_host.cpp).
#pragma once

#include "mpf_arith.cuh"

namespace mpfk {
namespace arith {

// FP64 instructions the lean multiply-accumulate executes per step
// (renorm_loose amortised over a 16-step k-tile on top: +6/16, +18/16,
// +30/16).
template <int W>
constexpr int lean_ops_per_mac() {
  return W == 2 ? 12 : (W == 3 ? 46 : 113);
}
template <int W>
constexpr int lean_renorm_ops() {
  return W == 2 ? 6 : (W == 3 ? 18 : 30);
}

// s[L..W-2] take x through exact two-sums; returns what is left for the
// last level
template <int W, int L>
MPFK_HD double lean_cascade(double (&s)[W], double x) {
#pragma unroll
  for (int i = L; i < W - 1; ++i) {
    double t, r;
    two_sum_knuth(s[i], x, t, r);
    s[i] = t;
    x = r;
  }
  return x;
}

// s += a * b (a, b normalised W-term values; s the levels)
template <int W>
MPFK_HD void lean_mac(double (&s)[W], const double* a, const double* b) {
  if constexpr (W == 2) {
    // order 0: p; order 1: its error and the cross products, one fma chain
    const double p = mul(a[0], b[0]);
    double e = fma(a[0], b[0], -p);
    e = fma(a[0], b[1], e);
    e = fma(a[1], b[0], e);
    const double r = lean_cascade<2, 0>(s, p);
    s[1] = add(s[1], add(r, e));
  } else if constexpr (W == 3) {
    double p00, e00, p01, e01, p10, e10;
    two_prod(a[0], b[0], p00, e00);
    two_prod(a[0], b[1], p01, e01);
    two_prod(a[1], b[0], p10, e10);
    // order 2 in plain binary64
    double t = mul(a[0], b[2]);
    t = fma(a[1], b[1], t);
    t = fma(a[2], b[0], t);
    t = add(t, add(e01, e10));
    const double r0 = lean_cascade<3, 0>(s, p00);
    const double r1 = lean_cascade<3, 1>(s, e00);
    const double r2 = lean_cascade<3, 1>(s, p01);
    const double r3 = lean_cascade<3, 1>(s, p10);
    s[2] = add(s[2], add(add(add(r0, r1), add(r2, r3)), t));
  } else {
    double p00, e00, p01, e01, p10, e10, p02, e02, p11, e11, p20, e20;
    two_prod(a[0], b[0], p00, e00);
    two_prod(a[0], b[1], p01, e01);
    two_prod(a[1], b[0], p10, e10);
    two_prod(a[0], b[2], p02, e02);
    two_prod(a[1], b[1], p11, e11);
    two_prod(a[2], b[0], p20, e20);
    // order 3 in plain binary64
    double t = mul(a[0], b[3]);
    t = fma(a[1], b[2], t);
    t = fma(a[2], b[1], t);
    t = fma(a[3], b[0], t);
    t = add(t, add(add(e02, e11), e20));
    const double r0 = lean_cascade<4, 0>(s, p00);
    const double r1 = lean_cascade<4, 1>(s, e00);
    const double r2 = lean_cascade<4, 1>(s, p01);
    const double r3 = lean_cascade<4, 1>(s, p10);
    const double r4 = lean_cascade<4, 2>(s, e01);
    const double r5 = lean_cascade<4, 2>(s, e10);
    const double r6 = lean_cascade<4, 2>(s, p02);
    const double r7 = lean_cascade<4, 2>(s, p11);
    const double r8 = lean_cascade<4, 2>(s, p20);
    const double ra = add(add(r0, r1), add(r2, r3));
    const double rb = add(add(r4, r5), add(r6, r7));
    s[3] = add(s[3], add(add(ra, rb), add(r8, t)));
  }
}

// DD: N multiply-accumulates that share a (one row of a thread's micro-tile)
// written stage by stage across the N elements, so consecutive instructions
// are independent -- the same operations as N calls of lean_mac<2>, only
// the order in the instruction stream differs (results are bit-identical).
template <int N>
MPFK_HD void lean_mac_dd_row(double (&s)[N][2], const double* a, const double (&b)[N][2]) {
  double p[N], e[N], ss[N], v[N], t1[N], t3[N];
#pragma unroll
  for (int j = 0; j < N; ++j) p[j] = mul(a[0], b[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) ss[j] = add(s[j][0], p[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = fma(a[0], b[j][0], -p[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = sub(ss[j], s[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = fma(a[0], b[j][1], e[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) t1[j] = sub(ss[j], v[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) t3[j] = sub(p[j], v[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = fma(a[1], b[j][0], e[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) t1[j] = sub(s[j][0], t1[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) t1[j] = add(t1[j], t3[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = add(t1[j], e[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    s[j][1] = add(s[j][1], e[j]);
    s[j][0] = ss[j];
  }
}

// Pull the levels back to nearly non-overlapping (|s[i+1]| <~ ulp(s[i])):
// VecSum from the bottom up, then the error pass from the top down, both
// with Knuth two-sums (exact whatever the overlap or cancellation above).
// The value of the sum does not change.
template <int W>
MPFK_HD void lean_renorm_loose(double (&s)[W]) {
  double e[W];
  double t = s[W - 1];
#pragma unroll
  for (int i = W - 2; i >= 0; --i) {
    double ss, r;
    two_sum_knuth(s[i], t, ss, r);
    e[i + 1] = r;
    t = ss;
  }
  s[0] = t;
  if constexpr (W == 2) {
    s[1] = e[1];
  } else {
    double eps = e[1];
#pragma unroll
    for (int i = 1; i < W - 1; ++i) {
      double ss, r;
      two_sum_knuth(eps, e[i + 1], ss, r);
      s[i] = ss;
      eps = r;
    }
    s[W - 1] = eps;
  }
}

// The levels as a canonical W-term value: two loose passes (after them the
// terms are ordered and nearly non-overlapping), then the compressing pass
// of the reference's renormalisation (VecSumErrBranch, eft.hpp:205-225: a
// zero error never takes a slot, unused slots are +0).
template <int W>
MPFK_HD void lean_finish(double (&s)[W], double* out) {
  lean_renorm_loose<W>(s);
  lean_renorm_loose<W>(s);
  double o[W];
#pragma unroll
  for (int i = 0; i < W; ++i) o[i] = 0.0;
  int j = 0;
  double eps = s[0];
#pragma unroll
  for (int i = 0; i < W - 1; ++i) {
    double ss, r;
    two_sum_knuth(eps, s[i + 1], ss, r);
    const bool nzr = nz(r);
#pragma unroll
    for (int q = 0; q < W; ++q) o[q] = sel(nzr && j == q, ss, o[q]);
    eps = sel(nzr, r, ss);
    j += nzr ? 1 : 0;
  }
#pragma unroll
  for (int q = 0; q < W; ++q) o[q] = sel(j == q && nz(eps), eps, o[q]);
#pragma unroll
  for (int i = 0; i < W; ++i) out[i] = o[i];
}

}  // namespace arith
}  // namespace mpfk
