// mpf_lean.cuh -- the MPFK_LEAN multiply-accumulate: C += a*b for DD/TD/QD
// with 10 / 42 / 107 FP64 operations instead of the reference sequence's
// 20 / 110 (132 counted) / 212 (218 counted).
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
//   * a product of the next-to-last order does not get a separate two_prod
//     error and two-sum error: both belong to the last level, and one fma
//     forms their sum in a single rounding (lean_last_prod; for DD this is
//     the leading product itself, lean_mac<2>).
//
// Every operation above the last level is exact, so the only rounding errors
// are the plain additions and fused corrections at the last level (each at
// most u * |s[W-1]| resp. u * ulp(s[W-2])) and the dropped product terms of
// order >= W (the same ones the reference drops).  |s[W-1]| is held near
// u^(W-1) * |C| by renorm_loose() once per k-tile (16 steps), so each step's
// error is a small multiple of u^W * |C| against a budget of 4*u_p = 16 u^2 /
// 32 u^3 / 64 u^4 per step (u = 2^-53, u_p = 2^-104 / 2^-156 / 2^-208).
// Measured against the exact dyadic oracle (tests/test_lean_host.py,
// tests/test_lean_gpu.py) on the BASELINE distributions at k = 2048..4096:
// 2e-4 .. 1.5e-3 of 4*k*u_p.  That is NOT as accurate as the reference
// sequence, which renormalises after every operation and lands at 4e-6 ..
// 2e-4 of the same tolerance (DD 1-3x, TD 14-72x, QD 36-290x smaller errors
// than the lean form): the lean form spends the tolerance the north star
// grants, it does not tighten it.  No worst-case proof at 4*k*u_p is claimed
// (a bound with every rounding residual of a k-tile aligned in sign exceeds
// it); DESIGN.md 9.2 lists what was measured instead.
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
  return W == 2 ? 10 : (W == 3 ? 42 : 107);
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

// A product x*y of the next-to-last order enters its level sl (the last one
// fed by two-sums): sl' = sl + p with p = RN(x*y).  Knuth's two-sum error is
// t2 + (p - v) (v = sl' - sl, t2 = sl - (sl' - v)) and the product's own
// error is x*y - p; both belong to the last level, where additions are plain
// anyway, so they are formed together: fma(x, y, -v) = (x*y - p) + (p - v) in
// one rounding (error <= u * |x*y - v|, of the last level's order times u).
// Returns what goes to the last level.  7 operations instead of 10.
MPFK_HD double lean_last_prod(double& sl, double x, double y) {
  const double p = mul(x, y);
  const double ss = add(sl, p);
  const double v = sub(ss, sl);
  const double t2 = sub(sl, sub(ss, v));
  const double g = fma(x, y, -v);
  sl = ss;
  return add(t2, g);
}

// s += a * b (a, b normalised W-term values; s the levels)
template <int W>
MPFK_HD void lean_mac(double (&s)[W], const double* a, const double* b) {
  if constexpr (W == 2) {
    // 10 operations.  Knuth's two-sum of (s0, p) is ss = s0 + p with the
    // exact error t2 + (p - v) (v = ss - s0, t2 = s0 - (ss - v)); the exact
    // product is p + (a0*b0 - p).  The two corrections are not formed one by
    // one: g = fma(a0, b0, -v) is (a0*b0 - p) + (p - v) in ONE rounding
    // (error <= u*|a0*b0 - v| <= u^2 (|p| + |ss|), second order like the
    // dropped a1*b1), and the cross products join the same fma chain.
    const double p = mul(a[0], b[0]);
    const double ss = add(s[0], p);
    const double v = sub(ss, s[0]);
    const double t2 = sub(s[0], sub(ss, v));
    double g = fma(a[0], b[0], -v);
    g = fma(a[0], b[1], g);
    g = fma(a[1], b[0], g);
    s[1] = add(s[1], add(t2, g));
    s[0] = ss;
  } else if constexpr (W == 3) {
    // 42 operations: order 0 exactly through s0, s1; its error exactly
    // through s1; the order-1 products through s1 with the fused correction
    // (lean_last_prod); order 2 in plain binary64
    double p00, e00;
    two_prod(a[0], b[0], p00, e00);
    double t = mul(a[0], b[2]);
    t = fma(a[1], b[1], t);
    t = fma(a[2], b[0], t);
    const double r0 = lean_cascade<3, 0>(s, p00);
    const double r1 = lean_cascade<3, 1>(s, e00);
    const double q01 = lean_last_prod(s[1], a[0], b[1]);
    const double q10 = lean_last_prod(s[1], a[1], b[0]);
    s[2] = add(s[2], add(add(add(r0, r1), add(q01, q10)), t));
  } else {
    // 107 operations: orders 0 and 1 exactly (two_prod errors included)
    // through every level above the last; the order-2 products through s2
    // with the fused correction; order 3 in plain binary64
    double p00, e00, p01, e01, p10, e10;
    two_prod(a[0], b[0], p00, e00);
    two_prod(a[0], b[1], p01, e01);
    two_prod(a[1], b[0], p10, e10);
    double t = mul(a[0], b[3]);
    t = fma(a[1], b[2], t);
    t = fma(a[2], b[1], t);
    t = fma(a[3], b[0], t);
    const double r0 = lean_cascade<4, 0>(s, p00);
    const double r1 = lean_cascade<4, 1>(s, e00);
    const double r2 = lean_cascade<4, 1>(s, p01);
    const double r3 = lean_cascade<4, 1>(s, p10);
    const double r4 = lean_cascade<4, 2>(s, e01);
    const double r5 = lean_cascade<4, 2>(s, e10);
    const double q02 = lean_last_prod(s[2], a[0], b[2]);
    const double q11 = lean_last_prod(s[2], a[1], b[1]);
    const double q20 = lean_last_prod(s[2], a[2], b[0]);
    const double ra = add(add(r0, r1), add(r2, r3));
    const double rb = add(add(r4, r5), add(q02, q11));
    s[3] = add(s[3], add(add(ra, rb), add(q20, t)));
  }
}

// DD: N multiply-accumulates that share a (one row of a thread's micro-tile)
// written stage by stage across the N elements, so consecutive instructions
// are independent -- the same operations as N calls of lean_mac<2>, only
// the order in the instruction stream differs (results are bit-identical).
template <int N>
MPFK_HD void lean_mac_dd_row(double (&s)[N][2], const double* a, const double (&b)[N][2]) {
  double p[N], ss[N], v[N], t[N], g[N];
#pragma unroll
  for (int j = 0; j < N; ++j) p[j] = mul(a[0], b[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) ss[j] = add(s[j][0], p[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = sub(ss[j], s[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = sub(ss[j], v[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) g[j] = fma(a[0], b[j][0], -v[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = sub(s[j][0], t[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) g[j] = fma(a[0], b[j][1], g[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) g[j] = fma(a[1], b[j][0], g[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) g[j] = add(t[j], g[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    s[j][1] = add(s[j][1], g[j]);
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
