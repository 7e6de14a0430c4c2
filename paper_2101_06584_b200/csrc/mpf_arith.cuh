// mpf_arith.cuh -- DD/TD/QD arithmetic as device-inlined SIMT FP64 code.
//
// B200-native restatement of the reference's error-free transformations and
// width kernels (mpfkit: proj/include/mpfkit/eft.hpp, mpf.hpp).  Every
// function reproduces the reference's operation sequence exactly, so results
// are bit-identical to the CPU library; the only structural change is that
// the branchy renormalisation steps (renorm5, vseb) are restated as
// predicated selects so a warp does not diverge on the common path.
//
// The same source compiles for the host (g++/nvcc host pass, with
// -ffp-contract=off) so tests/test_arith_host.py can check it bit-for-bit
// against the reference build before any GPU time is spent.  On the device
// every rounding operation is an explicit __dadd_rn/__dsub_rn/__dmul_rn/
// __fma_rn intrinsic: nvcc never contracts those into DFMA, regardless of
// -fmad (default contraction breaks the EFTs).
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define MPFK_HD __host__ __device__ __forceinline__
#else
#define MPFK_HD inline __attribute__((always_inline))
#endif

namespace mpfk {
namespace arith {

// ---------------------------------------------------------------------------
// Rounded binary64 operations (the "policy" of eft.hpp:29-31).
// ---------------------------------------------------------------------------
#if defined(__CUDA_ARCH__)
MPFK_HD double add(double a, double b) { return __dadd_rn(a, b); }
MPFK_HD double sub(double a, double b) { return __dsub_rn(a, b); }
MPFK_HD double mul(double a, double b) { return __dmul_rn(a, b); }
MPFK_HD double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
// x != 0 (either sign of zero counts as zero) as an integer test on the bit
// pattern: one LOP3 + ISETP on the ALU pipe instead of a DSETP on the FP64
// pipe, which is the bottleneck.
MPFK_HD bool nz(double x) {
  return ((__double2hiint(x) & 0x7fffffff) | __double2loint(x)) != 0;
}
#else
MPFK_HD double add(double a, double b) { return a + b; }
MPFK_HD double sub(double a, double b) { return a - b; }
MPFK_HD double mul(double a, double b) { return a * b; }
MPFK_HD double fma(double a, double b, double c) { return std::fma(a, b, c); }
MPFK_HD bool nz(double x) {
  uint64_t u;
  std::memcpy(&u, &x, sizeof u);
  return (u << 1) != 0;
}
#endif
MPFK_HD double sel(bool p, double a, double b) { return p ? a : b; }

// "a is at least in b's binade", conservatively: the high words with the
// sign bit dropped compare like magnitudes, and equal high words mean equal
// exponents.  On the device it is ONE instruction off the FP64 pipe: a
// binary32 compare of the high words with |.| operand modifiers.  High words
// that read as binary32 NaN (|x| >= 2^1017, infinities, NaNs) compare false:
// conservative (the caller then takes the exact form).
#if defined(__CUDA_ARCH__)
MPFK_HD bool mag_ge(double a, double b) {
  return fabsf(__int_as_float(__double2hiint(a))) >= fabsf(__int_as_float(__double2hiint(b)));
}
#else
MPFK_HD bool mag_ge(double a, double b) {
  uint64_t ua, ub;
  std::memcpy(&ua, &a, sizeof ua);
  std::memcpy(&ub, &b, sizeof ub);
  const uint32_t ha = static_cast<uint32_t>(ua >> 32) & 0x7fffffffu, hb = static_cast<uint32_t>(ub >> 32) & 0x7fffffffu;
  return ha <= 0x7f800000u && hb <= 0x7f800000u && ha >= hb;  // (binary32 NaN patterns are unordered)
}
#endif

// "This input left the fast form" accumulators for the GEMM inner loop (the
// `rare` argument of the *_t forms below): need_nz(x) records that x had to
// be nonzero, any() reports whether some recorded x was zero.
//
// RareBool: the exact test (one LOP3 into a predicate per value plus the
// predicate ORs).
struct RareBool {
  bool r = false;
  MPFK_HD void need_nz(double x) { r |= !nz(x); }
  MPFK_HD void need_nz(double x, double y) { r |= !(nz(x) & nz(y)); }
  MPFK_HD void need_nz(double x, double y, double z) { r |= !(nz(x) & nz(y) & nz(z)); }
  // a had to be at least b's binade (two_sum_ordered below)
  MPFK_HD void need_ge(double a, double b) { r |= !mag_ge(a, b); }
  MPFK_HD bool any() const { return r; }
};
// RareHi: the zero tests as binary32 compares of the high words too
// (|hi| == 0: conservative like RareMin's -- a subnormal below 2^-1042 reads
// as zero), so every test is ONE compare whose predicate update folds into
// the instruction (FSETP ... .OR), without RareBool's separate predicate ORs.
// MEASURED EQUAL (profiles/r02/tune_rarehi.log: 14-20 % fewer non-FP64
// instructions, -0.5 .. +0.3 % in time): kept as a measured alternative
// (TileCfg RAREMIN_ = 2), not the product's choice.
struct RareHi {
  bool r = false;
#if defined(__CUDA_ARCH__)
  static MPFK_HD bool hz(double x) { return fabsf(__int_as_float(__double2hiint(x))) == 0.0f; }
#else
  static MPFK_HD bool hz(double x) {
    uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    return (static_cast<uint32_t>(u >> 32) << 1) == 0;
  }
#endif
  MPFK_HD void need_nz(double x) { r |= hz(x); }
  MPFK_HD void need_nz(double x, double y) { r |= hz(x), r |= hz(y); }
  MPFK_HD void need_nz(double x, double y, double z) { r |= hz(x), r |= hz(y), r |= hz(z); }
  MPFK_HD void need_ge(double a, double b) { r |= !mag_ge(a, b); }
  MPFK_HD bool any() const { return r; }
};
// RareMin: a running minimum of |high word read as binary32| -- one FMNMX3
// with |.| operand modifiers per TWO values and nothing else, off the FP64
// pipe.  x = +-0 has a high word of +-0.0f, so the minimum reaches 0.0f
// whenever a recorded value was zero.  The test is conservative, never
// optimistic: a subnormal below 2^-1042 (zero high word, nonzero low word)
// also reads as zero, and the caller then merely recomputes with the exact
// form.  High words that read as binary32 NaN (|x| >= 2^1017, infinities,
// NaNs: nonzero) are skipped by fminf; binary32 subnormals (|x| < 2^-1015)
// compare as what they are (no flush-to-zero in this build; a flush would
// only be conservative).  MEASURED SLOWER than RareBool in the GEMMs
// (profiles/r02/tune_raremin.log: TD n=4096 472.6 vs 469.4 ms, QD 852.0 vs
// 848.2 ms) although the loop bodies shrink -- not the product's choice;
// tests/test_arith_host.py checks the contract of both.
struct RareMin {
#if defined(__CUDA_ARCH__)
  float m = 1.0f;
  static MPFK_HD float key(double x) { return fabsf(__int_as_float(__double2hiint(x))); }
  MPFK_HD void need_nz(double x) { m = fminf(m, key(x)); }
  MPFK_HD void need_nz(double x, double y) { m = fminf(fminf(m, key(x)), key(y)); }
  MPFK_HD void need_nz(double x, double y, double z) { need_nz(x, y), need_nz(z); }
  MPFK_HD void need_ge(double a, double b) { m = mag_ge(a, b) ? m : 0.0f; }
  MPFK_HD bool any() const { return m == 0.0f; }
#else
  bool r = false;
  static MPFK_HD bool hz(double x) {
    uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    return (static_cast<uint32_t>(u >> 32) << 1) == 0;
  }
  MPFK_HD void need_nz(double x) { r |= hz(x); }
  MPFK_HD void need_nz(double x, double y) { r |= hz(x) | hz(y); }
  MPFK_HD void need_nz(double x, double y, double z) { r |= hz(x) | hz(y) | hz(z); }
  MPFK_HD void need_ge(double a, double b) { r |= !mag_ge(a, b); }
  MPFK_HD bool any() const { return r; }
#endif
};

// ---------------------------------------------------------------------------
// EFT primitives, eft.hpp:46-113.
// ---------------------------------------------------------------------------

// Knuth two-sum, eft.hpp:46-51 (6 FP64 ops), literally.
MPFK_HD void two_sum_knuth(double a, double b, double& s, double& e) {
  const double ss = add(a, b);
  const double v = sub(ss, a);
  e = add(sub(a, sub(ss, v)), sub(b, v));
  s = ss;
}

// Magnitude key: the high word without its sign bit, shifted up -- exponent
// first, so key(x) >= key(y) implies exponent(x) >= exponent(y).
#if defined(__CUDA_ARCH__)
MPFK_HD uint32_t mag_key(double x) { return static_cast<uint32_t>(__double2hiint(x)) << 1; }
#else
MPFK_HD uint32_t mag_key(double x) {
  uint64_t u;
  std::memcpy(&u, &x, sizeof u);
  return static_cast<uint32_t>(u >> 32) << 1;
}
#endif

// The same (s, e) as two_sum_knuth with 3 FP64 ops: order the operands by
// exponent on the integer pipes, then Dekker's fast two-sum.  Why it is
// bit-identical for finite operands whose sum does not overflow:
//  * s = a + b is the same rounded sum (x + y = a + b, commutative);
//  * exponent(x) >= exponent(y) (Dekker's condition; equal exponents may go
//    either way, subnormals included), so x - s = -(s - x) is exact and
//    (x - s) + y = (a + b) - s is the exact rounding error, representable,
//    hence computed exactly -- the same real number Knuth's form yields;
//  * signed zeros: Knuth's e is never -0 (its last add is -0 only if both
//    addends are -0, i.e. b = -0 with v = s - a = +0, but then a - (s - v)
//    = +0).  (x - s) + y is -0 only if x - s = -0 and y = -0; x - s = -0
//    needs x = -0 and s = +0, and then y = s - x... = +0.  So both give +0
//    whenever the error is zero.
// The sort costs one compare, two key shifts and four 32-bit selects on the
// integer pipes.  MEASURED SLOWER on the B200 (profiles/r01_ceiling_two_sum.log):
// the DD register-resident ceiling drops from 0.975 to 0.940 of the DFMA
// peak (17 instead of 20 FP64 instructions per MAC, but the pipe then idles
// ~20 %), TD 0.972 -> 0.890, QD 0.916 -> 0.844; the GEMMs lose 3-8 %.  So the
// product keeps Knuth's form; this one is opt-in (-DMPFK_TWO_SUM_SORTED) and
// stays bit-identical (tests/test_arith_host.py checks it against Knuth's
// form on signed zeros, subnormals, ties and cancelling pairs).
MPFK_HD void two_sum_sorted(double a, double b, double& s, double& e) {
#if defined(MPFK_TWO_SUM_SORTED_FSETP)
  // experiment: the order from ONE binary32 compare of the high words
  // (mag_ge); NOT exact for |x| >= 2^1017, whose high words read as NaN
  const bool p = mag_ge(a, b);
#else
  const bool p = mag_key(a) >= mag_key(b);
#endif
  const double x = sel(p, a, b), y = sel(p, b, a);
  const double ss = add(a, b);
  e = add(sub(x, ss), y);
  s = ss;
}

// two_sum_sorted without the sort, for the GEMM's fast pass: where the
// operands' order is known with overwhelming probability (a leading product
// against the sum of its lower-order terms), take a as the larger one --
// 3 FP64 operations, the same bits as Knuth's form whenever exponent(a) >=
// exponent(b) (see above) -- and tell `rare` when that did not hold, so the
// caller recomputes exactly.  The test is one compare instruction off the
// FP64 pipe (mag_ge).
template <class Rare>
MPFK_HD void two_sum_ordered(double a, double b, double& s, double& e, Rare& rare) {
  rare.need_ge(a, b);
  const double ss = add(a, b);
  e = add(sub(a, ss), b);
  s = ss;
}

#ifdef MPFK_TWO_SUM_SORTED
MPFK_HD void two_sum(double a, double b, double& s, double& e) { two_sum_sorted(a, b, s, e); }
#else
MPFK_HD void two_sum(double a, double b, double& s, double& e) { two_sum_knuth(a, b, s, e); }
#endif

// Dekker fast-two-sum, eft.hpp:55-59 (3 ops).
MPFK_HD void qts(double a, double b, double& s, double& e) {
  const double ss = add(a, b);
  e = sub(b, sub(ss, a));
  s = ss;
}

// FMA two-product, eft.hpp:63-67: e = fma(a, b, -s).  The negation is an
// exact sign flip folded into the DFMA operand.
MPFK_HD void two_prod(double a, double b, double& s, double& e) {
  const double ss = mul(a, b);
  e = fma(a, b, -ss);
  s = ss;
}

// three-sum, eft.hpp:87-92.
MPFK_HD void three_sum(double a, double b, double c, double& s, double& e1, double& e2) {
  double ts, te, us, ue;
  two_sum(a, b, ts, te);
  two_sum(c, ts, us, ue);
  two_sum(te, ue, e1, e2);
  s = us;
}

// three-sum for the GEMM's fast pass when c is the rounding error of a sum
// that feeds a or b (so a + b is all but never below c's binade): the middle
// two-sum takes the ordered 3-operation form, larger operand first --
// two_sum(c, ts) and two_sum(ts, c) are the same bits (same rounded sum, same
// exact error, +0 when it vanishes) -- and `rare` hears when the order did
// not hold.
template <class Rare>
MPFK_HD void three_sum_c_small(double a, double b, double c, double& s, double& e1, double& e2, Rare& rare) {
  double ts, te, us, ue;
  two_sum(a, b, ts, te);
  two_sum_ordered(ts, c, us, ue, rare);
  two_sum(te, ue, e1, e2);
  s = us;
}

// three-sum2, eft.hpp:95-99.
MPFK_HD void three_sum2(double a, double b, double c, double& s, double& e) {
  double ts, te, us, ue;
  two_sum(a, b, ts, te);
  two_sum(c, ts, us, ue);
  s = us;
  e = add(te, ue);
}

// ---------------------------------------------------------------------------
// renorm5, eft.hpp:241-288.
//
// Backward quick-two-sum sweep, then the forward emission.  Paths A and B of
// the reference (first two forward residuals nonzero) cover >99% of GEMM MACs
// on random inputs; they differ only in where the last
// term lands, which is a select.  The remaining paths (a zero residual in the
// first two forward steps -- structured or sparse inputs) take the reference's
// branch structure verbatim.
//
// Signed zeros: every slot the reference leaves untouched keeps its exact
// value, including the +0 initialisers of s2/s3 (eft.hpp:251).
// ---------------------------------------------------------------------------
//
// kFast (the GEMM inner loop; the result is then NOT the reference's when
// `rare` gets set, and the caller recomputes with the exact form --
// gemm_kernel.cuh: a warp redoes its k-tile from a snapshot of C):
//   1: paths A/B, branch-free (two selects); `rare` for paths C/D, a zero
//      residual in the first two forward steps;
//   2: path A only, branch- and select-free; `rare` also for path B (a zero
//      third residual) -- a win when path B is rare (QD), a loss when it is
//      common (TD's zero-extended fourth lane makes it so).
// Without the branch the compiler interleaves a thread's independent chains
// across the renormalisation (TD/QD GEMM +2-3 %).
template <int kFast, bool kTrunc3 = false, class Rare = RareBool>
MPFK_HD void renorm5_t(double c0, double c1, double c2, double c3, double c4, double& r0,
                       double& r1, double& r2, double& r3, Rare& rare) {
  double t;
  qts(c3, c4, t, c4);
  qts(c2, t, t, c3);
  qts(c1, t, t, c2);
  qts(c0, t, c0, c1);

  double s0, s1, u, s2;
  qts(c0, c1, s0, s1);
  qts(s1, c2, u, s2);
  if (kFast == 1) rare.need_nz(s1, s2);
  if (kFast == 2) {
    // path A only (all three forward residuals nonzero, eft.hpp:255-257):
    // no selects; path B (s3 == 0) and C/D count as rare
    double v, s3;
    qts(s2, c3, v, s3);
    rare.need_nz(s1, s2, s3);
    r0 = s0;
    r1 = u;
    r2 = v;
    r3 = add(s3, c4);
    return;
  }
  if (kFast == 1 && kTrunc3) {
    // paths A/B when the fourth output is dropped (td_add_q): path A keeps
    // r2 = v, path B folds c4 into it -- the same add either way, one select
    double v, s3;
    qts(s2, c3, v, s3);
    r0 = s0;
    r1 = u;
    r2 = sel(nz(s3), v, add(v, c4));
    r3 = 0.0;  // not an output (the caller truncates)
    return;
  }
  if (kFast == 1 || (nz(s1) & nz(s2))) {
    // path A (s3 != 0: s3 += c4) or path B (s3 == 0: s2 += c4), eft.hpp:255-260
    double v, s3;
    qts(s2, c3, v, s3);
    const bool p = nz(s3);
    const double acc = add(sel(p, s3, v), c4);
    r0 = s0;
    r1 = u;
    r2 = sel(p, v, acc);
    r3 = sel(p, acc, s3);
    return;
  }
  // paths C/D and the zero-residual corners, eft.hpp:261-286, verbatim
  s2 = 0.0;
  double s3 = 0.0;
  if (nz(s1)) {
    // here the residual of qts(s1, c2) was zero: eft.hpp:261-268
    s1 = u;
    qts(s1, c3, s1, s2);
    if (nz(s2)) {
      qts(s2, c4, s2, s3);
    } else {
      qts(s1, c4, s1, s2);
    }
  } else {
    qts(s0, c2, s0, s1);
    if (nz(s1)) {
      qts(s1, c3, s1, s2);
      if (nz(s2)) {
        qts(s2, c4, s2, s3);
      } else {
        qts(s1, c4, s1, s2);
      }
    } else {
      qts(s0, c3, s0, s1);
      if (nz(s1)) {
        qts(s1, c4, s1, s2);
      } else {
        qts(s0, c4, s0, s1);
      }
    }
  }
  r0 = s0, r1 = s1, r2 = s2, r3 = s3;
}

MPFK_HD void renorm5(double c0, double c1, double c2, double c3, double c4, double& r0,
                     double& r1, double& r2, double& r3) {
  RareBool rare;
  renorm5_t<0>(c0, c1, c2, c3, c4, r0, r1, r2, r3, rare);
}

// vseb with k = 2 output slots over n = 3 inputs (the only use on the path:
// td_mul, mpf.hpp:162), eft.hpp:205-225 unrolled:
//   (a, r) = qts(e1, e2); eps = r != 0 ? r : a; (b, r2) = qts(eps, e3)
//   r != 0: out = (a, b)
//   r == 0: out = (b, r2 != 0 ? r2 : +0)    (a zero residual never lands)
MPFK_HD void vseb_2_3(double e1, double e2, double e3, double& o1, double& o2) {
  double a, r, b, r2;
  qts(e1, e2, a, r);
  const bool p = nz(r);
  qts(sel(p, r, a), e3, b, r2);
  o1 = sel(p, a, b);
  o2 = sel(p, b, sel(nz(r2), r2, 0.0));
}

// ---------------------------------------------------------------------------
// Width kernels, mpf.hpp:105-238.  Arrays are component-major (c[0] leads).
// ---------------------------------------------------------------------------

// dd_add, mpf.hpp:105-111 (11 ops).
MPFK_HD void dd_add(const double* x, const double* y, double* r) {
  double s, e;
  two_sum(x[0], y[0], s, e);
  const double w = add(x[1], y[1]);
  e = add(e, w);
  qts(s, e, r[0], r[1]);
}

// dd_mul, mpf.hpp:113-119 (9 ops; the cross terms are a plain mul+mul+add,
// not an fma).
MPFK_HD void dd_mul(const double* x, const double* y, double* r) {
  double p, e;
  two_prod(x[0], y[0], p, e);
  const double w = add(mul(x[0], y[1]), mul(x[1], y[0]));
  e = add(e, w);
  qts(p, e, r[0], r[1]);
}

// N DD multiply-adds acc[j] = dd_add(acc[j], dd_mul(a, b[j])) that share a
// (one row of a thread's micro-tile), written stage by stage across the N
// elements: the operations and their operands are exactly those of dd_mul
// followed by dd_add, element by element -- bit-identical -- only the order
// in the instruction stream differs (consecutive instructions independent,
// the shared operand a in the same slot).
template <int N>
MPFK_HD void dd_mac_row(double (&acc)[N][2], const double* a, const double (&b)[N][2]) {
  double p[N], e[N], t[N], r0[N], s[N], v[N];
#pragma unroll
  for (int j = 0; j < N; ++j) p[j] = mul(a[0], b[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = mul(a[0], b[j][1]);
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = mul(a[1], b[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = fma(a[0], b[j][0], -p[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = add(t[j], v[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = add(e[j], t[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) r0[j] = add(p[j], e[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) s[j] = add(acc[j][0], r0[j]);      // two_sum(acc0, r0): the sum
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = sub(e[j], sub(r0[j], p[j]));  // r1 of qts(p, e)
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = sub(s[j], acc[j][0]);
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = sub(s[j], v[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = add(acc[j][1], e[j]);         // w = x1 + y1
#pragma unroll
  for (int j = 0; j < N; ++j) t[j] = add(sub(acc[j][0], t[j]), sub(r0[j], v[j]));  // two_sum error
#pragma unroll
  for (int j = 0; j < N; ++j) e[j] = add(t[j], e[j]);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double hi = add(s[j], e[j]);
    acc[j][1] = sub(e[j], sub(hi, s[j]));
    acc[j][0] = hi;
  }
}

// qd_add, mpf.hpp:178-196 (63 ops + renorm5).  With Trunc3 the fourth
// output is not produced (td_add_q drops it, mpf.hpp:141), which lets the
// compiler delete the dead tail of renorm5.
template <bool Trunc3 = false, int kFast = 0, class Rare = RareBool>
MPFK_HD void qd_add(const double* x, const double* y, double* r, Rare& rare) {
  double s0, t0, s1, t1, s2, t2, s3, t3;
  two_sum(x[0], y[0], s0, t0);
  two_sum(x[1], y[1], s1, t1);
  two_sum(x[2], y[2], s2, t2);
  two_sum(x[3], y[3], s3, t3);
  two_sum(s1, t0, s1, t0);
  three_sum(s2, t0, t1, s2, t0, t1);
  three_sum2(s3, t0, t2, s3, t0);
  t0 = add(add(t0, t1), t3);
  double r3;
  renorm5_t<kFast>(s0, s1, s2, s3, t0, r[0], r[1], r[2], r3, rare);
  if (!Trunc3) r[3] = r3;
}
template <bool Trunc3 = false>
MPFK_HD void qd_add(const double* x, const double* y, double* r) {
  RareBool rare;
  qd_add<Trunc3, 0>(x, y, r, rare);
}

// qd_mul, mpf.hpp:198-238 (111 ops + renorm5), including the pre-combined
// operand pairs that keep it bitwise commutative (mpf.hpp:214-221).
template <int kFast, class Rare = RareBool>
MPFK_HD void qd_mul_t(const double* x, const double* y, double* r, Rare& rare) {
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5;
  two_prod(x[0], y[0], p0, q0);
  two_prod(x[0], y[1], p1, q1);
  two_prod(x[1], y[0], p2, q2);
  two_prod(x[0], y[2], p3, q3);
  two_prod(x[1], y[1], p4, q4);
  two_prod(x[2], y[0], p5, q5);

  three_sum(p1, p2, q0, p1, p2, q0);
  double gs, ge;
  two_sum(q1, q2, gs, ge);
  double hs, he;
  two_sum(p3, p5, hs, he);
  if (kFast) {
    // ge and he are the rounding errors of gs and hs: below p2 + gs and
    // hs + p4 unless those cancel to within an ulp
    three_sum_c_small(p2, gs, ge, p2, q1, q2, rare);
    three_sum_c_small(hs, p4, he, p3, p4, p5, rare);
  } else {
    three_sum(p2, gs, ge, p2, q1, q2);
    three_sum(hs, p4, he, p3, p4, p5);
  }

  double s0, t0, s1, t1;
  two_sum(p2, p3, s0, t0);
  two_sum(q1, p4, s1, t1);
  double s2 = add(q2, p5);
  two_sum(s1, t0, s1, t0);
  s2 = add(s2, add(t0, t1));
  s1 = add(s1, add(mul(x[0], y[3]), mul(x[3], y[0])));
  s1 = add(s1, add(mul(x[1], y[2]), mul(x[2], y[1])));
  s1 = add(s1, q0);
  s1 = add(s1, add(q3, q5));
  s1 = add(s1, q4);
  renorm5_t<kFast>(p0, p1, s0, s1, s2, r[0], r[1], r[2], r[3], rare);
}
MPFK_HD void qd_mul(const double* x, const double* y, double* r) {
  RareBool rare;
  qd_mul_t<0>(x, y, r, rare);
}

// td_add_q, mpf.hpp:135-142: zero-extend with +0, quad add, truncate.
//
// qd_add on (x0,x1,x2,+0) + (y0,y1,y2,+0) with the constant lane folded.
// Every fold is a bitwise identity of the reference sequence for finite
// operands (the EFT domain, eft.hpp:44-45):
//  * two_sum(+0, +0) = (+0, +0): s = +0, v = +0, e = (+0 - +0) + (+0 - +0).
//  * two_sum(+0, b) (first step of three_sum2(s3 = +0, t0, t2)):
//      s = +0 + b, v = s - +0 = s, s - v = +0, so
//      e = (+0 - +0) + (b - s) = +0 + (b - s), where b - s is +0 for b != -0
//      and -0 - +0 = -0 for b = -0; +0 + (+-0) = +0.  Hence (s, e) =
//      (+0 + b, +0): one add instead of six.
//  * three_sum2's error t.e + u.e = +0 + u.e, the +0 + t0 in front of it and
//    t0 + t3 with t3 = +0 only map -0 to +0, and their operands are never -0
//    (see the function body): identities too.
// 14 of td_add_q's 85 FP64 operations disappear; results are unchanged
// (tests/test_arith_host.py sweeps signed zeros against the reference).
template <int kFast, class Rare = RareBool>
MPFK_HD void td_add_q_t(const double* x, const double* y, double* r, Rare& rare) {
  double s0, t0, s1, t1, s2, t2;
  two_sum(x[0], y[0], s0, t0);
  two_sum(x[1], y[1], s1, t1);
  two_sum(x[2], y[2], s2, t2);
  two_sum(s1, t0, s1, t0);
  three_sum(s2, t0, t1, s2, t0, t1);
  // three_sum2(+0, t0, t2), eft.hpp:95-99, with the folds above.  The three
  // additions of +0 the folds leave (+0 + t0, +0 + u.e, (..) + t3) only map
  // -0 to +0, and none of their operands can be -0: a Knuth two-sum error is
  // never -0 (its last add is -0 only if both addends are, i.e. b = -0 with
  // v = s - a = +0, and then a - (s - v) = +0), so neither is a sum of two
  // such errors (t0 here is three_sum's e1 = te + ue; -0 needs both -0).
  // They are identities and are not executed: 116 operations per
  // multiply-add (tests/test_arith_host.py sweeps signed zeros against the
  // reference build).
  double s3, ue;
  two_sum(t2, t0, s3, ue);
  t0 = add(ue, t1);
  double r3;
  renorm5_t<kFast, true>(s0, s1, s2, s3, t0, r[0], r[1], r[2], r3, rare);
}
MPFK_HD void td_add_q(const double* x, const double* y, double* r) {
  RareBool rare;
  td_add_q_t<0>(x, y, r, rare);
}

// td_add_q without the folds (the literal zero-extend + qd_add); kept for
// the cross-check in tests (arith_host.cpp) and as documentation.
MPFK_HD void td_add_q_unfolded(const double* x, const double* y, double* r) {
  const double xx[4] = {x[0], x[1], x[2], 0.0};
  const double yy[4] = {y[0], y[1], y[2], 0.0};
  qd_add<true>(xx, yy, r);
}

// td_mul, mpf.hpp:146-163 (41 ops + vseb).  kFast: vseb's common case only
// (first residual nonzero: the two folds are the outputs), `rare` otherwise.
template <bool kFast, class Rare = RareBool>
MPFK_HD void td_mul_t(const double* x, const double* y, double* r, Rare& rare) {
  double z00s, z00e, z01s, z01e, z10s, z10e;
  two_prod(x[0], y[0], z00s, z00e);
  two_prod(x[0], y[1], z01s, z01e);
  two_prod(x[1], y[0], z10s, z10e);
  // vec_sum<3>(z00.e, z01.s, z10.s), eft.hpp:103-113
  double b0, b1, b2, s;
  two_sum(z01s, z10s, s, b2);
  two_sum(z00e, s, b0, b1);
  const double c = fma(x[1], y[1], b2);
  const double z31 = fma(x[0], y[2], z10e);
  const double z32 = fma(x[2], y[0], z01e);
  const double z3 = add(z31, z32);
  const double s3 = add(c, z3);
  // vec_sum<4>(z00.s, b0, b1, s3)
  double e0, e1, e2, e3;
  two_sum(b1, s3, s, e3);
  if (kFast) {
    // b0 leads the order-1 terms and z00.s is the leading product: each is
    // (all but never) at least in the binade of the sum of what lies below it
    two_sum_ordered(b0, s, s, e2, rare);
    two_sum_ordered(z00s, s, e0, e1, rare);
  } else {
    two_sum(b0, s, s, e2);
    two_sum(z00s, s, e0, e1);
  }
  r[0] = e0;
  if (kFast) {
    double a, rr, b, r2;
    qts(e1, e2, a, rr);
    rare.need_nz(rr);
    qts(rr, e3, b, r2);
    r[1] = a, r[2] = b;
  } else {
    vseb_2_3(e1, e2, e3, r[1], r[2]);
  }
}
MPFK_HD void td_mul(const double* x, const double* y, double* r) {
  RareBool rare;
  td_mul_t<false>(x, y, r, rare);
}

// merge_by_magnitude, eft.hpp:229-236: stable merge of two 3-term lists by
// nonincreasing magnitude (ties take x first), as the reference's loop
// executes it for ANY input order: take x[i] while i < 3 and (j == 3 or
// |x[i]| >= |y[j]|).
MPFK_HD void merge6(const double* x, const double* y, double* z) {
  int i = 0, j = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double xi = i == 0 ? x[0] : (i == 1 ? x[1] : x[2]);
    const double yj = j == 0 ? y[0] : (j == 1 ? y[1] : y[2]);
    const bool take_x = i < 3 && (j >= 3 || std::fabs(xi) >= std::fabs(yj));
    z[k] = take_x ? xi : yj;
    i += take_x ? 1 : 0;
    j += take_x ? 0 : 1;
  }
}

// VecSumErrBranch with k = 3 slots over n = 6 inputs (eft.hpp:205-225),
// including its early exit once the last slot is final.
// Branch-free: the slot writes are selects on (live, j); after the early
// exit the remaining quick-two-sums still execute but nothing they produce
// is kept, exactly as if the reference had returned.
MPFK_HD void vseb_3_6(const double* e, double* out) {
  double o0 = 0.0, o1 = 0.0, o2 = 0.0;
  int j = 0;
  bool live = true;  // !done
  double eps = e[0];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double s, r;
    qts(eps, e[i + 1], s, r);
    o0 = sel(live && j == 0, s, o0);
    o1 = sel(live && j == 1, s, o1);
    o2 = sel(live && j == 2, s, o2);
    const bool nzr = nz(r);
    const bool adv = live && nzr && j < 2;  // finalise slot j, open j + 1 with r
    eps = sel(live, sel(nzr, r, s), eps);   // (eps is dead once the slots are full)
    live = live && !(nzr && j >= 2);        // out of slots: drop the rest
    j += adv ? 1 : 0;
  }
  const bool tail = live && nz(eps);
  o0 = sel(tail && j == 0, eps, o0);
  o1 = sel(tail && j == 1, eps, o1);
  o2 = sel(tail && j == 2, eps, o2);
  out[0] = o0, out[1] = o1, out[2] = o2;
}

// td_add_merge, mpf.hpp:125-131: merge, distill (vec_sum<6>), compress.
MPFK_HD void td_add_merge(const double* x, const double* y, double* r) {
  double z[6], e[6];
  merge6(x, y, z);
  double s = z[5];
#pragma unroll
  for (int i = 4; i >= 0; --i) {
    double ss, ee;
    two_sum(z[i], s, ss, ee);
    e[i + 1] = ee;
    s = ss;
  }
  e[0] = s;
  vseb_3_6(e, r);
}

// td_add_merge with a ranked merge and a straight-line compress for the
// common case, the exact state machines otherwise (bit-identical):
//  * when both inputs are sorted by non-increasing magnitude (every
//    normalised TD value is), the reference's greedy merge (eft.hpp:229-236;
//    ties take x) is the stable merge: y[j] precedes x[i] iff |y[j]| >
//    |x[i]|, so each element's output slot is its index plus a count of
//    comparisons -- nine compares and a scatter through `zb` (slot k at
//    zb[k * zstride]: per-thread shared memory on the device) instead of six
//    rounds of data-dependent selects;
//  * vseb(3 of 6) (eft.hpp:205-225) with the first three residuals nonzero
//    emits the first three folds and returns: three quick-two-sums.
// Unsorted inputs or a zero residual take merge6 / vseb_3_6 above.
MPFK_HD void td_add_merge_ranked(const double* x, const double* y, double* r, double* zb, int zstride) {
  const double ax0 = std::fabs(x[0]), ax1 = std::fabs(x[1]), ax2 = std::fabs(x[2]);
  const double ay0 = std::fabs(y[0]), ay1 = std::fabs(y[1]), ay2 = std::fabs(y[2]);
  double z[6];
  if ((ax0 >= ax1) & (ax1 >= ax2) & (ay0 >= ay1) & (ay1 >= ay2)) {
    const int px0 = 0 + (ay0 > ax0) + (ay1 > ax0) + (ay2 > ax0);
    const int px1 = 1 + (ay0 > ax1) + (ay1 > ax1) + (ay2 > ax1);
    const int px2 = 2 + (ay0 > ax2) + (ay1 > ax2) + (ay2 > ax2);
    const int py0 = 0 + (ax0 >= ay0) + (ax1 >= ay0) + (ax2 >= ay0);
    const int py1 = 1 + (ax0 >= ay1) + (ax1 >= ay1) + (ax2 >= ay1);
    const int py2 = 2 + (ax0 >= ay2) + (ax1 >= ay2) + (ax2 >= ay2);
    zb[px0 * zstride] = x[0];
    zb[px1 * zstride] = x[1];
    zb[px2 * zstride] = x[2];
    zb[py0 * zstride] = y[0];
    zb[py1 * zstride] = y[1];
    zb[py2 * zstride] = y[2];
#pragma unroll
    for (int k = 0; k < 6; ++k) z[k] = zb[k * zstride];
  } else {
    merge6(x, y, z);
  }
  double e[6];
  double s = z[5];
#pragma unroll
  for (int i = 4; i >= 0; --i) {
    double ss, ee;
    two_sum(z[i], s, ss, ee);
    e[i + 1] = ee;
    s = ss;
  }
  e[0] = s;
  double o0, r1, o1, r2, o2, r3;
  qts(e[0], e[1], o0, r1);
  qts(r1, e[2], o1, r2);
  qts(r2, e[3], o2, r3);
  if (nz(r1) & nz(r2) & nz(r3)) {
    r[0] = o0, r[1] = o1, r[2] = o2;
  } else {
    vseb_3_6(e, r);
  }
}

// td_mul_q, mpf.hpp:167-174: zero-extend, quad multiply, truncate (not a
// library default; the comparison kernel of the paper's TD table).
MPFK_HD void td_mul_q(const double* x, const double* y, double* r) {
  const double xx[4] = {x[0], x[1], x[2], 0.0};
  const double yy[4] = {y[0], y[1], y[2], 0.0};
  double rr[4];
  qd_mul(xx, yy, rr);
  r[0] = rr[0], r[1] = rr[1], r[2] = rr[2];
}

// Library width defaults, mpf.hpp:242-260.
template <int W>
MPFK_HD void mp_add(const double* x, const double* y, double* r) {
  if constexpr (W == 2) dd_add(x, y, r);
  else if constexpr (W == 3) td_add_q(x, y, r);
  else qd_add<false>(x, y, r);
}

template <int W>
MPFK_HD void mp_mul(const double* x, const double* y, double* r) {
  if constexpr (W == 2) dd_mul(x, y, r);
  else if constexpr (W == 3) td_mul(x, y, r);
  else qd_mul(x, y, r);
}

// GEMM inner-loop forms: kRenorm = renorm5_t level (0 exact, 1 paths A/B,
// 2 path A), kVseb = td_mul's vseb common case only; `rare` reports an input
// that left the fast form (the result must then be recomputed exactly).  DD
// has no data-dependent branch, so its fast form is the exact one.
template <int W, int kRenorm, class Rare>
MPFK_HD void mp_add_f(const double* x, const double* y, double* r, Rare& rare) {
  if constexpr (W == 2) dd_add(x, y, r);
  else if constexpr (W == 3) td_add_q_t<kRenorm>(x, y, r, rare);
  else qd_add<false, kRenorm>(x, y, r, rare);
}

template <int W, int kRenorm, bool kVseb, class Rare>
MPFK_HD void mp_mul_f(const double* x, const double* y, double* r, Rare& rare) {
  if constexpr (W == 2) dd_mul(x, y, r);
  else if constexpr (W == 3) td_mul_t<kVseb>(x, y, r, rare);
  else qd_mul_t<kRenorm>(x, y, r, rare);
}

// Algorithmic FP64 operations per multiply-add (reference sequence, renorm5
// path A): the roofline numerator.
template <int W>
constexpr int ops_per_mac() {
  return W == 2 ? 20 : (W == 3 ? 132 : 218);
}

}  // namespace arith
}  // namespace mpfk
