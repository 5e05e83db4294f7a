// mcf_exp.cuh -- correctly rounded binary64 exp on the device.
//
// Exp-MCN's lead factor is the binary64 exponential of x_0 spread over nc
// components (mc_ops.hpp:303-313), and fl_exp<P> rounds a binary64 exp into P
// (precision.hpp:191-192).  The reference takes these from the host libm,
// which is not correctly rounded; CUDA's exp() is not either.  The GPU path
// computes the correctly rounded binary64 value instead:
//   fast path: x = m*ln2 + j*ln2/2048 + r, |r| <= ln2/4096, 2^(j/2048) from a
//   double-double table, exp(r) to ~2^-89 relative, then a rounding test
//   (Ziv): if the result is within the error bound of a binary64 midpoint,
//   or |x| > 704, the slow path re-evaluates with a full double-double
//   Taylor series (~2^-100) and rounds with explicit subnormal handling.
// The oracle's CR mode (oracle/mcf_oracle.c, binary128 expq + rounding test)
// is the matching checker; elements whose libm exp differs from the
// correctly rounded one are the only permitted differences from the
// unmodified reference (SURVEY 8a row E-exp).
#pragma once

#include <stdint.h>

namespace mcfg {

// 2^(j/2048) as (hi, lo), filled once per device from binary128 (capi.cpp)
static __device__ double2 g_exp_tab[2048];

namespace expd {

// ln2/2048 = L1 + L2 + L3, L1/L2 with 31 significant bits so k*L1, k*L2 are exact
constexpr double kL1 = 0x1.62e42fec00000p-12;
constexpr double kL2 = 0x1.d1cf79a800000p-43;
constexpr double kL3 = 0x1.e4f1d9cc01f98p-74;
constexpr double kInvL = 0x1.71547652b82fep+11;  // 2048/ln2

__device__ __forceinline__ void fast2(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}
__device__ __forceinline__ void two2(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bv = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bv)), __dsub_rn(b, bv));
}
__device__ __forceinline__ void dd_mul(double ah, double al, double bh, double bl, double& h,
                                       double& l) {
  const double p = __dmul_rn(ah, bh);
  double e = __fma_rn(ah, bh, -p);
  e = __fma_rn(ah, bl, e);
  e = __fma_rn(al, bh, e);
  fast2(p, e, h, l);
}
__device__ __forceinline__ void dd_add(double ah, double al, double bh, double bl, double& h,
                                       double& l) {
  double s, e;
  two2(ah, bh, s, e);
  e = __dadd_rn(e, __dadd_rn(al, bl));
  fast2(s, e, h, l);
}

// reduction x = (m*2048 + j) * ln2/2048 + (rh + rl)
__device__ __forceinline__ void reduce(double x, int& k, double& rh, double& rl) {
  const double kd = rint(__dmul_rn(x, kInvL));
  k = (int)kd;
  const double r0 = __fma_rn(-kd, kL1, x);  // exact (k*L1 exact, Sterbenz)
  const double p2 = __dmul_rn(kd, kL2);
  const double e2 = __fma_rn(kd, kL2, -p2);
  double s, e;
  two2(r0, -p2, s, e);
  e = __dsub_rn(e, e2);
  e = __fma_rn(-kd, kL3, e);
  fast2(s, e, rh, rl);
}

// true when (yh + yl) may round to a different binary64 than yh, given a
// relative error bound `rel` on yh + yl (yh normal, positive, yh = RN(yh+yl)).
__device__ __forceinline__ bool near_midpoint(double yh, double yl, double rel) {
  const int64_t bits = __double_as_longlong(yh);
  const int ex = (int)((bits >> 52) & 0x7ff);
  const double ulp = __longlong_as_double((int64_t)(ex - 52) << 52);  // 2^(e-52)
  const bool pow2 = (bits & ((1LL << 52) - 1)) == 0;
  const double half = (yl < 0.0 && pow2) ? 0.25 * ulp : 0.5 * ulp;
  return fabs(fabs(yl) - half) <= rel * yh;
}

static __device__ __noinline__ double slow(double x) {
  if (x > 709.7827128933841) return __longlong_as_double(0x7ff0000000000000LL);
  if (x < -745.2) return 0.0;
  int k;
  double rh, rl;
  reduce(x, k, rh, rl);
  // exp(r) = sum_{n<=13} r^n / n!, Horner in double-double
  double ph = 1.0, pl = 0.0;
  double fact = 6227020800.0;  // 13!
  {
    const double ch = __ddiv_rn(1.0, fact);
    ph = ch;
    pl = __ddiv_rn(__fma_rn(-ch, fact, 1.0), fact);
  }
  for (int n = 12; n >= 0; --n) {
    fact = fact / (double)(n + 1);  // exact: n! for n <= 13
    const double ch = __ddiv_rn(1.0, fact);
    const double cl = __ddiv_rn(__fma_rn(-ch, fact, 1.0), fact);
    double th, tl;
    dd_mul(ph, pl, rh, rl, th, tl);
    dd_add(th, tl, ch, cl, ph, pl);
  }
  const int j = k & 2047;
  const int m = (k - j) >> 11;
  const double2 t = g_exp_tab[j];
  double yh, yl;
  dd_mul(t.x, t.y, ph, pl, yh, yl);
  if (m >= -1021) {
    // normal result (or overflow): scale in two exact steps
    const int m1 = m / 2, m2 = m - m1;
    return scalbn(scalbn(yh, m1), m2);
  }
  // subnormal result: round (yh + yl) * 2^(m + 1074) to an integer, RN-even
  const int sc = m + 1074;
  if (sc < -60) return 0.0;
  const double vh = scalbn(yh, sc), vl = scalbn(yl, sc);
  double n = rint(vh);
  const double d = __dadd_rn(__dsub_rn(vh, n), vl);
  if (d > 0.5) n += 1.0;
  else if (d < -0.5) n -= 1.0;
  else if (d == 0.5 || d == -0.5) n = (fmod(n, 2.0) == 0.0) ? n : n + (d > 0 ? 1.0 : -1.0);
  return scalbn(n, -1074);
}

}  // namespace expd

// RN(ln2/2048 - kL1) to 53 bits: k * kL2F rounds once inside an fma
constexpr double kL2F = 0x1.d1cf79abc9e3bp-43;

// RN64(exp(x)) from a short evaluation (~2^-63.9 relative: reduction rounding
// 2^-65.5, degree-4 truncation 2^-69, evaluation 2^-66, table product 2^-66,
// dropped tl * p 2^-65.5) with no retry: returns false when the value could
// lie within 2^-61 of a binary64 midpoint (about 2^-8 of arguments) or
// |x| > 704; the caller then takes the correctly rounded path below.
__device__ __forceinline__ bool rn_exp_fast(double x, double& E) {
  using namespace expd;
  const double kd = rint(__dmul_rn(x, kInvL));
  const int k = (int)kd;
  const double rh = __fma_rn(-kd, kL1, x);  // exact
  const double r = __fma_rn(-kd, kL2F, rh);
  double p = __fma_rn(r, 1.0 / 24.0, 1.0 / 6.0);
  p = __fma_rn(r, p, 0.5);
  p = __fma_rn(__dmul_rn(r, r), p, r);  // exp(r) - 1
  const int j = k & 2047;
  const int m = (k - j) >> 11;
  const double2 t = g_exp_tab[j];
  double yh, yl;
  fast2(t.x, __fma_rn(t.x, p, t.y), yh, yl);
  E = __dmul_rn(yh, __longlong_as_double((long long)(m + 1023) << 52));
  return (fabs(x) <= 704.0) && !near_midpoint(yh, yl, 0x1p-61);
}

__device__ __forceinline__ double cr_exp(double x) {
  using namespace expd;
  if (!(fabs(x) <= 704.0)) {
    if (x != x) return __dadd_rn(x, x);
    return slow(x);
  }
  if (fabs(x) <= 0x1p-54) return 1.0;
  int k;
  double rh, rl;
  reduce(x, k, rh, rl);
  double ah = __dmul_rn(rh, rh);
  const double al = __fma_rn(rh, rh, -ah);
  const double sq_h = 0.5 * ah;                           // exact
  const double sq_l = __fma_rn(rh, rl, 0.5 * al);          // r^2/2 residue
  double poly = __fma_rn(rh, 1.0 / 720.0, 1.0 / 120.0);
  poly = __fma_rn(rh, poly, 1.0 / 24.0);
  poly = __fma_rn(rh, poly, 1.0 / 6.0);
  poly = __dmul_rn(__dmul_rn(ah, rh), poly);              // r^3/6 + r^4/24 + ...
  const double small = __dadd_rn(__dadd_rn(rl, sq_l), poly);
  double s, e1, e2;
  fast2(1.0, rh, s, e1);
  two2(s, sq_h, s, e2);
  const double lo = __dadd_rn(__dadd_rn(e1, e2), small);
  const int j = k & 2047;
  const int m = (k - j) >> 11;
  const double2 t = g_exp_tab[j];
  const double ph = __dmul_rn(t.x, s);
  double pl = __fma_rn(t.x, s, -ph);
  pl = __dadd_rn(pl, __fma_rn(t.x, lo, __dmul_rn(t.y, s)));
  double yh, yl;
  fast2(ph, pl, yh, yl);
  if (near_midpoint(yh, yl, 0x1p-88)) return slow(x);
  // |x| <= 704: |m| <= 1016, 2^m and the result are normal, so the product is exact
  return __dmul_rn(yh, __longlong_as_double((long long)(m + 1023) << 52));
}

}  // namespace mcfg
