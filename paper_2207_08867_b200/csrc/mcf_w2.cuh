// mcf_w2.cuh -- certified nc = 2 long division in a WIDE format (binary32
// components carried in binary64): Div-MCN, DivN and Mul-MCN (fast) of
// mc_ops.hpp:188-230 with every exact intermediate held in one wide value.
//
// Formats.  P = significand bits of the component format (24), W = those of
// the wide format (53 = 2 P + 5).  A wide value is "P-bit" when it is a
// component value.  rnp(t) rounds a wide t to P bits, nearest-even.
//
// What the reference computes (div_kernel, nc = 2; x, y compressed pairs, all
// renormalizations ending compressed -- tools/g2_verify.cpp checks that they
// do on these term sets -- and no component under- or overflowing):
//   r = x;  for d = 0, 1:  q_d = fl(r_0 / y_0)
//                          (s_0, s_1) = first two components of the compressed
//                                       expansion of q_d (y_0 + y_1)    [scale_raw + renorm]
//                          r = first two components of the compressed
//                              expansion of r - s_0 - s_1               [add_kernel]
//   q_2 = fl(r_0 / y_0);  out = first two components of q_0 + q_1 + q_2.
// renorm_kernel only applies error-free two_sums and drops zeros, so each of
// these expansions sums EXACTLY to the value named.  Two facts identify the
// first two components of the compressed expansion (c_0, c_1, ...) of an
// exactly known S (mcf_g2.cuh's argument, restated on wide values):
//   (M) margin: with A = rnp(S), if |S - A| < h (1 - 2^-(P-2)), h = half the gap
//       from A to its neighbour on S's side, then c_0 = A; an exact tie (|S - A|
//       = h with S exact) gives the even neighbour, which rnp returns.  On a
//       wide S this is a test on the low W - P bits L of S's own significand:
//       |L - 2^(W-P-1)| > 2^(W-2P+1) = 64 units (a value just below a power of
//       two lies in the lower binade, whose finer grid makes the test
//       conservative); one more unit covers a wide S known to half a unit.
//       (The device declines L - mid in [-m, 3 m): one mask test.)
//   (U) uniqueness: if S fits 2 P bits (the low W - 2P bits of its wide
//       significand are zero) then (rnp(S), S - rnp(S)) is its ONLY compressed
//       expansion: another one needs c_0 = the other neighbour, |c_1| = h and
//       a c_2 of 2^-P h beyond it, i.e. more than 2 P bits.  No margin needed.
// Exactness of the wide arithmetic: the product q Y (P x W bits) is ph + pl
// (one multiply, one fma); t = (ph - rnp(ph)) + pl spans at most W bits, so it
// is exact; r - s_0 is exact (Sterbenz: s_0 is within 2^-(P-2) of r); the one
// sum that can fail to fit, (r - s_0) - s_1, is verified by recomputing both
// operands from the result (exact iff both come back).  Quotient digits are
// rnp(r_0 rY) with rY = 1 / y_0 to 2^-(W-3) (verified by its residual): the
// true quotient of two P-bit values is never a P-bit midpoint, so 16 units of
// margin certify the digit.
// Anything else -- a failed test, operands outside a +-2^40 window (so that
// nothing over- or underflows: the reference's products must have exact low
// parts, |q y| >= 2^-100, and its digits must be normal), non-compressed or
// non-finite operands -- returns false and the caller falls back to the
// binary32 tier (mcf_g2.cuh), then the register and literal paths.
//
// Policy V: N (component type), W (wide type), wide(N), narrow(W) (exact on
// P-bit values), add/sub/mul/fma/neg/abs on W, rcp_seed(W) (any approximation
// of 1/y good to ~2^-16), rnpm(W, m, ok) (rnp, and ok &= L - mid outside [-m, 3 m)),
// rnpv(W, ref, lg, ok) (rnp with the absolute margin |ref| 2^(lg - (W-1))), span2p(W) (fits 2 P bits), eq/ge/le on W, c(double), two(k) = 2^k,
// rnpe (nearest-even), in_window / below_window / lead_window / tail_window on N, kP.
#pragma once

#include "mcf_g2.cuh"

namespace mcfg {
namespace w2 {

template <class V>
using W_ = typename V::W;
template <class V>
using N_ = typename V::N;

// 1 / y0 to within 2^-(W-3) relative (checked), from a seed good to 2^-16
template <class V>
G2_HD bool recip(W_<V> y0, W_<V> seed, W_<V>& r) {
  const W_<V> one = V::c(1.0);
  W_<V> e = V::fma(V::neg(y0), seed, one);
  r = V::fma(seed, e, seed);
  e = V::fma(V::neg(y0), r, one);
  r = V::fma(r, e, r);
  e = V::fma(V::neg(y0), r, one);
  return V::le(V::abs(e), V::tol_rcp());
}

// one digit of the long division: q = fl(r0 / y0), r <- r - trunc2(q (y0 + y1)).
// PAIR = false: Y = y0 + y1 is one wide value (Y1 unused) and the product's
// remainder t below s0 is exact.
// PAIR = true: the divisor stays a pair (y0 + y1 need not fit the wide
// format: Mul-MCN's reciprocal); q y0 and q y1 are exact wide products, their
// sum is (ph, pl) by a fast two-sum (|y1| <= 2^-P |y0|), and t is known to
// half a unit.  Either way 64 units of margin (strictly more: 65) certify s1.
template <class V, bool PAIR>
G2_HD bool digit(W_<V>& r, W_<V>& r0, W_<V> Y, W_<V> Y1, W_<V> rY, W_<V>& q) {
  using W = W_<V>;
  const W qt = V::mul(r0, rY);
  bool ok = true;
  q = V::rnpm(qt, 16, ok);
  W ph, pl;
  if constexpr (PAIR) {
    const W p0 = V::mul(q, Y), p1 = V::mul(q, Y1);  // exact (P x P bits)
    ph = V::add(p0, p1);
    pl = V::sub(p1, V::sub(ph, p0));               // exact (Dekker)
  } else {
    ph = V::mul(q, Y);
    pl = V::fma(q, Y, V::neg(ph));                 // q Y = ph + pl exactly
  }
  const W s0 = V::rnpm(ph, 64, ok);           // (M), |pl| <= half a unit
  const W t = V::add(V::sub(ph, s0), pl);     // q (y0 + y1) - s0 (exact unless PAIR: then to half a unit)
  const W s1 = V::rnpm(t, 64, ok);            // (M) below s0 (a tie is declined)
  const W u = V::sub(r, s0);                  // exact (Sterbenz); |u| <= 2^-(P-2) |r0| (1 + 2^-(P-3))
  const W v = V::sub(u, s1);
  // v is exact when s1's last place is within W bits of v's first:
  // |v| < 2^-(P-4) |r0| and u is a multiple of r's last place, so it is when
  // |s1| >= 2^-2P |r0| (or s1 = 0)
  ok &= V::ge(V::abs(s1), V::mul(V::abs(r0), V::two(-2 * V::kP))) | V::eq(s1, V::c(0.0));
  ok &= V::span2p(v);                         // (U): (rnpe(v), v - rnpe(v)) is the new remainder
  r = v;
  r0 = V::rnpe(v);
  return ok;
}

// x / y for wide X = x0 + x1 (x0 = X0 its lead) and the divisor as digit()
// takes it; Yl = the last nonzero component of y.  Results are P-bit wide values.
template <class V, bool PAIR>
G2_HD bool div_core(W_<V> X, W_<V> X0, W_<V> Y, W_<V> Y1, W_<V> Yl, W_<V> rY, W_<V>& o0, W_<V>& o1) {
  using W = W_<V>;
  W r = X, r0 = X0, q0, q1;
  bool ok = digit<V, PAIR>(r, r0, Y, Y1, rY, q0);
  ok &= digit<V, PAIR>(r, r0, Y, Y1, rY, q1);
  const W qt = V::mul(r0, rY);
  const W q2 = V::rnpm(qt, 16, ok);
  // out = first two components of S = q0 + q1 + q2.  u = fl(q1 + q2) and
  // Q = fl(q0 + u) are within 0.51 units of Q's last place of S; with
  // a = q0 - o0 (exact: zero or a step or two of q0's grid), a + q1 is exact
  // (a != 0 needs |q1 + q2| >= h(q0) (1 - 2^-20), so with |q2| <= |q1| both
  // are multiples of 2^-(2P+2) |q0| below 8 steps) and w = fl((a + q1) + q2)
  // is within half a unit of S - o0.
  ok &= V::ge(V::abs(q1), V::abs(q2));
  const W Q = V::add(q0, V::add(q1, q2));
  o0 = V::rnpm(Q, 64, ok);
  const W w = V::add(V::add(V::sub(q0, o0), q1), q2);
  o1 = V::rnpm(w, 64, ok);
  // range guards (the reference's arithmetic has a bounded exponent; the
  // callers keep |y0| and |x0| inside 2^+-40): every product q_d y_j must have
  // an exact low part and every digit must be normal.  The smallest product is
  // (last nonzero of q0, q1) x (last nonzero of y); at 2^-86 it also makes that
  // digit normal (|y| <= 2^40).  q2 is only ever divided out: normal or zero.
  const W zero = V::c(0.0);
  const W ql = V::eq(q1, zero) ? q0 : q1;
  ok &= V::ge(V::abs(V::mul(ql, Yl)), V::two(-86)) | V::eq(q0, zero);
  ok &= V::eq(q2, zero) | V::ge(V::abs(q2), V::two(-126));
  return ok;
}


// The same division with ONE explicit digit.  After digit 0 the reference holds
// r = X - trunc2(q0 (y0 + y1)) exactly (digit() checks it), and what it adds to
// q0 is q1 + q2 with q1 = fl(r_0 / y_0), r' = trunc2(r - trunc2(q1 Y)), q2 =
// fl(r'_0 / y_0).  With u = 2^-P (every rounding to P bits and every lead of a
// compressed pair is within u, relative; a two-component truncation within
// u^2 (1 + u)):  q1 = (r / Y)(1 + t1), |t1| <= 3 u;  r' = (r - q1 Y (1 + e1))(1 + e2);
// q2 = (r' / Y)(1 + t2), so
//   |q1 + q2 - r / Y| <= |r / Y| (|t1| (|e2| + |t2|) + |e1|) (1 + O(u)) <= 10 u^2 |r / Y| (1 + O(u)).
// R = r rY (1 - y1 rY) is r / Y to u^2 (the dropped (y1 / y0)^2) + 2^-(W-3) (rY)
// + three wide roundings, so S = q0 + q1 + q2 = q0 + R to within 11.3 u^2 |R|:
// at most 11.3 x 2 x 2^(W-1-2P) = 362 units of R's last wide place.  The two
// components of S then follow from (M) as in div_core, the second with an
// absolute margin of |R| 2^(10 - (W-1)) >= 2^10 units of R's last place: 362, plus
// the 64 units of (M) and the rounding of w = (q0 - o0) + R in w's own last
// place, which is at most twice R's (|w| <= half a step of o0 <= |R| (1 + 2^-20)
// whenever q0 != o0) -- and usually far below it: rnpv measures the margin
// against w's own P-bit grid.
// No q1, q2, second product or second remainder: ~2/3 of the instructions.
// Guards: |R| >= 2^-60 keeps q1 normal and makes a subnormal q2's rounding
// (<= 2^-150) invisible at w's resolution; |R Yl| >= 2^-85 is the exact-low-part
// guard for both digits' products (|q1| <= |q0|; R = q1 (1 + 2^-21)).
template <class V, bool PAIR>
G2_HD bool div_core1(W_<V> X, W_<V> X0, W_<V> Y, W_<V> Y1, W_<V> Yl, W_<V> rY, W_<V>& o0, W_<V>& o1) {
  using W = W_<V>;
  W r = X, r0 = X0, q0;
  bool ok = digit<V, PAIR>(r, r0, Y, Y1, rY, q0);
  const W c = V::mul(Y1, rY);
  const W R0 = V::mul(r, rY);
  const W R = V::fma(V::neg(R0), c, R0);
  const W Q = V::add(q0, R);
  o0 = V::rnpm(Q, 64, ok);
  const W w = V::add(V::sub(q0, o0), R);
  o1 = V::rnpv(w, R, V::lg1(), ok);
  ok &= V::ge(V::abs(R), V::two(-60));
  ok &= V::ge(V::abs(V::mul(R, Yl)), V::two(-85));
  return ok;
}

// mc_ops.hpp:188-207 div_kernel, nc = 2; cx / cy = the reference's compressed
// predicate fl(c0 + c1) == c0 evaluated by the caller in the component format
template <class V, bool X1ZERO, bool ONE = false>
G2_HD bool div(N_<V> x0, N_<V> x1, N_<V> y0, N_<V> y1, bool cx, bool cy, N_<V>& o0, N_<V>& o1) {
  using W = W_<V>;
  const W zero = V::c(0.0);
  const W X0 = V::wide(x0), Y0 = V::wide(y0), Y1 = V::wide(y1);
  W X = X0;
  bool ok = cx & cy;
  if constexpr (!X1ZERO) {
    const W X1 = V::wide(x1);
    X = V::add(X0, X1);
    ok &= V::eq(V::sub(X, X0), X1);           // x0 + x1 fits the wide format
  }
  const W Y = V::add(Y0, Y1);
  ok &= V::eq(V::sub(Y, Y0), Y1);
  ok &= V::in_window(y0) & V::below_window(x0);  // a tiny x0 fails the product guard of div_core
  W rY;
  ok &= recip<V>(Y0, V::rcp_seed(Y0), rY);
  const W Yl = V::eq(Y1, zero) ? Y0 : Y1;
  W w0, w1;
  if constexpr (ONE) ok &= div_core1<V, false>(X, X0, Y, Y1, Yl, rY, w0, w1);
  else ok &= div_core<V, false>(X, X0, Y, Y1, Yl, rY, w0, w1);
  o0 = V::canon(V::narrow(w0));
  o1 = V::canon(V::narrow(w1));
  return ok;
}

// mc_ops.hpp:216-230 Mul-MCN (fast): x / (1 / y), zero fast path decided by
// the caller (zx / zy: approx(x) == 0, approx(y) == 0)
template <class V, bool ONE = false>
G2_HD bool mul(N_<V> x0, N_<V> x1, N_<V> y0, N_<V> y1, bool cx, bool cy, N_<V>& o0, N_<V>& o1) {
  using W = W_<V>;
  const W zero = V::c(0.0), one = V::c(1.0);
  const W X0 = V::wide(x0), X1 = V::wide(x1), Y0 = V::wide(y0), Y1 = V::wide(y1);
  const W X = V::add(X0, X1), Y = V::add(Y0, Y1);
  bool ok = cx & cy & V::eq(V::sub(X, X0), X1) & V::eq(V::sub(Y, Y0), Y1);
  ok &= V::in_window(y0) & V::below_window(x0);  // a tiny x0 fails the product guard of div_core
  W rY;
  ok &= recip<V>(Y0, V::rcp_seed(Y0), rY);
  const W Yl = V::eq(Y1, zero) ? Y0 : Y1;
  W c0, c1;
  if constexpr (ONE) ok &= div_core1<V, false>(one, one, Y, Y1, Yl, rY, c0, c1);
  else ok &= div_core<V, false>(one, one, Y, Y1, Yl, rY, c0, c1);  // recip = 1 / y (compressed by construction)
  W rC;
  ok &= recip<V>(c0, Y0, rC);                           // 1 / c0 ~ y0 (to 2^-(P-1)): seed y0
  const W Cl = V::eq(c1, zero) ? c0 : c1;
  W w0, w1;
  if constexpr (ONE) ok &= div_core1<V, true>(X, X0, c0, c1, Cl, rC, w0, w1);
  else ok &= div_core<V, true>(X, X0, c0, c1, Cl, rC, w0, w1);
  o0 = V::canon(V::narrow(w0));
  o1 = V::canon(V::narrow(w1));
  return ok;
}

// First two components of the compressed expansion of X F (X = x0 + x1 exact in
// the wide format, F a P-bit value): scale_raw + renorm_kernel of
// mc_ops.hpp:143-169 for nc = 2 -> 2.  The product is ph + pl exactly, its
// remainder below o0 spans at most W bits (exact), (M) twice.
template <class V>
G2_HD bool scale_core(W_<V> X, W_<V> F, W_<V>& o0, W_<V>& o1) {
  using W = W_<V>;
  bool ok = true;
  const W ph = V::mul(X, F);
  const W pl = V::fma(X, F, V::neg(ph));
  o0 = V::rnpm(ph, 64, ok);
  const W t = V::add(V::sub(ph, o0), pl);
  o1 = V::rnpm(t, 64, ok);
  return ok;
}

// ScalingN nc = 2 -> 2 on component operands (cx = x compressed); products
// must have exact low parts: the smaller one, |x1 v| (or |x0 v| when x1 = 0),
// at least 2^-100, or zero because a factor is; the lead below 2^100
template <class V>
G2_HD bool scale(N_<V> x0, N_<V> x1, N_<V> v, bool cx, N_<V>& o0, N_<V>& o1) {
  using W = W_<V>;
  const W zero = V::c(0.0);
  const W X0 = V::wide(x0), X1 = V::wide(x1), F = V::wide(v);
  const W X = V::add(X0, X1);
  bool ok = cx & V::eq(V::sub(X, X0), X1);
  const W xs = V::eq(X1, zero) ? X0 : X1;
  const W sm = V::abs(V::mul(xs, F));
  ok &= V::ge(sm, V::two(-100)) | V::eq(sm, zero);
  ok &= V::le(V::abs(V::mul(X0, F)), V::two(100));
  W w0, w1;
  ok &= scale_core<V>(X, F, w0, w1);
  o0 = V::canon(V::narrow(w0));
  o1 = V::canon(V::narrow(w1));
  return ok;
}

// mc_ops.hpp:234-251 mul_slow_kernel, nc = 2 (Mul-MCN, the direct product): the
// seven terms two_prod(x0, y0), two_prod(x0, y1), two_prod(x1, y0) and the guard
// product fl(x1 y1) sum EXACTLY to S = X Y - x1 y1 + fl(x1 y1), and the result is
// the first two components of S's compressed expansion (renorm_kernel; (M)).
// Wide: X Y = ph + pl exactly (one multiply, one fma); x1 y1 is exact in the wide
// format (P x P bits), so c = rnpe(x1 y1) - x1 y1 is; pl + c rounds far below a
// unit of what is tested (|pl + c| <= 2^-(W-1) |ph| (1 + 2^-(P-4))), and t = (ph -
// o0) + (pl + c) is known to half a unit: 65 units of margin, as digit<PAIR>.
// Guards (cx / cy: compressed operands, by the caller): X and Y single wide
// values; every product with an exact low part and the guard product normal --
// leads inside 2^[-30, 40], second components zero or at least 2^-60.
template <class V>
G2_HD bool mul_slow(N_<V> x0, N_<V> x1, N_<V> y0, N_<V> y1, bool cx, bool cy, N_<V>& o0, N_<V>& o1) {
  using W = W_<V>;
  const W X0 = V::wide(x0), X1 = V::wide(x1), Y0 = V::wide(y0), Y1 = V::wide(y1);
  const W X = V::add(X0, X1), Y = V::add(Y0, Y1);
  bool ok = cx & cy & V::eq(V::sub(X, X0), X1) & V::eq(V::sub(Y, Y0), Y1);
  ok &= V::lead_window(x0) & V::lead_window(y0) & V::tail_window(x1) & V::tail_window(y1);
  const W ph = V::mul(X, Y);
  const W pl = V::fma(X, Y, V::neg(ph));
  const W g = V::mul(X1, Y1);                       // exact
  const W pc = V::add(pl, V::sub(V::rnpe(g), g));   // pl + (fl(x1 y1) - x1 y1)
  const W w0 = V::rnpm(ph, 64, ok);
  const W t = V::add(V::sub(ph, w0), pc);
  const W w1 = V::rnpm(t, 64, ok);
  o0 = V::canon(V::narrow(w0));
  o1 = V::canon(V::narrow(w1));
  return ok;
}

// mc_ops.hpp:256-282 square_kernel, nc = 2: two_prod(x0, x0), the doubled
// two_prod(x0, x1) and fl(x1 x1) sum exactly to S = X^2 - x1^2 + fl(x1^2) -- the
// direct product with y = x (five terms instead of seven; the same value, so
// the same first two components)
template <class V>
G2_HD bool square(N_<V> x0, N_<V> x1, bool cx, N_<V>& o0, N_<V>& o1) {
  return mul_slow<V>(x0, x1, x0, x1, cx, cx, o0, o1);
}

#if defined(__CUDACC__)
// binary32 components in binary64 on sm_100a
struct VD {
  using N = float;
  using W = double;
  __device__ __forceinline__ static W c(double v) { return v; }
  __device__ __forceinline__ static W two(int k) { return __hiloint2double((1023 + k) << 20, 0); }
  __device__ __forceinline__ static W tol_rcp() { return 0x1p-50; }
  __device__ __forceinline__ static W wide(N x) { return (double)x; }
  __device__ __forceinline__ static N narrow(W x) { return __double2float_rn(x); }
  __device__ __forceinline__ static N canon(N x) { return __fadd_rn(x, 0.0f); }
  __device__ __forceinline__ static W neg(W a) { return -a; }
  __device__ __forceinline__ static W abs(W a) { return fabs(a); }
  __device__ __forceinline__ static W add(W a, W b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static W sub(W a, W b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static W mul(W a, W b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static W fma(W a, W b, W c) { return __fma_rn(a, b, c); }
  __device__ __forceinline__ static bool eq(W a, W b) { return a == b; }
  __device__ __forceinline__ static bool ge(W a, W b) { return a >= b; }
  __device__ __forceinline__ static bool le(W a, W b) { return a <= b; }
  // MUFU.RCP64H: ~20 bits from the high word
  __device__ __forceinline__ static W rcp_seed(W y) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
    return r;
  }
  static constexpr int kP = 24;
  __device__ __forceinline__ static int lg1() { return 10; }  // div_core1's margin: 2^10 units of R's last place
  __device__ __forceinline__ static bool in_window(N a) { return (fabsf(a) >= 0x1p-40f) & (fabsf(a) <= 0x1p40f); }
  __device__ __forceinline__ static bool below_window(N a) { return fabsf(a) <= 0x1p40f; }
  __device__ __forceinline__ static bool lead_window(N a) { return (fabsf(a) >= 0x1p-30f) & (fabsf(a) <= 0x1p40f); }
  __device__ __forceinline__ static bool tail_window(N a) { return (a == 0.0f) | (fabsf(a) >= 0x1p-60f); }
  // round to 24 bits on the bit pattern (sign-magnitude: add half a step to
  // the magnitude, clear the 29 low bits; a carry runs into the exponent as
  // it should).  rnp: ties away from zero (every use declines near-ties);
  // rnpe: ties to even.
  // round to 24 bits AND test the margin m (a power of two) with one 64-bit
  // add: b' = b + half + m; (b' & ~low29) is t rounded to nearest whenever t
  // is not within m units of a midpoint (L in [mid - m, mid) would round the
  // wrong way -- and is declined); the low 29 bits of b' are below 4 m exactly
  // when L is in [mid - m, mid + 3 m): one LOP3 with a predicate result.
  __device__ __forceinline__ static W rnpm(W t, int m, bool& ok) {
    const long long b = __double_as_longlong(t) + (0x10000000LL + m);
    ok &= ((unsigned)b & (0x1fffffffu & ~(4u * (unsigned)m - 1u))) != 0u;
    return __longlong_as_double(b & ~0x1fffffffLL);
  }
  // rnp(t), accepted when t is farther than |ref| 2^(lg - 52) (>= 2^lg units of
  // ref's last place) from the nearest midpoint of ITS P-bit grid: the residual
  // e = t - rnp(t) is exact, half = 2^(e(t) - 24) is half a step of that grid
  // (one mask-and-subtract on the high word; a zero or tiny t gives a negative
  // or NaN half and declines), so the distance is half - |e| -- on the FP64
  // pipe, which has more room than the ALU pipe a variable shift would use
  __device__ __forceinline__ static W rnpv(W t, W ref, int lg, bool& ok) {
    const long long b = __double_as_longlong(t) + 0x10000000LL;
    const double o = __longlong_as_double(b & ~0x1fffffffLL);
    const double e = __dsub_rn(t, o);
    const double half = __hiloint2double((__double2hiint(t) & 0x7ff00000) - (24 << 20), 0);
    ok &= __dsub_rn(half, fabs(e)) > __dmul_rn(fabs(ref), __hiloint2double((1023 + lg - 52) << 20, 0));
    return o;
  }
  // ties to even: (t + M) - M with M = 1.5 2^(e + 29), e = t's exponent; the
  // sum lies in M's binade, whose spacing 2^(e - 23) is t's 24-bit grid.  M0 =
  // 1.5 2^e is one mask-or of t's high word; the 2^29 rides on two fmas.
  __device__ __forceinline__ static W rnpe(W t) {
    const double M0 = __hiloint2double((__double2hiint(t) & 0x7ff00000) | 0x00080000, 0);
    const double s = __fma_rn(M0, 0x1p29, t);
    return __fma_rn(M0, -0x1p29, s);
  }
  __device__ __forceinline__ static bool span2p(W t) { return ((unsigned)__double2loint(t) & 0x1fu) == 0u; }
};

// the correctly rounded exp out of line: taken by the few lanes whose short
// evaluation cannot decide the binary64 rounding
static __device__ __noinline__ double cr_exp_call(double x) { return cr_exp(x); }

// mc_ops.hpp:303-313 Exp-MCN, nc = 2, in the wide format: the greedy split of
// the correctly rounded binary64 exp(x0) (expansion_of_double: two
// nearest-even roundings, no renormalization in the reference either), then
// for x1 != 0 the scaling by f = fl_exp(x1) = RN32(exp(x1)) through
// scale_core.  f comes from a degree-4 polynomial in binary64 (|x1| <= 2^-12:
// truncation <= 2^-67, evaluation ~2^-64 absolute) rounded with 16 units
// (>= 2^-50) of margin, which the double rounding through binary64 and the
// approximation cannot cross.  Branch-free: both outcomes computed, selected.
__device__ __forceinline__ bool exp_b32(float x0, float x1, float& o0, float& o1) {
  using V = VD;
  double E;
  if (!rn_exp_fast((double)x0, E)) E = cr_exp_call((double)x0);  // near a binary64 midpoint (2^-8 of arguments)
  bool ok = (E >= 0x1p-60) & (E <= 0x1p100);   // every component and product normal, finite
  const double e0 = V::rnpe(E);
  const double e1 = V::rnpe(__dsub_rn(E, e0));
  const double d = (double)x1;
  double p = __fma_rn(d, 1.0 / 24.0, 1.0 / 6.0);
  p = __fma_rn(d, p, 0.5);
  p = __fma_rn(__dmul_rn(d, d), p, d);
  bool oks = fabsf(x1) <= 0x1p-12f;
  const double f = V::rnpm(__dadd_rn(1.0, p), 16, oks);
  double s0, s1;
  oks &= scale_core<V>(__dadd_rn(e0, e1), f, s0, s1);
  oks &= (fabs(__dmul_rn(e1, f)) >= 0x1p-100) | (e1 == 0.0);
  const bool z = x1 == 0.0f;
  o0 = V::canon(V::narrow(z ? e0 : s0));
  o1 = V::canon(V::narrow(z ? e1 : s1));
  return ok & (z | oks);
}
#endif

}  // namespace w2
}  // namespace mcfg
