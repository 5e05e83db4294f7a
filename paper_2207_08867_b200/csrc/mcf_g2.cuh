// mcf_g2.cuh -- certified shortcuts for nc = 2 MCF operators (binary32 fast tier).
//
// Why this is exact.  The reference's renorm_kernel (mc_ops.hpp:68-92) only
// uses error-free two_sum steps and zero compaction, so (no overflow, no
// underflowed products) the nonzero components c_0, c_1, ... it ends with sum
// EXACTLY to S, the exact sum of its input terms.  When the loop ends because
// the sequence is compressed (fl(c_i + c_{i+1}) == c_i, mc_ops.hpp:56-62),
// every |c_{i+1}| is at most h(c_i), half the gap from c_i to its neighbour
// on c_{i+1}'s side, and h(c) <= 2^-p |c|.  Hence |S - c_0| <= h(c_0) / (1 -
// 2^-p): S lies in c_0's rounding interval widened by a factor 1 + 2^-(p-1).
// If a candidate A satisfies |S - A| < h(A) (1 - 2^-(p-1)), S is strictly
// inside A's own interval and outside every neighbour's widened one, so
// c_0 = A.  The same argument on c_1, c_2, ... (sum S - c_0) certifies c_1.
// The reference output is the first two nonzeros padded with +0, so:
//
//     out = (A, B)   whenever  |S - A| and |S - A - B| pass those margins.
//
// Each operator below computes candidates A, B and the exact remainders with
// error-free transforms (ordered so the candidates are nearly always right),
// tests the two margins, and returns false when any precondition or margin
// fails; the caller then runs the register path (mcf_fast.cuh), which replays
// the reference's passes.  That the reference loop always ends compressed on
// these term sets (it never reaches its pass cap) and that the candidates
// equal its output whenever the margins pass is checked exhaustively in small
// precisions and by sampling at p = 24 by tools/g2_verify.cpp, which runs
// this same header on an emulated-precision policy.
//
// Policy Q: T, add, sub, mul, div, fma, abs, finite, hbd(t, d) = half the gap
// from t to its neighbour on d's side, hb(t) = the smaller of the two half
// gaps (both 0 for zero / subnormal t), shrink(h) = h (1 - 2^-(p-2)), big(p) (|p| >= 2^-100:
// a product that large has an exact low part, and a quotient that large is
// normal), canon(x) (-0 -> +0, the reference's padding).
#pragma once

#if defined(__CUDACC__)
#include "mcf_exp.cuh"
#define G2_HD __host__ __device__ __forceinline__
#else
#define G2_HD inline
#endif

namespace mcfg {
namespace g2 {

template <class Q>
using T_ = typename Q::T;
template <class Q>
using B_ = typename Q::B;  // per-element flags (bool, or a pair of bools)

// eft.hpp:31-38
template <class Q>
G2_HD void two_sum(T_<Q> a, T_<Q> b, T_<Q>& s, T_<Q>& e) {
  s = Q::add(a, b);
  const T_<Q> bv = Q::sub(s, a);
  const T_<Q> av = Q::sub(s, bv);
  e = Q::add(Q::sub(a, av), Q::sub(b, bv));
}

// Dekker: exact when |a| >= |b| (or a == 0)
template <class Q>
G2_HD void fast_two_sum(T_<Q> a, T_<Q> b, T_<Q>& s, T_<Q>& e) {
  s = Q::add(a, b);
  e = Q::sub(b, Q::sub(s, a));
}

// eft.hpp:75-80
template <class Q>
G2_HD void two_prod(T_<Q> a, T_<Q> b, T_<Q>& p, T_<Q>& e) {
  p = Q::mul(a, b);
  e = Q::fma(a, b, Q::neg(p));
}

// fl(x0 + x1) == x0: the reference's compressed predicate for a pair
template <class Q>
G2_HD B_<Q> compressed(T_<Q> x0, T_<Q> x1) {
  return Q::eq(Q::add(x0, x1), x0);
}

// Certify out = (A, C1) from S = A + B + R0 + rest exactly, rest_abs >= |rest|
// (a rounded-to-nearest sum of magnitudes: the (1 - 2^-(p-2)) factor of thr
// absorbs its rounding).
//   (C1, F) = two_sum(B, R0);  S = A + C1 + F + rest
// Margins: |C1| < thr(A) certifies c_0 = A (|S - A| <= |C1| (1 + 2^-p));
//          |F| + rest < thr(C1) certifies c_1 = C1.
// Exact midpoints (frequent: a sum of two binary32 values one binade apart
// rounds with an error of exactly half an ulp): if S is exactly halfway between
// two neighbours, the only compressed expansion of S starts with the EVEN
// neighbour (an odd c_0 would need |c_1| = h, which fl(c_0 + c_1) rounds
// away, or |c_1| < h with a tail too small to reach h), i.e. c_0 = fl(A + C1)
// under ties-to-even, c_1 = the exact rest.  Same at the second level with
// C1 = fl(B + R0).  A zero candidate is only accepted when everything below it
// is zero (the reference pads +0).
// REST: a remainder beyond R0 exists; DIR: use the exact half gap on C1's
// side at the top (needed where the lead is often a power of two: the
// division's partial products q (y0 + y1) ~ r0, e.g. 1 / y); CANON: final
// output (a zero component is the reference's +0 padding).
// The all-zero case passes through the tie clauses (h = 0 for a zero lead).
// TIE0 = false drops the top-level tie clause where exact midpoints are rare
// (an exact tie there then takes the fallback).  B is usually much larger than
// R0, so (C1, F) comes from a fast two-sum guarded by |B| >= |R0|.
// SWAP: no structural order between B and R0: the fast two-sum takes the
// larger magnitude first instead of guarding.
template <class Q, bool REST, bool DIR, bool CANON, bool TIE0 = true, bool SWAP = false>
G2_HD B_<Q> finish(T_<Q> A, T_<Q> B, T_<Q> R0, T_<Q> rest_abs, T_<Q>& o0, T_<Q>& o1) {
  T_<Q> C1, F;
  const B_<Q> ge = Q::ge(Q::abs(B), Q::abs(R0));
  if (SWAP) fast_two_sum<Q>(Q::sel(ge, B, R0), Q::sel(ge, R0, B), C1, F);
  else fast_two_sum<Q>(B, R0, C1, F);
  const T_<Q> zero = Q::c(0.0);
  // tie at the top: fl(A + C1) is the even neighbour; otherwise it is A
  T_<Q> A2 = A, C2 = C1;
  if (TIE0) {
    A2 = Q::add(A, C1);
    C2 = Q::sel(Q::eq(A2, A), C1, Q::neg(C1));
  }
  const T_<Q> below = REST ? Q::add(Q::abs(F), rest_abs) : Q::abs(F);
  // half gaps: toward C2 at the top (S - A2 has C2's sign) or the smaller
  // one, and the smaller one below (exact unless C2 is a power of two)
  const T_<Q> h0 = DIR ? Q::hbd(A2, C2) : Q::hb(A2), h1 = Q::hb(C2);
  const B_<Q> z0 = Q::eq(below, zero);
  B_<Q> ok0 = Q::lt(Q::abs(C2), Q::shrink(h0));
  if (TIE0) ok0 = ok0 | (z0 & Q::eq(Q::abs(C2), h0));
  else ok0 = ok0 | (Q::eq(A2, zero) & Q::eq(C2, zero) & z0);
  B_<Q> tie1 = Q::eq(below, h1);
  if (REST) tie1 = tie1 & Q::eq(rest_abs, zero);
  const B_<Q> ok1 = Q::lt(below, Q::shrink(h1)) | tie1;
  o0 = CANON ? Q::canon(A2) : A2;
  o1 = CANON ? Q::canon(C2) : C2;
  return SWAP ? ok0 & ok1 : ok0 & ok1 & ge;
}

// exact product x v (x a compressed pair, underflow guarded by the caller)
// rounded to two components: S = A + U + w + ew after the sweep below.
// |fl(e0 + p1)| <= 2^-22 |p0| (x compressed), so the top sum is a fast one.
template <class Q, bool DIR, bool CANON, bool TIE0 = true>
G2_HD B_<Q> scale_core(T_<Q> x0, T_<Q> x1, T_<Q> v, T_<Q>& o0, T_<Q>& o1) {
  T_<Q> p0, e0, p1, e1, a, ea, A, U;
  two_prod<Q>(x0, v, p0, e0);
  two_prod<Q>(x1, v, p1, e1);
  two_sum<Q>(e0, p1, a, ea);
  fast_two_sum<Q>(p0, a, A, U);  // S = A + U + ea + e1
  // w = fl(ea + e1) (both ~2^-48 |A|) is exact up to |ew| <= 2^-p |w|; that
  // bound stands in for the exact rest (0 exactly when w == 0: the sum was exact)
  const T_<Q> w = Q::add(ea, e1);
  return finish<Q, true, DIR, CANON, TIE0>(A, U, w, Q::ulpb(w), o0, o1);
}

// mc_ops.hpp:143-169 ScalingN, nc = 2 -> 2: renorm(scale_raw(x, v)), S = x v.
// Products are exact when the smaller one, |x1 v| (or |x0 v| when x1 = 0), is
// at least 2^-100 or zero because a factor is.
template <class Q>
G2_HD B_<Q> scale(T_<Q> x0, T_<Q> x1, T_<Q> v, T_<Q>& o0, T_<Q>& o1) {
  const T_<Q> zero = Q::c(0.0);
  const T_<Q> xs = Q::sel(Q::eq(x1, zero), x0, x1);
  const B_<Q> ok = compressed<Q>(x0, x1) & (Q::big(Q::mul(xs, v)) | Q::eq(xs, zero) | Q::eq(v, zero));
  return scale_core<Q, false, true>(x0, x1, v, o0, o1) & ok & Q::finite(o0);
}

// mc_ops.hpp:118-138 Grow-ExpN, nc = 2: the ladder (two exact two-sums from
// the smallest component up) gives S = h0 + h1 + h2 exactly; its compressed
// shortcut equals renorm_kernel whenever it applies, so the certificate on
// (h0, h1, h2) is the reference's result.
// (h1 + h2 can reach past h0's rounding interval when v is as large as x0:
// the top is re-rounded with the tail first, as in add.)
template <class Q>
G2_HD B_<Q> grow(T_<Q> x0, T_<Q> x1, T_<Q> v, T_<Q>& o0, T_<Q>& o1) {
  T_<Q> q, h0, h1, h2, u, g, A, U;
  two_sum<Q>(x1, v, q, h2);
  two_sum<Q>(x0, q, h0, h1);
  two_sum<Q>(h1, h2, u, g);
  two_sum<Q>(h0, u, A, U);  // S = A + U + g
  return finish<Q, false, false, true, true, true>(A, U, g, Q::c(0.0), o0, o1) & compressed<Q>(x0, x1) &
         Q::finite(o0);
}

// mc_ops.hpp:173-184 add_kernel, nc = 2 -> 2 (Add-MCN; also the MLP's bias
// add): S = x0 + x1 + y0 + y1 through four exact two-sums, the top candidate
// re-rounded with the tail (A = fl(s + u)), the last two error terms bounded.
template <class Q, bool CANON = true>
G2_HD B_<Q> add(T_<Q> x0, T_<Q> x1, T_<Q> y0, T_<Q> y1, T_<Q>& o0, T_<Q>& o1) {
  T_<Q> s, e, t, f, u, g, A, U;
  two_sum<Q>(x0, y0, s, e);
  two_sum<Q>(x1, y1, t, f);
  two_sum<Q>(e, t, u, g);  // S = s + u + g + f
  two_sum<Q>(s, u, A, U);  // S = A + U + g + f
  // w = fl(g + f) is exact when either term is zero (frequent: f is often
  // an exact half-ulp tie residue with g = 0), else within 2^-p |w|
  const T_<Q> zero = Q::c(0.0);
  const T_<Q> w = Q::add(g, f);
  const T_<Q> rest = Q::sel(Q::eq(g, zero) | Q::eq(f, zero), zero, Q::ulpb(w));
  const B_<Q> ok = compressed<Q>(x0, x1) & compressed<Q>(y0, y1);
  return finish<Q, true, false, CANON, true, true>(A, U, w, rest, o0, o1) & ok & Q::finite(o0);
}

// mc_ops.hpp:256-282 Square-MCN, nc = 2: terms x0^2 (p, e), 2 x0 x1 (2p', 2e'),
// fl(x1^2).  x compressed => |e + 2p'| <= 2^-22 |p| (fast sum).
template <class Q>
G2_HD B_<Q> square(T_<Q> x0, T_<Q> x1, T_<Q>& o0, T_<Q>& o1) {
  T_<Q> p, e, pp, ep, a, ea, A, U, w, ew, w2, ew2;
  two_prod<Q>(x0, x0, p, e);
  two_prod<Q>(x0, x1, pp, ep);
  const T_<Q> g = Q::mul(x1, x1);
  pp = Q::add(pp, pp);  // exact doubling (mc_ops.hpp:270); overflow -> non-finite -> declined
  ep = Q::add(ep, ep);
  two_sum<Q>(e, pp, a, ea);
  fast_two_sum<Q>(p, a, A, U);  // S = A + U + ea + 2e' + g
  two_sum<Q>(ep, g, w, ew);
  two_sum<Q>(ea, w, w2, ew2);   // S = A + U + w2 + ew2 + ew
  const T_<Q> zero = Q::c(0.0);
  const T_<Q> xs = Q::sel(Q::eq(x1, zero), x0, x1);
  const B_<Q> ok = compressed<Q>(x0, x1) & (Q::big(Q::mul(x0, xs)) | Q::eq(x0, zero));
  return finish<Q, true, false, true>(A, U, w2, Q::add(Q::abs(ew2), Q::abs(ew)), o0, o1) & ok & Q::finite(o0);
}

// add_kernel(r, sc) -> 2 for the division step: D = r0 + sc0 is exact
// (Sterbenz: sc0 = -RN(q (y0 + y1)) with q = RN(r0 / y0), so |sc0| is within
// (1 +- 2^-24)^3 of |r0|), S = D + r1 + sc1.
// R1ZERO: the remainder's second component is known to be zero (the first
// step of a division whose numerator is a single binary32, e.g. div_n, 1 / y):
// S = D + s1 is one exact two-sum, and finish re-rounds its top.
template <class Q, bool R1ZERO = false>
G2_HD B_<Q> add_step(T_<Q> D, T_<Q> r1, T_<Q> s1, T_<Q>& o0, T_<Q>& o1) {
  T_<Q> a, ea, A, U, V, eV, A2, V2;
  if constexpr (R1ZERO) {
    two_sum<Q>(D, s1, A, U);  // S = A + U exactly
    return finish<Q, false, false, false>(A, U, Q::c(0.0), Q::c(0.0), o0, o1);
  }
  two_sum<Q>(r1, s1, a, ea);
  two_sum<Q>(D, a, A, U);      // S = A + U + ea
  two_sum<Q>(U, ea, V, eV);    // S = A + V + eV
  fast_two_sum<Q>(A, V, A2, V2);  // S = A2 + V2 + eV  (A2 = RN(A + V); |A| >= |V| checked)
  return finish<Q, false, false, false>(A2, V2, eV, Q::c(0.0), o0, o1) & Q::ge(Q::abs(A), Q::abs(V));
}

// mc_ops.hpp:188-207 div_kernel, nc = 2 (x, y compressed pairs).  Underflow
// guard: every product is q_d y_j with |q_1| < |q_0| and |y1| < |y0|, so the
// smallest nonzero one is the last nonzero digit times the last nonzero
// divisor component; it must be >= 2^-100, and a nonzero digit >= 2^-100
// (normal with margin: the Sterbenz step relies on its relative rounding).
template <class Q, bool X1ZERO = false>
G2_HD B_<Q> div(T_<Q> x0, T_<Q> x1, T_<Q> y0, T_<Q> y1, T_<Q>& o0, T_<Q>& o1) {
  // digit 0
  const T_<Q> q0 = Q::div(x0, y0);
  T_<Q> s0, s1, r0, r1;
  B_<Q> ok = scale_core<Q, true, false, false>(y0, y1, Q::neg(q0), s0, s1);
  ok = ok & add_step<Q, X1ZERO>(Q::add(x0, s0), x1, s1, r0, r1);
  // digit 1
  const T_<Q> q1 = Q::div(r0, y0);
  ok = ok & scale_core<Q, true, false, false>(y0, y1, Q::neg(q1), s0, s1);
  ok = ok & add_step<Q>(Q::add(r0, s0), r1, s1, r0, r1);
  // guard digit, then renorm(q0, q1, q2 -> 2)
  const T_<Q> q2 = Q::div(r0, y0);
  T_<Q> a, ea, A, U;
  fast_two_sum<Q>(q1, q2, a, ea);  // |q2| < |q1| < |q0| (checked)
  fast_two_sum<Q>(q0, a, A, U);    // S = A + U + ea
  ok = ok & finish<Q, false, false, true>(A, U, ea, Q::c(0.0), o0, o1) & Q::ge(Q::abs(q1), Q::abs(q2)) &
       Q::ge(Q::abs(q0), Q::abs(a));
  const T_<Q> zero = Q::c(0.0);
  const B_<Q> q0z = Q::eq(q0, zero);
  const T_<Q> ql = Q::sel(Q::eq(q1, zero), q0, q1), yl = Q::sel(Q::eq(y1, zero), y0, y1);
  ok = ok & compressed<Q>(x0, x1) & compressed<Q>(y0, y1) & (Q::big(ql) | q0z) & (Q::big(Q::mul(ql, yl)) | q0z);
  return ok & Q::finite(o0);
}

// mc_ops.hpp:216-230 Mul-MCN (fast): x / (1 / y), zero fast path
template <class Q>
G2_HD B_<Q> mul(T_<Q> x0, T_<Q> x1, T_<Q> y0, T_<Q> y1, T_<Q>& o0, T_<Q>& o1) {
  const T_<Q> zero = Q::c(0.0);
  const B_<Q> z = Q::eq(Q::add(y1, y0), zero) | Q::eq(Q::add(x1, x0), zero);
  T_<Q> c0, c1;
  B_<Q> ok = div<Q, true>(Q::c(1.0), zero, y0, y1, c0, c1);
  ok = ok & div<Q>(x0, x1, c0, c1, o0, o1);
  o0 = Q::sel(z, zero, o0);
  o1 = Q::sel(z, zero, o1);
  return ok | z;
}

#if defined(__CUDACC__)
// binary32 on sm_100a: native round-to-nearest intrinsics (never contracted),
// no FTZ (the library builds with -ftz=false)
struct QF32 {
  using T = float;
  using B = bool;
  __device__ __forceinline__ static T c(double v) { return (float)v; }
  __device__ __forceinline__ static T neg(T a) { return -a; }
  __device__ __forceinline__ static T sel(B m, T a, T b) { return m ? a : b; }
  __device__ __forceinline__ static B eq(T a, T b) { return a == b; }
  __device__ __forceinline__ static B lt(T a, T b) { return a < b; }
  __device__ __forceinline__ static B ge(T a, T b) { return a >= b; }
  __device__ __forceinline__ static T add(T a, T b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static T sub(T a, T b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static T mul(T a, T b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static T div(T a, T b) { return __fdiv_rn(a, b); }
  __device__ __forceinline__ static T fma(T a, T b, T c) { return __fmaf_rn(a, b, c); }
  __device__ __forceinline__ static T abs(T a) { return fabsf(a); }
  __device__ __forceinline__ static bool finite(T a) { return isfinite(a); }
  __device__ __forceinline__ static bool big(T a) { return fabsf(a) >= 0x1p-100f; }
  __device__ __forceinline__ static T canon(T a) { return __fadd_rn(a, 0.0f); }
  // 2^floor(log2 RN(|t| f)) 2^-24 with f = 1 - 2^-24, which drops a power of
  // two into the binade below: ulp(t)/2, or ulp(t)/4 at a power of two (the
  // gap below); 0 for zero and subnormal t
  __device__ __forceinline__ static T hb(T t) {
    const float u = __fmul_rn(fabsf(t), 1.0f - 0x1p-24f);
    return __fmul_rn(__uint_as_float(__float_as_uint(u) & 0x7f800000u), 0x1p-24f);
  }
  // the same toward d's side: f = 1 when d has t's sign (the gap above)
  __device__ __forceinline__ static T hbd(T t, T d) {
    const bool away = (int)(__float_as_uint(d) ^ __float_as_uint(t)) >= 0;
    const float u = __fmul_rn(fabsf(t), away ? 1.0f : 1.0f - 0x1p-24f);
    return __fmul_rn(__uint_as_float(__float_as_uint(u) & 0x7f800000u), 0x1p-24f);
  }
  __device__ __forceinline__ static T shrink(T h) { return __fmul_rn(h, 1.0f - 0x1p-22f); }
  // bound on the rounding error of a binary32 result w: 2^-24 |w| >= h(w)
  __device__ __forceinline__ static T ulpb(T w) { return __fmul_rn(fabsf(w), 0x1p-24f); }
};

// Two elements in lockstep on the packed binary32 pipes (FADD2 / FMUL2 /
// FFMA2: one instruction per pair, IEEE round-to-nearest per lane, no FTZ);
// divisions, comparisons and selects stay per element.
struct M2 {
  bool x, y;
};
__device__ __forceinline__ M2 operator&(M2 a, M2 b) { return {a.x && b.x, a.y && b.y}; }
__device__ __forceinline__ M2 operator|(M2 a, M2 b) { return {a.x || b.x, a.y || b.y}; }

struct QF32x2 {
  using T = float2;
  using B = M2;
  __device__ __forceinline__ static T c(double v) { return make_float2((float)v, (float)v); }
  __device__ __forceinline__ static T neg(T a) { return make_float2(-a.x, -a.y); }
  __device__ __forceinline__ static T add(T a, T b) { return __fadd2_rn(a, b); }
  __device__ __forceinline__ static T sub(T a, T b) { return __fadd2_rn(a, neg(b)); }
  __device__ __forceinline__ static T mul(T a, T b) { return __fmul2_rn(a, b); }
  __device__ __forceinline__ static T fma(T a, T b, T c) { return __ffma2_rn(a, b, c); }
  __device__ __forceinline__ static T div(T a, T b) { return make_float2(__fdiv_rn(a.x, b.x), __fdiv_rn(a.y, b.y)); }
  __device__ __forceinline__ static T abs(T a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
  __device__ __forceinline__ static T sel(B m, T a, T b) { return make_float2(m.x ? a.x : b.x, m.y ? a.y : b.y); }
  __device__ __forceinline__ static B eq(T a, T b) { return {a.x == b.x, a.y == b.y}; }
  __device__ __forceinline__ static B lt(T a, T b) { return {a.x < b.x, a.y < b.y}; }
  __device__ __forceinline__ static B ge(T a, T b) { return {a.x >= b.x, a.y >= b.y}; }
  __device__ __forceinline__ static B finite(T a) { return {(bool)isfinite(a.x), (bool)isfinite(a.y)}; }
  __device__ __forceinline__ static B big(T a) { return {fabsf(a.x) >= 0x1p-100f, fabsf(a.y) >= 0x1p-100f}; }
  __device__ __forceinline__ static T canon(T a) { return __fadd2_rn(a, c(0.0)); }
  __device__ __forceinline__ static float exp_mask(float u) {
    return __uint_as_float(__float_as_uint(u) & 0x7f800000u);
  }
  __device__ __forceinline__ static T hb(T t) {
    const float2 u = __fmul2_rn(abs(t), c(1.0 - 0x1p-24));
    return __fmul2_rn(make_float2(exp_mask(u.x), exp_mask(u.y)), c(0x1p-24));
  }
  __device__ __forceinline__ static T hbd(T t, T d) {
    const float fx = (int)(__float_as_uint(d.x) ^ __float_as_uint(t.x)) >= 0 ? 1.0f : 1.0f - 0x1p-24f;
    const float fy = (int)(__float_as_uint(d.y) ^ __float_as_uint(t.y)) >= 0 ? 1.0f : 1.0f - 0x1p-24f;
    const float2 u = __fmul2_rn(abs(t), make_float2(fx, fy));
    return __fmul2_rn(make_float2(exp_mask(u.x), exp_mask(u.y)), c(0x1p-24));
  }
  __device__ __forceinline__ static T shrink(T h) { return __fmul2_rn(h, c(1.0 - 0x1p-22)); }
  __device__ __forceinline__ static T ulpb(T w) { return __fmul2_rn(abs(w), c(0x1p-24)); }
};

#endif

}  // namespace g2
}  // namespace mcfg
