// mcf_accum.cuh -- compensated binary64 accumulators for the MCF_FAST
// contractions (mm_fast.cu tiled kernels, stream_fast.cu row kernels).
//
// Every product of two binary32 components is exact in binary64, so an
// output is carried as a short binary64 expansion: level 0 takes the leading
// product through an error-free two_sum, lower levels take products and
// rounding errors ~2^-24 / 2^-48 smaller.  Policies (FP64 ops per MAD):
//   AccP2<NB>  nc=2 x T / MC(2), offset accumulation on (sum, err) pairs   4
//   AccP2X<NB> same, err terms folded in (used when the widening flag is set) 5/7
//   AccT2  MC(nc=2) x T      (S, C)      6  (streaming kernels)
//   AccT3  MC(nc=3) x T      (S, C, D)  14
//   AccM2  MC(nc=2) x MC(2)  (S, C)      8
//   AccM3  MC(nc=3) x MC(3)  (S, C, D)  23
//   AccH3  MC(nc=3, binary16) x MC(3, binary16), operands pre-summed into one
//          binary64 each (<= 33 significant bits): S = fma(a, b, S), 1 op
// merge() combines two partial expansions (warp reductions); the final value
// is split greedily into nc components (mc_ops.hpp:286-297 on the extended
// value) by split_out().
#pragma once

#include <cuda_fp16.h>

namespace mcfg {

__device__ __forceinline__ void dsum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bv = __dsub_rn(s, a);
  const double av = __dsub_rn(s, bv);
  e = __dadd_rn(__dsub_rn(a, av), __dsub_rn(b, bv));
}

// Fast2Sum with the operand order chosen by the high words: s = a + b, and
// the exact error with 3 FP64 ops instead of two_sum's 6.  Dekker's
// condition is exponent(big) >= exponent(small); comparing |hi32| of the two
// binary64 patterns as binary32 magnitudes (one FSETP on the FP32 side,
// monotone in the binary64 magnitude, equal high words => equal exponents)
// picks a valid order.  The selects run on the integer pipe (small = a^b^big).
__device__ __forceinline__ void dsum_fast(double a, double b, double& s, double& e) {
  const float ha = __int_as_float(__double2hiint(a)), hb = __int_as_float(__double2hiint(b));
  const bool b_big = fabsf(hb) > fabsf(ha);
  const long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
  const long long ibig = b_big ? ib : ia;
  const double big = __longlong_as_double(ibig);
  const double small = __longlong_as_double(ia ^ ib ^ ibig);
  s = __dadd_rn(a, b);
  e = __dsub_rn(small, __dsub_rn(s, big));
}

struct AccT2 {
  static constexpr int kNA = 2, kNB = 1, kLv = 2, kOps = 6;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double p = __dmul_rn(a[0], b[0]);
    double e;
    dsum_fast(acc[0], p, acc[0], e);
    acc[1] = __fma_rn(a[1], b[0], __dadd_rn(acc[1], e));
  }
  __device__ static void merge(double (&acc)[kLv], const double (&o)[kLv]) {
    double e;
    dsum(acc[0], o[0], acc[0], e);
    acc[1] = __dadd_rn(acc[1], __dadd_rn(o[1], e));
  }
};

// Offset accumulation (Rump-style extraction folded into the running sum):
// with operands pre-scaled so every product has |a0*b| <= 1 and tau
// initialised to sigma = 2^(ceil(log2 K) + 1), the running value
// tau = sigma + S stays in [sigma/2, 2*sigma), so
//   tau' = fma(a0, b, tau)      (one rounding)
//   q    = tau' - tau           (exact: Sterbenz)
//   r    = fma(a0, b, -q)       (exact: the rounding residual of tau + a0*b)
// carries the product exactly as q (into tau) + r (into C).  C also takes
// the a1*b terms (~2^-24 smaller).  5 FP64 ops per MAD, no compare/select.
struct AccT2S {
  static constexpr int kNA = 2, kNB = 1, kLv = 2, kOps = 5;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double t = __fma_rn(a[0], b[0], acc[0]);
    const double q = __dsub_rn(t, acc[0]);
    const double r = __fma_rn(a[0], b[0], -q);
    acc[0] = t;
    acc[1] = __fma_rn(a[1], b[0], __dadd_rn(acc[1], r));
  }
};

// Offset accumulation on pre-summed operands: a = fl(a0 + a1) (exact for
// expansions whose components span <= 53 bits, e.g. every split of a
// binary64; otherwise a 2^-53 relative perturbation), same for b when it is
// an MC operand.  The product a*b stays exact inside the fma; the residual r
// of tau + a*b is rounded once (|r| <= ulp(sigma)/2, so the loss is
// ~2^-106 sigma per MAD).  4 FP64 ops per MAD for MC x T and MC x MC alike.
// Operands are stored as (sum, err) pairs with sum + err exactly the MC value
// (err = two_sum residual, zero for expansions spanning <= 53 bits).  The
// widening pass raises a flag if any err is nonzero; the exact-sum kernel
// (AccP2, 4 ops) runs when the flag is clear, AccP2X (err terms folded into
// C by fma, +1 op per nonzero-err operand pairing) when it is set.
template <int NB>
struct AccP2 {
  static constexpr int kNA = 2, kNB = NB, kLv = 2, kOps = 4;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double t = __fma_rn(a[0], b[0], acc[0]);
    const double q = __dsub_rn(t, acc[0]);
    acc[0] = t;
    acc[1] = __dadd_rn(acc[1], __fma_rn(a[0], b[0], -q));
  }
};

template <int NB>
struct AccP2X {
  static constexpr int kNA = 2, kNB = NB, kLv = 2, kOps = NB == 2 ? 7 : 5;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double t = __fma_rn(a[0], b[0], acc[0]);
    const double q = __dsub_rn(t, acc[0]);
    acc[0] = t;
    double c = __dadd_rn(acc[1], __fma_rn(a[0], b[0], -q));
    c = __fma_rn(a[1], b[0], c);
    if constexpr (NB == 2) {
      c = __fma_rn(a[0], b[1], c);
      c = __fma_rn(a[1], b[1], c);
    }
    acc[1] = c;
  }
};

struct AccM2S {  // MC(nc=2) x MC(nc=2), same offset scheme: 7 FP64 ops / MAD
  static constexpr int kNA = 2, kNB = 2, kLv = 2, kOps = 7;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double t = __fma_rn(a[0], b[0], acc[0]);
    const double q = __dsub_rn(t, acc[0]);
    const double r = __fma_rn(a[0], b[0], -q);
    acc[0] = t;
    double c = __fma_rn(a[0], b[1], __dadd_rn(acc[1], r));
    c = __fma_rn(a[1], b[0], c);
    acc[1] = __fma_rn(a[1], b[1], c);
  }
};

struct AccT3 {
  static constexpr int kNA = 3, kNB = 1, kLv = 3, kOps = 14;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double p0 = __dmul_rn(a[0], b[0]);
    const double p1 = __dmul_rn(a[1], b[0]);
    double e0, e1, e2;
    dsum_fast(acc[0], p0, acc[0], e0);
    dsum_fast(acc[1], e0, acc[1], e1);
    dsum_fast(acc[1], p1, acc[1], e2);
    acc[2] = __fma_rn(a[2], b[0], __dadd_rn(acc[2], __dadd_rn(e1, e2)));
  }
  __device__ static void merge(double (&acc)[kLv], const double (&o)[kLv]) {
    double e0, e1, e2;
    dsum(acc[0], o[0], acc[0], e0);
    dsum(acc[1], o[1], acc[1], e1);
    dsum(acc[1], e0, acc[1], e2);
    acc[2] = __dadd_rn(__dadd_rn(acc[2], o[2]), __dadd_rn(e1, e2));
  }
};

struct AccM2 {
  static constexpr int kNA = 2, kNB = 2, kLv = 2, kOps = 8;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double p = __dmul_rn(a[0], b[0]);
    double e;
    dsum_fast(acc[0], p, acc[0], e);
    double c = __dadd_rn(acc[1], e);
    c = __fma_rn(a[0], b[1], c);
    c = __fma_rn(a[1], b[0], c);
    acc[1] = __fma_rn(a[1], b[1], c);
  }
  __device__ static void merge(double (&acc)[kLv], const double (&o)[kLv]) { AccT2::merge(acc, o); }
};

struct AccM3 {
  static constexpr int kNA = 3, kNB = 3, kLv = 3, kOps = 23;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    const double p00 = __dmul_rn(a[0], b[0]);
    const double p01 = __dmul_rn(a[0], b[1]);
    const double p10 = __dmul_rn(a[1], b[0]);
    double e0, e1, e2, e3;
    dsum_fast(acc[0], p00, acc[0], e0);
    dsum_fast(acc[1], e0, acc[1], e1);
    dsum_fast(acc[1], p01, acc[1], e2);
    dsum_fast(acc[1], p10, acc[1], e3);
    double d = __dadd_rn(acc[2], __dadd_rn(e1, __dadd_rn(e2, e3)));
    d = __fma_rn(a[0], b[2], d);
    d = __fma_rn(a[1], b[1], d);
    d = __fma_rn(a[2], b[0], d);
    d = __fma_rn(a[1], b[2], d);
    d = __fma_rn(a[2], b[1], d);
    acc[2] = __fma_rn(a[2], b[2], d);
  }
  __device__ static void merge(double (&acc)[kLv], const double (&o)[kLv]) { AccT3::merge(acc, o); }
};

struct AccH3 {
  static constexpr int kNA = 1, kNB = 1, kLv = 1, kOps = 1;
  __device__ static void mad(double (&acc)[kLv], const double* a, const double* b) {
    acc[0] = __fma_rn(a[0], b[0], acc[0]);
  }
  __device__ static void merge(double (&acc)[kLv], const double (&o)[kLv]) {
    acc[0] = __dadd_rn(acc[0], o[0]);
  }
};

template <class S>
__device__ __forceinline__ double to_d(S v) { return (double)v; }
template <>
__device__ __forceinline__ double to_d<__half>(__half v) { return (double)__half2float(v); }

template <class S>
__device__ __forceinline__ S from_d(double v);
template <>
__device__ __forceinline__ float from_d<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ __half from_d<__half>(double v) { return __double2half(v); }

// greedy split of S + C (+ D) into nc components of type ST
template <class ST, int NC, int LV>
__device__ __forceinline__ void split_out(const double (&acc)[LV], ST* out) {
  double hi = acc[0], lo = 0.0;
  if constexpr (LV >= 2) {
    dsum(acc[0], acc[1], hi, lo);
    if constexpr (LV >= 3) lo = __dadd_rn(lo, acc[2]);
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const ST c = from_d<ST>(__dadd_rn(hi, lo));
    out[i] = c;
    const double r = __dsub_rn(hi, to_d<ST>(c));  // exact
    dsum(r, lo, hi, lo);
  }
}

}  // namespace mcfg
