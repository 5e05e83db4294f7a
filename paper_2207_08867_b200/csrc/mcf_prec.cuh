// mcf_prec.cuh -- device precision policies for MCF components.
//
// The reference stores every component as a binary64 holding a value exactly
// representable in the working format P and emulates P by rounding each
// binary64 result once (precision.hpp:3-14, fl_* at :165-187).  On sm_100a
// the same results come from native IEEE round-to-nearest instructions:
//   B32: __fadd_rn/__fsub_rn/__fmul_rn/__fdiv_rn/__fmaf_rn (no FTZ: the
//        library is compiled with -ftz=false -prec-div=true -fmad=false)
//   B64: __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn/__fma_rn
//   B16: computed in binary32 and rounded once to binary16; double rounding
//        is innocuous for + - * / because 24 >= 2*11+2 (precision.hpp:9-12),
//        and the only fma use (two_prod) is exact in binary32.
// The _rn intrinsics are never contracted or reassociated by the compiler,
// which is what the error-free transforms need.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace mcfg {

struct PB32 {
  using st = float;   // storage in HBM
  using rt = float;   // register type
  static constexpr int kSig = 24;
  __device__ __forceinline__ static rt ld(st v) { return v; }
  __device__ __forceinline__ static st sv(rt v) { return v; }
  __device__ __forceinline__ static rt add(rt a, rt b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static rt sub(rt a, rt b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static rt mul(rt a, rt b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static rt div(rt a, rt b) { return __fdiv_rn(a, b); }
  __device__ __forceinline__ static rt fma(rt a, rt b, rt c) { return __fmaf_rn(a, b, c); }
  // exact doubling kept in the register type (square_kernel's 2.0 * p, mc_ops.hpp:270)
  __device__ __forceinline__ static rt twice(rt a) { return __fmul_rn(2.0f, a); }
  __device__ __forceinline__ static rt rd(double d) { return __double2float_rn(d); }
  __device__ __forceinline__ static double to_d(rt v) { return (double)v; }
  __device__ __forceinline__ static rt mag(rt v) { return fabsf(v); }
  __device__ __forceinline__ static bool finite(rt v) { return isfinite(v); }
};

struct PB64 {
  using st = double;
  using rt = double;
  static constexpr int kSig = 53;
  __device__ __forceinline__ static rt ld(st v) { return v; }
  __device__ __forceinline__ static st sv(rt v) { return v; }
  __device__ __forceinline__ static rt add(rt a, rt b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static rt sub(rt a, rt b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static rt mul(rt a, rt b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static rt div(rt a, rt b) { return __ddiv_rn(a, b); }
  __device__ __forceinline__ static rt fma(rt a, rt b, rt c) { return __fma_rn(a, b, c); }
  __device__ __forceinline__ static rt twice(rt a) { return __dmul_rn(2.0, a); }
  __device__ __forceinline__ static rt rd(double d) { return d; }
  __device__ __forceinline__ static double to_d(rt v) { return v; }
  __device__ __forceinline__ static rt mag(rt v) { return fabs(v); }
  __device__ __forceinline__ static bool finite(rt v) { return isfinite(v); }
};

struct PB16 {
  using st = __half;
  using rt = float;
  static constexpr int kSig = 11;
  __device__ __forceinline__ static rt r16(float v) { return __half2float(__float2half_rn(v)); }
  __device__ __forceinline__ static rt ld(st v) { return __half2float(v); }
  __device__ __forceinline__ static st sv(rt v) { return __float2half_rn(v); }
  __device__ __forceinline__ static rt add(rt a, rt b) { return r16(__fadd_rn(a, b)); }
  __device__ __forceinline__ static rt sub(rt a, rt b) { return r16(__fsub_rn(a, b)); }
  __device__ __forceinline__ static rt mul(rt a, rt b) { return r16(__fmul_rn(a, b)); }
  __device__ __forceinline__ static rt div(rt a, rt b) { return r16(__fdiv_rn(a, b)); }
  __device__ __forceinline__ static rt fma(rt a, rt b, rt c) { return r16(__fmaf_rn(a, b, c)); }
  // the reference doubles in binary64 without rounding to P; binary32 holds 2p exactly
  __device__ __forceinline__ static rt twice(rt a) { return __fmul_rn(2.0f, a); }
  __device__ __forceinline__ static rt rd(double d) { return __half2float(__double2half(d)); }
  __device__ __forceinline__ static double to_d(rt v) { return (double)v; }
  __device__ __forceinline__ static rt mag(rt v) { return fabsf(v); }
  __device__ __forceinline__ static bool finite(rt v) { return isfinite(v); }
};

// ---- error-free transforms (eft.hpp) ---------------------------------------

// eft.hpp:31-38 -- Knuth two-sum, 6 rounded operations
template <class P>
__device__ __forceinline__ void two_sum(typename P::rt a, typename P::rt b, typename P::rt& s,
                                        typename P::rt& e) {
  s = P::add(a, b);
  const typename P::rt bv = P::sub(s, a);
  const typename P::rt av = P::sub(s, bv);
  e = P::add(P::sub(a, av), P::sub(b, bv));
}

// eft.hpp:75-80 -- p = fl(ab), e = fma(a, b, -p)  (the reference's default route;
// the split route eft.hpp:62-72 is pinned bitwise equal, T/test_eft.cpp:167-182)
template <class P>
__device__ __forceinline__ void two_prod(typename P::rt a, typename P::rt b, typename P::rt& p,
                                         typename P::rt& e) {
  p = P::mul(a, b);
  e = P::fma(a, b, -p);
}

}  // namespace mcfg
