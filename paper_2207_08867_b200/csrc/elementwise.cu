// elementwise.cu -- the elementwise MCF operators (mc_ops.hpp) on sm_100a.
//
// One thread owns EPT consecutive elements; with binary32 components the
// (…, nc) layout makes an EPT-element slice a multiple of 16 bytes, so every
// operand moves with 128-bit streaming loads/stores (ld.global.cs /
// st.global.cs: each byte is touched once, keep L2 for the next operand).
// All nc components live in registers; the operator bodies are the
// register fast paths of mcf_fast.cuh, and any element whose fast-path
// preconditions fail re-runs the literal restatement (mcf_lit.cuh).
// Precisions / nc without an instantiated fast path run the literal kernel.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "mcf_exp.cuh"
#include "mcf_fast.cuh"
#include "mcf_g2.cuh"
#include "mcf_w2.cuh"
#include "mcf_lit.cuh"
#include "mcf_prec.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

template <class P>
using RT = typename P::rt;
template <class P>
using ST = typename P::st;

constexpr int kThreads = 256;

// ---- vector IO ---------------------------------------------------------------

template <int B>
struct VecOf;
template <>
struct VecOf<16> { using T = uint4; };
template <>
struct VecOf<8> { using T = uint2; };
template <>
struct VecOf<4> { using T = unsigned int; };
template <>
struct VecOf<2> { using T = unsigned short; };

template <class T, int N>
__device__ __forceinline__ void load_stream(const T* __restrict__ p, T (&d)[N]) {
  constexpr int B = N * (int)sizeof(T);
  constexpr int V = (B % 16 == 0) ? 16 : (B % 8 == 0) ? 8 : (B % 4 == 0) ? 4 : 2;
  using VT = typename VecOf<V>::T;
  VT tmp[B / V];
#pragma unroll
  for (int i = 0; i < B / V; ++i) tmp[i] = __ldcs(reinterpret_cast<const VT*>(p) + i);
  memcpy(&d[0], &tmp[0], B);
}

template <class T, int N>
__device__ __forceinline__ void store_stream(T* __restrict__ p, const T (&d)[N]) {
  constexpr int B = N * (int)sizeof(T);
  constexpr int V = (B % 16 == 0) ? 16 : (B % 8 == 0) ? 8 : (B % 4 == 0) ? 4 : 2;
  using VT = typename VecOf<V>::T;
  VT tmp[B / V];
  memcpy(&tmp[0], &d[0], B);
#pragma unroll
  for (int i = 0; i < B / V; ++i) __stcs(reinterpret_cast<VT*>(p) + i, tmp[i]);
}

// elements per thread so that one thread's slice of an nc-component operand
// is a whole number of 16-byte vectors when possible
template <class P, int NC>
constexpr int ept_for() {
  constexpr int b = (int)sizeof(ST<P>) * NC;
  return b % 16 == 0 ? 1 : (2 * b) % 16 == 0 ? 2 : (4 * b) % 16 == 0 ? 4 : 8;
}

// ---- operator table -------------------------------------------------------------
// Each op supplies the register fast path (compile-time nc) and the literal
// restatement (runtime nc).  Flags say which operands it reads.
enum OpId {
  kGrow, kScale, kScaleX, kDivN, kAdd, kDiv, kMul, kMulSlow, kSquare, kExp, kNeg, kApprox,
  kRenorm, kSimple
};

template <int OP>
struct OpTraits {
  static constexpr bool kY = OP == kAdd || OP == kDiv || OP == kMul || OP == kMulSlow;
  static constexpr bool kV = OP == kGrow || OP == kScale || OP == kScaleX || OP == kDivN;
};

// binary32 nc = 2 operators with a certified shortcut (mcf_g2.cuh); an element
// it declines runs the register path below, then the literal one
template <int OP, class P, int NC, int ONC>
constexpr bool kG2 = std::is_same<P, PB32>::value && NC == 2 && ONC == 2 &&
                     (OP == kScale || OP == kSquare || OP == kDiv || OP == kDivN || OP == kMul || OP == kMulSlow ||
                      OP == kExp || OP == kAdd || OP == kGrow);

// the ops whose certified shortcut runs two elements at once (FADD2 / FMUL2 /
// FFMA2); exp keeps a per-element binary64 exp and runs one at a time
// (measured on B200, 2^24 config-0 elements: Mul-MCN's chained divisions
// need 79 registers packed, one ring per SM, 294 us against 275 us scalar at
// two rings, so it stays scalar)
// the division-based ones and the direct product first try the wide tier
// (mcf_w2.cuh: binary64 carries every exact intermediate, one element at a
// time).  Square-MCN stays on the packed binary32 shortcut: its wide form
// (w2::square) measured the same 54 us -- the operator is bound by its 8 B in /
// 8 B out stream, not by instructions
template <int OP, class P, int NC, int ONC>
constexpr bool kW2 = kG2<OP, P, NC, ONC> && (OP == kDiv || OP == kDivN || OP == kMul || OP == kMulSlow);

template <int OP, class P, int NC, int ONC>
constexpr bool kG2Pair = kG2<OP, P, NC, ONC> && OP != kExp && !kW2<OP, P, NC, ONC>;

// two binary32 nc = 2 elements (x = e0c0 e0c1 e1c0 e1c1, v = v0 v1) through the
// packed certified shortcut; returns which were accepted
template <int OP>
__device__ __forceinline__ g2::M2 run_g2_pair(const float (&x)[4], const float (&y)[4], float v0, float v1,
                                              float (&o)[4]) {
  using Q = g2::QF32x2;
  const float2 x0 = make_float2(x[0], x[2]), x1 = make_float2(x[1], x[3]);
  const float2 y0 = make_float2(y[0], y[2]), y1 = make_float2(y[1], y[3]);
  const float2 v = make_float2(v0, v1);
  float2 o0, o1;
  g2::M2 ok;
  if constexpr (OP == kScale) ok = g2::scale<Q>(x0, x1, v, o0, o1);
  else if constexpr (OP == kSquare) ok = g2::square<Q>(x0, x1, o0, o1);
  else if constexpr (OP == kDiv) ok = g2::div<Q>(x0, x1, y0, y1, o0, o1);
  else if constexpr (OP == kDivN) ok = g2::div<Q, true>(v, Q::c(0.0), x0, x1, o0, o1);  // x holds the divisor
  else if constexpr (OP == kMul) ok = g2::mul<Q>(x0, x1, y0, y1, o0, o1);
  else if constexpr (OP == kGrow) ok = g2::grow<Q>(x0, x1, v, o0, o1);
  else ok = g2::add<Q>(x0, x1, y0, y1, o0, o1);
  o[0] = o0.x, o[1] = o1.x, o[2] = o0.y, o[3] = o1.y;
  return ok;
}

// the wide tier alone (binary32 nc = 2 Div-MCN / DivN / Mul-MCN fast and slow), branch-free:
// the TMA kernel runs it for all of a thread's elements before it looks at any
// verdict, so their independent chains interleave
template <int OP>
__device__ __forceinline__ bool run_w2(const float (&x)[2], const float (&y)[2], float v, float (&o)[2]) {
  using V = w2::VD;
  bool ok;
  if constexpr (OP == kDivN) {  // x holds the divisor
    ok = w2::div<V, true, true>(v, 0.0f, x[0], x[1], true, __fadd_rn(x[0], x[1]) == x[0], o[0], o[1]);
  } else {
    const bool cx = __fadd_rn(x[0], x[1]) == x[0], cy = __fadd_rn(y[0], y[1]) == y[0];
    if constexpr (OP == kDiv) ok = w2::div<V, false, true>(x[0], x[1], y[0], y[1], cx, cy, o[0], o[1]);
    else if constexpr (OP == kMulSlow) ok = w2::mul_slow<V>(x[0], x[1], y[0], y[1], cx, cy, o[0], o[1]);
    else {
      ok = w2::mul<V, true>(x[0], x[1], y[0], y[1], cx, cy, o[0], o[1]);
      if (__fadd_rn(y[1], y[0]) == 0.0f || __fadd_rn(x[1], x[0]) == 0.0f) o[0] = o[1] = 0.0f, ok = true;
    }
  }
  return ok;
}

template <int OP, class P, int NC, int ONC, bool TRY_G2 = true, bool TRY_W2 = true>
__device__ __forceinline__ bool run_fast(const RT<P> (&x)[NC], const RT<P> (&y)[NC], RT<P> v,
                                         RT<P> (&o)[ONC]) {
  if constexpr (TRY_G2 && TRY_W2 && kW2<OP, P, NC, ONC>) {
    if (__builtin_expect(run_w2<OP>(x, y, v, o), 1)) return true;
  }
  if constexpr (TRY_G2 && kG2<OP, P, NC, ONC>) {
    using Q = g2::QF32;
    bool ok;
    if constexpr (OP == kScale) ok = g2::scale<Q>(x[0], x[1], v, o[0], o[1]);
    else if constexpr (OP == kSquare) ok = g2::square<Q>(x[0], x[1], o[0], o[1]);
    else if constexpr (OP == kDiv) ok = g2::div<Q>(x[0], x[1], y[0], y[1], o[0], o[1]);
    else if constexpr (OP == kDivN) ok = g2::div<Q, true>(v, 0.0f, x[0], x[1], o[0], o[1]);  // x holds the divisor
    else if constexpr (OP == kMul) ok = g2::mul<Q>(x[0], x[1], y[0], y[1], o[0], o[1]);
    else if constexpr (OP == kAdd) ok = g2::add<Q>(x[0], x[1], y[0], y[1], o[0], o[1]);
    else if constexpr (OP == kGrow) ok = g2::grow<Q>(x[0], x[1], v, o[0], o[1]);
    else if constexpr (OP == kMulSlow) ok = false;  // no binary32 shortcut: the register path is next
    else ok = w2::exp_b32(x[0], x[1], o[0], o[1]);
    if (__builtin_expect(ok, 1)) return true;
  }
  if constexpr (OP == kGrow) return fast::grow<P, NC>(x, v, o);
  else if constexpr (OP == kScale || OP == kScaleX) return fast::scale<P, NC, ONC>(x, v, o);
  else if constexpr (OP == kDivN) {
    RT<P> num[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) num[i] = i == 0 ? v : RT<P>(0);
    return fast::div<P, NC>(num, x, o);  // x holds the MC divisor y
  } else if constexpr (OP == kAdd) return fast::add<P, NC>(x, y, o);
  else if constexpr (OP == kDiv) return fast::div<P, NC>(x, y, o);
  else if constexpr (OP == kMul) return fast::mul_fast<P, NC>(x, y, o);
  else if constexpr (OP == kMulSlow) return fast::mul_slow<P, NC>(x, y, o);
  else if constexpr (OP == kSquare) return fast::square<P, NC>(x, o);
  else if constexpr (OP == kExp) return fast::exp<P, NC>(x, o);
  else if constexpr (OP == kNeg) {
#pragma unroll
    for (int i = 0; i < NC; ++i) o[i] = -x[i];
    return true;
  } else if constexpr (OP == kRenorm) {
    RT<P> h[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) h[i] = x[i];
    return fast::renorm<P, NC, ONC>(h, o);
  } else {
    return false;
  }
}

// literal restatement with runtime component counts (padded operands)
template <int OP, class P>
__device__ __noinline__ void run_lit(const RT<P>* x, const RT<P>* y, RT<P> v, RT<P>* o, int nc,
                                     int onc) {
  if constexpr (OP == kGrow) lit::grow<P>(x, nc, v, o);
  else if constexpr (OP == kScale || OP == kScaleX) lit::scale<P>(x, nc, v, o, onc);
  else if constexpr (OP == kDivN) {
    RT<P> num[lit::kMaxNc];
    for (int i = 0; i < nc; ++i) num[i] = i == 0 ? v : RT<P>(0);
    lit::div<P>(num, x, nc, o);
  } else if constexpr (OP == kAdd) lit::add<P>(x, nc, y, nc, o, nc);
  else if constexpr (OP == kDiv) lit::div<P>(x, y, nc, o);
  else if constexpr (OP == kMul) lit::mul_fast<P>(x, y, nc, o);
  else if constexpr (OP == kMulSlow) lit::mul_slow<P>(x, y, nc, o);
  else if constexpr (OP == kSquare) lit::square<P>(x, nc, o);
  else if constexpr (OP == kExp) lit::exp<P>(x, nc, o);
  else if constexpr (OP == kNeg) {
    for (int i = 0; i < nc; ++i) o[i] = -x[i];
  } else if constexpr (OP == kApprox) {
    o[0] = lit::approx<P>(x, nc);
  } else if constexpr (OP == kRenorm) lit::renorm<P>(x, nc, o, onc);
  else if constexpr (OP == kSimple) lit::simple_renorm<P>(x, nc, o, onc);
}

// one element through the literal path, operands read from memory (global or
// shared) and the result written to memory: nothing of the caller's register
// state escapes to the stack on the fast path
template <int OP, class P>
__device__ __noinline__ void lit_element(const ST<P>* xe, const ST<P>* ye, RT<P> v, ST<P>* oe, int nc,
                                         int onc) {
  RT<P> xa[lit::kMaxNc], ya[lit::kMaxNc], oa[lit::kMaxNc + 1];
  for (int c = 0; c < nc; ++c) {
    xa[c] = P::ld(xe[c]);
    ya[c] = ye ? P::ld(ye[c]) : RT<P>(0);
  }
  run_lit<OP, P>(xa, ya, v, oa, nc, onc);
  for (int c = 0; c < onc; ++c) oe[c] = P::sv(oa[c]);
}

// v[e % vn]: vmode 0 = per-element (vn == numel), 1 = scalar, 2 = general suffix
template <class P>
__device__ __forceinline__ RT<P> v_at(const ST<P>* v, int64_t vn, int vmode, int64_t e) {
  if (vmode == 0) return P::ld(v[e]);
  if (vmode == 1) return P::ld(v[0]);
  return P::ld(v[e % vn]);
}

// ---- fast kernel ----------------------------------------------------------------

template <int OP, class P, int NC, int ONC>
__global__ void __launch_bounds__(kThreads) k_fast(const ST<P>* __restrict__ x,
                                                   const ST<P>* __restrict__ y,
                                                   const ST<P>* __restrict__ v, int64_t vn,
                                                   int vmode, ST<P>* __restrict__ out,
                                                   int64_t numel) {
  constexpr int EPT = ept_for<P, NC>();
  constexpr bool kY = OpTraits<OP>::kY, kV = OpTraits<OP>::kV;
  struct Frag {
    ST<P> xs[EPT * NC];
    ST<P> ys[kY ? EPT * NC : 1];
    RT<P> vs[kV ? EPT : 1];
  };
  // full EPT-element groups, vector IO
  auto load = [&](Frag& f, int64_t e0) {
    load_stream<ST<P>, EPT * NC>(x + e0 * NC, f.xs);
    if constexpr (kY) load_stream<ST<P>, EPT * NC>(y + e0 * NC, f.ys);
    if constexpr (kV) {
      if (vmode == 0 && (EPT * sizeof(ST<P>)) % 4 == 0) {
        ST<P> vv[EPT];
        load_stream<ST<P>, EPT>(v + e0, vv);
#pragma unroll
        for (int i = 0; i < EPT; ++i) f.vs[i] = P::ld(vv[i]);
      } else {
#pragma unroll
        for (int i = 0; i < EPT; ++i) f.vs[i] = v_at<P>(v, vn, vmode, e0 + i);
      }
    }
  };
  // returns a mask of elements whose fast path declined (re-run by redo())
  auto compute = [&](const Frag& f, ST<P> (&os)[EPT * ONC], int count) -> unsigned {
    unsigned bail = 0;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      if (i >= count) break;
      RT<P> xa[NC], ya[NC], oa[ONC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        xa[c] = P::ld(f.xs[i * NC + c]);
        ya[c] = kY ? P::ld(f.ys[i * NC + c]) : RT<P>(0);
      }
      const RT<P> vv = kV ? f.vs[i] : RT<P>(0);
      if (!run_fast<OP, P, NC, ONC>(xa, ya, vv, oa)) bail |= 1u << i;
#pragma unroll
      for (int c = 0; c < ONC; ++c) os[i * ONC + c] = P::sv(oa[c]);
    }
    return bail;
  };
  // literal re-run of declined elements straight from/to global memory, after
  // the vector store (same thread, later store wins)
  auto redo = [&](unsigned bail, int64_t e0, const Frag& f) {
#pragma unroll 1
    for (int i = 0; i < EPT; ++i)
      if (bail >> i & 1u)
        lit_element<OP, P>(x + (e0 + i) * NC, kY ? y + (e0 + i) * NC : nullptr, kV ? f.vs[i] : RT<P>(0),
                           out + (e0 + i) * ONC, NC, ONC);
  };
  const int64_t groups = numel / EPT;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // software pipeline: the next group's loads are in flight while this one computes
  Frag cur;
  if (g < groups) load(cur, g * EPT);
  for (; g < groups; g += stride) {
    Frag nxt;
    const bool more = g + stride < groups;
    if (more) load(nxt, (g + stride) * EPT);
    ST<P> os[EPT * ONC];
    const unsigned bail = compute(cur, os, EPT);
    store_stream<ST<P>, EPT * ONC>(out + g * EPT * ONC, os);
    if (bail) redo(bail, g * EPT, cur);
    if (more) cur = nxt;
  }
  // ragged tail (< EPT elements): one thread, scalar IO
  if (blockIdx.x == 0 && threadIdx.x == 0 && groups * EPT < numel) {
    const int64_t e0 = groups * EPT;
    const int cnt = (int)(numel - e0);
    Frag f;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const bool in = i < cnt;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        f.xs[i * NC + c] = in ? x[(e0 + i) * NC + c] : P::sv(RT<P>(0));
        if constexpr (kY) f.ys[i * NC + c] = in ? y[(e0 + i) * NC + c] : P::sv(RT<P>(0));
      }
      if constexpr (kV) f.vs[i] = in ? v_at<P>(v, vn, vmode, e0 + i) : RT<P>(0);
    }
    ST<P> os[EPT * ONC];
    const unsigned bail = compute(f, os, cnt);
    for (int i = 0; i < cnt; ++i)
#pragma unroll
      for (int c = 0; c < ONC; ++c) out[(e0 + i) * ONC + c] = os[i * ONC + c];
    if (bail) redo(bail, e0, f);
  }
}

// ---- TMA-staged kernel (bulk copies into a shared-memory ring) ---------------
//
// One persistent CTA per SM.  A producer warp streams whole tiles of every
// operand into a kStages-deep ring with cp.async.bulk (TMA, 1-D), completion
// tracked by mbarrier transaction counts; 16 consumer warps read their
// elements from shared memory (LDS.128), run the same register fast path and
// store with 128-bit streaming stores.  Bytes in flight per SM are set by the
// ring (kStages x ~40 KiB), not by registers, which keeps HBM busy while the
// consumers spend their issue slots on the operator itself.

namespace tma {

constexpr int kConsumerWarps = 16;
constexpr int kCtasPerSm = 2;  // two rings per SM: 32 consumer warps hide FP latency
constexpr int kSmemBudget = 100 * 1024;
#ifndef MCF_W2_CTAS
#define MCF_W2_CTAS 2
#endif
// rings per SM an operator is compiled for (the wide-tier ops are set below)
template <int OP>
constexpr int kCtasFor = (OP == kDiv || OP == kDivN || OP == kMul) ? MCF_W2_CTAS : kCtasPerSm;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// the suspend-time hint parks the waiting warp instead of spinning on the
// barrier (spinning costs issue slots the computing warps need)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <class P, int NC, int OP>
struct Geo {
  static constexpr int EPT = ept_for<P, NC>();
  static constexpr int kThreads = kConsumerWarps * 32;
  static constexpr int kRound = kThreads * EPT;                 // elements per round
  static constexpr int kRounds = 1;
  static constexpr int kTile = kRound * kRounds;                // elements per tile
  static constexpr bool kY = OpTraits<OP>::kY, kV = OpTraits<OP>::kV;
  static constexpr int kXBytes = kTile * NC * (int)sizeof(typename P::st);
  static constexpr int kYBytes = kY ? kXBytes : 0;
  static constexpr int kVBytes = kV ? kTile * (int)sizeof(typename P::st) : 0;
  static constexpr int kStageBytes = kXBytes + kYBytes + kVBytes;
  static constexpr int kFit = (kCtasFor<OP> > 2 ? 72 * 1024 : kSmemBudget) / kStageBytes;
  static constexpr int kStages = kFit >= 8 ? 8 : (kFit >= 4 ? 4 : 2);  // power of two: cheap ring index
  static constexpr int kSmem = kStages * kStageBytes + 2 * kStages * 8;
};

}  // namespace tma

// the packed certified ops need the registers of one ring per SM: at two
// rings (56 registers) ptxas splits FADD2 / FMUL2 / FFMA2 back into scalars
template <int OP, class P, int NC, int ONC>
constexpr int kTmaCtas = kG2Pair<OP, P, NC, ONC> ? 1 : kW2<OP, P, NC, ONC> ? MCF_W2_CTAS : tma::kCtasPerSm;

// vmode here is 0 (v per element) or 1 (scalar v); `tiles` full tiles only
template <int OP, class P, int NC, int ONC>
__global__ void __launch_bounds__(tma::kConsumerWarps * 32 + 32, (kTmaCtas<OP, P, NC, ONC>))
    k_tma(const ST<P>* __restrict__ x, const ST<P>* __restrict__ y, const ST<P>* __restrict__ v,
          int vmode, ST<P>* __restrict__ out, int64_t tiles) {
  using G = tma::Geo<P, NC, OP>;
  constexpr int EPT = G::EPT;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int S = G::kStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * G::kStageBytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], tma::kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == tma::kConsumerWarps) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int s = it % S;
        const unsigned ph = (unsigned)(it / S) & 1u;
        tma::mbar_wait(&empty[s], ph ^ 1u);
        unsigned char* st = smem + s * G::kStageBytes;
        tma::mbar_expect_tx(&full[s], G::kStageBytes);
        const int64_t e0 = t * G::kTile;
        tma::bulk_g2s(st, x + e0 * NC, G::kXBytes, &full[s]);
        if constexpr (G::kY) tma::bulk_g2s(st + G::kXBytes, y + e0 * NC, G::kYBytes, &full[s]);
        if constexpr (G::kV) tma::bulk_g2s(st + G::kXBytes + G::kYBytes, v + e0, G::kVBytes, &full[s]);
      }
    }
    return;
  }

  RT<P> vscalar = RT<P>(0);
  if constexpr (G::kV) {
    if (vmode == 1) vscalar = P::ld(v[0]);
  }
  int it = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int s = it % S;
    const unsigned ph = (unsigned)(it / S) & 1u;
    tma::mbar_wait(&full[s], ph);
    const unsigned char* st = smem + s * G::kStageBytes;
    const ST<P>* xs_s = reinterpret_cast<const ST<P>*>(st);
    const ST<P>* ys_s = reinterpret_cast<const ST<P>*>(st + G::kXBytes);
    const ST<P>* vs_s = reinterpret_cast<const ST<P>*>(st + G::kXBytes + G::kYBytes);
#pragma unroll
    for (int r = 0; r < G::kRounds; ++r) {
      const int l0 = r * G::kRound + threadIdx.x * EPT;  // element offset inside the tile
      ST<P> xs[EPT * NC], ys[G::kY ? EPT * NC : 1], vv[G::kV ? EPT : 1];
      memcpy(xs, xs_s + l0 * NC, sizeof(xs));
      if constexpr (G::kY) memcpy(ys, ys_s + l0 * NC, sizeof(ys));
      if constexpr (G::kV) {
        if (vmode == 0) memcpy(vv, vs_s + l0, sizeof(vv));
      }
      ST<P> os[EPT * ONC];
      unsigned bail = 0;
      if constexpr (kG2Pair<OP, P, NC, ONC> && EPT == 2) {
        // both elements through the packed certified shortcut; a declined one
        // re-runs the register path alone
        float xp[4], yp[4], op[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          xp[c] = xs[c];
          yp[c] = G::kY ? ys[c] : 0.0f;
        }
        float v0 = 0.0f, v1 = 0.0f;
        if constexpr (G::kV) {
          v0 = vmode == 0 ? vv[0] : vscalar;
          v1 = vmode == 0 ? vv[1] : vscalar;
        }
        const g2::M2 ok = run_g2_pair<OP>(xp, yp, v0, v1, op);
#pragma unroll
        for (int c = 0; c < 4; ++c) os[c] = op[c];
        const bool acc[2] = {ok.x, ok.y};
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (!acc[i]) {
            RT<P> xa[NC], ya[NC], oa[ONC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              xa[c] = P::ld(xs[i * NC + c]);
              ya[c] = G::kY ? P::ld(ys[i * NC + c]) : RT<P>(0);
            }
            const RT<P> ve = i == 0 ? v0 : v1;
            if (!run_fast<OP, P, NC, ONC, false>(xa, ya, ve, oa)) bail |= 1u << i;
#pragma unroll
            for (int c = 0; c < ONC; ++c) os[i * ONC + c] = P::sv(oa[c]);
          }
      } else if constexpr (kW2<OP, P, NC, ONC>) {
        // the wide tier for every element first (no branch between them), then
        // the lower tiers for the declined ones
        bool acc[EPT];
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          float xa[2], ya[2], oa[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            xa[c] = xs[i * 2 + c];
            ya[c] = G::kY ? ys[i * 2 + c] : 0.0f;
          }
          float ve = 0.0f;
          if constexpr (G::kV) ve = vmode == 0 ? vv[i] : vscalar;
          acc[i] = run_w2<OP>(xa, ya, ve, oa);
          os[i * 2] = oa[0], os[i * 2 + 1] = oa[1];
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i)
          if (__builtin_expect(!acc[i], 0)) {
            RT<P> xa[NC], ya[NC], oa[ONC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              xa[c] = P::ld(xs[i * NC + c]);
              ya[c] = G::kY ? P::ld(ys[i * NC + c]) : RT<P>(0);
            }
            RT<P> ve = RT<P>(0);
            if constexpr (G::kV) ve = vmode == 0 ? P::ld(vv[i]) : vscalar;
            if (!run_fast<OP, P, NC, ONC, true, false>(xa, ya, ve, oa)) bail |= 1u << i;
#pragma unroll
            for (int c = 0; c < ONC; ++c) os[i * ONC + c] = P::sv(oa[c]);
          }
      } else {
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
          RT<P> xa[NC], ya[NC], oa[ONC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            xa[c] = P::ld(xs[i * NC + c]);
            ya[c] = G::kY ? P::ld(ys[i * NC + c]) : RT<P>(0);
          }
          RT<P> ve = RT<P>(0);
          if constexpr (G::kV) ve = vmode == 0 ? P::ld(vv[i]) : vscalar;
          if (!run_fast<OP, P, NC, ONC>(xa, ya, ve, oa)) bail |= 1u << i;
#pragma unroll
          for (int c = 0; c < ONC; ++c) os[i * ONC + c] = P::sv(oa[c]);
        }
      }
      ST<P>* og = out + (t * G::kTile + l0) * ONC;
      store_stream<ST<P>, EPT * ONC>(og, os);
      if (bail) {  // literal re-run from the staged operands (stage not yet released)
#pragma unroll 1
        for (int i = 0; i < EPT; ++i)
          if (bail >> i & 1u) {
            RT<P> ve = RT<P>(0);
            if constexpr (G::kV) ve = vmode == 0 ? P::ld(vs_s[l0 + i]) : vscalar;
            lit_element<OP, P>(xs_s + (l0 + i) * NC, G::kY ? ys_s + (l0 + i) * NC : nullptr, ve,
                               og + i * ONC, NC, ONC);
          }
      }
    }
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty[s]);
  }
}

// ---- literal kernel (any precision, any nc, mixed-nc padding) ----------------

template <int OP, class P>
__global__ void __launch_bounds__(kThreads) k_lit(const ST<P>* __restrict__ x, int ncx,
                                                  const ST<P>* __restrict__ y, int ncy,
                                                  const ST<P>* __restrict__ v, int64_t vn,
                                                  int vmode, ST<P>* __restrict__ out, int onc,
                                                  int64_t numel) {
  constexpr bool kY = OpTraits<OP>::kY, kV = OpTraits<OP>::kV;
  const int nc = kY ? (ncx > ncy ? ncx : ncy) : ncx;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += stride) {
    RT<P> xa[lit::kMaxNc], ya[lit::kMaxNc], oa[lit::kMaxNc + 1];
    for (int c = 0; c < nc; ++c) {
      xa[c] = c < ncx ? P::ld(x[e * ncx + c]) : RT<P>(0);
      ya[c] = (kY && c < ncy) ? P::ld(y[e * ncy + c]) : RT<P>(0);
    }
    const RT<P> vv = kV ? v_at<P>(v, vn, vmode, e) : RT<P>(0);
    run_lit<OP, P>(xa, ya, vv, oa, nc, onc);
    for (int c = 0; c < onc; ++c) out[e * onc + c] = P::sv(oa[c]);
  }
}

// ---- EFT array kernels (eft.hpp:89-111) -------------------------------------------

template <class P, bool PROD>
__global__ void __launch_bounds__(kThreads) k_eft(const ST<P>* __restrict__ a,
                                                  const ST<P>* __restrict__ b,
                                                  ST<P>* __restrict__ s, ST<P>* __restrict__ e,
                                                  int64_t n) {
  constexpr int EPT = ept_for<P, 1>();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g * EPT < n; g += stride) {
    const int64_t i0 = g * EPT;
    ST<P> as[EPT], bs[EPT], ss[EPT], es[EPT];
    const bool full = i0 + EPT <= n;
    if (full) {
      load_stream<ST<P>, EPT>(a + i0, as);
      load_stream<ST<P>, EPT>(b + i0, bs);
    } else {
#pragma unroll
      for (int i = 0; i < EPT; ++i) {
        as[i] = i0 + i < n ? a[i0 + i] : P::sv(RT<P>(0));
        bs[i] = i0 + i < n ? b[i0 + i] : P::sv(RT<P>(0));
      }
    }
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      RT<P> hi, lo;
      if constexpr (PROD) two_prod<P>(P::ld(as[i]), P::ld(bs[i]), hi, lo);
      else two_sum<P>(P::ld(as[i]), P::ld(bs[i]), hi, lo);
      ss[i] = P::sv(hi);
      es[i] = P::sv(lo);
    }
    if (full) {
      store_stream<ST<P>, EPT>(s + i0, ss);
      store_stream<ST<P>, EPT>(e + i0, es);
    } else {
#pragma unroll
      for (int i = 0; i < EPT; ++i)
        if (i0 + i < n) {
          s[i0 + i] = ss[i];
          e[i0 + i] = es[i];
        }
    }
  }
}

// approx: MC -> one working-precision value per element (smallest first)
template <class P, int NC>
__global__ void __launch_bounds__(kThreads) k_approx(const ST<P>* __restrict__ x,
                                                     ST<P>* __restrict__ out, int64_t numel) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += stride) {
    RT<P> acc = P::ld(x[e * NC + NC - 1]);
#pragma unroll
    for (int i = NC - 2; i >= 0; --i) acc = P::add(acc, P::ld(x[e * NC + i]));
    out[e] = P::sv(acc);
  }
}

// ---- host launch helpers -----------------------------------------------------

template <class K>
int per_sm(K kernel) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kThreads, 0) != cudaSuccess || n < 1) n = 1;
  return n;
}

struct Args {
  const void* x;
  int ncx;
  const void* y;
  int ncy;
  const void* v;
  int64_t vn;
  void* out;
  int onc;
  int64_t numel;
  cudaStream_t stream;
};

int vmode_of(int64_t vn, int64_t numel) { return vn == numel ? 0 : (vn == 1 ? 1 : 2); }

template <int OP, class P, int NC, int ONC>
mcf_status launch_fast(const Args& a) {
  using G = tma::Geo<P, NC, OP>;
  const int vmode = vmode_of(a.vn, a.numel);
  const ST<P>* x = static_cast<const ST<P>*>(a.x);
  const ST<P>* y = static_cast<const ST<P>*>(a.y);
  const ST<P>* v = static_cast<const ST<P>*>(a.v);
  ST<P>* out = static_cast<ST<P>*>(a.out);
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  static const bool tma_on = [] {
    const char* e = getenv("MCF_EW_TMA");
    return !(e && e[0] == '0');
  }();
  int64_t done = 0;
  const int64_t tiles = a.numel / G::kTile;
  if (tma_on && vmode != 2 && tiles > 0 && al16(x) && (!G::kY || al16(y)) && (!G::kV || vmode != 0 || al16(v)) &&
      al16(out) && ((int64_t)G::kTile * ONC * sizeof(ST<P>)) % 16 == 0) {
    auto kt = k_tma<OP, P, NC, ONC>;
    {
      const mcf_status ast = mcfr::ensure_smem_attr<k_tma<OP, P, NC, ONC>>(
          G::kSmem, "mcf: cannot reserve shared memory for the TMA ring");
      if (ast != MCF_OK) return ast;
    }
    // two rings per SM, except packed ScalingN and Grow-ExpN (measured 59 us
    // at one ring, 66 us at two): the packed ops are compiled for one ring (so
    // ptxas keeps FADD2 / FMUL2 / FFMA2) and fit two at their register counts
    const int64_t slots = (int64_t)mcfr::sm_count() * (kG2Pair<OP, P, NC, ONC> && (OP == kScale || OP == kGrow) ? 1
                                                        : kW2<OP, P, NC, ONC>                                  ? MCF_W2_CTAS
                                                                                                               : tma::kCtasPerSm);
    const int grid = (int)(tiles < slots ? tiles : slots);
    kt<<<grid, tma::kConsumerWarps * 32 + 32, G::kSmem, a.stream>>>(x, y, v, vmode, out, tiles);
    mcfr::note_launch();
    const mcf_status st = mcfr::check_launch("mcf elementwise kernel (TMA)");
    if (st != MCF_OK) return st;
    done = tiles * G::kTile;
    if (done == a.numel) return MCF_OK;
  }
  // remaining elements (or everything): register-pipelined grid-stride kernel
  const int64_t rest = a.numel - done;
  auto k = k_fast<OP, P, NC, ONC>;
  static const int occ = per_sm(k);
  constexpr int EPT = ept_for<P, NC>();
  const int grid = mcfr::grid_for((rest + EPT - 1) / EPT, kThreads, occ);
  k<<<grid, kThreads, 0, a.stream>>>(x + done * NC, G::kY ? y + done * NC : y,
                                      (G::kV && vmode == 0) ? v + done : v, vmode == 0 ? rest : a.vn, vmode,
                                      out + done * ONC, rest);
  mcfr::note_launch();
  return mcfr::check_launch("mcf elementwise kernel");
}

template <int OP, class P>
mcf_status launch_lit(const Args& a) {
  auto k = k_lit<OP, P>;
  static const int occ = per_sm(k);
  const int grid = mcfr::grid_for(a.numel, kThreads, occ);
  k<<<grid, kThreads, 0, a.stream>>>(static_cast<const ST<P>*>(a.x), a.ncx,
                                      static_cast<const ST<P>*>(a.y), a.ncy,
                                      static_cast<const ST<P>*>(a.v), a.vn, vmode_of(a.vn, a.numel),
                                      static_cast<ST<P>*>(a.out), a.onc, a.numel);
  mcfr::note_launch();
  return mcfr::check_launch("mcf elementwise kernel (literal)");
}

// register fast paths: binary32 with nc 1..4 and binary64 with nc 1..3
// (SURVEY 8f row 3), equal operand nc; everything else runs the literal
// kernels.  The fast paths' preconditions are checked per element at run
// time with the literal restatement as the fallback, so they are exact for
// any precision; binary16 keeps the literal kernels (one rounding per op).
template <int OP, class P>
mcf_status dispatch(const Args& a) {
  if (a.numel == 0) return MCF_OK;
  if constexpr (std::is_same<P, PB64>::value) {
    if constexpr (OP != kApprox && OP != kSimple && OP != kRenorm && OP != kScaleX) {
      const bool same_nc = !OpTraits<OP>::kY || a.ncx == a.ncy;
      if (same_nc) {
        switch (a.ncx) {
          case 1: return launch_fast<OP, P, 1, 1>(a);
          case 2: return launch_fast<OP, P, 2, 2>(a);
          case 3: return launch_fast<OP, P, 3, 3>(a);
          default: break;
        }
      }
    }
  }
  if constexpr (std::is_same<P, PB32>::value) {
    if constexpr (OP == kRenorm) {
      if (a.ncx == a.onc) {
        switch (a.ncx) {
          case 2: return launch_fast<kRenorm, P, 2, 2>(a);
          case 3: return launch_fast<kRenorm, P, 3, 3>(a);
          case 4: return launch_fast<kRenorm, P, 4, 4>(a);
          default: break;
        }
      } else if (a.ncx == a.onc + 1) {
        switch (a.onc) {
          case 2: return launch_fast<kRenorm, P, 3, 2>(a);
          case 3: return launch_fast<kRenorm, P, 4, 3>(a);
          default: break;
        }
      }
    } else if constexpr (OP == kScaleX) {
      switch (a.ncx) {
        case 1: return launch_fast<OP, P, 1, 2>(a);
        case 2: return launch_fast<OP, P, 2, 3>(a);
        case 3: return launch_fast<OP, P, 3, 4>(a);
        default: break;
      }
    } else if constexpr (OP != kApprox && OP != kSimple) {
      const bool same_nc = !OpTraits<OP>::kY || a.ncx == a.ncy;
      if (same_nc) {
        switch (a.ncx) {
          case 1: return launch_fast<OP, P, 1, 1>(a);
          case 2: return launch_fast<OP, P, 2, 2>(a);
          case 3: return launch_fast<OP, P, 3, 3>(a);
          case 4:
            if constexpr (OP != kMulSlow && OP != kSquare) return launch_fast<OP, P, 4, 4>(a);
            break;
          default: break;
        }
      }
    }
  }
  return launch_lit<OP, P>(a);
}

template <int OP>
mcf_status dispatch_prec(mcf_prec p, const Args& a) {
  const mcf_status ready = mcfr::ensure_device_tables();
  if (ready != MCF_OK) return ready;
  switch (p) {
    case MCF_B16: return dispatch<OP, PB16>(a);
    case MCF_B32: return dispatch<OP, PB32>(a);
    case MCF_B64: return dispatch<OP, PB64>(a);
  }
  return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "unknown precision");
}

mcf_status approx_dispatch(mcf_prec p, const void* x, int nc, void* out, int64_t numel,
                           cudaStream_t s) {
  if (numel == 0) return MCF_OK;
  auto go = [&](auto tag, auto nct) -> mcf_status {
    using P = decltype(tag);
    constexpr int NC = decltype(nct)::value;
    auto k = k_approx<P, NC>;
    static const int occ = per_sm(k);
    k<<<mcfr::grid_for(numel, kThreads, occ), kThreads, 0, s>>>(static_cast<const ST<P>*>(x),
                                                                static_cast<ST<P>*>(out), numel);
    mcfr::note_launch();
    return mcfr::check_launch("mcf approx kernel");
  };
  if (p == MCF_B32) {
    switch (nc) {
      case 1: return go(PB32{}, std::integral_constant<int, 1>{});
      case 2: return go(PB32{}, std::integral_constant<int, 2>{});
      case 3: return go(PB32{}, std::integral_constant<int, 3>{});
      case 4: return go(PB32{}, std::integral_constant<int, 4>{});
    }
  }
  Args a{x, nc, nullptr, nc, nullptr, 1, out, 1, numel, s};
  return dispatch_prec<kApprox>(p, a);
}

std::mutex g_tab_mu;
bool g_tab_done[64];

}  // namespace
}  // namespace mcfg

namespace mcfr {
mcf_status ensure_device_tables() {
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) d = 0;
  std::lock_guard<std::mutex> lk(mcfg::g_tab_mu);
  if (mcfg::g_tab_done[d]) return MCF_OK;
  // The literal fallback path keeps reference-sized staging arrays in local
  // memory (binary64 renorm stages are 640 B per frame and the deepest chain,
  // mul_mcn -> div -> add -> renorm, exceeds the 1 KiB default stack).
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitStackSize);
  if (cur < 4096 && cudaDeviceSetLimit(cudaLimitStackSize, 4096) != cudaSuccess)
    return fail(MCF_ERR_CUDA, "mcf: cannot raise the device stack limit");
  double tab[4096];
  exp2_table(tab);
  if (cudaMemcpyToSymbol(mcfg::g_exp_tab, tab, sizeof(tab)) != cudaSuccess)
    return fail(MCF_ERR_CUDA, "mcf: cannot upload the exp table to the device");
  mcfg::g_tab_done[d] = true;
  return MCF_OK;
}
}  // namespace mcfr

// ---- C-ABI ---------------------------------------------------------------------

using mcfg::Args;

namespace {

mcf_status check_common(mcf_prec p, int64_t numel, const char* op) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, std::string(op) + ": unknown precision");
  if (numel < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, std::string(op) + ": negative element count");
  return MCF_OK;
}

mcf_status check_nc(int nc) {
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  return MCF_OK;
}

mcf_status check_vn(int64_t vn, int64_t numel, const char* op) {
  if (vn < 1 || (numel > 0 && numel % vn != 0))
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT,
                      std::string(op) + ": operand of " + std::to_string(vn) +
                          " elements does not broadcast over " + std::to_string(numel));
  return MCF_OK;
}

#define MCF_TRY(expr)                  \
  do {                                 \
    const mcf_status _s = (expr);      \
    if (_s != MCF_OK) return _s;       \
  } while (0)

template <int OP>
mcf_status binary(const char* name, mcf_prec p, const void* x, int ncx, const void* y, int ncy,
                  void* out, int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, name));
  MCF_TRY(check_nc(ncx));
  MCF_TRY(check_nc(ncy));
  const int nc = ncx > ncy ? ncx : ncy;
  Args a{x, ncx, y, ncy, nullptr, 1, out, nc, numel, s};
  return mcfg::dispatch_prec<OP>(p, a);
}

}  // namespace

extern "C" {

mcf_status mcf_two_sum(mcf_prec p, const void* a, const void* b, void* s, void* e, int64_t n,
                       mcf_stream stream) {
  MCF_TRY(check_common(p, n, "two_sum"));
  if (n == 0) return MCF_OK;
  auto go = [&](auto tag) -> mcf_status {
    using P = decltype(tag);
    using S = typename P::st;
    auto k = mcfg::k_eft<P, false>;
    static const int occ = mcfg::per_sm(k);
    constexpr int EPT = mcfg::ept_for<P, 1>();
    k<<<mcfr::grid_for((n + EPT - 1) / EPT, mcfg::kThreads, occ), mcfg::kThreads, 0, stream>>>(
        static_cast<const S*>(a), static_cast<const S*>(b), static_cast<S*>(s), static_cast<S*>(e), n);
    mcfr::note_launch();
    return mcfr::check_launch("two_sum kernel");
  };
  return p == MCF_B16 ? go(mcfg::PB16{}) : p == MCF_B32 ? go(mcfg::PB32{}) : go(mcfg::PB64{});
}

mcf_status mcf_two_prod(mcf_prec p, const void* a, const void* b, void* prod, void* e, int64_t n,
                        mcf_stream stream) {
  MCF_TRY(check_common(p, n, "two_prod"));
  if (n == 0) return MCF_OK;
  auto go = [&](auto tag) -> mcf_status {
    using P = decltype(tag);
    using S = typename P::st;
    auto k = mcfg::k_eft<P, true>;
    static const int occ = mcfg::per_sm(k);
    constexpr int EPT = mcfg::ept_for<P, 1>();
    k<<<mcfr::grid_for((n + EPT - 1) / EPT, mcfg::kThreads, occ), mcfg::kThreads, 0, stream>>>(
        static_cast<const S*>(a), static_cast<const S*>(b), static_cast<S*>(prod), static_cast<S*>(e), n);
    mcfr::note_launch();
    return mcfr::check_launch("two_prod kernel");
  };
  return p == MCF_B16 ? go(mcfg::PB16{}) : p == MCF_B32 ? go(mcfg::PB32{}) : go(mcfg::PB64{});
}

mcf_status mcf_renormalize(mcf_prec p, const void* h, int nc, void* out, int r_nc, int64_t numel,
                           mcf_stream s) {
  MCF_TRY(check_common(p, numel, "renormalize"));
  MCF_TRY(check_nc(nc));
  MCF_TRY(check_nc(r_nc));
  return mcfg::dispatch_prec<mcfg::kRenorm>(p, Args{h, nc, nullptr, nc, nullptr, 1, out, r_nc, numel, s});
}

mcf_status mcf_simple_renorm(mcf_prec p, const void* h, int nc, void* out, int r_nc,
                             int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "simple_renorm"));
  MCF_TRY(check_nc(nc));
  MCF_TRY(check_nc(r_nc));
  return mcfg::dispatch_prec<mcfg::kSimple>(p, Args{h, nc, nullptr, nc, nullptr, 1, out, r_nc, numel, s});
}

mcf_status mcf_approx(mcf_prec p, const void* x, int nc, void* out, int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "approx"));
  MCF_TRY(check_nc(nc));
  return mcfg::approx_dispatch(p, x, nc, out, numel, s);
}

mcf_status mcf_negate(mcf_prec p, const void* x, int nc, void* out, int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "negate"));
  MCF_TRY(check_nc(nc));
  return mcfg::dispatch_prec<mcfg::kNeg>(p, Args{x, nc, nullptr, nc, nullptr, 1, out, nc, numel, s});
}

mcf_status mcf_grow_expn(mcf_prec p, const void* x, int nc, const void* v, int64_t vn, void* out,
                         int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "grow_expn"));
  MCF_TRY(check_nc(nc));
  MCF_TRY(check_vn(vn, numel, "grow_expn"));
  return mcfg::dispatch_prec<mcfg::kGrow>(p, Args{x, nc, nullptr, nc, v, vn, out, nc, numel, s});
}

mcf_status mcf_scaling_n(mcf_prec p, const void* x, int nc, const void* v, int64_t vn, int expanded,
                         void* out, int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "scaling_n"));
  MCF_TRY(check_nc(nc));
  MCF_TRY(check_vn(vn, numel, "scaling_n"));
  if (expanded) {
    MCF_TRY(check_nc(nc + 1));
    return mcfg::dispatch_prec<mcfg::kScaleX>(p, Args{x, nc, nullptr, nc, v, vn, out, nc + 1, numel, s});
  }
  return mcfg::dispatch_prec<mcfg::kScale>(p, Args{x, nc, nullptr, nc, v, vn, out, nc, numel, s});
}

mcf_status mcf_div_n(mcf_prec p, const void* v, int64_t vn, const void* y, int nc, void* out,
                     int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "div_n"));
  MCF_TRY(check_nc(nc));
  MCF_TRY(check_vn(vn, numel, "div_n"));
  return mcfg::dispatch_prec<mcfg::kDivN>(p, Args{y, nc, nullptr, nc, v, vn, out, nc, numel, s});
}

mcf_status mcf_add_mcn(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                       int64_t numel, mcf_stream s) {
  return binary<mcfg::kAdd>("add_mcn", p, x, ncx, y, ncy, out, numel, s);
}
mcf_status mcf_div_mcn(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                       int64_t numel, mcf_stream s) {
  return binary<mcfg::kDiv>("div_mcn", p, x, ncx, y, ncy, out, numel, s);
}
mcf_status mcf_mul_mcn(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                       int64_t numel, mcf_stream s) {
  return binary<mcfg::kMul>("mul_mcn", p, x, ncx, y, ncy, out, numel, s);
}
mcf_status mcf_mul_mcn_slow(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                            int64_t numel, mcf_stream s) {
  return binary<mcfg::kMulSlow>("mul_mcn_slow", p, x, ncx, y, ncy, out, numel, s);
}

mcf_status mcf_square_mcn(mcf_prec p, const void* x, int nc, void* out, int64_t numel,
                          mcf_stream s) {
  MCF_TRY(check_common(p, numel, "square_mcn"));
  MCF_TRY(check_nc(nc));
  return mcfg::dispatch_prec<mcfg::kSquare>(p, Args{x, nc, nullptr, nc, nullptr, 1, out, nc, numel, s});
}

mcf_status mcf_exp_mcn(mcf_prec p, const void* x, int nc, void* out, int64_t numel, mcf_stream s) {
  MCF_TRY(check_common(p, numel, "exp_mcn"));
  MCF_TRY(check_nc(nc));
  MCF_TRY(mcfr::ensure_device_tables());
  return mcfg::dispatch_prec<mcfg::kExp>(p, Args{x, nc, nullptr, nc, nullptr, 1, out, nc, numel, s});
}

}  // extern "C"
