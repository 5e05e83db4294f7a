// mcf_fast.cuh -- register-resident MCF kernels, bit-exact with the reference.
//
// The reference's renormalization (mc_ops.hpp:68-92) drops zeros, sorts by
// magnitude, then repeats {bottom-up two_sum sweep; compact zeros} while the
// sequence is not "compressed" and pass < m + 4.  With nc fixed at compile
// time this becomes straight-line register code:
//
//  * zeros are not compacted between sweeps.  two_sum(0, q) = (q, 0) and
//    two_sum(a, 0) = (a, 0), so a sweep over a sequence with interleaved zeros
//    produces the same nonzero subsequence as the sweep over the compacted
//    one; only the final output compacts (first r_nc nonzeros, +0 padding).
//  * the sort is a stable adjacent-transposition (insertion) network; zeros
//    sink to the end exactly as if they had been dropped first.
//  * each sweep also decides whether its INPUT was compressed: walking up,
//    as long as every step leaves h[i] unchanged (fl(h[i] + q) == h[i]) the
//    carry q is exactly the next nonzero below, i.e. the step performs the
//    reference's is_compressed test.  A sweep over a compressed, finite
//    sequence is the identity on its nonzero subsequence, so "sweep, and stop
//    when nothing changed" equals the reference loop.
//  * the pass cap m + 4 cannot bind before pass 6 (m >= 2 while a sweep is
//    still needed), so up to 6 changing sweeps are always the reference's;
//    a 7th changing sweep, an unordered operand where the reference merges,
//    or a non-finite result makes the element fall back to the literal path
//    (mcf_lit.cuh), which restates the reference line by line.
#pragma once

#include "mcf_exp.cuh"
#include "mcf_prec.cuh"

namespace mcfg {
namespace fast {

template <class P>
using RT = typename P::rt;

constexpr int kSafeSweeps = 7;  // 6 reference passes + 1 confirming sweep

// stable insertion network over h[0..N), elements [0, PRE) already ordered
template <class P, int N, int PRE>
__device__ __forceinline__ void sort_net(RT<P> (&h)[N]) {
#pragma unroll
  for (int i = (PRE < 1 ? 1 : PRE); i < N; ++i) {
#pragma unroll
    for (int j = i - 1; j >= 0; --j) {
      const RT<P> a = h[j], b = h[j + 1];
      const bool sw = P::mag(a) < P::mag(b);
      h[j] = sw ? b : a;
      h[j + 1] = sw ? a : b;
    }
  }
}

// one bottom-up two_sum sweep; true when it changed the nonzero subsequence
// (i.e. its input was not compressed)
template <class P, int N>
__device__ __forceinline__ bool sweep_once(RT<P> (&h)[N]) {
  bool changed = false;
  RT<P> q = h[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; --i) {
    RT<P> s, e;
    two_sum<P>(h[i], q, s, e);
    changed |= (h[i] != RT<P>(0)) & (s != h[i]);
    h[i + 1] = e;
    q = s;
  }
  h[0] = q;
  return changed;
}

// the same sweep without the change test
template <class P, int N>
__device__ __forceinline__ void sweep_blind(RT<P> (&h)[N]) {
  RT<P> q = h[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; --i) {
    RT<P> s, e;
    two_sum<P>(h[i], q, s, e);
    h[i + 1] = e;
    q = s;
  }
  h[0] = q;
}

// repeated sweeps until one leaves the sequence unchanged (fully unrolled:
// no loop counter, one early exit per sweep).  The first PU sweeps skip the
// change test: a sweep over a compressed finite sequence is the identity on
// its nonzero subsequence, and no pass before the 7th can hit the reference's
// cap, so PU <= 6 blind sweeps followed by tested ones give the reference's
// result.  PU is chosen per operator from the measured pass distribution
// (the warp pays for its slowest lane).
template <class P, int N, int PU = 0>
__device__ __forceinline__ bool sweeps(RT<P> (&h)[N]) {
  static_assert(PU < kSafeSweeps, "blind sweeps must stay below the pass cap");
  if constexpr (N < 2) {
    return true;
  } else {
#pragma unroll
    for (int pass = 0; pass < PU; ++pass) sweep_blind<P, N>(h);
#pragma unroll
    for (int pass = PU; pass < kSafeSweeps; ++pass)
      if (!sweep_once<P, N>(h)) return true;
    return false;
  }
}

// first R nonzeros of h in order, +0 padded (mc_ops.hpp:91)
template <class P, int N, int R>
__device__ __forceinline__ void compact(const RT<P> (&h)[N], RT<P> (&out)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = RT<P>(0);
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const bool nz = h[i] != RT<P>(0);
#pragma unroll
    for (int r = R - 1; r > 0; --r) out[r] = nz ? out[r - 1] : out[r];
    out[0] = nz ? h[i] : out[0];
  }
}

// One backward scan that both compacts (first R nonzeros, +0 padded) and
// evaluates the reference's is_compressed over the nonzero subsequence:
// out[0] always holds the nearest nonzero below position i, i.e. the
// successor the reference compares h[i] with.
template <class P, int N, int R>
__device__ __forceinline__ bool scan(const RT<P> (&h)[N], RT<P> (&out)[R]) {
  bool comp = true;
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = RT<P>(0);
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const bool nz = h[i] != RT<P>(0);
    if (i < N - 1) comp &= !nz | (P::add(h[i], out[0]) == h[i]);
#pragma unroll
    for (int r = R - 1; r > 0; --r) out[r] = nz ? out[r - 1] : out[r];
    out[0] = nz ? h[i] : out[0];
  }
  return comp;
}

// renorm_kernel(h, N, out, R); PRE leading terms are known to be ordered.
// PU blind sweeps (see sweeps()), then scan; while the scan finds the
// sequence not compressed, one more sweep (a real reference pass: pass
// index PU + extra < 6 keeps it below the cap) and scan again.
template <class P, int N, int R, int PRE = 1, int PU = 0>
__device__ __forceinline__ bool renorm(RT<P> (&h)[N], RT<P> (&out)[R]) {
  static_assert(PU < kSafeSweeps - 1, "blind sweeps must stay below the pass cap");
  sort_net<P, N, PRE>(h);
  if constexpr (N >= 2) {
#pragma unroll
    for (int pass = 0; pass < PU; ++pass) sweep_blind<P, N>(h);
  }
  bool comp = scan<P, N, R>(h, out);
  if constexpr (N >= 2) {
#pragma unroll 1
    for (int extra = PU; !comp; ++extra) {
      if (extra >= kSafeSweeps - 1) return false;  // a 7th pass could hit the cap: literal path
      sweep_blind<P, N>(h);
      comp = scan<P, N, R>(h, out);
    }
  }
  return P::finite(out[0]);
}

template <class P, int NC>
__device__ __forceinline__ bool ordered(const RT<P> (&x)[NC]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i + 1 < NC; ++i) ok &= P::mag(x[i]) >= P::mag(x[i + 1]);
  return ok;
}

// mc_ops.hpp:105-110
template <class P, int NC>
__device__ __forceinline__ RT<P> approx(const RT<P> (&x)[NC]) {
  RT<P> acc = x[NC - 1];
#pragma unroll
  for (int i = NC - 2; i >= 0; --i) acc = P::add(acc, x[i]);
  return acc;
}

// mc_ops.hpp:118-138  Grow-ExpN
template <class P, int NC>
__device__ __forceinline__ bool grow(const RT<P> (&x)[NC], RT<P> v, RT<P> (&out)[NC]) {
  RT<P> h[NC + 1];
  RT<P> q = v;
#pragma unroll
  for (int k = NC; k >= 1; --k) two_sum<P>(x[k - 1], q, q, h[k]);
  h[0] = q;
  // The reference returns the compacted ladder when it is compressed and
  // renorm_kernel(h, nc+1, out, nc) otherwise.  The two agree whenever the
  // ladder is compressed (compressed => strictly magnitude-ordered => the
  // sort is the identity and the pass loop never runs), so renorm always.
  // (config 0: <= 2 passes, warp maximum 1 or 2 -> one blind sweep)
  return renorm<P, NC + 1, NC, 1, 1>(h, out);
}

// mc_ops.hpp:143-158
template <class P, int NC>
__device__ __forceinline__ void scale_raw(const RT<P> (&x)[NC], RT<P> v, RT<P> (&st)[2 * NC]) {
  RT<P> q;
  two_prod<P>(x[NC - 1], v, q, st[0]);
  int k = 1;
#pragma unroll
  for (int i = NC - 2; i >= 0; --i) {
    RT<P> t, tl, s1, s2;
    two_prod<P>(x[i], v, t, tl);
    two_sum<P>(q, tl, s1, st[k++]);
    two_sum<P>(t, s1, s2, st[k++]);
    q = s2;
  }
  st[2 * NC - 1] = q;
}

// mc_ops.hpp:160-169  ScalingN (ONC = NC, or NC+1 when expanded)
template <class P, int NC, int ONC>
__device__ __forceinline__ bool scale(const RT<P> (&x)[NC], RT<P> v, RT<P> (&out)[ONC]) {
  if constexpr (NC == 1 && ONC == 1) {
    out[0] = P::mul(x[0], v);
    return true;
  } else {
    RT<P> st[2 * NC];
    scale_raw<P, NC>(x, v, st);
    return renorm<P, 2 * NC, ONC, 1, 1>(st, out);  // config 0: <= 2 passes
  }
}

// mc_ops.hpp:173-184 for ordered operands: the magnitude merge with x winning
// ties equals the stable sort of the concatenation x ++ y.
template <class P, int NC, int ONC, int PU = 2>
__device__ __forceinline__ bool add_ordered(const RT<P> (&x)[NC], const RT<P> (&y)[NC],
                                            RT<P> (&out)[ONC]) {
  RT<P> h[2 * NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    h[i] = x[i];
    h[NC + i] = y[i];
  }
  return renorm<P, 2 * NC, ONC, NC, PU>(h, out);
}

template <class P, int NC>
__device__ __forceinline__ bool add(const RT<P> (&x)[NC], const RT<P> (&y)[NC],
                                    RT<P> (&out)[NC]) {
  const bool ord = ordered<P, NC>(x) & ordered<P, NC>(y);
  // config 0: 1-3 passes, the warp maximum is 3 for 99.7% of warps
  return add_ordered<P, NC, NC, 3>(x, y, out) && ord;
}

// mc_ops.hpp:188-207  long division, nc digits + 1 guard digit
template <class P, int NC>
__device__ __forceinline__ bool div(const RT<P> (&x)[NC], const RT<P> (&y)[NC],
                                    RT<P> (&out)[NC]) {
  if constexpr (NC == 1) {
    out[0] = P::div(x[0], y[0]);
    return true;
  } else {
    bool ok = ordered<P, NC>(x);  // r = x is merged by add_kernel
    RT<P> r[NC], q[NC + 1];
#pragma unroll
    for (int i = 0; i < NC; ++i) r[i] = x[i];
#pragma unroll
    for (int d = 0; d <= NC; ++d) {
      q[d] = P::div(r[0], y[0]);
      if (d == NC) break;
      RT<P> st[2 * NC], sc[NC];
      scale_raw<P, NC>(y, -q[d], st);
      ok &= renorm<P, 2 * NC, NC, 1, 1>(st, sc);
      ok &= add_ordered<P, NC, NC, 2>(r, sc, r);  // both are renorm outputs: ordered
    }
    ok &= renorm<P, NC + 1, NC, 1, 1>(q, out);
    return ok;
  }
}

// mc_ops.hpp:216-230  Mul-MCN fast
template <class P, int NC>
__device__ __forceinline__ bool mul_fast(const RT<P> (&x)[NC], const RT<P> (&y)[NC],
                                         RT<P> (&out)[NC]) {
  if constexpr (NC == 1) {
    out[0] = P::mul(x[0], y[0]);
    return true;
  } else {
    if (approx<P, NC>(y) == RT<P>(0) || approx<P, NC>(x) == RT<P>(0)) {
#pragma unroll
      for (int i = 0; i < NC; ++i) out[i] = RT<P>(0);
      return true;
    }
    RT<P> one[NC], rec[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) one[i] = RT<P>(i == 0 ? 1 : 0);
    bool ok = div<P, NC>(one, y, rec);
    ok &= div<P, NC>(x, rec, out);
    return ok;
  }
}

constexpr int mul_slow_terms(int nc) { return nc * (nc + 1) + nc - 1; }
constexpr int square_terms(int nc) {
  int m = 0;
  for (int i = 0; i < nc; ++i)
    for (int j = i; i + j < nc; ++j) m += 2;
  for (int i = 1; i < nc; ++i) {
    if (nc - i < i) break;
    m += 1;
  }
  return m;
}

// mc_ops.hpp:235-251  Mul-MCN slow
template <class P, int NC>
__device__ __forceinline__ bool mul_slow(const RT<P> (&x)[NC], const RT<P> (&y)[NC],
                                         RT<P> (&out)[NC]) {
  if constexpr (NC == 1) {
    out[0] = P::mul(x[0], y[0]);
    return true;
  } else {
    RT<P> h[mul_slow_terms(NC)];
    int m = 0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int j = 0; i + j < NC; ++j) {
        two_prod<P>(x[i], y[j], h[m], h[m + 1]);
        m += 2;
      }
#pragma unroll
    for (int i = 1; i < NC; ++i) h[m++] = P::mul(x[i], y[NC - i]);
    return renorm<P, mul_slow_terms(NC), NC, 1, 2>(h, out);
  }
}

// mc_ops.hpp:256-282  Square-MCN
template <class P, int NC>
__device__ __forceinline__ bool square(const RT<P> (&x)[NC], RT<P> (&out)[NC]) {
  if constexpr (NC == 1) {
    out[0] = P::mul(x[0], x[0]);
    return true;
  } else {
    RT<P> h[square_terms(NC)];
    int m = 0;
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int j = i; i + j < NC; ++j) {
        RT<P> p, e;
        two_prod<P>(x[i], x[j], p, e);
        h[m++] = i == j ? p : P::twice(p);
        h[m++] = i == j ? e : P::twice(e);
      }
#pragma unroll
    for (int i = 1; i < NC; ++i) {
      const int j = NC - i;
      if (j < i) break;
      const RT<P> p = P::mul(x[i], x[j]);
      h[m++] = i == j ? p : P::twice(p);
    }
    return renorm<P, square_terms(NC), NC, 1, 3>(h, out);  // config 0: warp max 3 passes
  }
}

// mc_ops.hpp:286-297
template <class P, int NC>
__device__ __forceinline__ void expand_double(double v, RT<P> (&out)[NC]) {
  double rest = v;
  bool live = true;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const RT<P> c = P::rd(rest);
    out[i] = live ? c : RT<P>(0);
    live &= P::finite(c);
    rest = __dsub_rn(rest, P::to_d(c));
  }
}

// mc_ops.hpp:303-313  Exp-MCN (correctly rounded binary64 exp, mcf_exp.cuh)
template <class P, int NC>
__device__ __forceinline__ bool exp(const RT<P> (&x)[NC], RT<P> (&out)[NC]) {
  expand_double<P, NC>(cr_exp(P::to_d(x[0])), out);
  bool ok = true;
#pragma unroll
  for (int i = 1; i < NC; ++i) {
    if (x[i] != RT<P>(0)) {
      const RT<P> f = P::rd(cr_exp(P::to_d(x[i])));
      RT<P> tmp[NC];
      ok &= scale<P, NC, NC>(out, f, tmp);
#pragma unroll
      for (int j = 0; j < NC; ++j) out[j] = tmp[j];
    }
  }
  // a non-finite lead (overflow) is legal reference output; let the literal
  // path reproduce the reference's exact handling of it
  return ok && P::finite(out[0]);
}

}  // namespace fast
}  // namespace mcfg
