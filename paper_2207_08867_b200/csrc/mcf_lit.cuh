// mcf_lit.cuh -- the "literal" per-element MCF kernels.
//
// Runtime component count (1..8), local staging arrays, and control flow that
// follows the reference statement by statement (cited per function).  This
// path is bit-exact for every input the reference accepts -- including
// unordered/overlapping components, zeros anywhere and non-finite values --
// and serves two roles:
//   * the kernel for precisions / nc without a register fast path, and
//   * the per-element fallback a fast kernel takes when its own preconditions
//     (ordered inputs, convergence within the safe pass count, finite values)
//     do not hold for that element.
#pragma once

#include "mcf_exp.cuh"
#include "mcf_prec.cuh"

namespace mcfg {
namespace lit {

constexpr int kMaxNc = 8;   // mc_ops.hpp:27
constexpr int kStage = 80;  // largest term count fed to renorm: mul_slow at nc=8 (79)

template <class P>
using R = typename P::rt;

// mc_ops.hpp:41-52
template <class P>
__device__ void sort_mag(R<P>* h, int n) {
  for (int i = 1; i < n; ++i) {
    const R<P> cur = h[i];
    const R<P> cm = P::mag(cur);
    int j = i - 1;
    for (; j >= 0 && P::mag(h[j]) < cm; --j) h[j + 1] = h[j];
    h[j + 1] = cur;
  }
}

// mc_ops.hpp:56-62
template <class P>
__device__ bool compressed(const R<P>* h, int n) {
  for (int i = 0; i + 1 < n; ++i)
    if (P::add(h[i], h[i + 1]) != h[i]) return false;
  return true;
}

// mc_ops.hpp:68-92
template <class P>
__device__ __noinline__ void renorm(const R<P>* in, int n, R<P>* out, int r_nc) {
  R<P> h[kStage];
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (in[i] != R<P>(0)) h[m++] = in[i];
  if (m > 1) {
    sort_mag<P>(h, m);
    for (int pass = 0; pass < m + 4 && !compressed<P>(h, m); ++pass) {
      for (int i = m - 2; i >= 0; --i) two_sum<P>(h[i], h[i + 1], h[i], h[i + 1]);
      int k = 0;
      for (int i = 0; i < m; ++i)
        if (h[i] != R<P>(0)) h[k++] = h[i];
      m = k;
      if (m <= 1) break;
    }
  }
  for (int i = 0; i < r_nc; ++i) out[i] = i < m ? h[i] : R<P>(0);
}

// mc_ops.hpp:96-103
template <class P>
__device__ void simple_renorm(const R<P>* in, int n, R<P>* out, int r_nc) {
  int k = 0;
  for (int i = 0; i < n && k < r_nc; ++i)
    if (in[i] != R<P>(0)) out[k++] = in[i];
  for (; k < r_nc; ++k) out[k] = R<P>(0);
}

// mc_ops.hpp:105-110
template <class P>
__device__ R<P> approx(const R<P>* x, int nc) {
  R<P> acc = x[nc - 1];
  for (int i = nc - 2; i >= 0; --i) acc = P::add(acc, x[i]);
  return acc;
}

// mc_ops.hpp:118-138
template <class P>
__device__ __noinline__ void grow(const R<P>* x, int nc, R<P> v, R<P>* out) {
  R<P> h[kMaxNc + 1], c[kMaxNc + 1];
  R<P> q = v;
  for (int k = nc; k >= 1; --k) two_sum<P>(x[k - 1], q, q, h[k]);
  h[0] = q;
  int m = 0;
  for (int i = 0; i <= nc; ++i)
    if (h[i] != R<P>(0)) c[m++] = h[i];
  if (compressed<P>(c, m)) {
    for (int i = 0; i < nc; ++i) out[i] = i < m ? c[i] : R<P>(0);
  } else {
    renorm<P>(h, nc + 1, out, nc);
  }
}

// mc_ops.hpp:143-158
template <class P>
__device__ int scale_raw(const R<P>* x, int nc, R<P> v, R<P>* out) {
  R<P> q, h0;
  two_prod<P>(x[nc - 1], v, q, h0);
  out[0] = h0;
  int k = 1;
  for (int i = nc - 2; i >= 0; --i) {
    R<P> t, tl, s1, e1, s2, e2;
    two_prod<P>(x[i], v, t, tl);
    two_sum<P>(q, tl, s1, e1);
    out[k++] = e1;
    two_sum<P>(t, s1, s2, e2);
    out[k++] = e2;
    q = s2;
  }
  out[k++] = q;
  return k;
}

// mc_ops.hpp:160-169
template <class P>
__device__ __noinline__ void scale(const R<P>* x, int nc, R<P> v, R<P>* out, int out_nc) {
  if (nc == 1 && out_nc == 1) {
    out[0] = P::mul(x[0], v);
    return;
  }
  R<P> st[2 * kMaxNc];
  const int m = scale_raw<P>(x, nc, v, st);
  renorm<P>(st, m, out, out_nc);
}

// mc_ops.hpp:173-184
template <class P>
__device__ __noinline__ void add(const R<P>* x, int ncx, const R<P>* y, int ncy, R<P>* out, int out_nc) {
  R<P> h[2 * kMaxNc + 2];
  int i = 0, j = 0, k = 0;
  while (i < ncx && j < ncy) h[k++] = P::mag(x[i]) >= P::mag(y[j]) ? x[i++] : y[j++];
  while (i < ncx) h[k++] = x[i++];
  while (j < ncy) h[k++] = y[j++];
  renorm<P>(h, k, out, out_nc);
}

// mc_ops.hpp:188-207
// (kept out of line: with two inlined copies under mul_fast, binary64 code
// generation produced wrong low components on sm_100a -- see DESIGN.md)
template <class P>
__device__ __noinline__ void div(const R<P>* x, const R<P>* y, int nc, R<P>* out) {
  if (nc == 1) {
    out[0] = P::div(x[0], y[0]);
    return;
  }
  R<P> q[kMaxNc + 1], r[kMaxNc], st[2 * kMaxNc], sc[kMaxNc];
  for (int i = 0; i < nc; ++i) r[i] = x[i];
  for (int d = 0;; ++d) {
    q[d] = P::div(r[0], y[0]);
    if (d == nc) break;
    const int m = scale_raw<P>(y, nc, -q[d], st);
    renorm<P>(st, m, sc, nc);
    add<P>(r, nc, sc, nc, r, nc);
  }
  renorm<P>(q, nc + 1, out, nc);
}

// mc_ops.hpp:216-230
template <class P>
__device__ __noinline__ void mul_fast(const R<P>* x, const R<P>* y, int nc, R<P>* out) {
  if (nc == 1) {
    out[0] = P::mul(x[0], y[0]);
    return;
  }
  if (approx<P>(y, nc) == R<P>(0) || approx<P>(x, nc) == R<P>(0)) {
    for (int i = 0; i < nc; ++i) out[i] = R<P>(0);
    return;
  }
  R<P> one[kMaxNc], rec[kMaxNc];
  for (int i = 0; i < nc; ++i) one[i] = R<P>(i == 0 ? 1 : 0);
  div<P>(one, y, nc, rec);
  div<P>(x, rec, nc, out);
}

// mc_ops.hpp:235-251
template <class P>
__device__ __noinline__ void mul_slow(const R<P>* x, const R<P>* y, int nc, R<P>* out) {
  if (nc == 1) {
    out[0] = P::mul(x[0], y[0]);
    return;
  }
  R<P> h[kStage];
  int m = 0;
  for (int i = 0; i < nc; ++i)
    for (int j = 0; i + j < nc; ++j) {
      two_prod<P>(x[i], y[j], h[m], h[m + 1]);
      m += 2;
    }
  for (int i = 1; i < nc; ++i) h[m++] = P::mul(x[i], y[nc - i]);
  renorm<P>(h, m, out, nc);
}

// mc_ops.hpp:256-282
template <class P>
__device__ __noinline__ void square(const R<P>* x, int nc, R<P>* out) {
  if (nc == 1) {
    out[0] = P::mul(x[0], x[0]);
    return;
  }
  R<P> h[kStage];
  int m = 0;
  for (int i = 0; i < nc; ++i)
    for (int j = i; i + j < nc; ++j) {
      R<P> p, e;
      two_prod<P>(x[i], x[j], p, e);
      h[m++] = i == j ? p : P::twice(p);
      h[m++] = i == j ? e : P::twice(e);
    }
  for (int i = 1; i < nc; ++i) {
    const int j = nc - i;
    if (j < i) break;
    const R<P> p = P::mul(x[i], x[j]);
    h[m++] = i == j ? p : P::twice(p);
  }
  renorm<P>(h, m, out, nc);
}

// mc_ops.hpp:286-297
template <class P>
__device__ void expand_double(double v, R<P>* out, int nc) {
  double rest = v;
  for (int i = 0; i < nc; ++i) {
    out[i] = P::rd(rest);
    if (!isfinite(P::to_d(out[i]))) {
      for (int j = i + 1; j < nc; ++j) out[j] = R<P>(0);
      return;
    }
    rest = __dsub_rn(rest, P::to_d(out[i]));
  }
}

// mc_ops.hpp:303-313, with a correctly rounded binary64 exp (see mcf_exp.cuh)
template <class P>
__device__ __noinline__ void exp(const R<P>* x, int nc, R<P>* out) {
  expand_double<P>(cr_exp(P::to_d(x[0])), out, nc);
  for (int i = 1; i < nc; ++i) {
    if (x[i] == R<P>(0)) continue;
    const R<P> f = P::rd(cr_exp(P::to_d(x[i])));  // fl_exp<P>, precision.hpp:191-192
    R<P> tmp[kMaxNc];
    scale<P>(out, nc, f, tmp, nc);
    for (int j = 0; j < nc; ++j) out[j] = tmp[j];
  }
}

}  // namespace lit
}  // namespace mcfg
