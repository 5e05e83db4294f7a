// linalg.cu -- MC contractions (linalg.hpp) on sm_100a.
//
// Reference-order kernels (this file, "exact"): every output element runs the
// reference's DotCore (linalg.hpp:38-91) with the register fast paths --
// term(k) = ScalingN expanded to nc+1 (:55-57), sequential add_kernel at
// nc+1 (:63-69) or the pairwise tree (:71-75), final renorm to nc (:89) --
// so results are bit-identical to the reference.  nc == 1 is the plain
// fl-MAC chain (:47-53).  An output whose fast-path preconditions fail is
// recomputed by the literal restatement (mcf_lit.cuh).
//
// MC x MC (the reference refuses it, linalg.hpp:159-166) uses the same
// DotCore with SURVEY 8c "recipe B" terms: the mul_mcn_slow term set
// (mc_ops.hpp:240-250) renormalized to nc+1.
//
// The throughput kernels (compensated register accumulators on tiled
// operands) live in mm_fast.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <type_traits>

#include "mcf_fast.cuh"
#include "mcf_lit.cuh"
#include "mcf_prec.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

template <class P>
using RT = typename P::rt;
template <class P>
using ST = typename P::st;

constexpr int kThreads = 128;
#ifndef MCF_DOT_PU
#define MCF_DOT_PU 2
#endif
// blind sweeps before the tested ones in the DotCore accumulation (see
// mcf_fast.cuh sweeps(): any value below the pass cap gives the same bits)
constexpr int kDotPU = MCF_DOT_PU;

// ---- literal DotCore (runtime nc; fallback and non-instantiated shapes) ----

template <class P>
__device__ __noinline__ void lit_term(const ST<P>* x, int64_t xi, const ST<P>* w, int64_t wi, int nc,
                         RT<P>* out) {
  RT<P> xc[lit::kMaxNc];
  for (int c = 0; c < nc; ++c) xc[c] = P::ld(x[xi * nc + c]);
  lit::scale<P>(xc, nc, P::ld(w[wi]), out, nc + 1);
}

template <class P>
__device__ void lit_reduce(const ST<P>* x, int64_t xa, const ST<P>* w, int64_t wa, int64_t ws,
                           int nc, int64_t lo, int64_t hi, int strategy, int leaf, RT<P>* acc) {
  const int64_t leafn = leaf > 1 ? leaf : 1;
  if (strategy == MCF_SEQUENTIAL || hi - lo <= leafn) {
    lit_term<P>(x, xa + lo, w, wa + lo * ws, nc, acc);
    RT<P> t[lit::kMaxNc + 1];
    for (int64_t k = lo + 1; k < hi; ++k) {
      lit_term<P>(x, xa + k, w, wa + k * ws, nc, t);
      lit::add<P>(acc, nc + 1, t, nc + 1, acc, nc + 1);
    }
    return;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  RT<P> rhs[lit::kMaxNc + 1];
  lit_reduce<P>(x, xa, w, wa, ws, nc, lo, mid, strategy, leaf, acc);
  lit_reduce<P>(x, xa, w, wa, ws, nc, mid, hi, strategy, leaf, rhs);
  lit::add<P>(acc, nc + 1, rhs, nc + 1, acc, nc + 1);
}

template <class P>
__device__ __noinline__ void lit_dot(const ST<P>* x, int64_t xa, const ST<P>* w, int64_t wa,
                                     int64_t ws, int nc, int64_t len, int strategy, int leaf,
                                     RT<P>* out) {
  if (len == 0) {
    for (int c = 0; c < nc; ++c) out[c] = RT<P>(0);
    return;
  }
  if (nc == 1 && strategy == MCF_SEQUENTIAL) {
    RT<P> acc = RT<P>(0);
    for (int64_t k = 0; k < len; ++k)
      acc = P::add(acc, P::mul(P::ld(x[xa + k]), P::ld(w[wa + k * ws])));
    out[0] = acc;
    return;
  }
  RT<P> acc[lit::kMaxNc + 1];
  lit_reduce<P>(x, xa, w, wa, ws, nc, 0, len, strategy, leaf, acc);
  lit::renorm<P>(acc, nc + 1, out, nc);
}

// recipe B, literal
template <class P>
__device__ __noinline__ void lit_mcmc_term(const ST<P>* x, int64_t xi, const ST<P>* y, int64_t yi, int nc,
                              RT<P>* out) {
  RT<P> a[lit::kMaxNc], b[lit::kMaxNc], h[lit::kStage];
  for (int c = 0; c < nc; ++c) {
    a[c] = P::ld(x[xi * nc + c]);
    b[c] = P::ld(y[yi * nc + c]);
  }
  int m = 0;
  for (int i = 0; i < nc; ++i)
    for (int j = 0; i + j < nc; ++j) {
      two_prod<P>(a[i], b[j], h[m], h[m + 1]);
      m += 2;
    }
  for (int i = 1; i < nc; ++i) h[m++] = P::mul(a[i], b[nc - i]);
  lit::renorm<P>(h, m, out, nc + 1);
}

template <class P>
__device__ __noinline__ void lit_mcmc(const ST<P>* x, int64_t xa, int64_t xs, const ST<P>* y,
                                      int64_t ya, int64_t ys, int nc, int64_t len, RT<P>* out) {
  if (len == 0) {
    for (int c = 0; c < nc; ++c) out[c] = RT<P>(0);
    return;
  }
  if (nc == 1) {
    RT<P> acc = RT<P>(0);
    for (int64_t k = 0; k < len; ++k)
      acc = P::add(acc, P::mul(P::ld(x[xa + k * xs]), P::ld(y[ya + k * ys])));
    out[0] = acc;
    return;
  }
  RT<P> acc[lit::kMaxNc + 1], t[lit::kMaxNc + 1];
  lit_mcmc_term<P>(x, xa, y, ya, nc, acc);
  for (int64_t k = 1; k < len; ++k) {
    lit_mcmc_term<P>(x, xa + k * xs, y, ya + k * ys, nc, t);
    lit::add<P>(acc, nc + 1, t, nc + 1, acc, nc + 1);
  }
  lit::renorm<P>(acc, nc + 1, out, nc);
}

// ---- register DotCore (compile-time nc) ---------------------------------------

template <class P, int NC>
__device__ __forceinline__ bool fast_term(const ST<P>* x, int64_t xi, RT<P> v,
                                          RT<P> (&t)[NC + 1]) {
  RT<P> xc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) xc[c] = P::ld(x[xi * NC + c]);
  return fast::scale<P, NC, NC + 1>(xc, v, t);
}

// sequential DotCore over k in [0, len); false -> recompute with lit_dot
template <class P, int NC>
__device__ __forceinline__ bool fast_dot_seq(const ST<P>* x, int64_t xa, const ST<P>* w,
                                             int64_t wa, int64_t ws, int64_t len,
                                             RT<P> (&out)[NC]) {
  RT<P> acc[NC + 1], t[NC + 1];
  bool ok = fast_term<P, NC>(x, xa, P::ld(w[wa]), acc);
  for (int64_t k = 1; k < len; ++k) {
    ok &= fast_term<P, NC>(x, xa + k, P::ld(w[wa + k * ws]), t);
    ok &= fast::add_ordered<P, NC + 1, NC + 1, kDotPU>(acc, t, acc);
  }
  ok &= fast::renorm<P, NC + 1, NC>(acc, out);
  return ok;
}

template <class P, int NC>
__device__ __forceinline__ bool fast_mcmc_term(const ST<P>* x, int64_t xi, const ST<P>* y,
                                               int64_t yi, RT<P> (&t)[NC + 1]) {
  RT<P> a[NC], b[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    a[c] = P::ld(x[xi * NC + c]);
    b[c] = P::ld(y[yi * NC + c]);
  }
  RT<P> h[fast::mul_slow_terms(NC)];
  int m = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int j = 0; i + j < NC; ++j) {
      two_prod<P>(a[i], b[j], h[m], h[m + 1]);
      m += 2;
    }
#pragma unroll
  for (int i = 1; i < NC; ++i) h[m++] = P::mul(a[i], b[NC - i]);
  return fast::renorm<P, fast::mul_slow_terms(NC), NC + 1>(h, t);
}

// ---- kernels -----------------------------------------------------------------------

// out[b, i, j] for a batch of MC x Tensor products; one thread per output,
// consecutive threads on consecutive j (coalesced w reads, broadcast x reads)
template <class P, int NC>
__global__ void __launch_bounds__(kThreads) k_bmm_exact(const ST<P>* __restrict__ x, int nc,
                                                        const ST<P>* __restrict__ w,
                                                        int64_t batch, int64_t m, int64_t k,
                                                        int64_t n, int w_batched,
                                                        ST<P>* __restrict__ out, int strategy,
                                                        int leaf) {
  const int64_t total = batch * m * n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += stride) {
    const int64_t b = o / (m * n), r = o % (m * n), i = r / n, j = r % n;
    const int64_t xa = (b * m + i) * k;              // element index of x[b, i, 0]
    const int64_t wa = (w_batched ? b * k * n : 0) + j;
    RT<P> res[lit::kMaxNc];
    bool done = false;
    if constexpr (NC > 0) {
      if (strategy == MCF_SEQUENTIAL && k > 0) {
        if constexpr (NC == 1) {
          RT<P> acc = RT<P>(0);
          for (int64_t t = 0; t < k; ++t)
            acc = P::add(acc, P::mul(P::ld(x[xa + t]), P::ld(w[wa + t * n])));
          res[0] = acc;
          done = true;
        } else {
          RT<P> o2[NC];
          done = fast_dot_seq<P, NC>(x, xa, w, wa, n, k, o2);
#pragma unroll
          for (int c = 0; c < NC; ++c) res[c] = o2[c];
        }
      }
    }
    const int ncr = NC > 0 ? NC : nc;
    if (!done) lit_dot<P>(x, xa, w, wa, n, ncr, k, strategy, leaf, res);
    for (int c = 0; c < ncr; ++c) out[o * ncr + c] = P::sv(res[c]);
  }
}

// ---- pairwise tree as a warp-parallel split-K ------------
// DotCore::reduce_range (linalg.hpp:59-76) halves [lo, hi) at mid = lo +
// (hi - lo) / 2 down to runs of <= leaf_arity terms and merges with
// add_kernel(left, right).  A warp per output reproduces that tree exactly:
// lane l takes the depth-5 node its bits select (MSB = the root's choice),
// reduces it with the same recursion, and the lanes merge back up the five
// top levels with shuffles -- left child (lower lane) as add_kernel's x --
// skipping levels whose node was already a leaf.  32-way parallel per output
// for long K / few outputs; bit-identical to the reference's tree.

template <class P, int NC>
__device__ __noinline__ bool tree_range(const ST<P>* x, int64_t xa, const ST<P>* w, int64_t wa, int64_t ws,
                                        int64_t lo, int64_t hi, int64_t leafn, RT<P> (&acc)[NC + 1]) {
  if (hi - lo <= leafn) {
    bool ok = fast_term<P, NC>(x, xa + lo, P::ld(w[wa + lo * ws]), acc);
    RT<P> t[NC + 1];
    for (int64_t k = lo + 1; k < hi; ++k) {
      ok &= fast_term<P, NC>(x, xa + k, P::ld(w[wa + k * ws]), t);
      ok &= fast::add_ordered<P, NC + 1, NC + 1>(acc, t, acc);
    }
    return ok;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  RT<P> rhs[NC + 1];
  bool ok = tree_range<P, NC>(x, xa, w, wa, ws, lo, mid, leafn, acc);
  ok &= tree_range<P, NC>(x, xa, w, wa, ws, mid, hi, leafn, rhs);
  ok &= fast::add_ordered<P, NC + 1, NC + 1>(acc, rhs, acc);
  return ok;
}

template <class P, int NC>
__global__ void __launch_bounds__(kThreads) k_bmm_tree(const ST<P>* __restrict__ x, const ST<P>* __restrict__ w,
                                                       int64_t batch, int64_t m, int64_t k, int64_t n,
                                                       int w_batched, ST<P>* __restrict__ out, int leaf) {
  constexpr int D = 5;  // top levels resolved across the 32 lanes
  const int lane = threadIdx.x & 31;
  const int64_t total = batch * m * n;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t leafn = leaf > 1 ? leaf : 1;
  for (int64_t o = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < total; o += warps) {
    const int64_t b = o / (m * n), r = o % (m * n), i = r / n, j = r % n;
    const int64_t xa = (b * m + i) * k;
    const int64_t wa = (w_batched ? b * k * n : 0) + j;
    RT<P> res[NC];
    bool ok = true;
    if (k == 0) {
#pragma unroll
      for (int c = 0; c < NC; ++c) res[c] = RT<P>(0);
    } else {
      // descend to this lane's depth-5 node; internal[d] = node at depth d split
      int64_t lo = 0, hi = k;
      unsigned internal = 0;
      int depth = 0;
      for (; depth < D; ++depth) {
        if (hi - lo <= leafn) break;
        internal |= 1u << depth;
        const int64_t mid = lo + (hi - lo) / 2;
        if ((lane >> (D - 1 - depth)) & 1) lo = mid;
        else hi = mid;
      }
      // a node that stopped splitting above depth 5 is held by the lane whose
      // remaining bits are zero; the other lanes of its subtree carry nothing
      const bool holder = depth == D || (lane & ((1 << (D - depth)) - 1)) == 0;
      RT<P> acc[NC + 1];
#pragma unroll
      for (int c = 0; c <= NC; ++c) acc[c] = RT<P>(0);
      if (holder) ok = tree_range<P, NC>(x, xa, w, wa, n, lo, hi, leafn, acc);
      // merge up: level d (depth D-1 .. 0), partner differs in bit (D-1-d)
      for (int d = D - 1; d >= 0; --d) {
        const int bit = 1 << (D - 1 - d);
        RT<P> rhs[NC + 1];
#pragma unroll
        for (int c = 0; c <= NC; ++c) rhs[c] = __shfl_xor_sync(0xffffffffu, acc[c], bit);
        // the depth-d node on this lane's path; only meaningful on lanes whose
        // bits below (D-1-d) are zero, which hold its left child
        if ((internal >> d) & 1 && (lane & (2 * bit - 1)) == 0) ok &= fast::add_ordered<P, NC + 1, NC + 1>(acc, rhs, acc);
      }
      ok &= fast::renorm<P, NC + 1, NC>(acc, res);
    }
    const unsigned bad = __ballot_sync(0xffffffffu, !ok);
    if (lane == 0) {
      if (bad != 0) {
        RT<P> r2[lit::kMaxNc];
        lit_dot<P>(x, xa, w, wa, n, NC, k, MCF_PAIRWISE_TREE, leaf, r2);
        for (int c = 0; c < NC; ++c) out[o * NC + c] = P::sv(r2[c]);
      } else {
        for (int c = 0; c < NC; ++c) out[o * NC + c] = P::sv(res[c]);
      }
    }
  }
}

// MC x MC, recipe B: out[i, j] = sum_k x[xa_i + k*xs] * y[ya_j + k*ys]
// dot: (x, y both (batch, k, nc)); mm: x (m, k, nc), y (k, n, nc)
template <class P, int NC>
__global__ void __launch_bounds__(kThreads) k_mcmc_exact(const ST<P>* __restrict__ x,
                                                         const ST<P>* __restrict__ y, int nc,
                                                         int64_t rows, int64_t cols, int64_t k,
                                                         int mm_layout, ST<P>* __restrict__ out) {
  const int64_t total = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += stride) {
    const int64_t i = o / cols, j = o % cols;
    // mm: x row i (xa=i*k, xs=1), y column j (ya=j, ys=cols); dot: both row o
    const int64_t xa = mm_layout ? i * k : o * k, xs = 1;
    const int64_t ya = mm_layout ? j : o * k, ys = mm_layout ? cols : 1;
    RT<P> res[lit::kMaxNc];
    bool done = false;
    if constexpr (NC > 1) {
      if (k > 0) {
        RT<P> acc[NC + 1], t[NC + 1];
        done = fast_mcmc_term<P, NC>(x, xa, y, ya, acc);
        for (int64_t kk = 1; kk < k; ++kk) {
          done &= fast_mcmc_term<P, NC>(x, xa + kk * xs, y, ya + kk * ys, t);
          done &= fast::add_ordered<P, NC + 1, NC + 1>(acc, t, acc);
        }
        RT<P> o2[NC];
        done &= fast::renorm<P, NC + 1, NC>(acc, o2);
#pragma unroll
        for (int c = 0; c < NC; ++c) res[c] = o2[c];
      }
    }
    const int ncr = NC > 0 ? NC : nc;
    if (!done) lit_mcmc<P>(x, xa, xs, y, ya, ys, ncr, k, res);
    for (int c = 0; c < ncr; ++c) out[o * ncr + c] = P::sv(res[c]);
  }
}

template <class K>
int per_sm(K kernel) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kThreads, 0) != cudaSuccess || n < 1) n = 1;
  return n;
}

template <class P, int NC>
mcf_status launch_bmm(const void* x, int nc, const void* w, int64_t batch, int64_t m, int64_t k,
                      int64_t n, int w_batched, void* out, int strategy, int leaf, cudaStream_t s) {
  if constexpr (NC >= 2) {
    if (strategy == MCF_PAIRWISE_TREE) {
      auto tk = k_bmm_tree<P, NC>;
      const int grid = mcfr::grid_for(batch * m * n * 32, kThreads, 8);
      tk<<<grid, kThreads, 0, s>>>(static_cast<const ST<P>*>(x), static_cast<const ST<P>*>(w), batch, m, k, n,
                                   w_batched, static_cast<ST<P>*>(out), leaf);
      mcfr::note_launch();
      return mcfr::check_launch("mcf bmm tree kernel");
    }
  }
  auto kern = k_bmm_exact<P, NC>;
  static const int occ = per_sm(kern);
  const int grid = mcfr::grid_for(batch * m * n, kThreads, occ);
  kern<<<grid, kThreads, 0, s>>>(static_cast<const ST<P>*>(x), nc, static_cast<const ST<P>*>(w), batch,
                                 m, k, n, w_batched, static_cast<ST<P>*>(out), strategy, leaf);
  mcfr::note_launch();
  return mcfr::check_launch("mcf bmm kernel");
}

template <class P, int NC>
mcf_status launch_mcmc(const void* x, const void* y, int nc, int64_t rows, int64_t cols, int64_t k,
                       int mm_layout, void* out, cudaStream_t s) {
  auto kern = k_mcmc_exact<P, NC>;
  static const int occ = per_sm(kern);
  const int grid = mcfr::grid_for(rows * cols, kThreads, occ);
  kern<<<grid, kThreads, 0, s>>>(static_cast<const ST<P>*>(x), static_cast<const ST<P>*>(y), nc, rows,
                                 cols, k, mm_layout, static_cast<ST<P>*>(out));
  mcfr::note_launch();
  return mcfr::check_launch("mcf mc x mc kernel");
}

template <class P>
mcf_status bmm_prec(const void* x, int nc, const void* w, int64_t batch, int64_t m, int64_t k,
                    int64_t n, int w_batched, void* out, int strategy, int leaf, cudaStream_t s) {
  if constexpr (std::is_same<P, PB32>::value) {
    switch (nc) {
      case 1: return launch_bmm<P, 1>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf, s);
      case 2: return launch_bmm<P, 2>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf, s);
      case 3: return launch_bmm<P, 3>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf, s);
      default: break;
    }
  }
  if (nc == 1) return launch_bmm<P, 1>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf, s);
  return launch_bmm<P, 0>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf, s);
}

template <class P>
mcf_status mcmc_prec(const void* x, const void* y, int nc, int64_t rows, int64_t cols, int64_t k,
                     int mm_layout, void* out, cudaStream_t s) {
  if constexpr (std::is_same<P, PB32>::value || std::is_same<P, PB16>::value) {
    switch (nc) {
      case 2: return launch_mcmc<P, 2>(x, y, nc, rows, cols, k, mm_layout, out, s);
      case 3: return launch_mcmc<P, 3>(x, y, nc, rows, cols, k, mm_layout, out, s);
      default: break;
    }
  }
  return launch_mcmc<P, 0>(x, y, nc, rows, cols, k, mm_layout, out, s);
}

}  // namespace
}  // namespace mcfg

// ---- C-ABI ---------------------------------------------------------------------

namespace {
mcf_status check_lin(mcf_prec p, int nc, const char* op) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, std::string(op) + ": unknown precision");
  if (mcfr::bad_nc(nc) || mcfr::bad_nc(nc + 1))
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  return MCF_OK;
}
}  // namespace

namespace {
// component-preserving transpose (linalg.hpp:301-315): out[j, i, :] = x[i, j, :],
// elements of W 32-bit words moved as a 32 x 32 tile through shared memory
template <int W>
__global__ void __launch_bounds__(256) k_mc_transpose(const uint32_t* __restrict__ x, int64_t m, int64_t n,
                                                      uint32_t* __restrict__ out) {
  __shared__ uint32_t t[32][32 * W + 1];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.x >> 5; r < 32; r += 8) {
    const int64_t i = i0 + r;
    for (int c = threadIdx.x & 31; c < 32 * W; c += 32) {
      const int64_t j = j0 + c / W;
      if (i < m && j < n) t[r][c] = x[(i * n + j) * W + c % W];
    }
  }
  __syncthreads();
  for (int r = threadIdx.x >> 5; r < 32; r += 8) {
    const int64_t j = j0 + r;
    for (int c = threadIdx.x & 31; c < 32 * W; c += 32) {
      const int64_t i = i0 + c / W;
      if (i < m && j < n) out[(j * m + i) * W + c % W] = t[c / W][r * W + c % W];
    }
  }
}
// binary16 components of odd count: 16-bit words
__global__ void __launch_bounds__(256) k_mc_transpose16(const uint16_t* __restrict__ x, int64_t m, int64_t n, int w,
                                                        uint16_t* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e / n, j = e - i * n;
  for (int c = 0; c < w; ++c) out[(j * m + i) * w + c] = x[e * w + c];
}
}  // namespace

extern "C" {

mcf_status mcf_bmm_mcn(mcf_prec p, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                       int64_t k, int64_t n, int w_batched, void* out, int strategy, int leaf_arity,
                       mcf_stream stream) {
  const mcf_status st = check_lin(p, nc, "mm_mcn");
  if (st != MCF_OK) return st;
  if (batch < 0 || m < 0 || k < 0 || n < 0)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_mcn: negative dimension");
  if (strategy != MCF_SEQUENTIAL && strategy != MCF_PAIRWISE_TREE && strategy != MCF_FAST &&
      strategy != MCF_FAST_FP64)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_mcn: unknown reduction strategy");
  if (batch * m * n == 0) return MCF_OK;
  if (mcfr::ensure_device_tables() != MCF_OK) return MCF_ERR_CUDA;
  if (strategy == MCF_FAST || strategy == MCF_FAST_FP64) {
    if (nc >= 2 && k > 0) {
      const bool tc = strategy == MCF_FAST;
      const mcf_status fs = n == 1 ? mcfr::mv_fast_mct(p, x, nc, w, batch, m, k, w_batched, out, stream)
                                   : mcfr::mm_fast_mct(p, x, nc, w, batch, m, k, n, w_batched, out, stream, tc);
      if (fs != MCF_ERR_UNSUPPORTED) return fs;
    }
    strategy = MCF_SEQUENTIAL;  // no fast kernel for this shape: reference order
  }
  // the literal pairwise tree recurses ceil(log2 k) deep (linalg.hpp:59-76)
  if (strategy == MCF_PAIRWISE_TREE && mcfr::ensure_stack(16384) != MCF_OK) return MCF_ERR_CUDA;
  switch (p) {
    case MCF_B16: return mcfg::bmm_prec<mcfg::PB16>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf_arity, stream);
    case MCF_B32: return mcfg::bmm_prec<mcfg::PB32>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf_arity, stream);
    default: return mcfg::bmm_prec<mcfg::PB64>(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf_arity, stream);
  }
}

mcf_status mcf_mm_mcn_mcmc_refusal(void) {
  return mcfr::fail(MCF_ERR_UNSUPPORTED,
                    "mm_mcn: matrix products of two MCTensors are not supported; convert one "
                    "operand to a working-precision tensor first");
}

mcf_status mcf_mm_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t m, int64_t k,
                       int64_t n, void* out, int strategy, mcf_stream stream) {
  const mcf_status st = check_lin(p, nc, "mm_mcmc");
  if (st != MCF_OK) return st;
  if (m < 0 || k < 0 || n < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_mcmc: negative dimension");
  if (strategy != MCF_SEQUENTIAL && strategy != MCF_FAST && strategy != MCF_FAST_FP64)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_mcmc: unknown reduction strategy");
  if (m * n == 0) return MCF_OK;
  if (mcfr::ensure_device_tables() != MCF_OK) return MCF_ERR_CUDA;
  if ((strategy == MCF_FAST || strategy == MCF_FAST_FP64) && k > 0) {
    const mcf_status fs = mcfr::mm_fast_mcmc(p, x, y, nc, m, k, n, out, stream, strategy == MCF_FAST);
    if (fs != MCF_ERR_UNSUPPORTED) return fs;
  }
  switch (p) {
    case MCF_B16: return mcfg::mcmc_prec<mcfg::PB16>(x, y, nc, m, n, k, 1, out, stream);
    case MCF_B32: return mcfg::mcmc_prec<mcfg::PB32>(x, y, nc, m, n, k, 1, out, stream);
    default: return mcfg::mcmc_prec<mcfg::PB64>(x, y, nc, m, n, k, 1, out, stream);
  }
}

mcf_status mcf_dot_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t batch, int64_t k,
                        void* out, int strategy, mcf_stream stream) {
  const mcf_status st = check_lin(p, nc, "dot_mcmc");
  if (st != MCF_OK) return st;
  if (batch < 0 || k < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "dot_mcmc: negative dimension");
  if (strategy != MCF_SEQUENTIAL && strategy != MCF_FAST && strategy != MCF_FAST_FP64)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "dot_mcmc: unknown reduction strategy");
  if (batch == 0) return MCF_OK;
  if (mcfr::ensure_device_tables() != MCF_OK) return MCF_ERR_CUDA;
  if ((strategy == MCF_FAST || strategy == MCF_FAST_FP64) && k > 0) {
    const mcf_status fs = mcfr::dot_fast_mcmc(p, x, y, nc, batch, k, out, stream);
    if (fs != MCF_ERR_UNSUPPORTED) return fs;
  }
  switch (p) {
    case MCF_B16: return mcfg::mcmc_prec<mcfg::PB16>(x, y, nc, batch, 1, k, 0, out, stream);
    case MCF_B32: return mcfg::mcmc_prec<mcfg::PB32>(x, y, nc, batch, 1, k, 0, out, stream);
    default: return mcfg::mcmc_prec<mcfg::PB64>(x, y, nc, batch, 1, k, 0, out, stream);
  }
}

int mcf_fast_ops_per_mad(int mcmc, mcf_prec p, int nc) { return mcfr::mm_fast_ops_per_mad(mcmc, p, nc); }

mcf_status mcf_mc_transpose2d(mcf_prec p, const void* x, int nc, int64_t m, int64_t n, void* out, mcf_stream stream) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_transpose2d: unknown precision");
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (m < 0 || n < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_transpose2d: negative dimension");
  if (m * n == 0) return MCF_OK;
  const int64_t bytes = (int64_t)nc * (int64_t)mcfr::elem_bytes(p);
  const dim3 g((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
  const auto* xu = static_cast<const uint32_t*>(x);
  auto* ou = static_cast<uint32_t*>(out);
  switch (bytes % 4 == 0 ? bytes / 4 : 0) {
    case 1: k_mc_transpose<1><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 2: k_mc_transpose<2><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 3: k_mc_transpose<3><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 4: k_mc_transpose<4><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 6: k_mc_transpose<6><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 8: k_mc_transpose<8><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 5: k_mc_transpose<5><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    case 7: k_mc_transpose<7><<<g, 256, 0, stream>>>(xu, m, n, ou); break;
    default:  // wide binary64 elements, or binary16 with an odd component count: 16-bit words
      k_mc_transpose16<<<(unsigned)((m * n + 255) / 256), 256, 0, stream>>>(static_cast<const uint16_t*>(x), m, n,
                                                                          (int)(bytes / 2),
                                                                          static_cast<uint16_t*>(out));
  }
  mcfr::note_launch();
  return mcfr::check_launch("mc_transpose2d kernel");
}

int mcf_fast_tc_digits(void) { return mcfr::ozaki_digits(); }

int mcf_fast_tc_gemm_equivalents(int b_components, int64_t k) {
  return mcfr::ozaki_gemm_equivalents(b_components, k);
}

int mcf_fast_tc_plan(int64_t k, int b_components, int* moduli, int* bits_a, int* bits_b) {
  return mcfr::ozaki_crt_info(k, b_components, moduli, bits_a, bits_b);
}

int mcf_fast_tc_crt_table(int n, int* moduli, float* w_slices, float* m_slices, float* q_scale, int* m_bits) {
  return mcfr::ozaki_crt_table(n, moduli, w_slices, m_slices, q_scale, m_bits);
}

mcf_status mcf_fast_mm_reserve(int64_t m, int64_t k, int64_t n, int b_components, mcf_stream stream) {
  if (mcfr::ensure_device_tables() != MCF_OK) return MCF_ERR_CUDA;
  return mcfr::ozaki_reserve(m, k, n, b_components, stream);
}

mcf_status mcf_fast_mm_phases(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out,
                              double* phase_ms, int64_t* fallback_outputs, mcf_stream stream) {
  if (!x || !w || !out || !phase_ms || !fallback_outputs)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_phases: null argument");
  if (mcfr::ensure_device_tables() != MCF_OK) return MCF_ERR_CUDA;
  return mcfr::ozaki_phases(x, w, m, k, n, out, phase_ms, fallback_outputs, stream);
}

}  // extern "C"
