// mlp.cu -- the MC-MLP training step around the MC contractions (config 3).
//
// The reference composes MCLinear / ReLU / cross-entropy / MC-SGD from its
// library (nn.hpp:49-92, autodiff.hpp:133-144, 255-298, 541-582, optim.hpp:54-77,
// mc_ops.hpp:509-513).  The GPU keeps activations feature-major, (features x
// batch), so every layer's forward is the MC x Tensor product
//   Z_l (out x N, MC) = W_l (out x in, MC) . A_{l-1} (in x N)
// exactly as the reference computes matmul_mcn(W, transpose2d(X)) before its
// transpose (autodiff.hpp:265).  This file adds the kernels around it, each
// reproducing the reference's rounding sequence:
//   k_bias_act  z + bias (add_mcn, x = product, y = bias), approx(), ReLU
//   k_ce        max-shifted softmax, log-sum-exp, per-sample loss terms and
//               the gradient (softmax - onehot) / N, all rounded in binary32
//   k_seqsum    the loss's left-to-right binary32 sum (autodiff.hpp:572)
//   k_gemm      matmul2d (ndarray.hpp:147-165): fl_mul then fl_add, reduction
//               index in increasing order, no fma -- used for dW = G A^T and
//               dA = approx(W)^T G (+ ReLU mask) of mc_linear_op's backward
//   k_rowsum    the bias gradient, rows summed in order
//   k_sgd_grow  MC-SGD (momentum 0): u = 0*u + g, delta = -lr*u, and the
//               Grow-ExpN update of the MC parameter in place
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "mcf_fast.cuh"
#include "mcf_lit.cuh"
#include "mcf_prec.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

using P = PB32;

template <int NC>
__global__ void __launch_bounds__(256) k_bias_act(const float* __restrict__ z, const float* __restrict__ bias,
                                                  int64_t out_dim, int64_t n, int relu,
                                                  float* __restrict__ h, float* __restrict__ act) {
  const int64_t total = out_dim * n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t o = e / n;
    float zx[NC], by[NC], r[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      zx[c] = z[e * NC + c];
      by[c] = bias[o * NC + c];
    }
    if (!fast::add<P, NC>(zx, by, r)) lit::add<P>(zx, NC, by, NC, r, NC);
    const float v = fast::approx<P, NC>(r);
    h[e] = v;
    if (act) act[e] = relu ? (v > 0.0f ? v : 0.0f) : v;  // Tape::relu, autodiff.hpp:134
  }
}

// one thread per sample (column n of the C x n logits)
__global__ void __launch_bounds__(256) k_ce(const float* __restrict__ logits, const int* __restrict__ labels,
                                            int64_t classes, int64_t n, float n_global,
                                            float* __restrict__ grad, float* __restrict__ terms) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  float m = logits[s];
  for (int64_t c = 1; c < classes; ++c) {
    const float z = logits[c * n + s];
    m = m < z ? z : m;  // std::max
  }
  float sum = 0.0f;
  for (int64_t c = 0; c < classes; ++c) {
    const float d = __fsub_rn(logits[c * n + s], m);
    const float ex = __double2float_rn(cr_exp((double)d));  // P::round(std::exp(...))
    grad[c * n + s] = ex;
    sum = __fadd_rn(sum, ex);
  }
  const int lab = labels[s];
  for (int64_t c = 0; c < classes; ++c) {
    float sm = __fdiv_rn(grad[c * n + s], sum);
    if (c == lab) sm = __fsub_rn(sm, 1.0f);
    // fl_mul(1, fl_div(d, n)), accumulated into a zero gradient (fl_add(0, .))
    grad[c * n + s] = __fadd_rn(0.0f, __fmul_rn(1.0f, __fdiv_rn(sm, n_global)));
  }
  const float lse = __fadd_rn(m, __double2float_rn(log((double)sum)));
  terms[s] = __fsub_rn(lse, logits[(int64_t)lab * n + s]);
}

// the loss sum, left to right from 0; the block stages 2048-term slabs in
// shared memory so thread 0's chain reads them at shared-memory latency
__global__ void __launch_bounds__(256) k_seqsum(const float* __restrict__ terms, int64_t n, float* __restrict__ out) {
  __shared__ float buf[2048];
  float acc = 0.0f;
  for (int64_t j0 = 0; j0 < n; j0 += 2048) {
    const int cnt = (int)((n - j0) < 2048 ? (n - j0) : 2048);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) buf[t] = terms[j0 + t];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int t = 0; t < cnt; ++t) acc = __fadd_rn(acc, buf[t]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = acc;
}

// C[i, j] = sum_k A(i, k) * B(k, j), k increasing, fl_mul then fl_add.
// A(i, k) = TA ? a[k * lda + i] : a[i * lda + k];  B(k, j) = TB ? b[j * ldb + k] : b[k * ldb + j]
// mask (optional): C[i, j] = mask[i * ldc + j] > 0 ? (0 + c) : 0  (ReLU backward)
// The chain per output is fixed by the reference (no split-K, no fma), so
// the parallelism is the outputs: BM x BN tiles, 256 threads as 16 x 16,
// each thread TM x TN outputs in two row halves and two column halves
// (rows ty*TM/2 + u and BM/2 + ty*TM/2 + u; columns likewise), so a warp's
// fragment loads are 128-bit and conflict-free.  K tiles of 16 staged
// through shared memory (k-major, both operands), the next tile prefetched
// into registers while the current one is consumed.
constexpr int GT = 256;

// (a b0, a b1), each product rounded to binary32 (mul.rn.f32x2 on sm_100a;
// ptxas issues FMUL2 with the scalar a as a broadcast operand).  The result
// feeds separate FADDs: no contraction into FFMA2 is possible there.
__device__ __forceinline__ void mul2_bcast(float a, float b0, float b1, float& p0, float& p1) {
  unsigned long long ap, bp, pp;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(a), "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bp) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(pp) : "l"(ap), "l"(bp));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(p0), "=f"(p1) : "l"(pp));
}

// row (col) of the tile owned by fragment index u of thread t (T per thread):
// T == 1 -> t; else two halves of T/2, at t*T/2 and B/2 + t*T/2
template <int T, int B>
__device__ __forceinline__ int frag_pos(int t, int u) {
  if constexpr (T == 1) return t;
  else return u < T / 2 ? t * (T / 2) + u : B / 2 + t * (T / 2) + (u - T / 2);
}

template <bool TA, bool TB, int BM, int BN, int TM, int TN, int GK>
__global__ void __launch_bounds__(GT) k_gemm(const float* __restrict__ a, int64_t lda, const float* __restrict__ b,
                                             int64_t ldb, float* __restrict__ c, int64_t ldc, int64_t M, int64_t N,
                                             int64_t K, const float* __restrict__ mask) {
  static_assert(BM == 16 * TM && BN == 16 * TN, "16 x 16 threads");
  constexpr int PA = BM + 4, PB = BN + 4;              // rows stay 16-byte aligned
  constexpr int LA = BM * GK / GT, LB = BN * GK / GT;  // elements per thread per tile
  static_assert(LA * GT == BM * GK && LB * GT == BN * GK, "whole tiles per thread");
  __shared__ __align__(16) float As[2][GK][PA];
  __shared__ __align__(16) float Bs[2][GK][PB];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
  float ra[LA], rb[LB];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < LA; ++r) {
      const int e = tid + r * GT;
      const int kk = TA ? e / BM : e % GK, ii = TA ? e % BM : e / GK;
      const int64_t gi = i0 + ii, gk = k0 + kk;
      ra[r] = (gi < M && gk < K) ? (TA ? a[gk * lda + gi] : a[gi * lda + gk]) : 0.0f;
    }
#pragma unroll
    for (int r = 0; r < LB; ++r) {
      const int e = tid + r * GT;
      const int kk = TB ? e % GK : e / BN, jj = TB ? e / GK : e % BN;
      const int64_t gj = j0 + jj, gk = k0 + kk;
      rb[r] = (gj < N && gk < K) ? (TB ? b[gj * ldb + gk] : b[gk * ldb + gj]) : 0.0f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int r = 0; r < LA; ++r) {
      const int e = tid + r * GT;
      As[buf][TA ? e / BM : e % GK][TA ? e % BM : e / GK] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < LB; ++r) {
      const int e = tid + r * GT;
      Bs[buf][TB ? e % GK : e / BN][TB ? e / GK : e % BN] = rb[r];
    }
  };
  float acc[TM][TN];
#pragma unroll
  for (int u = 0; u < TM; ++u)
#pragma unroll
    for (int v = 0; v < TN; ++v) acc[u][v] = 0.0f;
  auto step = [&](int buf, int kk) {
    float av[TM], bv[TN];
#pragma unroll
    for (int u = 0; u < TM; ++u) av[u] = As[buf][kk][frag_pos<TM, BM>(ty, u)];
#pragma unroll
    for (int v = 0; v < TN; ++v) bv[v] = Bs[buf][kk][frag_pos<TN, BN>(tx, v)];
    if constexpr (TN % 2 == 0) {
      // packed products: one FMUL2 (scalar a broadcast against a pair of b)
      // per two multiply-adds, then the two ordered FADDs -- the roundings
      // are the scalar ones (fl_mul then fl_add), three instructions
      // instead of four
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; v += 2) {
          float p0, p1;
          mul2_bcast(av[u], bv[v], bv[v + 1], p0, p1);
          acc[u][v] = __fadd_rn(acc[u][v], p0);
          acc[u][v + 1] = __fadd_rn(acc[u][v + 1], p1);
        }
    } else {
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = __fadd_rn(acc[u][v], __fmul_rn(av[u], bv[v]));
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < K; k0 += GK) {
    const bool more = k0 + GK < K;
    if (more) fetch(k0 + GK);
    if (K - k0 >= GK) {
#pragma unroll
      for (int kk = 0; kk < GK; ++kk) step(buf, kk);
    } else {
      // exactly K terms per chain: the last partial tile stops at K
      const int kmax = (int)(K - k0);
      for (int kk = 0; kk < kmax; ++kk) step(buf, kk);
    }
    if (more) {
      stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    const int64_t gi = i0 + frag_pos<TM, BM>(ty, u);
    if (gi >= M) continue;
#pragma unroll
    for (int v = 0; v < TN; ++v) {
      const int64_t gj = j0 + frag_pos<TN, BN>(tx, v);
      if (gj >= N) continue;
      float r = __fadd_rn(0.0f, acc[u][v]);
      if (mask) r = mask[gi * ldc + gj] > 0.0f ? __fadd_rn(0.0f, r) : 0.0f;
      c[gi * ldc + gj] = r;
    }
  }
}

// g (rows x n): out[r] = sum_j g[r, j], j increasing, starting from 0.
// 32 rows per CTA; the 8 warps stage 32 x 128 slabs (coalesced: rows of g are
// contiguous) into a double-buffered shared tile, and lane l of warp 0 adds
// row l's values in order -- the reference's left-to-right chain -- while the
// other warps fetch the next slab.
constexpr int RS_ROWS = 32, RS_COLS = 128;

__global__ void __launch_bounds__(256) k_rowsum(const float* __restrict__ g, int64_t rows, int64_t n,
                                                float* __restrict__ out) {
  __shared__ float tile[2][RS_ROWS][RS_COLS + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * RS_ROWS;
  auto load = [&](int64_t j0, int buf) {
    // warp w loads rows w, w+8, w+16, w+24; lane covers 8 columns strided by 32
#pragma unroll
    for (int q = 0; q < RS_ROWS / 8; ++q) {
      const int rr = warp + 8 * q;
      const int64_t r = r0 + rr;
#pragma unroll
      for (int cc = 0; cc < RS_COLS / 32; ++cc) {
        const int64_t j = j0 + cc * 32 + lane;
        tile[buf][rr][cc * 32 + lane] = (r < rows && j < n) ? g[r * n + j] : 0.0f;
      }
    }
  };
  float acc = 0.0f;
  load(0, 0);
  __syncthreads();
  int buf = 0;
  for (int64_t j0 = 0; j0 < n; j0 += RS_COLS) {
    if (j0 + RS_COLS < n && warp != 0) load(j0 + RS_COLS, buf ^ 1);
    if (warp == 0) {
      const int cnt = (int)((n - j0) < RS_COLS ? (n - j0) : RS_COLS);
      for (int c = 0; c < cnt; ++c) acc = __fadd_rn(acc, tile[buf][lane][c]);
    }
    __syncthreads();
    if (j0 + RS_COLS < n && warp == 0) {
      // warp 0 was summing; fetch its share of the next slab now
#pragma unroll
      for (int q = 0; q < RS_ROWS / 8; ++q) {
        const int rr = 8 * q;
        const int64_t r = r0 + rr;
#pragma unroll
        for (int cc = 0; cc < RS_COLS / 32; ++cc) {
          const int64_t j = j0 + RS_COLS + cc * 32 + lane;
          tile[buf ^ 1][rr][cc * 32 + lane] = (r < rows && j < n) ? g[r * n + j] : 0.0f;
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  if (warp == 0 && r0 + lane < rows) out[r0 + lane] = acc;
}

template <int NC>
__global__ void __launch_bounds__(256) k_sgd_grow(float* __restrict__ w, const float* __restrict__ g, int64_t numel,
                                                  float lr) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += stride) {
    // optim.hpp:70-73 with momentum 0: u = fl_add(fl_mul(0, 0), g); update = -fl_mul(lr, u)
    const float u = __fadd_rn(__fmul_rn(0.0f, 0.0f), g[e]);
    const float delta = -__fmul_rn(lr, u);
    float x[NC], o[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) x[c] = w[e * NC + c];
    if (!fast::grow<P, NC>(x, delta, o)) lit::grow<P>(x, NC, delta, o);
#pragma unroll
    for (int c = 0; c < NC; ++c) w[e * NC + c] = o[c];
  }
}

}  // namespace
}  // namespace mcfg

// ---- C-ABI ---------------------------------------------------------------------

namespace {
mcf_status launched(const char* what) {
  mcfr::note_launch();
  return mcfr::check_launch(what);
}
int grid_of(int64_t n) { return mcfr::grid_for(n, 256, 8); }

// this translation unit's copy of the device exp table (mcf_exp.cuh keeps the
// table per translation unit; k_ce's cr_exp reads this one)
std::mutex g_tab_mu;
bool g_tab_done[64];
mcf_status ensure_tables_here() {
  const mcf_status st = mcfr::ensure_device_tables();  // stack limit + elementwise copy
  if (st != MCF_OK) return st;
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) d = 0;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (g_tab_done[d]) return MCF_OK;
  double tab[4096];
  mcfr::exp2_table(tab);
  if (cudaMemcpyToSymbol(mcfg::g_exp_tab, tab, sizeof(tab)) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot upload the exp table (mlp)");
  g_tab_done[d] = true;
  return MCF_OK;
}

template <bool TA, bool TB, int BM, int BN, int TM, int TN, int GK>
mcf_status gemm_launch(const float* a, int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, int64_t m,
                       int64_t n, int64_t k, const float* mask, cudaStream_t s) {
  const dim3 grid((unsigned)((n + BN - 1) / BN), (unsigned)((m + BM - 1) / BM));
  mcfg::k_gemm<TA, TB, BM, BN, TM, TN, GK><<<grid, mcfg::GT, 0, s>>>(a, lda, b, ldb, c, ldc, m, n, k, mask);
  return launched("ordered fp32 gemm kernel");
}

// the largest tile that still gives ~one CTA per SM (the chains cannot be
// split, so small outputs take small tiles, with longer K tiles to cover
// the load latency)
template <bool TA, bool TB>
mcf_status gemm_shape(const float* a, int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, int64_t m,
                      int64_t n, int64_t k, const float* mask, cudaStream_t s) {
  const int64_t want = (int64_t)mcfr::sm_count() * 4 / 5;
  auto ctas = [&](int bm, int bn) { return ((m + bm - 1) / bm) * ((n + bn - 1) / bn); };
  if (ctas(128, 128) >= want) return gemm_launch<TA, TB, 128, 128, 8, 8, 16>(a, lda, b, ldb, c, ldc, m, n, k, mask, s);
  if (ctas(128, 64) >= want) return gemm_launch<TA, TB, 128, 64, 8, 4, 16>(a, lda, b, ldb, c, ldc, m, n, k, mask, s);
  if (ctas(64, 64) >= want) return gemm_launch<TA, TB, 64, 64, 4, 4, 32>(a, lda, b, ldb, c, ldc, m, n, k, mask, s);
  if (ctas(32, 32) >= want) return gemm_launch<TA, TB, 32, 32, 2, 2, 64>(a, lda, b, ldb, c, ldc, m, n, k, mask, s);
  return gemm_launch<TA, TB, 16, 16, 1, 1, 64>(a, lda, b, ldb, c, ldc, m, n, k, mask, s);
}
}  // namespace

extern "C" {

mcf_status mcf_mlp_bias_act(const float* z, int nc, const float* bias, int64_t out_dim, int64_t n, int relu,
                            float* h, float* act, mcf_stream s) {
  if (nc != 2 && nc != 3) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mlp_bias_act: nc must be 2 or 3");
  if (out_dim * n == 0) return MCF_OK;
  if (nc == 2) mcfg::k_bias_act<2><<<grid_of(out_dim * n), 256, 0, s>>>(z, bias, out_dim, n, relu, h, act);
  else mcfg::k_bias_act<3><<<grid_of(out_dim * n), 256, 0, s>>>(z, bias, out_dim, n, relu, h, act);
  return launched("mlp_bias_act kernel");
}

// one MCLinear forward (mc_linear_op, autodiff.hpp:255-268) + Tape::relu:
// Z = W (out x in, MC) . A_prev (in x n), h = approx(add_mcn(Z, bias)),
// act = relu ? max(h, 0) : h.  Plan MCF_FAST on the tensor-core shapes fuses
// the bias / approx / ReLU into the product's recombination (Z is never
// written); otherwise Z (out x n x nc) is the caller's buffer.
mcf_status mcf_mlp_linear_fwd(const float* w, int nc, const float* a_prev, int64_t out_dim, int64_t in_dim,
                              int64_t n, const float* bias, int relu, float* z, float* h, float* act, int strategy,
                              mcf_stream s) {
  if (strategy == MCF_FAST && nc == 2) {
    const mcf_status st = mcfr::mm_ozaki_bias_act(w, a_prev, out_dim, in_dim, n, bias, relu, h, act, s);
    if (st != MCF_ERR_UNSUPPORTED) return st;
  }
  const mcf_status st = mcf_bmm_mcn(MCF_B32, w, nc, a_prev, 1, out_dim, in_dim, n, 0, z, strategy, 1, s);
  if (st != MCF_OK) return st;
  return mcf_mlp_bias_act(z, nc, bias, out_dim, n, relu, h, act, s);
}

mcf_status mcf_mlp_cross_entropy(const float* logits, const int* labels, int64_t classes, int64_t n,
                                 int64_t n_global, float* grad, float* terms, float* term_sum, mcf_stream s) {
  if (n == 0) return MCF_OK;
  const mcf_status ok = ensure_tables_here();
  if (ok != MCF_OK) return ok;
  mcfg::k_ce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(logits, labels, classes, n, (float)n_global, grad, terms);
  mcf_status st = launched("mlp cross-entropy kernel");
  if (st != MCF_OK || !term_sum) return st;
  mcfg::k_seqsum<<<1, 256, 0, s>>>(terms, n, term_sum);
  return launched("mlp loss sum kernel");
}

mcf_status mcf_mlp_loss_sum(const float* terms, int64_t n, float* term_sum, mcf_stream s) {
  if (n < 0 || !terms || !term_sum) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mlp_loss_sum: bad arguments");
  mcfg::k_seqsum<<<1, 256, 0, s>>>(terms, n, term_sum);
  return launched("mlp loss sum kernel");
}

mcf_status mcf_gemm_f32_ordered(int trans_a, int trans_b, const float* a, int64_t lda, const float* b, int64_t ldb,
                                float* c, int64_t ldc, int64_t m, int64_t n, int64_t k, const float* relu_mask,
                                mcf_stream s) {
  if (m * n == 0) return MCF_OK;
  if (trans_a && trans_b) return gemm_shape<true, true>(a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
  if (trans_a) return gemm_shape<true, false>(a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
  if (trans_b) return gemm_shape<false, true>(a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
  return gemm_shape<false, false>(a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
}

mcf_status mcf_rowsum_f32_ordered(const float* g, int64_t rows, int64_t n, float* out, mcf_stream s) {
  if (rows == 0) return MCF_OK;
  mcfg::k_rowsum<<<(unsigned)((rows + mcfg::RS_ROWS - 1) / mcfg::RS_ROWS), 256, 0, s>>>(g, rows, n, out);
  return launched("row-sum kernel");
}

mcf_status mcf_sgd_grow(float* w, int nc, const float* g, int64_t numel, float lr, mcf_stream s) {
  if (nc != 2 && nc != 3) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "sgd_grow: nc must be 2 or 3");
  if (numel == 0) return MCF_OK;
  const mcf_status ok = mcfr::ensure_device_tables();
  if (ok != MCF_OK) return ok;
  if (nc == 2) mcfg::k_sgd_grow<2><<<grid_of(numel), 256, 0, s>>>(w, g, numel, lr);
  else mcfg::k_sgd_grow<3><<<grid_of(numel), 256, 0, s>>>(w, g, numel, lr);
  return launched("sgd grow kernel");
}

}  // extern "C"
