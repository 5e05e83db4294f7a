// mm_fast.cu -- throughput MC contractions on the FP64 pipe (plan MCF_FAST).
//
// Each product of two binary32 (or binary16) components is exact in
// binary64 (24+24 <= 53 bits).  The GPU therefore carries every output as an
// extended binary64 accumulator in registers through the K loop (policies in
// mcf_accum.cuh):
//
//   nc=2 (MC x T and MC x MC): operands widened to (sum, err) pairs and scaled
//     by powers of two per row of A / column of B; offset accumulation
//     t = fma(a,b,tau), q = t - tau, C += fma(a,b,-q)   -> 4 FP64 ops / MAD
//     (5-7 when some err is nonzero: AccP2X, chosen by a device flag)
//   MC x T, nc=3:  three levels (S, C, D)                 -> 14 ops / MAD
//   MC x MC, fp16 nc=3: components summed into one binary64 per operand
//                  (<= 33 significant bits), S = fma(a, b, S) -> 1 op / MAD
//
// so the error before the final split into nc components is ~2^-100 x cond
// (2^-47 x cond for the binary16 case, whose format resolves 2^-33) -- below
// the reference's own error, which is dominated by the nc-component output
// (2^-51.7 median at nc=2).  The value is then split greedily
// (round-and-residual, mc_ops.hpp:286-297) into nc components.
//
// B200 mapping: FP64 runs at half the FP32 lane rate (measured 63 vs 119
// lanes/clk/SM, profiles/pipe_bench.txt), and one compensated FP64 MAD
// replaces ~32 FP32 error-free ops, so the FP64 pipe is the faster exact
// path.  Operands are widened once to binary64 (a streaming pass into a
// per-stream workspace), tiles are staged global->shared with cp.async
// (LDGSTS, 16-byte chunks, 3-stage ring), and each thread owns a TM x TN
// block of outputs with interleaved rows and columns (conflict-free LDS).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "mcf_accum.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

// ---- widening pass: components -> binary64 (optionally summed) --------------------

template <class ST, int NC, bool SUM>
__global__ void __launch_bounds__(256) k_widen(const ST* __restrict__ in, double* __restrict__ out,
                                                int64_t elems) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < elems; e += stride) {
    if constexpr (SUM) {
      double s = 0.0;
#pragma unroll
      for (int c = NC - 1; c >= 0; --c) s = __dadd_rn(s, to_d<ST>(in[e * NC + c]));
      out[e] = s;
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) out[e * NC + c] = to_d<ST>(in[e * NC + c]);
    }
  }
}

// ---- power-of-two operand scaling for the offset-accumulation policies ---------------
// Row i of A is scaled by 2^-ea[i], column j of B by 2^-eb[j], with 2^e the
// smallest power of two above the largest leading component, so every
// leading product is below 1 in magnitude.  Scaling by powers of two is exact
// in binary64 and undone on the output.

// (non-finite maxima leave the row / column unscaled: Inf and NaN propagate)
__device__ __forceinline__ int exp_above(float m) { return m > 0.0f && isfinite(m) ? ilogbf(m) + 1 : 0; }
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

template <class ST, int NC>
__global__ void __launch_bounds__(256) k_rowexp(const ST* __restrict__ a, int64_t rows, int64_t k,
                                                 int* __restrict__ e) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float m = 0.0f;
  for (int64_t t = lane; t < k; t += 32) m = fmaxf(m, fabsf((float)to_d<ST>(a[(r * k + t) * NC])));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) e[r] = exp_above(m);
}

// column maxima of B (k x n, row-major): CTA (x, y) covers 256 columns of a
// kColRows-row slab, coalesced along n; slabs meet through atomicMax on the
// bit pattern (monotone in the magnitude for non-negative binary32; e must
// start at 0).  k_colexp_fin turns the maxima into exponents in place.
constexpr int kColRows = 64;

template <class ST, int NC>
__global__ void __launch_bounds__(256) k_colmax(const ST* __restrict__ b, int64_t k, int64_t n,
                                                 int* __restrict__ e) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t t0 = (int64_t)blockIdx.y * kColRows;
  const int64_t t1 = t0 + kColRows < k ? t0 + kColRows : k;
  float m = 0.0f;
  for (int64_t t = t0; t < t1; ++t) m = fmaxf(m, fabsf((float)to_d<ST>(b[(t * n + j) * NC])));
  if (m > 0.0f) atomicMax(e + j, __float_as_int(m));
}

__global__ void __launch_bounds__(256) k_colexp_fin(int* __restrict__ e, int64_t n) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) e[j] = exp_above(__int_as_float(e[j]));
}

// out = in * 2^-e[row] (BY_ROW, rows of `cols` elements) or * 2^-e[col].
// PAIR: each nc=2 element becomes (sum, err) = two_sum(c0, c1) in binary64
// (sum + err == c0 + c1 exactly); any nonzero err raises *inexact.
template <class ST, int NC, bool BY_ROW, bool PAIR>
__global__ void __launch_bounds__(256) k_widen_scaled(const ST* __restrict__ in, double* __restrict__ out,
                                                       int64_t rows, int64_t cols, const int* __restrict__ e,
                                                       int* __restrict__ inexact) {
  const int64_t elems = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < elems; x += stride) {
    const double s = pow2(-(BY_ROW ? e[x / cols] : e[x % cols]));
    if constexpr (PAIR) {
      static_assert(NC == 2, "pairs are formed from two components");
      double sum, err;
      dsum(to_d<ST>(in[x * 2]), to_d<ST>(in[x * 2 + 1]), sum, err);
      out[x * 2] = __dmul_rn(sum, s);
      out[x * 2 + 1] = __dmul_rn(err, s);
      if (err != 0.0) atomicOr(inexact, 1);
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) out[x * NC + c] = __dmul_rn(to_d<ST>(in[x * NC + c]), s);
    }
  }
}

// ---- cp.async helpers ------------------------------------------------------------------

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- the tiled kernel ------------------------------------------------------------------

template <int NA, int NB, int BM, int BN, int BK, int TM, int TN>
struct Tile {
  static constexpr int kThreads = (BM / TM) * (BN / TN);
  static constexpr int kStages = 3;
  static constexpr int kRowA = BK * NA + 2;  // doubles; +16 B staggers rows across banks
  static constexpr int kRowB = BN * NB;
  static constexpr int kStageElems = BM * kRowA + BK * kRowB;
  static constexpr int kSmem = kStages * kStageElems * 8;
};

// A: (batch, M, K, NA) binary64; B: (batch, K, N, NB) binary64 (b_bstride 0 =
// broadcast); out: (batch, M, N, NCO) components of type OST.
// Thread (ty, tx) owns rows ty + i*(BM/TM) and columns tx + j*(BN/TN): a
// warp's B loads are consecutive doubles (conflict-free), its A loads two
// broadcast rows 16 B apart in bank space.
template <class Acc, class OST, int NCO, int BM, int BN, int BK, int TM, int TN, int MINB = 1>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
    k_mm_fast(const double* __restrict__ A, const double* __restrict__ B, OST* __restrict__ Cout,
              int64_t M, int64_t N, int64_t K, int64_t a_bstride, int64_t b_bstride,
              int64_t c_bstride, const int* __restrict__ row_e, const int* __restrict__ col_e,
              double sigma, const int* __restrict__ inexact, int want_inexact) {
  // the exact-sum and the err-carrying variants are both launched; the
  // widening pass's flag decides which one runs (the other exits here)
  if (inexact && ((*inexact != 0) != (want_inexact != 0))) return;
  constexpr int NA = Acc::kNA, NB = Acc::kNB;
  using T = Tile<NA, NB, BM, BN, BK, TM, TN>;
  constexpr int RS = BM / TM;  // row stride between a thread's rows
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int64_t bz = blockIdx.z;
  A += bz * a_bstride;
  B += bz * b_bstride;
  Cout += bz * c_bstride;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int ktiles = (int)((K + BK - 1) / BK);

  auto load_tile = [&](int kt, int slot) {
    double* As = smem + slot * T::kStageElems;
    double* Bs = As + BM * T::kRowA;
    const int64_t k0 = (int64_t)kt * BK;
    constexpr int kChA = BK * NA / 2;  // 16-byte chunks per A row
    for (int c = tid; c < BM * kChA; c += T::kThreads) {
      const int r = c / kChA, q = c % kChA;
      const int64_t gr = m0 + r;
      const int64_t ge = k0 * NA + 2 * q;
      const bool ok = gr < M && ge < K * NA;
      cp16(As + r * T::kRowA + 2 * q, ok ? A + gr * K * NA + ge : A, ok);
    }
    constexpr int kChB = BN * NB / 2;
    for (int c = tid; c < BK * kChB; c += T::kThreads) {
      const int r = c / kChB, q = c % kChB;
      const int64_t gk = k0 + r;
      const int64_t ge = n0 * NB + 2 * q;
      const bool ok = gk < K && ge < N * NB;
      cp16(Bs + r * T::kRowB + 2 * q, ok ? B + gk * N * NB + ge : B, ok);
    }
  };

  double acc[TM][TN][Acc::kLv];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int l = 0; l < Acc::kLv; ++l) acc[i][j][l] = l == 0 ? sigma : 0.0;

#pragma unroll
  for (int s = 0; s < T::kStages - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<T::kStages - 2>();
    __syncthreads();
    {
      const int nk = kt + T::kStages - 1;
      if (nk < ktiles) load_tile(nk, nk % T::kStages);
      cp_commit();
    }
    const double* As = smem + (kt % T::kStages) * T::kStageElems;
    const double* Bs = As + BM * T::kRowA;
    // unrolled by 2 so the running value's old and new registers alternate
    // instead of being copied (IMAD.MOV pairs) every step
#pragma unroll 2
    for (int k = 0; k < BK; ++k) {
      double a[TM][NA], b[TN * NB];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int c = 0; c < NA; ++c) a[i][c] = As[(ty + i * RS) * T::kRowA + k * NA + c];
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int c = 0; c < NB; ++c) b[j * NB + c] = Bs[k * T::kRowB + (tx + j * (BN / TN)) * NB + c];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) Acc::mad(acc[i][j], a[i], b + j * NB);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t r = m0 + ty + i * RS;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t c = n0 + tx + j * (BN / TN);
      if (c >= N) continue;
      if (row_e) {
        // offset policies: S = tau - sigma (exact), undo the operand scaling
        const double sc = pow2(row_e[bz * M + r] + col_e[(b_bstride ? bz * N : 0) + c]);
        double v[Acc::kLv];
#pragma unroll
        for (int l = 0; l < Acc::kLv; ++l) v[l] = __dmul_rn(l == 0 ? __dsub_rn(acc[i][j][0], sigma) : acc[i][j][l], sc);
        split_out<OST, NCO, Acc::kLv>(v, Cout + (r * N + c) * NCO);
      } else {
        split_out<OST, NCO, Acc::kLv>(acc[i][j], Cout + (r * N + c) * NCO);
      }
    }
  }
}

template <class Acc, class OST, int NCO, int BM, int BN, int BK, int TM, int TN, int MINB = 1>
mcf_status launch_mm(const double* A, const double* B, void* C, int64_t batch, int64_t M,
                     int64_t N, int64_t K, int64_t a_bs, int64_t b_bs, int64_t c_bs,
                     cudaStream_t s, const int* row_e = nullptr, const int* col_e = nullptr,
                     double sigma = 0.0, const int* inexact = nullptr, int want_inexact = 0) {
  using T = Tile<Acc::kNA, Acc::kNB, BM, BN, BK, TM, TN>;
  auto kern = k_mm_fast<Acc, OST, NCO, BM, BN, BK, TM, TN, MINB>;
  {
    const mcf_status ast = mcfr::ensure_smem_attr<k_mm_fast<Acc, OST, NCO, BM, BN, BK, TM, TN, MINB>>(
        T::kSmem, "mm_fast: cannot reserve shared memory");
    if (ast != MCF_OK) return ast;
  }
  const dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)batch);
  kern<<<grid, T::kThreads, T::kSmem, s>>>(A, B, static_cast<OST*>(C), M, N, K, a_bs, b_bs, c_bs, row_e,
                                            col_e, sigma, inexact, want_inexact);
  mcfr::note_launch();
  return mcfr::check_launch("mm_fast kernel");
}

// sigma = 2^(ceil(log2 K) + 1): every partial sum of products below 1 in
// magnitude stays below sigma / 2
double offset_sigma(int64_t k) {
  int e = 0;
  while ((int64_t(1) << e) < k) ++e;
  return ldexp(1.0, e + 1);
}

// exponents + scaled widening of A (rows of k elements, nca comps) and B
// (k x n, ncb comps); nc=2 operands become (sum, err) pairs, *inexact is
// cleared first and raised if any err is nonzero
// B side: column exponents and the scaled widening of B (raises *inexact,
// which the caller has cleared)
template <int NCB>
mcf_status widen_scaled_b(const float* w, int64_t brows, int64_t n, double* wd, int* eb, int* inexact,
                          cudaStream_t s) {
  if (cudaMemsetAsync(eb, 0, n * sizeof(int), s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the column maxima");
  const dim3 g((unsigned)((n + 255) / 256), (unsigned)((brows + kColRows - 1) / kColRows));
  if (brows > 0) {
    k_colmax<float, NCB><<<g, 256, 0, s>>>(w, brows, n, eb);
    mcfr::note_launch();
  }
  k_colexp_fin<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(eb, n);
  mcfr::note_launch();
  k_widen_scaled<float, NCB, false, NCB == 2><<<mcfr::grid_for(brows * n, 256, 8), 256, 0, s>>>(w, wd, brows, n, eb,
                                                                                                inexact);
  mcfr::note_launch();
  return mcfr::check_launch("mm_fast B scaling kernels");
}

// A side: row exponents and the scaled widening of A (rows x k)
template <int NCA>
mcf_status widen_scaled_a(const float* x, int64_t rows, int64_t k, double* xd, int* ea, int* inexact,
                          cudaStream_t s) {
  k_rowexp<float, NCA><<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(x, rows, k, ea);
  mcfr::note_launch();
  k_widen_scaled<float, NCA, true, NCA == 2><<<mcfr::grid_for(rows * k, 256, 8), 256, 0, s>>>(x, xd, rows, k, ea,
                                                                                              inexact);
  mcfr::note_launch();
  return mcfr::check_launch("mm_fast A scaling kernels");
}

template <int NCA, int NCB>
mcf_status widen_scaled(const float* x, const float* w, int64_t rows, int64_t k, int64_t brows, int64_t n,
                        double* xd, double* wd, int* ea, int* eb, int* inexact, cudaStream_t s) {
  if (cudaMemsetAsync(inexact, 0, sizeof(int), s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the exactness flag");
  const mcf_status st = widen_scaled_a<NCA>(x, rows, k, xd, ea, inexact, s);
  if (st != MCF_OK) return st;
  return widen_scaled_b<NCB>(w, brows, n, wd, eb, inexact, s);
}

template <class ST, int NC, bool SUM>
mcf_status widen(const void* in, double* out, int64_t elems, cudaStream_t s) {
  if (elems == 0) return MCF_OK;
  const int grid = mcfr::grid_for(elems, 256, 8);
  k_widen<ST, NC, SUM><<<grid, 256, 0, s>>>(static_cast<const ST*>(in), out, elems);
  mcfr::note_launch();
  return mcfr::check_launch("mm_fast widen kernel");
}

// per-(device, stream) binary64 operand workspace
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, std::pair<void*, std::size_t>> g_ws;

double* stream_workspace(std::size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& slot = g_ws[{dev, s}];
  if (slot.second < bytes) {
    if (slot.first) {
      cudaStreamSynchronize(s);
      cudaFree(slot.first);
    }
    slot = {nullptr, 0};
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    slot = {p, bytes};
  }
  return static_cast<double*>(slot.first);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// pipe-rate probe: 8 independent FMA chains per thread, all SMs, 8 CTAs/SM
template <bool F64>
__global__ void __launch_bounds__(256) k_probe(double* out, int iters, double a) {
  double d[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    d[i] = a + i + threadIdx.x;
    f[i] = (float)d[i];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (F64) d[i] = __fma_rn(d[i], a, d[(i + 1) & 7]);
      else f[i] = __fmaf_rn(f[i], (float)a, f[(i + 1) & 7]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace
}  // namespace mcfg

extern "C" int mcf_probe_pipe_rates(double* fp64_ops_per_s, double* fp32_ops_per_s) {
  using namespace mcfg;
  const int sms = mcfr::sm_count(), blocks = sms * 8, threads = 256, iters = 8192;
  double* buf = nullptr;
  if (cudaMalloc(&buf, (size_t)blocks * threads * sizeof(double)) != cudaSuccess) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double rates[2] = {0, 0};
  for (int kind = 0; kind < 2; ++kind) {
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_probe<true><<<blocks, threads>>>(buf, iters, 0.999999);
      else k_probe<false><<<blocks, threads>>>(buf, iters, 0.999999);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double r = (double)blocks * threads * iters * 8 / (ms * 1e-3);
      if (r > rates[kind]) rates[kind] = r;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  if (fp64_ops_per_s) *fp64_ops_per_s = rates[0];
  if (fp32_ops_per_s) *fp32_ops_per_s = rates[1];
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// ---- entry points used by the C-ABI (linalg.cu routes MCF_FAST here) -------------------

namespace mcfr {

// the offset-accumulation pair (AccP2 runs when the widening flag is clear,
// AccP2X when it is set; the other exits at once), tile chosen by shape.
// MCF_MM_TILE (tuning knob) forces a tile: a = 128x64/8x4 (256 thr),
// b = 64x64/4x4 (256 thr, 2 CTAs/SM), c = 128x64/4x4 (512 thr).
template <int NB>
mcf_status launch_p2(const double* xd, const double* wd, void* out, int64_t batch, int64_t m, int64_t n, int64_t k,
                     int64_t a_bs, int64_t b_bs, int64_t c_bs, cudaStream_t s, const int* ea, const int* eb,
                     double sg, const int* flag) {
  using namespace mcfg;
  static const char tile = [] {
    const char* e = getenv("MCF_MM_TILE");
    return e && *e ? e[0] : 'a';
  }();
#define MCF_P2(BM, BN, TM, TN, MINB)                                                                              \
  do {                                                                                                            \
    mcf_status st = launch_mm<AccP2<NB>, float, 2, BM, BN, 16, TM, TN, MINB>(xd, wd, out, batch, m, n, k, a_bs,   \
                                                                            b_bs, c_bs, s, ea, eb, sg, flag, 0);  \
    if (st != MCF_OK) return st;                                                                                  \
    return launch_mm<AccP2X<NB>, float, 2, BM, BN, 16, TM, TN, MINB>(xd, wd, out, batch, m, n, k, a_bs, b_bs,     \
                                                                     c_bs, s, ea, eb, sg, flag, 1);               \
  } while (0)
  // short A (e.g. an MLP's 10-class output layer): 16-row tiles, so the
  // outputs spread over ~one CTA per SM instead of one mostly empty row block
  if (m <= 32) MCF_P2(16, 64, 2, 4, 1);
  if (tile == 'b') MCF_P2(64, 64, 4, 4, 2);
  if (tile == 'c') MCF_P2(128, 64, 4, 4, 1);
  MCF_P2(128, 64, 8, 4, 1);
#undef MCF_P2
}

// FP64-pipe instructions per multiply-add of the kernel a fast call uses
int mm_fast_ops_per_mad(int mcmc, mcf_prec p, int nc) {
  using namespace mcfg;
  if (p == MCF_B32 && !mcmc) return nc == 2 ? AccP2<1>::kOps : nc == 3 ? AccT3::kOps : 0;
  if (p == MCF_B32 && mcmc) return nc == 2 ? AccP2<2>::kOps : nc == 3 ? AccM3::kOps : 0;
  return (p == MCF_B16 && mcmc && nc == 3) ? AccH3::kOps : 0;
}

// MC x Tensor; MCF_ERR_UNSUPPORTED (no message) when no fast instantiation
// covers the call, so the caller can fall back to the reference-order kernel.
mcf_status mm_fast_mct(mcf_prec p, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                       int64_t k, int64_t n, int w_batched, void* out, cudaStream_t s, bool tc) {
  using namespace mcfg;
  // INT8 tensor-core path (mm_ozaki.cu), one product per batch entry.  Short
  // A (m < 64, e.g. an MLP's 10-class layer) stays on the FP64 pipe: the int8
  // GEMMs degenerate to GEMV kernels there (measured 0.68 ms vs 0.09 ms).
  if (tc && p == MCF_B32 && nc == 2 && m >= 64 && ozaki_supported(m, k, n)) {
    const float* xf = static_cast<const float*>(x);
    const float* wf = static_cast<const float*>(w);
    float* of = static_cast<float*>(out);
    for (int64_t b = 0; b < batch; ++b) {
      const mcf_status st = mm_ozaki(xf + b * m * k * 2, 2, wf + (w_batched ? b * k * n : 0), 1, m, k, n,
                                     of + b * m * n * 2, s);
      if (st == MCF_ERR_UNSUPPORTED) break;  // no int8 GEMM for the shape: FP64 pipe below
      if (st != MCF_OK) return st;
      if (b + 1 == batch) return MCF_OK;
    }
  }
  // short A (an MLP's class layer): one kernel, no binary64 workspace (mm_skinny.cu)
  static const bool skinny_on = [] {
    const char* e = getenv("MCF_MM_SKINNY");
    return !(e && e[0] == '0');
  }();
  if (skinny_on && p == MCF_B32 && nc == 2 && m <= 16) {
    const float* xf = static_cast<const float*>(x);
    const float* wf = static_cast<const float*>(w);
    float* of = static_cast<float*>(out);
    for (int64_t b = 0; b < batch; ++b) {
      const mcf_status st = mm_skinny_mct(xf + b * m * k * 2, wf + (w_batched ? b * k * n : 0), m, k, n,
                                          of + b * m * n * 2, s);
      if (st == MCF_ERR_UNSUPPORTED) {
        if (b == 0) break;  // alignment / shape outside the kernel: the general path below
        return fail(MCF_ERR_CUDA, "mm_fast: the short-A kernel refused a later batch entry");
      }
      if (st != MCF_OK) return st;
      if (b + 1 == batch) return MCF_OK;
    }
  }
  if (p != MCF_B32 || (nc != 2 && nc != 3) || n % 2 != 0 || (k * nc) % 2 != 0)
    return MCF_ERR_UNSUPPORTED;
  const int64_t xa = batch * m * k * nc, wb = (w_batched ? batch : 1) * k * n;
  const int64_t ne = batch * m + (w_batched ? batch : 1) * n;  // scale exponents
  double* ws = stream_workspace((xa + wb) * sizeof(double) + ne * sizeof(int) + 512, s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the binary64 workspace");
  double* xd = ws;
  double* wd = ws + ((xa + 1) / 2) * 2;  // 16-byte aligned
  const int64_t a_bs = m * k * nc, b_bs = w_batched ? k * n : 0, c_bs = m * n * nc;
  if (nc == 2 && !w_batched) {
    // offset accumulation on (sum, err) operands: rows of A and columns of B
    // scaled by powers of two (AccP2 / AccP2X, see mcf_accum.cuh)
    int* ea = reinterpret_cast<int*>(wd + ((wb + 1) / 2) * 2);
    int* eb = ea + batch * m;
    int* flag = eb + n;
    mcf_status st = widen_scaled<2, 1>(static_cast<const float*>(x), static_cast<const float*>(w), batch * m, k, k,
                                       n, xd, wd, ea, eb, flag, s);
    if (st != MCF_OK) return st;
    return launch_p2<1>(xd, wd, out, batch, m, n, k, a_bs, b_bs, c_bs, s, ea, eb, offset_sigma(k), flag);
  }
  mcf_status st = nc == 2 ? widen<float, 2, false>(x, xd, batch * m * k, s)
                          : widen<float, 3, false>(x, xd, batch * m * k, s);
  if (st != MCF_OK) return st;
  st = widen<float, 1, false>(w, wd, wb, s);
  if (st != MCF_OK) return st;
  if (nc == 2) return launch_mm<AccT2, float, 2, 128, 64, 16, 8, 4>(xd, wd, out, batch, m, n, k, a_bs, b_bs, c_bs, s);
  return launch_mm<AccT3, float, 3, 64, 64, 16, 4, 4>(xd, wd, out, batch, m, n, k, a_bs, b_bs, c_bs, s);
}

// Host-buffer MC(nc=2, binary32) x T product, pipelined over row chunks of A:
// B is copied, scaled and widened once; then chunk c's H2D copy (stream cin),
// its widening and mm (alternating comp[0] / comp[1], so one chunk's tail CTAs
// overlap the next chunk's first ones) and its D2H copy (cout) overlap the
// neighbouring chunks.  dx / dw / dout are device buffers of the full sizes.
mcf_status mm_fast_mct_host(const float* hx, const float* hw, int64_t m, int64_t k, int64_t n, float* hout,
                            float* dx, float* dw, float* dout, cudaStream_t cin, const cudaStream_t comp[2],
                            cudaStream_t cout) {
  using namespace mcfg;
  if (m <= 0 || k <= 0 || n <= 0 || n % 2 != 0) return MCF_ERR_UNSUPPORTED;
  const int64_t rc = std::max<int64_t>(512, ((m + 7) / 8 + 127) / 128 * 128);
  const int nch = (int)((m + rc - 1) / rc);
  double* ws = stream_workspace((m * k * 2 + k * n) * sizeof(double) + (m + n + nch + 1) * sizeof(int) + 512,
                                comp[0]);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the binary64 workspace");
  double* xd = ws;
  double* wd = ws + m * k * 2;
  int* ea = reinterpret_cast<int*>(wd + ((k * n + 1) / 2) * 2);
  int* eb = ea + m;
  int* flag_b = eb + n;  // then one flag per chunk
  std::vector<cudaEvent_t> ev(2 * nch + 2, nullptr);
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return fail(MCF_ERR_CUDA, "mm_fast: cannot create pipeline events");
  auto done = [&](mcf_status st) {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    return st;
  };
  auto cu = [&](cudaError_t e, const char* what) {
    return e == cudaSuccess ? MCF_OK : fail(MCF_ERR_CUDA, std::string("mm_mcn pipeline: ") + what + ": " +
                                                              cudaGetErrorString(e));
  };
#define PIPE_TRY(expr)                    \
  do {                                    \
    const mcf_status _s = (expr);         \
    if (_s != MCF_OK) return done(_s);    \
  } while (0)
  const double sg = offset_sigma(k);
  PIPE_TRY(cu(cudaMemcpyAsync(dw, hw, k * n * sizeof(float), cudaMemcpyHostToDevice, cin), "H2D w"));
  PIPE_TRY(cu(cudaEventRecord(ev[0], cin), "event"));
  PIPE_TRY(cu(cudaStreamWaitEvent(comp[0], ev[0], 0), "wait"));
  PIPE_TRY(cu(cudaMemsetAsync(flag_b, 0, sizeof(int), comp[0]), "flag"));
  PIPE_TRY(widen_scaled_b<1>(dw, k, n, wd, eb, flag_b, comp[0]));
  PIPE_TRY(cu(cudaEventRecord(ev[1], comp[0]), "event"));
  PIPE_TRY(cu(cudaStreamWaitEvent(comp[1], ev[1], 0), "wait"));
  for (int c = 0; c < nch; ++c) {
    const int64_t r0 = c * rc, rows = std::min<int64_t>(rc, m - r0);
    cudaStream_t cs = comp[c & 1];
    cudaEvent_t ex = ev[2 + 2 * c], em = ev[3 + 2 * c];
    int* fl = flag_b + 1 + c;
    PIPE_TRY(cu(cudaMemcpyAsync(dx + r0 * k * 2, hx + r0 * k * 2, rows * k * 2 * sizeof(float),
                                cudaMemcpyHostToDevice, cin), "H2D x"));
    PIPE_TRY(cu(cudaEventRecord(ex, cin), "event"));
    PIPE_TRY(cu(cudaStreamWaitEvent(cs, ex, 0), "wait"));
    PIPE_TRY(cu(cudaMemcpyAsync(fl, flag_b, sizeof(int), cudaMemcpyDeviceToDevice, cs), "flag"));
    PIPE_TRY(widen_scaled_a<2>(dx + r0 * k * 2, rows, k, xd + r0 * k * 2, ea + r0, fl, cs));
    PIPE_TRY(launch_p2<1>(xd + r0 * k * 2, wd, dout + r0 * n * 2, 1, rows, n, k, 0, 0, 0, cs, ea + r0, eb, sg, fl));
    PIPE_TRY(cu(cudaEventRecord(em, cs), "event"));
    PIPE_TRY(cu(cudaStreamWaitEvent(cout, em, 0), "wait"));
    PIPE_TRY(cu(cudaMemcpyAsync(hout + r0 * n * 2, dout + r0 * n * 2, rows * n * 2 * sizeof(float),
                                cudaMemcpyDeviceToHost, cout), "D2H out"));
  }
#undef PIPE_TRY
  return done(cu(cudaStreamSynchronize(cout), "sync"));
}

mcf_status mm_fast_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t m, int64_t k,
                        int64_t n, void* out, cudaStream_t s, bool tc) {
  using namespace mcfg;
  if (tc && p == MCF_B32 && nc == 2 && ozaki_supported(m, k, n)) {
    const mcf_status st = mm_ozaki(static_cast<const float*>(x), 2, static_cast<const float*>(y), 2, m, k, n,
                                   static_cast<float*>(out), s);
    if (st != MCF_ERR_UNSUPPORTED) return st;
  }
  if (tc && p == MCF_B16 && nc <= 3) {
    const mcf_status st = mm_b16_i8(x, y, nc, m, k, n, out, s);
    if (st != MCF_ERR_UNSUPPORTED) return st;
  }
  const bool f32 = p == MCF_B32 && nc == 2, f16 = p == MCF_B16 && nc == 3;
  if ((!f32 && !f16) || n % 2 != 0 || k % 2 != 0) return MCF_ERR_UNSUPPORTED;
  const int w = f32 ? 2 : 1;  // binary64 words per element after widening
  const int64_t xa = m * k * w, yb = k * n * w;
  double* ws = stream_workspace((xa + yb) * sizeof(double) + (m + n) * sizeof(int) + 512, s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the binary64 workspace");
  double* xd = ws;
  double* yd = ws + ((xa + 1) / 2) * 2;
  mcf_status st;
  if (f32) {
    int* ea = reinterpret_cast<int*>(yd + ((yb + 1) / 2) * 2);
    int* eb = ea + m;
    int* flag = eb + n;
    st = widen_scaled<2, 2>(static_cast<const float*>(x), static_cast<const float*>(y), m, k, k, n, xd, yd, ea, eb,
                            flag, s);
    if (st != MCF_OK) return st;
    return launch_p2<2>(xd, yd, out, 1, m, n, k, 0, 0, 0, s, ea, eb, offset_sigma(k), flag);
  }
  st = widen<__half, 3, true>(x, xd, m * k, s);
  if (st == MCF_OK) st = widen<__half, 3, true>(y, yd, k * n, s);
  if (st != MCF_OK) return st;
  return launch_mm<AccH3, __half, 3, 128, 128, 16, 8, 8>(xd, yd, out, 1, m, n, k, 0, 0, 0, s);
}

}  // namespace mcfr
