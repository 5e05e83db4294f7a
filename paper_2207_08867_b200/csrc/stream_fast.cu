// stream_fast.cu -- memory-bound MCF_FAST contractions: one output per warp.
//
// dot_mcn / mv_mcn (MC x Tensor, n = 1) and batched MC x MC dots read each
// operand byte once, so they are HBM-bound (12 B/MAD at nc=3 fp32 MC x T,
// 24 B/MAD for MC x MC).  A warp owns one output row; each lane streams four
// consecutive elements per step with 128-bit loads (the row is contiguous,
// nc components fastest), widens them to binary64 and feeds the compensated
// expansion of mcf_accum.cuh.  The 32 lane partials are merged with
// error-free two_sums through register shuffles in a fixed order, so results
// are deterministic run to run.
#include <cuda_runtime.h>

#include <cstdint>

#include "mcf_accum.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

constexpr int kWarps = 8;
constexpr int kV = 4;  // elements per lane per step

template <int N>
__device__ __forceinline__ void ld_f32(const float* __restrict__ p, float (&d)[N]) {
  static_assert(N % 4 == 0, "16-byte vectors");
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(p) + i);
    d[4 * i] = v.x;
    d[4 * i + 1] = v.y;
    d[4 * i + 2] = v.z;
    d[4 * i + 3] = v.w;
  }
}

// out[r] = sum_k x[r, k, :] * y[r', k, :]; r' = r (y_rstride = row length) or
// 0 (a broadcast vector, y_rstride = 0).  Rows are K*NA (x) and K*NB (y)
// floats; both must be 16-byte aligned with K % 4 == 0.
template <class Acc>
__global__ void __launch_bounds__(kWarps * 32) k_rowdot(const float* __restrict__ x,
                                                        const float* __restrict__ y,
                                                        int64_t y_rstride, float* __restrict__ out,
                                                        int onc, int64_t rows, int64_t K) {
  constexpr int NA = Acc::kNA, NB = Acc::kNB;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float* xr = x + row * K * NA;
  const float* yr = y + row * y_rstride;
  double acc[Acc::kLv];
#pragma unroll
  for (int l = 0; l < Acc::kLv; ++l) acc[l] = 0.0;
  for (int64_t k0 = (int64_t)lane * kV; k0 < K; k0 += 32 * kV) {
    float xa[kV * NA], ya[kV * NB];
    ld_f32<kV * NA>(xr + k0 * NA, xa);
    if (y_rstride == 0) {  // broadcast vector: keep it cached
#pragma unroll
      for (int i = 0; i < kV * NB; ++i) ya[i] = __ldg(yr + k0 * NB + i);
    } else {
      ld_f32<kV * NB>(yr + k0 * NB, ya);
    }
#pragma unroll
    for (int e = 0; e < kV; ++e) {
      double a[NA], b[NB];
#pragma unroll
      for (int c = 0; c < NA; ++c) a[c] = (double)xa[e * NA + c];
#pragma unroll
      for (int c = 0; c < NB; ++c) b[c] = (double)ya[e * NB + c];
      Acc::mad(acc, a, b);
    }
  }
  // butterfly merge of the 32 lane expansions (fixed pairing -> deterministic)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double o[Acc::kLv];
#pragma unroll
    for (int l = 0; l < Acc::kLv; ++l) o[l] = __shfl_xor_sync(0xffffffffu, acc[l], off);
    // both lanes of a pair must form the same sum: order the operands by lane
    if (lane & off) {
      double t[Acc::kLv];
#pragma unroll
      for (int l = 0; l < Acc::kLv; ++l) t[l] = o[l];
#pragma unroll
      for (int l = 0; l < Acc::kLv; ++l) o[l] = acc[l];
#pragma unroll
      for (int l = 0; l < Acc::kLv; ++l) acc[l] = t[l];
    }
    Acc::merge(acc, o);
  }
  if (lane == 0) {
    float res[4];
    if (onc == 2) split_out<float, 2, Acc::kLv>(acc, res);
    else split_out<float, 3, Acc::kLv>(acc, res);
    for (int c = 0; c < onc; ++c) out[row * onc + c] = res[c];
  }
}

template <class Acc>
mcf_status launch_rowdot(const void* x, const void* y, int64_t y_rstride, void* out, int onc,
                         int64_t rows, int64_t K, cudaStream_t s) {
  const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
  k_rowdot<Acc><<<grid, kWarps * 32, 0, s>>>(static_cast<const float*>(x), static_cast<const float*>(y),
                                             y_rstride, static_cast<float*>(out), onc, rows, K);
  mcfr::note_launch();
  return mcfr::check_launch("rowdot kernel");
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace mcfg

namespace mcfr {

// MC x Tensor with n == 1: rows = batch * m, w is a k-vector per batch (or one
// broadcast vector).  MCF_ERR_UNSUPPORTED -> caller falls back.
mcf_status mv_fast_mct(mcf_prec p, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                       int64_t k, int w_batched, void* out, cudaStream_t s) {
  using namespace mcfg;
  if (p != MCF_B32 || (nc != 2 && nc != 3) || k % kV != 0 || !al16(x) || !al16(w))
    return MCF_ERR_UNSUPPORTED;
  if (w_batched && batch > 1 && m > 1) return MCF_ERR_UNSUPPORTED;  // per-batch vector, several rows
  const int64_t rows = batch * m;
  const int64_t ys = (w_batched && batch > 1) ? k : 0;
  return nc == 2 ? launch_rowdot<AccT2>(x, w, ys, out, 2, rows, k, s)
                 : launch_rowdot<AccT3>(x, w, ys, out, 3, rows, k, s);
}

mcf_status dot_fast_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t batch, int64_t k,
                         void* out, cudaStream_t s) {
  using namespace mcfg;
  if (p != MCF_B32 || (nc != 2 && nc != 3) || k % kV != 0 || !al16(x) || !al16(y))
    return MCF_ERR_UNSUPPORTED;
  return nc == 2 ? launch_rowdot<AccM2>(x, y, k * 2, out, 2, batch, k, s)
                 : launch_rowdot<AccM3>(x, y, k * 3, out, 3, batch, k, s);
}

}  // namespace mcfr
