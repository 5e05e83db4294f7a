// mm_skinny.cu -- MC(nc = 2, binary32) x Tensor for a SHORT A (m <= 16 rows:
// an MLP's class layer W (10 x 1024) . activations (1024 x batch)) on the FP64
// pipe, one kernel.
//
// The general FP64-pipe product (mm_fast.cu) widens both operands into a
// binary64 workspace first (column maxima, scaled widening of B: four
// launches and 3x B's bytes of traffic) and then runs 16-row tiles that are
// mostly empty for ten rows.  Here a CTA owns 64 columns and every row:
//   0. row exponents of A (2^e above the largest leading component),
//   1. column maxima of its B columns (one pass over the tile; the second
//      pass below hits L2),
//   2. per 512-deep K chunk, A's rows as scaled (sum, err) binary64 pairs in
//      shared memory; B's rows stream through a 4-stage shared-memory ring
//      filled by TMA bulk copies (cp.async.bulk, one 256-byte row segment per
//      lane of a producer warp, mbarrier transaction counts); a consumer
//      thread owns one column and half the rows and carries each output's
//      extended accumulator (tau, C) in registers through the K loop: the
//      offset accumulation of mcf_accum.cuh (AccP2X: 5 FP64 ops per
//      multiply-add, products of binary32 components exact in binary64),
//   3. the greedy split of each accumulator into two binary32 components.
// Accuracy is that of the general FP64-pipe path (~2^-100 x cond before the
// split).  Non-finite rows / columns stay unscaled and propagate.
#include <cuda_runtime.h>

#include <cstdint>

#include "mcf_accum.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

constexpr int kCols = 64;        // columns per CTA
constexpr int kGroups = 2;       // row groups (a thread: one column, one group's rows)
constexpr int kConsumers = kCols * kGroups;
constexpr int kThreads = kConsumers + 32;  // + one producer warp
constexpr int kChunk = 512;      // K rows of A staged at a time
constexpr int kStageRows = 32;   // B rows per ring stage (one per producer lane)
constexpr int kStages = 4;

__device__ __forceinline__ unsigned s_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(s_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumers) : "memory"); }

__device__ __forceinline__ int exp_above(float m) { return m > 0.0f && isfinite(m) ? ilogbf(m) + 1 : 0; }
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// x: (m, k, 2) binary32 MC, w: (k, n) binary32, out: (m, n, 2).  RPT rows per
// thread (m <= 2 RPT).  Dynamic shared memory: A chunk, B ring, barriers.
template <int RPT>
__global__ void __launch_bounds__(kThreads, 1)
    k_mm_skinny(const float* __restrict__ x, const float* __restrict__ w, float* __restrict__ out, int m, int64_t k,
                int64_t n, double sigma) {
  extern __shared__ __align__(128) unsigned char smem[];
  double2* As = reinterpret_cast<double2*>(smem);                                   // [2 RPT][kChunk]
  float* Bs = reinterpret_cast<float*>(smem + (size_t)2 * RPT * kChunk * 16);        // [kStages][kStageRows][kCols]
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + kStages * kStageRows * kCols);
  uint64_t* empty = full + kStages;
  float* cmax = reinterpret_cast<float*>(empty + kStages);                           // [kGroups][kCols]
  int* ea = reinterpret_cast<int*>(cmax + kGroups * kCols);                          // [2 RPT]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t j0 = (int64_t)blockIdx.x * kCols;
  const int ncols = (int)(n - j0 < kCols ? n - j0 : kCols);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // 0. row exponents of A (the leading components' maximum), a warp per row
  for (int i = warp; i < m; i += kThreads / 32) {
    float mx = 0.0f;
    for (int64_t t = lane; t < k; t += 32) mx = fmaxf(mx, fabsf(x[((int64_t)i * k + t) * 2]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (lane == 0) ea[i] = exp_above(mx);
  }
  // 1. column maxima of this CTA's columns (both row groups share a column)
  const int c = tid & (kCols - 1), g = tid >> 6;  // consumers: g in {0, 1}
  if (tid < kConsumers) {
    float mx = 0.0f;
    if (c < ncols)
      for (int64_t t = g; t < k; t += kGroups) mx = fmaxf(mx, fabsf(__ldg(w + t * n + j0 + c)));
    cmax[g * kCols + c] = mx;
  }
  __syncthreads();

  const int64_t stages_total = (k + kStageRows - 1) / kStageRows;
  if (warp == kConsumers / 32) {  // producer: B's rows, one row segment per lane
    for (int64_t it = 0; it < stages_total; ++it) {
      const int s = (int)(it % kStages);
      const unsigned ph = (unsigned)(it / kStages) & 1u;
      mbar_wait(&empty[s], ph ^ 1u);
      const int64_t r0 = it * kStageRows;
      const int rows = (int)(k - r0 < kStageRows ? k - r0 : kStageRows);
      if (lane == 0) mbar_expect_tx(&full[s], (unsigned)(rows * ncols * 4));
      __syncwarp();
      if (lane < rows)
        bulk_g2s(Bs + ((size_t)s * kStageRows + lane) * kCols, w + (r0 + lane) * n + j0, (unsigned)(ncols * 4), &full[s]);
    }
    return;
  }

  // consumers
  const int eb = exp_above(fmaxf(cmax[c], cmax[kCols + c]));
  const double sb = pow2(-eb);
  double tau[RPT], cc[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) tau[i] = sigma, cc[i] = 0.0;
  int64_t it = 0;
  for (int64_t kc0 = 0; kc0 < k; kc0 += kChunk) {
    const int klen = (int)(k - kc0 < kChunk ? k - kc0 : kChunk);
    consumer_sync();  // the previous chunk's rows are no longer read
    // 2a. A's rows of this chunk as scaled (sum, err) pairs
    for (int e = tid; e < m * klen; e += kConsumers) {
      const int i = e / klen, t = e - i * klen;
      const float2 v = *reinterpret_cast<const float2*>(x + ((int64_t)i * k + kc0 + t) * 2);
      double sum, err;
      dsum((double)v.x, (double)v.y, sum, err);
      const double sa = pow2(-ea[i]);
      As[i * kChunk + t] = make_double2(__dmul_rn(sum, sa), __dmul_rn(err, sa));
    }
    consumer_sync();
    // 2b. the chunk's B rows through the ring
    for (int t0 = 0; t0 < klen; t0 += kStageRows, ++it) {
      const int s = (int)(it % kStages);
      const unsigned ph = (unsigned)(it / kStages) & 1u;
      mbar_wait(&full[s], ph);
      const int rows = klen - t0 < kStageRows ? klen - t0 : kStageRows;
      if (c < ncols) {
        const float* bs = Bs + (size_t)s * kStageRows * kCols + c;
        for (int r = 0; r < rows; ++r) {
          const double b = __dmul_rn((double)bs[r * kCols], sb);
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int row = g * RPT + i;
            if (row < m) {
              const double2 a = As[row * kChunk + t0 + r];
              const double t = __fma_rn(a.x, b, tau[i]);
              const double q = __dsub_rn(t, tau[i]);
              tau[i] = t;
              cc[i] = __fma_rn(a.y, b, __dadd_rn(cc[i], __fma_rn(a.x, b, -q)));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  // 3. undo the scaling, split into two binary32 components
  if (c < ncols) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int row = g * RPT + i;
      if (row < m) {
        const double sc = pow2(ea[row] + eb);
        const double v[2] = {__dmul_rn(__dsub_rn(tau[i], sigma), sc), __dmul_rn(cc[i], sc)};
        float o[2];
        split_out<float, 2, 2>(v, o);
        *reinterpret_cast<float2*>(out + ((int64_t)row * n + j0 + c) * 2) = make_float2(o[0], o[1]);
      }
    }
  }
}

template <int RPT>
mcf_status launch_skinny(const float* x, const float* w, float* out, int m, int64_t k, int64_t n, double sigma,
                         cudaStream_t s) {
  constexpr int smem = 2 * RPT * kChunk * 16 + kStages * kStageRows * kCols * 4 + 2 * kStages * 8 +
                       kGroups * kCols * 4 + 2 * RPT * 4 + 64;
  const mcf_status ast = mcfr::ensure_smem_attr<k_mm_skinny<RPT>>(smem, "mm_skinny: cannot reserve shared memory");
  if (ast != MCF_OK) return ast;
  const unsigned grid = (unsigned)((n + kCols - 1) / kCols);
  k_mm_skinny<RPT><<<grid, kThreads, smem, s>>>(x, w, out, m, k, n, sigma);
  mcfr::note_launch();
  return mcfr::check_launch("mm_skinny kernel");
}

}  // namespace
}  // namespace mcfg

namespace mcfr {

// out (m, n, 2) = x (m, k, 2) . w (k, n) for m <= 16; MCF_ERR_UNSUPPORTED (no
// message) when the shape or the alignment is outside this kernel.
mcf_status mm_skinny_mct(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out, cudaStream_t s) {
  using namespace mcfg;
  if (m < 1 || m > 16 || k < 1 || n < 1 || n % 4 != 0 || k >= (int64_t(1) << 40) ||
      (reinterpret_cast<uintptr_t>(w) & 15) || (reinterpret_cast<uintptr_t>(x) & 7) ||
      (reinterpret_cast<uintptr_t>(out) & 7))
    return MCF_ERR_UNSUPPORTED;
  int e = 0;
  while ((int64_t(1) << e) < k) ++e;
  const double sigma = ldexp(1.0, e + 1);  // mm_fast.cu's offset_sigma
  switch ((int)((m + 1) / 2)) {
    case 1: return launch_skinny<1>(x, w, out, (int)m, k, n, sigma, s);
    case 2: return launch_skinny<2>(x, w, out, (int)m, k, n, sigma, s);
    case 3: return launch_skinny<3>(x, w, out, (int)m, k, n, sigma, s);
    case 4: return launch_skinny<4>(x, w, out, (int)m, k, n, sigma, s);
    case 5: return launch_skinny<5>(x, w, out, (int)m, k, n, sigma, s);
    case 6: return launch_skinny<6>(x, w, out, (int)m, k, n, sigma, s);
    case 7: return launch_skinny<7>(x, w, out, (int)m, k, n, sigma, s);
    default: return launch_skinny<8>(x, w, out, (int)m, k, n, sigma, s);
  }
}

}  // namespace mcfr
