// mm_skinny.cu -- MC(nc = 2, binary32) x Tensor for a SHORT A (m <= 16 rows:
// an MLP's class layer W (10 x 1024) . activations (1024 x batch)) on the FP64
// pipe, one kernel.
//
// The general FP64-pipe product (mm_fast.cu) widens both operands into a
// binary64 workspace first (column maxima, scaled widening of B: four
// launches and 3x B's bytes of traffic) and then runs 16-row tiles that are
// mostly empty for ten rows.  Here a CTA owns 64 columns and every row:
//   0. row exponents of A (2^e above the largest leading component),
//   1. column maxima of its B columns (a first pass of the tile through the
//      same ring; the second pass below hits L2),
//   2. per 512-deep K chunk, A's rows as scaled (sum, err) binary64 pairs in
//      shared memory; B's rows stream through an 8-stage shared-memory ring
//      filled by TMA tensor copies (cp.async.bulk.tensor.2d: one 32-row x 64-
//      column box per stage from a tensor map of B, out-of-range rows and
//      columns zero-filled, mbarrier transaction counts; 256-byte row
//      segments as separate bulk copies took ~130 cycles each); a consumer
//      thread owns one column and a quarter of the rows and carries each output's
//      extended accumulator (tau, C) in registers through the K loop: the
//      offset accumulation of mcf_accum.cuh (AccP2X: 5 FP64 ops per
//      multiply-add, products of binary32 components exact in binary64),
//   3. the greedy split of each accumulator into two binary32 components.
// Accuracy is that of the general FP64-pipe path (~2^-100 x cond before the
// split).  Non-finite rows / columns stay unscaled and propagate.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mcf_accum.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

constexpr int kCols = 64;        // columns per CTA
// row groups G (a thread: one column, one group's RPT rows): 4 or 5, whichever
// wastes fewer row slots (ten rows: 5 x 2); 64 G consumer threads + a producer warp
constexpr int kChunk = 512;      // K rows of A staged at a time
constexpr int kStageRows = 32;   // B rows per ring stage (one per producer lane)
constexpr int kStages = 8;      // 64 KB of B in flight per SM

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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(s_u32(bar))
      : "memory");
}
template <int N>
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ int exp_above(float m) { return m > 0.0f && isfinite(m) ? ilogbf(m) + 1 : 0; }
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// x: (m, k, 2) binary32 MC, w: (k, n) binary32, out: (m, n, 2).  RPT rows per
// thread (m <= G RPT).  Dynamic shared memory: A chunk, B ring, barriers.
template <int G, int RPT>
__global__ void __launch_bounds__(kCols * G + 32, 1)
    k_mm_skinny(const float* __restrict__ x, const __grid_constant__ CUtensorMap tw, float* __restrict__ out, int m,
                int64_t k, int64_t n, double sigma) {
  constexpr int kGroups = G, kConsumers = kCols * G, kThreads = kConsumers + 32;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* As = reinterpret_cast<double2*>(smem);                                   // [kGroups RPT][kChunk]
  float* Bs = reinterpret_cast<float*>(smem + (size_t)kGroups * RPT * kChunk * 16);  // [kStages][kStageRows][kCols]
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + kStages * kStageRows * kCols);
  uint64_t* empty = full + kStages;
  float* cmax = reinterpret_cast<float*>(empty + kStages);                           // [kGroups][kCols]
  int* ea = reinterpret_cast<int*>(cmax + kGroups * kCols);                          // [kGroups RPT]
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
  const int c = tid & (kCols - 1), g = tid >> 6;  // consumers: g < kGroups
  __syncthreads();

  // B's rows, a 32 x 64 box per stage, streamed twice: once for the column
  // maxima, once for the products (the second pass hits L2)
  const int64_t stages_total = (k + kStageRows - 1) / kStageRows;
  if (warp == kConsumers / 32) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
      for (int64_t it = 0; it < 2 * stages_total; ++it) {
        const int s = (int)(it % kStages);
        const unsigned ph = (unsigned)(it / kStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        const int64_t r0 = (it < stages_total ? it : it - stages_total) * kStageRows;
        mbar_expect_tx(&full[s], kStageRows * kCols * 4);  // the whole box: out-of-range parts arrive as zeros
        tma_load_2d(Bs + (size_t)s * kStageRows * kCols, &tw, (int)j0, (int)r0, &full[s]);
      }
    }
    return;
  }

  // consumers
  // 1. column maxima of this CTA's columns (the row groups share a column)
  int64_t it = 0;
  {
    float mx = 0.0f;
    for (; it < stages_total; ++it) {
      const int s = (int)(it % kStages);
      const unsigned ph = (unsigned)(it / kStages) & 1u;
      mbar_wait(&full[s], ph);
      const int64_t r0 = it * kStageRows;
      const int rows = (int)(k - r0 < kStageRows ? k - r0 : kStageRows);
      if (c < ncols) {
        const float* bs = Bs + (size_t)s * kStageRows * kCols + c;
        for (int r = g; r < rows; r += kGroups) mx = fmaxf(mx, fabsf(bs[r * kCols]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    cmax[g * kCols + c] = mx;
    consumer_sync<kConsumers>();
  }
  float cm = cmax[c];
#pragma unroll
  for (int q = 1; q < kGroups; ++q) cm = fmaxf(cm, cmax[q * kCols + c]);
  const int eb = exp_above(cm);
  const double sb = pow2(-eb);
  double tau[RPT], cc[RPT];
  int arow[RPT];  // offset of the thread's rows in As
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    tau[i] = sigma, cc[i] = 0.0;
    arow[i] = (g * RPT + i < m ? g * RPT + i : m - 1) * kChunk;
  }
  for (int64_t kc0 = 0; kc0 < k; kc0 += kChunk) {
    const int klen = (int)(k - kc0 < kChunk ? k - kc0 : kChunk);
    consumer_sync<kConsumers>();  // the previous chunk's rows are no longer read
    // 2a. A's rows of this chunk as scaled (sum, err) pairs
    // (zeros up to a whole ring stage: B's rows past K arrive as zeros, and
    // 0 x 0 keeps the inner loop free of tail tests)
    const int kpad = (klen + kStageRows - 1) / kStageRows * kStageRows;
    for (int e = tid; e < m * kpad; e += kConsumers) {
      const int i = e / kpad, t = e - i * kpad;
      double2 av = make_double2(0.0, 0.0);
      if (t < klen) {
        const float2 v = *reinterpret_cast<const float2*>(x + ((int64_t)i * k + kc0 + t) * 2);
        double sum, err;
        dsum((double)v.x, (double)v.y, sum, err);
        const double sa = pow2(-ea[i]);
        av = make_double2(__dmul_rn(sum, sa), __dmul_rn(err, sa));
      }
      As[i * kChunk + t] = av;
    }
    consumer_sync<kConsumers>();
    // 2b. the chunk's B rows through the ring
    for (int t0 = 0; t0 < klen; t0 += kStageRows, ++it) {
      const int s = (int)(it % kStages);
      const unsigned ph = (unsigned)(it / kStages) & 1u;
      mbar_wait(&full[s], ph);
      if (c < ncols) {
        const float* bs = Bs + (size_t)s * kStageRows * kCols + c;
        // four k at a time: the loads and conversions of the next steps are
        // in flight while the accumulators' dependent fmas run; branch-free
        // over the thread's rows (a row index past m repeats row m - 1 and is
        // dropped at the end), so the rows' dependent chains interleave: with
        // a branch per row they ran one after the other and the kernel was
        // latency-bound (FP64 pipe 26% active)
#pragma unroll 2
        for (int r0 = 0; r0 < kStageRows; r0 += 4) {
          double b[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) b[u] = __dmul_rn((double)bs[(r0 + u) * kCols], sb);
          double2 a[RPT][4];
#pragma unroll
          for (int i = 0; i < RPT; ++i)
#pragma unroll
            for (int u = 0; u < 4; ++u) a[i][u] = As[arow[i] + t0 + r0 + u];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              const double t = __fma_rn(a[i][u].x, b[u], tau[i]);
              const double q = __dsub_rn(t, tau[i]);
              tau[i] = t;
              cc[i] = __fma_rn(a[i][u].y, b[u], __dadd_rn(cc[i], __fma_rn(a[i][u].x, b[u], -q)));
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

template <int G, int RPT>
mcf_status launch_skinny(const float* x, const CUtensorMap& tw, float* out, int m, int64_t k, int64_t n, double sigma,
                         cudaStream_t s) {
  constexpr int smem = G * RPT * kChunk * 16 + kStages * kStageRows * kCols * 4 + 2 * kStages * 8 + G * kCols * 4 +
                       G * RPT * 4 + 64;
  const mcf_status ast = mcfr::ensure_smem_attr<k_mm_skinny<G, RPT>>(smem, "mm_skinny: cannot reserve shared memory");
  if (ast != MCF_OK) return ast;
  const unsigned grid = (unsigned)((n + kCols - 1) / kCols);
  k_mm_skinny<G, RPT><<<grid, kCols * G + 32, smem, s>>>(x, tw, out, m, k, n, sigma);
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
  auto enc = encode_fn();
  if (!enc || k >= (int64_t(1) << 31) || n >= (int64_t(1) << 31)) return MCF_ERR_UNSUPPORTED;
  CUtensorMap tw;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)k};
    const cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    const cuuint32_t box[2] = {(cuuint32_t)kCols, (cuuint32_t)kStageRows};
    const cuuint32_t estr[2] = {1u, 1u};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(w), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return MCF_ERR_UNSUPPORTED;
  }
  int e = 0;
  while ((int64_t(1) << e) < k) ++e;
  const double sigma = ldexp(1.0, e + 1);  // mm_fast.cu's offset_sigma
  // row groups x rows per thread: 4 x ceil(m / 4) or 5 x ceil(m / 5), the fewer slots
  const int r4 = (int)((m + 3) / 4), r5 = (int)((m + 4) / 5);
  if (5 * r5 < 4 * r4) {
    switch (r5) {
      case 1: return launch_skinny<5, 1>(x, tw, out, (int)m, k, n, sigma, s);
      case 2: return launch_skinny<5, 2>(x, tw, out, (int)m, k, n, sigma, s);
      default: return launch_skinny<5, 3>(x, tw, out, (int)m, k, n, sigma, s);
    }
  }
  switch (r4) {
    case 1: return launch_skinny<4, 1>(x, tw, out, (int)m, k, n, sigma, s);
    case 2: return launch_skinny<4, 2>(x, tw, out, (int)m, k, n, sigma, s);
    case 3: return launch_skinny<4, 3>(x, tw, out, (int)m, k, n, sigma, s);
    default: return launch_skinny<4, 4>(x, tw, out, (int)m, k, n, sigma, s);
  }
}

}  // namespace mcfr
