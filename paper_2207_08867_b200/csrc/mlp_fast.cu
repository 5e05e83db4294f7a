// mlp_fast.cu -- the MC-MLP backward pass under plan MCF_FAST.
//
// The reference computes the backward products of mc_linear_op in plain
// binary32 (matmul2d, ndarray.hpp:147-165: fl_mul then fl_add, k in order),
// and the reference-order plan reproduces that bit for bit (mlp.cu).  Plan
// MCF_FAST only promises the reference's error level, so there the gradient
// GEMMs run on the int8 tensor cores (four-digit int8 products, binary32
// accuracy, mm_ozaki.cu: gemm_f32_i8) and the bias gradient is a tree
// reduction.  Shapes the int8 path does not take (a dimension below 64: the
// 10-class layer's dW and dA) run the library's own ordered FFMA GEMM
// (mlp.cu, matmul2d order) -- no vendor BLAS on the path.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "mcf_runtime.h"

namespace {


// C (m x n) = A B^T for short A (m <= 32 rows, K contiguous: the 10-class
// layer's dW = G A_prev^T, K = the batch): a warp per (row j of B, K chunk)
// streams B's row with 16-byte loads, A's chunk staged in shared memory; each
// lane keeps one partial sum per row of A; the lanes are merged by a
// butterfly and the chunks by k_splitk_reduce in chunk order (deterministic).
constexpr int kSkChunk = 1024;
constexpr int kSkRows = 32;
__global__ void __launch_bounds__(256) k_gemm_abt_splitk(const float* __restrict__ a, int64_t lda,
                                                         const float* __restrict__ b, int64_t ldb, int64_t m, int64_t n,
                                                         int64_t k, float* __restrict__ part) {
  extern __shared__ float4 as4[];  // [m][kSkChunk / 4]
  const int64_t k0 = (int64_t)blockIdx.y * kSkChunk, k1 = k0 + kSkChunk < k ? k0 + kSkChunk : k;
  for (int idx = threadIdx.x; idx < m * kSkChunk; idx += blockDim.x) {
    const int i = idx / kSkChunk, kk = idx - i * kSkChunk;
    reinterpret_cast<float*>(as4)[idx] = k0 + kk < k1 ? a[i * lda + k0 + kk] : 0.0f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 8 + warp;
  if (j >= n) return;
  float acc[kSkRows];
#pragma unroll
  for (int i = 0; i < kSkRows; ++i) acc[i] = 0.0f;
  const float* br = b + j * ldb + k0;
  const int len = (int)(k1 - k0);
  const bool vec = ((reinterpret_cast<uintptr_t>(br) & 15) == 0);
  for (int kk = lane * 4; kk < len; kk += 128) {
    float4 q;
    if (vec && kk + 3 < len) {
      q = __ldg(reinterpret_cast<const float4*>(br + kk));
    } else {
      q.x = br[kk];
      q.y = kk + 1 < len ? br[kk + 1] : 0.0f;
      q.z = kk + 2 < len ? br[kk + 2] : 0.0f;
      q.w = kk + 3 < len ? br[kk + 3] : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < kSkRows; ++i) {
      if (i >= m) break;
      const float4 av = as4[i * (kSkChunk / 4) + kk / 4];  // 16-byte shared loads, conflict-free
      acc[i] = __fmaf_rn(av.x, q.x, acc[i]);
      acc[i] = __fmaf_rn(av.y, q.y, acc[i]);
      acc[i] = __fmaf_rn(av.z, q.z, acc[i]);
      acc[i] = __fmaf_rn(av.w, q.w, acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < kSkRows; ++i) {
    if (i >= m) break;
    float v = acc[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) part[((int64_t)blockIdx.y * m + i) * n + j] = v;
  }
}

__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ part, int chunks, int64_t m,
                                                       int64_t n, float* __restrict__ c, int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e / n, j = e - i * n;
  float v = 0.0f;
  for (int q = 0; q < chunks; ++q) v = __fadd_rn(v, part[(int64_t)q * m * n + e]);
  c[i * ldc + j] = v;
}

// C (m x n) = op(A) B for a SHORT K (k <= 16, B's rows contiguous: the
// 10-class layer's dA = approx(W)^T G, K = 10 classes): memory-bound (one
// mask load and one store per output), so a thread keeps its four columns of
// B (k x 4 values) in registers and walks a strip of rows with op(A)'s strip
// in shared memory; 16-byte mask loads and stores.  The arithmetic is the
// ordered kernel's (fl_mul then fl_add, k increasing, mask applied as 0 + c):
// bit-identical to mcf_gemm_f32_ordered.
constexpr int kSmallK = 16;
constexpr int kSmallRows = 32;  // rows per CTA
template <bool TA>
__global__ void __launch_bounds__(256) k_gemm_smallk(const float* __restrict__ a, int64_t lda,
                                                     const float* __restrict__ b, int64_t ldb, float* __restrict__ c,
                                                     int64_t ldc, int64_t m, int64_t n, int k,
                                                     const float* __restrict__ mask) {
  __shared__ float as[kSmallK][kSmallRows];
  const int64_t i0 = (int64_t)blockIdx.y * kSmallRows;
  for (int e = threadIdx.x; e < k * kSmallRows; e += blockDim.x) {
    const int kk = e / kSmallRows, r = e - kk * kSmallRows;
    const int64_t gi = i0 + r;
    as[kk][r] = gi < m ? (TA ? a[kk * lda + gi] : a[gi * lda + kk]) : 0.0f;
  }
  __syncthreads();
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (j >= n) return;
  float4 bv[kSmallK];
#pragma unroll
  for (int kk = 0; kk < kSmallK; ++kk)
    bv[kk] = kk < k ? __ldg(reinterpret_cast<const float4*>(b + kk * ldb + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
  const int rows = (int)(m - i0 < kSmallRows ? m - i0 : kSmallRows);
  for (int r = 0; r < rows; ++r) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int kk = 0; kk < kSmallK; ++kk)
      if (kk < k) {
        const float av = as[kk][r];
        acc.x = __fadd_rn(acc.x, __fmul_rn(av, bv[kk].x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(av, bv[kk].y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(av, bv[kk].z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(av, bv[kk].w));
      }
    float* cr = c + (i0 + r) * ldc + j;
    if (mask) {
      const float4 mk = __ldcs(reinterpret_cast<const float4*>(mask + (i0 + r) * ldc + j));
      acc.x = mk.x > 0.0f ? __fadd_rn(0.0f, acc.x) : 0.0f;
      acc.y = mk.y > 0.0f ? __fadd_rn(0.0f, acc.y) : 0.0f;
      acc.z = mk.z > 0.0f ? __fadd_rn(0.0f, acc.z) : 0.0f;
      acc.w = mk.w > 0.0f ? __fadd_rn(0.0f, acc.w) : 0.0f;
    }
    *reinterpret_cast<float4*>(cr) = acc;
  }
}

// out[r] = sum_j g[r, j]: a CTA per row, tree reduction
__global__ void __launch_bounds__(256) k_rowsum_tree(const float* __restrict__ g, int64_t n, float* __restrict__ out) {
  __shared__ float part[8];
  const int64_t r = blockIdx.x;
  float acc = 0.0f;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) acc += g[r * n + j];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < 8 ? part[threadIdx.x] : 0.0f;
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (threadIdx.x == 0) out[r] = acc;
  }
}

}  // namespace

extern "C" {

// Same operands and layout as mcf_gemm_f32_ordered (row-major C = op(A) op(B),
// optional ReLU mask), binary32 accuracy in the GPU's summation order.
mcf_status mcf_gemm_f32_fast(int trans_a, int trans_b, const float* a, int64_t lda, const float* b, int64_t ldb,
                             float* c, int64_t ldc, int64_t m, int64_t n, int64_t k, const float* relu_mask,
                             mcf_stream s) {
  if (m < 0 || n < 0 || k < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "gemm_f32: negative dimension");
  if (m * n == 0) return MCF_OK;
  // int8 tensor cores (four balanced digits per operand, exact int32 sums:
  // mm_ozaki.cu) unless the shape is outside them; MCF_GEMM_F32_I8=0 forces
  // the FFMA GEMM
  static const bool i8 = [] {
    const char* e = getenv("MCF_GEMM_F32_I8");
    return !(e && e[0] == '0');
  }();
  if (i8) {
    const mcf_status st = mcfr::gemm_f32_i8(trans_a, trans_b, a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
    if (st != MCF_ERR_UNSUPPORTED) return st;
  }
  // short A with a long K and no mask (the 10-class layer's dW: 10 x 1024, K =
  // the batch): split-K FFMA, chunks merged in order
  if (!trans_a && trans_b && !relu_mask && m <= kSkRows && k >= 2 * kSkChunk) {
    const int chunks = (int)((k + kSkChunk - 1) / kSkChunk);
    float* part = static_cast<float*>(mcfr::workspace((std::size_t)chunks * m * n * sizeof(float) + 256, 8));
    if (!part) return mcfr::fail(MCF_ERR_CUDA, "gemm_f32: cannot allocate the split-K workspace");
    const int smem = (int)(m * kSkChunk * sizeof(float));
    if (smem > (48 << 10)) {
      const mcf_status ast = mcfr::ensure_smem_attr<k_gemm_abt_splitk>(kSkRows * kSkChunk * (int)sizeof(float),
                                                                       "gemm_f32: cannot reserve shared memory");
      if (ast != MCF_OK) return ast;
    }
    k_gemm_abt_splitk<<<dim3((unsigned)((n + 7) / 8), (unsigned)chunks), 256, smem, s>>>(a, lda, b, ldb, m, n, k,
                                                                                       part);
    k_splitk_reduce<<<(unsigned)((m * n + 255) / 256), 256, 0, s>>>(part, chunks, m, n, c, ldc);
    mcfr::note_launch();
    mcfr::note_launch();
    return mcfr::check_launch("gemm_f32 split-K kernels");
  }
  // a short K with B's rows contiguous (the 10-class layer's dA, K = 10):
  // the register-resident small-K kernel (bit-identical to the ordered GEMM)
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!trans_b && k >= 1 && k <= kSmallK && n % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && al16(b) && al16(c) &&
      (!relu_mask || al16(relu_mask))) {
    const dim3 grid((unsigned)((n / 4 + 255) / 256), (unsigned)((m + kSmallRows - 1) / kSmallRows));
    if (trans_a) k_gemm_smallk<true><<<grid, 256, 0, s>>>(a, lda, b, ldb, c, ldc, m, n, (int)k, relu_mask);
    else k_gemm_smallk<false><<<grid, 256, 0, s>>>(a, lda, b, ldb, c, ldc, m, n, (int)k, relu_mask);
    mcfr::note_launch();
    return mcfr::check_launch("gemm_f32 small-K kernel");
  }
  // the other shapes outside the int8 path (a dimension below 64): the ordered FFMA GEMM
  return mcf_gemm_f32_ordered(trans_a, trans_b, a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
}

mcf_status mcf_rowsum_f32_fast(const float* g, int64_t rows, int64_t n, float* out, mcf_stream s) {
  if (rows <= 0) return MCF_OK;
  k_rowsum_tree<<<(unsigned)rows, 256, 0, s>>>(g, n, out);
  mcfr::note_launch();
  return mcfr::check_launch("row-sum kernel");
}

}  // extern "C"
