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
  // outside the int8 path's shapes: the ordered FFMA GEMM (same operands,
  // same optional ReLU mask; small here: k or m is 10)
  return mcf_gemm_f32_ordered(trans_a, trans_b, a, lda, b, ldb, c, ldc, m, n, k, relu_mask, s);
}

mcf_status mcf_rowsum_f32_fast(const float* g, int64_t rows, int64_t n, float* out, mcf_stream s) {
  if (rows <= 0) return MCF_OK;
  k_rowsum_tree<<<(unsigned)rows, 256, 0, s>>>(g, n, out);
  mcfr::note_launch();
  return mcfr::check_launch("row-sum kernel");
}

}  // extern "C"
