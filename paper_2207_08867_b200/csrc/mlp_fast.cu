// mlp_fast.cu -- the MC-MLP backward pass under plan MCF_FAST.
//
// The reference computes the backward products of mc_linear_op in plain
// binary32 (matmul2d, ndarray.hpp:147-165: fl_mul then fl_add, k in order),
// and the reference-order plan reproduces that bit for bit (mlp.cu).  Plan
// MCF_FAST only promises the reference's error level, so there the gradient
// GEMMs are ordinary FP32 GEMMs (cuBLAS SGEMM, FFMA accumulation, no TF32:
// a plain library GEMM) and the bias gradient a tree reduction -- the
// contraction work of the step that is not an MC product.  Shapes the int8
// tensor cores take go through four-digit int8 products instead (binary32
// accuracy, mm_ozaki.cu: gemm_f32_i8).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "mcf_runtime.h"

namespace {

std::mutex g_mu;
std::map<int, cublasHandle_t> g_handles;

cublasHandle_t handle() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  cublasHandle_t& h = g_handles[dev];
  if (!h) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);  // binary32 FFMA, no TF32
  }
  return h;
}

// C[i, j] = mask[i, j] > 0 ? C[i, j] : 0
__global__ void __launch_bounds__(256) k_relu_mask(float* __restrict__ c, const float* __restrict__ mask,
                                                    int64_t m, int64_t n, int64_t ldc) {
  const int64_t total = m * n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    const int64_t i = x / n, j = x - i * n;
    if (!(mask[i * ldc + j] > 0.0f)) c[i * ldc + j] = 0.0f;
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
// optional ReLU mask), FP32 GEMM in cuBLAS order.
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
  cublasHandle_t h = handle();
  if (!h) return mcfr::fail(MCF_ERR_CUDA, "gemm_f32: cannot create a cuBLAS handle");
  cublasSetStream(h, s);
  // row-major C (m x n) is column-major C^T (n x m) = op(B)^T op(A)^T; the
  // row-major operand arrays seen column-major are B^T / A^T (no transpose)
  // or B / A (transposed storage)
  const cublasOperation_t tx = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t ty = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
  const float one = 1.0f, zero = 0.0f;
  const cublasStatus_t st = cublasSgemm(h, tx, ty, (int)n, (int)m, (int)k, &one, b, (int)ldb, a, (int)lda, &zero, c,
                                        (int)ldc);
  if (st != CUBLAS_STATUS_SUCCESS)
    return mcfr::fail(MCF_ERR_CUDA, "gemm_f32: cublasSgemm failed (status " + std::to_string((int)st) + ")");
  mcfr::note_launch();
  if (relu_mask) {
    k_relu_mask<<<mcfr::grid_for(m * n, 256, 8), 256, 0, s>>>(c, relu_mask, m, n, ldc);
    mcfr::note_launch();
  }
  return mcfr::check_launch("gemm_f32 kernels");
}

mcf_status mcf_rowsum_f32_fast(const float* g, int64_t rows, int64_t n, float* out, mcf_stream s) {
  if (rows <= 0) return MCF_OK;
  k_rowsum_tree<<<(unsigned)rows, 256, 0, s>>>(g, n, out);
  mcfr::note_launch();
  return mcfr::check_launch("row-sum kernel");
}

}  // extern "C"
