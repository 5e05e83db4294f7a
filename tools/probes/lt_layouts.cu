// Probe: which int8 layouts cuBLASLt accepts on this GPU and how fast (4096^3).
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

int main() {
  cublasLtHandle_t h;
  cublasLtCreate(&h);
  const int64_t M = 4096, N = 4096, K = 4096 * 6;
  int8_t *A, *B;
  int32_t* C;
  cudaMalloc(&A, M * K);
  cudaMalloc(&B, K * N);
  cudaMalloc(&C, M * N * 4);
  cudaMemset(A, 1, M * K);
  cudaMemset(B, 1, K * N);
  void* ws;
  size_t wsb = 64 << 20;
  cudaMalloc(&ws, wsb);
  for (int ta = 0; ta < 2; ++ta)
    for (int tb = 0; tb < 2; ++tb) {
      cublasLtMatmulDesc_t op;
      cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I);
      cublasOperation_t oa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, ob = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
      cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &oa, sizeof(oa));
      cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &ob, sizeof(ob));
      cublasLtMatrixLayout_t la, lb, lc;
      cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, ta ? K : M, ta ? M : K, ta ? K : M);
      cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, tb ? N : K, tb ? K : N, tb ? N : K);
      cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, M, N, M);
      cublasLtMatmulPreference_t pref;
      cublasLtMatmulPreferenceCreate(&pref);
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
      cublasLtMatmulHeuristicResult_t res;
      int found = 0;
      cublasStatus_t st = cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 1, &res, &found);
      float ms = -1;
      if (st == CUBLAS_STATUS_SUCCESS && found) {
        int32_t one = 1, zero = 0;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cublasLtMatmul(h, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res.algo, ws, wsb, 0);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) cublasLtMatmul(h, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res.algo, ws, wsb, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
      }
      printf("transa=%c transb=%c: %s %.3f ms %.0f TOPS\n", ta ? 'T' : 'N', tb ? 'T' : 'N',
             found ? "supported" : "NOT supported", ms, ms > 0 ? 2.0 * M * N * K / ms / 1e9 : 0.0);
    }
  return 0;
}
