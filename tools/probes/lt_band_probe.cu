// lt_band_probe.cu -- time a config-4-sized int8 digit GEMM (C = A^T B, s8 x s8 -> s32,
// the layout of mm_ozaki.cu's gemm_s8) as one cuBLASLt call vs. column bands
// of B (each band's operand slab small enough to stay in L2), and over the
// heuristic's top algorithms.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/lt_band_probe.cu -lcublasLt -o /tmp/ltb
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    auto _e = (x);                                                             \
    if ((int)_e != 0) {                                                        \
      printf("error %d at %s:%d\n", (int)_e, __FILE__, __LINE__);              \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void fill(int8_t* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    p[i] = (int8_t)((h >> 8) & 0xff) >> 1;
  }
}

int main(int argc, char** argv) {
  static int reps = 3;
  if (getenv("REPS")) reps = atoi(getenv("REPS"));
  const long M = argc > 1 ? atol(argv[1]) : 16384, N = argc > 2 ? atol(argv[2]) : 16384,
             K = argc > 3 ? atol(argv[3]) : 21760, LD = argc > 4 ? atol(argv[4]) : K;
  cublasLtHandle_t h;
  CK(cublasLtCreate(&h));
  int8_t *A, *B;
  int* C;
  CK(cudaMalloc(&A, (size_t)M * LD));
  CK(cudaMalloc(&B, (size_t)N * LD));
  CK(cudaMalloc(&C, (size_t)M * N * 4));
  fill<<<1024, 256>>>(A, (size_t)M * LD, 1);
  fill<<<1024, 256>>>(B, (size_t)N * LD, 2);
  size_t wsb = 64u << 20;
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](long bands, int which) -> float {
    const long nb = N / bands;
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I));
    cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
    cublasLtMatrixLayout_t la, lb, lc;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, K, M, LD));
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, K, nb, LD));
    CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, M, nb, M));
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
    cublasLtMatmulHeuristicResult_t res[16];
    int found = 0;
    CK(cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 16, res, &found));
    if (which >= found) return -1.f;
    const int alpha = 1, beta = 0;
    auto go = [&]() {
      for (long b = 0; b < bands; ++b)
        cublasLtMatmul(h, op, &alpha, A, la, B + (size_t)b * nb * LD, lb, &beta, C + (size_t)b * nb * M, lc,
                       C + (size_t)b * nb * M, lc, &res[which].algo, ws, wsb, 0);
    };
    go();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) go();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (which == 0 && bands == 1) printf("heuristic returned %d algorithms\n", found);
    cublasLtMatmulPreferenceDestroy(pref);
    cublasLtMatrixLayoutDestroy(la);
    cublasLtMatrixLayoutDestroy(lb);
    cublasLtMatrixLayoutDestroy(lc);
    cublasLtMatmulDescDestroy(op);
    return ms / reps;
  };
  const int nalg = argc > 5 ? atoi(argv[5]) : 2;
  for (long bands : {1L, 4L, 16L})
    for (int w = 0; w < nalg; ++w) {
      const float ms = run(bands, w);
      if (ms < 0) break;
      printf("M=%ld N=%ld K=%ld ld=%ld bands=%ld algo#%d: %.3f ms  %.0f TOPS\n", M, N, K, LD, bands, w, ms,
             2.0 * M * N * K / ms / 1e9);
    }
  return 0;
}
