// acc_bench.cu -- throughput of the compensated MAD bodies in registers only
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2207_08867_b200/csrc/mcf_accum.cuh"
using namespace mcfg;
struct Old9 { static __device__ void mad(double (&acc)[2], const double* a, const double* b) {
  const double p = __dmul_rn(a[0], b[0]); double e; dsum(acc[0], p, acc[0], e); acc[1] = __fma_rn(a[1], b[0], __dadd_rn(acc[1], e)); } };
struct Plain { static __device__ void mad(double (&acc)[2], const double* a, const double* b) { acc[0] = __fma_rn(a[0], b[0], acc[0]); } };
template <class A, int NACC>
__global__ void k(double* out, int iters, double s) {
  double acc[NACC][2]; double a[NACC][2]; double b[4];
  for (int i = 0; i < NACC; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = 0; a[i][0] = s + i; a[i][1] = s * 1e-9 * i; }
  for (int j = 0; j < 4; ++j) b[j] = 1.0 / (j + 3 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) A::mad(acc[i], a[i], &b[i & 3]);
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = -b[j];
  }
  double t = 0; for (int i = 0; i < NACC; ++i) t += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <class A, int NACC>
void run(const char* name, int blocks_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm, threads = 256, iters = 512;
  double* o; cudaMalloc(&o, blocks * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); k<A, NACC><<<blocks, threads>>>(o, iters, 1.0001); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  const double mads = (double)blocks * threads * iters * NACC;
  printf("%-8s nacc=%2d blk/sm=%d: %.3f T MAD/s\n", name, NACC, blocks_per_sm, mads / best / 1e9);
  cudaFree(o);
}
int main() {
  run<Old9, 16>("old9", 2); run<AccT2, 16>("fast6", 2); run<Plain, 16>("dfma", 2);
  run<Old9, 32>("old9", 1); run<AccT2, 32>("fast6", 1);
  run<Old9, 8>("old9", 4); run<AccT2, 8>("fast6", 4);
  return 0;
}
