// pipe_bench.cu -- measured instruction throughput of the pipes the MC
// contractions and the certified elementwise tier can use (FP32 add/fma,
// FP64 add/fma/mul/setp, FP16x2 fma, packed FP32x2 add, binary32 <-> binary64
// conversions), per SM per clock, so rooflines are measured numbers, not
// datasheet ones.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int KIND>
__global__ void k(float* outf, double* outd, int iters, float a, float b) {
  float f[8]; double d[8]; __half2 h[8];
  for (int i = 0; i < 8; ++i) { f[i] = a + i + threadIdx.x; d[i] = b + i + threadIdx.x; h[i] = __floats2half2_rn(a + i, b); }
  const __half2 hb = __floats2half2_rn(b, a);
  float2 p2[8];
  for (int i = 0; i < 8; ++i) p2[i] = make_float2(f[i], a);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) f[i] = __fadd_rn(f[i], b);
      if (KIND == 1) f[i] = __fmaf_rn(f[i], a, f[(i + 1) & 7]);
      if (KIND == 2) d[i] = __dadd_rn(d[i], (double)b);
      if (KIND == 3) d[i] = __fma_rn(d[i], (double)a, d[(i + 1) & 7]);
      if (KIND == 4) h[i] = __hfma2(h[i], hb, h[(i + 1) & 7]);
      if (KIND == 5) f[i] = __fadd_rn(f[i], f[(i + 3) & 7]);
      if (KIND == 6) asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d[i]) : "f"(f[i]));
      if (KIND == 7) asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[i]) : "d"(d[i]));
      if (KIND == 8) d[i] = __dmul_rn(d[i], (double)a);
      if (KIND == 9) {
        unsigned u;
        asm volatile("{.reg .pred p; setp.lt.f64 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(u) : "d"(d[i]), "d"(d[(i + 1) & 7]));
        f[i] += __uint_as_float(u);
      }
      if (KIND == 10) {
        p2[i] = __fadd2_rn(p2[i], make_float2(b, a));
      }
    }
  }
  float s = 0; double t = 0;
  for (int i = 0; i < 8; ++i) { s += f[i] + __low2float(h[i]) + p2[i].x + p2[i].y; t += d[i]; }
  outf[blockIdx.x * blockDim.x + threadIdx.x] = s;
  outd[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float* of; double* od;
  cudaMalloc(&of, blocks * threads * 4); cudaMalloc(&od, blocks * threads * 8);
  const char* names[] = {"FADD", "FFMA", "DADD", "DFMA", "HFMA2", "FADD(reg,reg)", "F2F.F64.F32", "F2F.F32.F64",
                         "DMUL", "DSETP+SEL+FADD", "FADD2 (pairs)"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int kind = 0; kind < 11; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      switch (kind) {
        case 0: k<0><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 1: k<1><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 2: k<2><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 3: k<3><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 4: k<4><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 5: k<5><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 6: k<6><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 7: k<7><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 8: k<8><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 9: k<9><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
        case 10: k<10><<<blocks, threads>>>(of, od, iters, 1.0001f, 0.999); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;
      if (rep) printf("%-14s %8.2f Tinstr/s  (%.1f lane-ops/clk/SM at %d MHz nominal)\n", names[kind],
                      ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  printf("SMs %d\n", sms);
  return 0;
}
