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
      if (KIND == 6) { d[i] = (double)f[i]; f[i] = __int_as_float(__double2hiint(d[i]) + it); }   // F2F.F64.F32 + IADD
      if (KIND == 7) { f[i] = __double2float_rn(d[i]); d[i] = __hiloint2double(__float_as_int(f[i]), it); }  // F2F.F32.F64 + mov
      if (KIND == 8) d[i] = __dmul_rn(d[i], (double)a);
      if (KIND == 9) {
        unsigned u;
        asm volatile("{.reg .pred p; setp.lt.f64 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(u) : "d"(d[i]), "d"(d[(i + 1) & 7]));
        f[i] += __uint_as_float(u);
      }
      if (KIND == 10) {
        p2[i] = __fadd2_rn(p2[i], make_float2(b, a));
      }
      if (KIND == 11) p2[i] = __ffma2_rn(p2[i], make_float2(a, a), p2[(i + 1) & 7]);
      if (KIND == 12) f[i] = f[i] < f[(i + 1) & 7] ? f[(i + 2) & 7] : f[(i + 3) & 7];
      if (KIND == 13) {
        unsigned u = __float_as_uint(f[i]), v = __float_as_uint(f[(i + 1) & 7]);
        asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(u) : "r"(u), "r"(v), "r"(0x7f800000u));
        f[i] = __uint_as_float(u);
      }
      if (KIND == 14) {
        int u = __float_as_int(f[i]), v = __float_as_int(f[(i + 1) & 7]);
        asm volatile("add.s32 %0, %1, %2;" : "=r"(u) : "r"(u), "r"(v));
        f[i] = __int_as_float(u);
      }
      if (KIND == 15) { f[i] = __fadd_rn(f[i], b); p2[i].x = __fadd_rn(p2[i].x, b); d[i] = __dadd_rn(d[i], (double)b); }
      if (KIND == 16) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(f[i]) : "f"(f[i] + 1.0f));
      if (KIND == 17) f[i] = __fdiv_rn(f[(i + 1) & 7] + 3.0f, f[i] + 1.5f);
      if (KIND == 18) { p2[i] = __fadd2_rn(p2[i], make_float2(b, a)); d[i] = __dadd_rn(d[i], (double)b); }
      if (KIND == 19) f[i] = fmaxf(f[i], f[(i + 1) & 7]);
      if (KIND == 20) { f[i] = __fadd_rn(f[i], b); int u = __float_as_int(p2[i].x); asm volatile("add.s32 %0, %1, %2;" : "=r"(u) : "r"(u), "r"(it)); p2[i].x = __int_as_float(u); }
      if (KIND == 21) d[i] = __ddiv_rn(d[(i + 1) & 7] + 3.0, d[i] + 1.5);
      if (KIND == 22) { long long u = __double_as_longlong(d[i]); u += 0x10000000LL; u &= ~0x1fffffffLL; d[i] = __longlong_as_double(u); }
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
                         "DMUL", "DSETP+SEL+FADD", "FADD2 (pairs)", "FFMA2 (pairs)", "FSETP+FSEL", "LOP3", "IADD", "2FADD+1DADD (x3)",
                         "MUFU.RCP", "fdiv_rn f32", "FADD2+DADD (x2)", "FMNMX", "FADD+IADD (x2)", "ddiv_rn", "int64 add+and"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int kind = 0; kind < 23; ++kind) {
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
#define C(n) case n: k<n><<<blocks, threads>>>(of, od, n == 17 || n == 21 ? iters / 16 : iters, 1.0001f, 0.999); break;
        C(11) C(12) C(13) C(14) C(15) C(16) C(17) C(18) C(19) C(20) C(21) C(22)
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * (kind == 17 || kind == 21 ? iters / 16 : iters) * 8;
      if (rep) printf("%-14s %8.2f Tinstr/s  (%.1f lane-ops/clk/SM at %d MHz nominal)\n", names[kind],
                      ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  printf("SMs %d\n", sms);
  return 0;
}
