// mm_ozaki.cu -- MCF_FAST MC contractions on the INT8 tensor cores.
//
// The reference's mm_mcn (linalg.hpp:138-157) accumulates every output in MC
// arithmetic; its error is set by the nc-component result (2^-51.7
// median / 2^-49.1 max at nc=2 fp32).  On B200 the fastest exact arithmetic
// for a GEMM is the INT8 tensor core (int32 accumulation is exact), so the
// product is computed as an exact integer product by Chinese remaindering
// (the modular integer splitting known as Ozaki scheme II):
//
//   * every row i of A is scaled by 2^-ea[i] and every column j of B by
//     2^-eb[j] (powers of two above twice the line's max |c0 + c1|, exact), so
//     all values lie in (-1/2, 1/2), and rounded to integers
//     A' = round(A 2^pa) (|A'| < 2^(pa-1), error <= 0.51 units) and
//     B' = round(B 2^pb); a binary32 B keeps pb = 48 bits, exact for every
//     element within 2^23 binades of its column's scale (the others are
//     counted per column and their rounding enters that column's bound);
//   * n pairwise coprime moduli m_t <= 256 with M = prod m_t >= 4 K 2^(pa+pb-2)
//     (17 at config 2): for each t one int8 GEMM of the symmetric residues
//     A' mod m_t, B' mod m_t (|r| <= 128, exact int32 sums for K < 2^17) gives
//     C' mod m_t;
//   * C' = sum_t r_t w_t - q M (w_t the CRT weights, q = round(T / M)) is
//     formed exactly: the weights are cut into eight balanced 12-bit slices, so
//     every slice sum T_j = sum_t r_t w_tj and D_j = T_j - q M_j is an exact
//     binary32 integer, and the slices are joined by a binary64 Horner pass
//     whose partial sums are exact while they matter (|C'| <= M/4);
//   * C = C' 2^(ea+eb-pa-pb), split greedily into the binary32 components.
//
// Error per output: A's rounding against the column's sum of |B'| and (MC B) B's
// against the row's sum of |A'| -- the operands' own magnitude sums, taken in
// the exponent pre-passes -- at most K 2^-(pa+1) scaled: 2^-62 at config 2, ~30x
// tighter than the nine-digit splitting this replaced, with 17 int8 GEMMs
// instead of 39 GEMM-equivalents.  Binary32 B elements that do not fit the
// column's 48-bit fixed point are listed per column and the part their
// rounding dropped is added back in the reconstruction.  Outputs whose
// magnitude is not at least 2^50 times their bound (cancellation) and rows /
// columns holding Inf or NaN are listed per row and recomputed by the
// fallback kernel in double-double from the binary32 operands, so every
// output has relative error <= 2^-50 before the final split -- the resolution
// of the reference's own nc=2 result (its measured max is 2^-49.1).
//
// The int8 GEMMs run on the hand-written tcgen05 kernel of tc_gemm.cu (one
// launch over the moduli, int8 residues out of the epilogue); a strided-batched
// cuBLASLt IMMA GEMM (int32 sums, reduced here) is kept behind
// MCF_OZ_GEMM=cublaslt for A/B measurement.  The scaling, residue extraction,
// transposes, CRT reconstruction + split and the cancellation fallback are
// this file's kernels.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "mcf_accum.cuh"
#include "mcf_fast.cuh"
#include "mcf_g2.cuh"
#include "mcf_lit.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace oz {
namespace {

constexpr int kSlab = 32;  // transpose tile of the column kernels

__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// 2^e > 2 m (m >= 0 finite): scaled values lie in (-1/2, 1/2); 0 for m == 0
// or non-finite (those rows / columns go to the fallback list)
__device__ __forceinline__ int exp_above_d(double m) { return m > 0.0 && isfinite(m) ? ilogb(m) + 2 : 0; }

template <int NC>
__device__ __forceinline__ void load_pair(const float* p, double& hi, double& lo, double& mag) {
  if constexpr (NC == 1) {
    hi = (double)p[0];
    lo = 0.0;
    mag = fabs(hi);
  } else {
    const double a = (double)p[0], b = (double)p[1];
    dsum(a, b, hi, lo);
    mag = __dadd_ru(fabs(a), fabs(b));
  }
}

// ---- moduli and CRT constants ------------------------------------------------------------

constexpr int kMaxMod = 22;
// pairwise coprime, largest first (256 = 2^8, 255 = 3 5 17, 253 = 11 23,
// 247 = 13 19, 217 = 7 31, the rest prime); n moduli = the first n
constexpr int kModuli[kMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223,
                                  217, 211, 199, 197, 193, 191, 181, 179, 173, 167, 163};
constexpr int kMinMod = 16;     // instantiated moduli counts: kMinMod .. kMaxMod
constexpr int kSlices = 8;      // balanced 12-bit slices of the CRT weights
constexpr int kSliceBits = 12;
constexpr int kYShift = kSlices * kSliceBits;  // Y = C' / 2^(L - kYShift)
constexpr int kMaxInx = 128;   // listed inexact elements per binary32 B column (more: the column falls back)
constexpr float kMagic = 12582912.0f;  // 1.5 2^23: x + kMagic has x in its low mantissa bits (|x| < 2^22)

struct CrtTab {
  float w[kMaxMod][kSlices];  // slice j of the symmetric CRT weight w_t (weight 2^(L - 12 (j + 1)))
  float mh[kSlices];          // slices of M
  float cq;                   // RN32(2^(L - 12) / M)
  int L;                      // bit length of M
};
__constant__ float c_pw[kMaxMod][6];  // 2^(12 j) mod m_t, symmetric (limb weights of the residue sums)
__constant__ float c_c14[kMaxMod];    // 2^14 mod m_t, symmetric
__constant__ float c_inv[kMaxMod];    // RN32(1 / m_t)
__constant__ float c_mod[kMaxMod];
__constant__ CrtTab c_crt[kMaxMod + 1];  // by moduli count

// ---- host: exact CRT constants (small unsigned big integers) ----

struct Big {  // non-negative, 32-bit words little-endian
  uint32_t w[8] = {};
};
void big_mul(Big& x, uint32_t k) {
  uint64_t c = 0;
  for (auto& v : x.w) {
    const uint64_t t = (uint64_t)v * k + c;
    v = (uint32_t)t;
    c = t >> 32;
  }
}
uint32_t big_divmod(Big& x, uint32_t m) {  // x /= m; returns x mod m
  uint64_t r = 0;
  for (int i = 7; i >= 0; --i) {
    const uint64_t t = (r << 32) | x.w[i];
    x.w[i] = (uint32_t)(t / m);
    r = t % m;
  }
  return (uint32_t)r;
}
int big_bitlen(const Big& x) {
  for (int i = 7; i >= 0; --i)
    if (x.w[i]) return 32 * i + 32 - __builtin_clz(x.w[i]);
  return 0;
}
int big_bit(const Big& x, int b) { return b < 0 || b >= 256 ? 0 : (int)((x.w[b >> 5] >> (b & 31)) & 1u); }
int big_bits(const Big& x, int lo, int cnt) {
  int v = 0;
  for (int i = cnt - 1; i >= 0; --i) v = 2 * v + big_bit(x, lo + i);
  return v;
}
bool big_le(const Big& a, const Big& b) {
  for (int i = 7; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  return true;
}
void big_sub(Big& a, const Big& b) {  // a -= b, b <= a
  int64_t br = 0;
  for (int i = 0; i < 8; ++i) {
    int64_t t = (int64_t)a.w[i] - (int64_t)b.w[i] - br;
    br = t < 0 ? 1 : 0;
    a.w[i] = (uint32_t)(t + (br << 32));
  }
}
double big_double(const Big& x) {
  double d = 0.0;
  for (int i = 7; i >= 0; --i) d = d * 4294967296.0 + (double)x.w[i];
  return d;
}
int modinv(int a, int m) {  // a^-1 mod m (gcd(a, m) = 1)
  int t = 0, nt = 1, r = m, nr = a % m;
  while (nr) {
    const int q = r / nr, t2 = t - q * nt, r2 = r - q * nr;
    t = nt, nt = t2, r = nr, nr = r2;
  }
  return t < 0 ? t + m : t;
}
int sym(int v, int m) {  // symmetric representative of v mod m
  v %= m;
  if (v < 0) v += m;
  return v > m / 2 ? v - m : v;
}
// balanced slices of x (0 <= x < 2^L) at weights 2^(L - 12 (j + 1)), the last
// one rounded: |x - sum_j d_j 2^(L - 12 (j + 1))| <= 2^(L - 12 kSlices - 1);
// |d_j| <= 2^11 for j >= 1, d_0 <= 2^12 (x < 2^(L-1) gives d_0 <= 2^11)
void slices(const Big& x, int L, float* out) {
  int d[kSlices];
  for (int j = 0; j < kSlices; ++j) d[j] = big_bits(x, L - kSliceBits * (j + 1), kSliceBits);
  if (big_bit(x, L - kYShift - 1)) ++d[kSlices - 1];
  for (int j = kSlices - 1; j > 0; --j)
    if (d[j] >= (1 << (kSliceBits - 1))) {
      d[j] -= 1 << kSliceBits;
      ++d[j - 1];
    }
  for (int j = 0; j < kSlices; ++j) out[j] = (float)d[j];
}

struct HostCrt {
  CrtTab tab[kMaxMod + 1];
  double log2m[kMaxMod + 1];
  float pw[kMaxMod][6], c14[kMaxMod], inv[kMaxMod], mod[kMaxMod];
};
const HostCrt& host_crt() {
  static const HostCrt h = [] {
    HostCrt h{};
    for (int t = 0; t < kMaxMod; ++t) {
      const int m = kModuli[t];
      int p = 1 % m;
      for (int j = 0; j < 6; ++j) {
        h.pw[t][j] = (float)sym(p, m);
        for (int b = 0; b < 12; ++b) p = p * 2 % m;
      }
      int p14 = 1;
      for (int b = 0; b < 14; ++b) p14 = p14 * 2 % m;
      h.c14[t] = (float)sym(p14, m);
      h.inv[t] = 1.0f / (float)m;
      h.mod[t] = (float)m;
    }
    for (int n = 1; n <= kMaxMod; ++n) {
      Big M;
      M.w[0] = 1;
      for (int t = 0; t < n; ++t) big_mul(M, (uint32_t)kModuli[t]);
      const int L = big_bitlen(M);
      CrtTab& tb = h.tab[n];
      tb.L = L;
      const double md = big_double(M);
      h.log2m[n] = std::log2(md);
      tb.cq = (float)(std::ldexp(1.0, L - kSliceBits) / md);
      slices(M, L, tb.mh);
      for (int t = 0; t < n; ++t) {
        Big mt = M;
        big_divmod(mt, (uint32_t)kModuli[t]);  // M / m_t
        Big tmp = mt;
        const int inv = modinv((int)big_divmod(tmp, (uint32_t)kModuli[t]), kModuli[t]);
        Big w = mt;
        big_mul(w, (uint32_t)inv);  // w_t = (M / m_t) ((M / m_t)^-1 mod m_t) < M
        Big w2 = w;
        big_mul(w2, 2);
        const bool neg = !big_le(w2, M);  // symmetric: w_t - M when w_t > M / 2
        if (neg) {
          Big d = M;
          big_sub(d, w);
          w = d;
        }
        slices(w, L, tb.w[t]);
        if (neg)
          for (auto& v : tb.w[t]) v = -v;
      }
    }
    return h;
  }();
  return h;
}

mcf_status upload_crt_tables() {
  mcf_status st = MCF_OK;
  mcfr::per_device_once(mcfr::kOnceCrtTables, [&] {
    const HostCrt& h = host_crt();
    if (cudaMemcpyToSymbol(c_pw, h.pw, sizeof(h.pw)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_c14, h.c14, sizeof(h.c14)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_inv, h.inv, sizeof(h.inv)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_mod, h.mod, sizeof(h.mod)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_crt, h.tab, sizeof(h.tab)) != cudaSuccess)
      st = mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot upload the CRT tables");
  });
  return st;
}

// Moduli count and operand precisions of a K-long product.  A binary32 B keeps
// pb = 48 bits; MC operands pa (= pb for an MC B).  Needs |C'| <= K 2^(pa-1)
// 2^(pb-1) <= M / 4 (the reconstruction's margin) and a per-output bound
// K 2^-(pa+1) (scaled) <= 2^-57, i.e. pa >= log2 K + 56; the limbs allow pa <= 73.
struct CrtPlan {
  int n = 0, pa = 0, pb = 0;
};
CrtPlan crt_plan(int64_t k, int ncb) {
  int lk = 0;
  while ((int64_t(1) << lk) < k) ++lk;
  for (int n = kMinMod; n <= kMaxMod; ++n) {
    const double avail = host_crt().log2m[n] - lk;  // >= pa + pb
    int pa, pb;
    if (ncb == 1) {
      pb = 48;
      pa = std::min(73, (int)std::floor(avail - pb));
    } else {
      pa = pb = std::min(73, (int)std::floor(avail / 2));
    }
    if (pa >= lk + 56) return CrtPlan{n, pa, pb};
  }
  return CrtPlan{};
}

// ---- device: residues ----

// 2^v as a binary32 (v in [-126, 127])
__device__ __forceinline__ float pow2f(int v) { return __int_as_float((127 + v) << 23); }

// Six balanced 12-bit limbs of round(x 2^s) for two binary32 values at once
// (x finite; 2^s applied as two exact binary32 products sa sb, so that
// |x 2^s| < 2^72 never overflows): from the top, t_j = rint(r 2^-12j) by
// magic-constant rounding (exact while |r 2^-12j| < 2^22), r -= t_j 2^12j
// (exact: the remainder is a multiple of r's ulp and no larger than r), all
// packed FFMA2 / FADD2 -- no binary64 work.  The last step rounds the
// fraction (error <= 1/2); rem is what is left (nonzero: inexact), scaled the
// input as scaled (zero with x nonzero: underflow, also inexact).  |t_j| <=
// 2^11 for j < 5, |t_5| <= 2^12.
// NL limbs hold |x 2^s| < 2^(12 NL - 1) (4 for a binary32 B's 48 bits; the
// limbs above stay untouched and unused).
template <int NL = 6>
__device__ __forceinline__ void limbs2(float2 x, float sa, float sb, float2 (&l)[6], float2& rem, float2& xs) {
  float2 r = __fmul2_rn(__fmul2_rn(x, make_float2(sa, sa)), make_float2(sb, sb));
  xs = r;
  const float2 mg = make_float2(kMagic, kMagic), nmg = make_float2(-kMagic, -kMagic);
#pragma unroll
  for (int j = NL - 1; j >= 0; --j) {
    const float dn = pow2f(-12 * j), up = -pow2f(12 * j);
    const float2 t = __fadd2_rn(__ffma2_rn(r, make_float2(dn, dn), mg), nmg);
    r = __ffma2_rn(t, make_float2(up, up), r);
    l[j] = t;
  }
  rem = r;
}

// the limbs of X = round(c0 2^s) + round(c1 2^s) (each rounding <= 1/2; c1 = 0
// for NC = 1) for two elements; returns the number of inexact elements
template <int NC, int NL = 6>
__device__ __forceinline__ int limbs_pair(const float (&c0)[2], const float (&c1)[2], float sa, float sb,
                                          float2 (&l)[6]) {
  float2 rem, xs;
  limbs2<NL>(make_float2(c0[0], c0[1]), sa, sb, l, rem, xs);
  int inexact = (rem.x != 0.0f || (xs.x == 0.0f && c0[0] != 0.0f)) + (rem.y != 0.0f || (xs.y == 0.0f && c0[1] != 0.0f));
  if constexpr (NC == 2) {
    float2 l1[6], rem1, xs1;
    limbs2<NL>(make_float2(c1[0], c1[1]), sa, sb, l1, rem1, xs1);
#pragma unroll
    for (int j = 0; j < NL; ++j) l[j] = __fadd2_rn(l[j], l1[j]);  // |sum| <= 2^12 (2^13 for j = 5): exact
    inexact += (rem1.x != 0.0f || (xs1.x == 0.0f && c1[0] != 0.0f)) + (rem1.y != 0.0f || (xs1.y == 0.0f && c1[1] != 0.0f));
  }
  return inexact;
}

// the lowest limb as an integer (X mod 256 is its low byte; |l0| < 2^22)
__device__ __forceinline__ int limb_int(float v) { return __float_as_int(__fadd_rn(v, kMagic)) - 0x4B400000; }

// scale factors 2^(p - e) as two binary32 powers of two
__device__ __forceinline__ void scale_pair(int p, int e, float& sa, float& sb) {
  const int s = p - e, s1 = s < 127 ? s : 127;
  sa = pow2f(s1);
  sb = pow2f(s - s1);
}

// kMagic + (X mod m_t), symmetric, for modulus t >= 1 (odd m_t): the limb sum
// s (|s| <= 127 (2^13 + 5 2^12) < 2^22, exact in binary32, and s + kMagic
// exact) reduced by q = rint(s / m_t) from one FFMA (|s RN(1/m) - s / m| <=
// |s| 2^-24 / m < 1 / (2 m), and s / m is never a half integer for odd m, so
// q is exact); the low byte of the result's bits is the residue as int8.
template <int T>
__device__ __forceinline__ unsigned res_bits(const float (&l)[6]) {
  float s = __fmaf_rn(l[0], c_pw[T][0], kMagic);
#pragma unroll
  for (int j = 1; j < 6; ++j) s = __fmaf_rn(l[j], c_pw[T][j], s);
  const float q = __fsub_rn(__fmaf_rn(__fsub_rn(s, kMagic), c_inv[T], kMagic), kMagic);
  return __float_as_uint(__fmaf_rn(-q, c_mod[T], s));
}

// res_bits for two elements at once: packed FFMA2 / FADD2 with the weights
// as scalar (broadcast) operands, the same roundings per lane -- half the
// issue slots of the scalar form (the residue kernels are issue-bound)
template <int T, int NL = 6>
__device__ __forceinline__ float2 res_bits2(const float2 (&l)[6]) {
  const float2 mg = make_float2(kMagic, kMagic), nmg = make_float2(-kMagic, -kMagic);
  float2 s = __ffma2_rn(l[0], make_float2(c_pw[T][0], c_pw[T][0]), mg);
#pragma unroll
  for (int j = 1; j < NL; ++j) s = __ffma2_rn(l[j], make_float2(c_pw[T][j], c_pw[T][j]), s);
  const float2 q = __fadd2_rn(__ffma2_rn(__fadd2_rn(s, nmg), make_float2(c_inv[T], c_inv[T]), mg), nmg);
  return __ffma2_rn(q, make_float2(-c_mod[T], -c_mod[T]), s);
}

// low bytes of four words -> one word (byte u = word u's low byte)
__device__ __forceinline__ unsigned pack4(unsigned w0, unsigned w1, unsigned w2, unsigned w3) {
  return __byte_perm(__byte_perm(w0, w1, 0x0040), __byte_perm(w2, w3, 0x0040), 0x5410);
}

template <int NMOD, int T = 0, int NL = 6>
__device__ __forceinline__ void residue_words(const float2 (&l01)[6], const float2 (&l23)[6], const int (&l0i)[4],
                                              unsigned (&wd)[NMOD]) {
  if constexpr (T < NMOD) {
    if constexpr (T == 0) {  // m = 256: X mod 256 is the lowest limb's low byte
      wd[0] = pack4((unsigned)l0i[0], (unsigned)l0i[1], (unsigned)l0i[2], (unsigned)l0i[3]);
    } else {
      const float2 a = res_bits2<T, NL>(l01), b = res_bits2<T, NL>(l23);
      wd[T] = pack4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(b.x), __float_as_uint(b.y));
    }
    residue_words<NMOD, T + 1, NL>(l01, l23, l0i, wd);
  }
}

// A (rows x k, NC comps) -> residue planes [t][i][kp] (int8, zero for k >= K
// and for non-finite elements; those rows are listed anyway).  Each thread
// makes 4 consecutive k (one 32-bit store per plane); rows strided over y.
template <int NC, int NMOD>
__global__ void __launch_bounds__(256) k_res_rows(const float* __restrict__ a, int64_t rows, int64_t k, int64_t kp,
                                                   int pa, const int* __restrict__ e, int8_t* __restrict__ out) {
  const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k0 >= kp) return;
  const int64_t plane = rows * kp;
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    float sa, sb;
    scale_pair(pa, e[i], sa, sb);
    float c[NC][4];
    const float* ar = a + i * k * NC;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bool fin = k0 + u < k;
#pragma unroll
      for (int q = 0; q < NC; ++q) c[q][u] = fin ? __ldg(ar + (k0 + u) * NC + q) : 0.0f;
#pragma unroll
      for (int q = 0; q < NC; ++q) fin = fin && isfinite(c[q][u]);
      if (!fin)
#pragma unroll
        for (int q = 0; q < NC; ++q) c[q][u] = 0.0f;
    }
    float2 l01[6], l23[6];
    {
      const float a0[2] = {c[0][0], c[0][1]}, a1[2] = {c[NC - 1][0], c[NC - 1][1]};
      const float b0[2] = {c[0][2], c[0][3]}, b1[2] = {c[NC - 1][2], c[NC - 1][3]};
      limbs_pair<NC>(a0, a1, sa, sb, l01);
      limbs_pair<NC>(b0, b1, sa, sb, l23);
    }
    const int l0i[4] = {limb_int(l01[0].x), limb_int(l01[0].y), limb_int(l23[0].x), limb_int(l23[0].y)};
    unsigned wd[NMOD];
    residue_words<NMOD>(l01, l23, l0i, wd);
    unsigned* o = reinterpret_cast<unsigned*>(out + i * kp + k0);
    if ((uint64_t)NMOD * (uint64_t)plane < (uint64_t(1) << 33)) {  // word offsets of the planes fit 32 bits
      const unsigned pw = (unsigned)(plane >> 2);
#pragma unroll
      for (int t = 0; t < NMOD; ++t) o[(unsigned)t * pw] = wd[t];
    } else {
#pragma unroll
      for (int t = 0; t < NMOD; ++t) o[(int64_t)t * (plane >> 2)] = wd[t];
    }
  }
}

// B (k x n, NC comps, row stride ldb elements) -> residue planes transposed,
// [t][j][kp] (K contiguous per column: the int8 GEMM's TN layout), and
// bt[j, k, :] = B[k, j, :] (binary32, for the fallback list); per column the
// count of elements whose rounding to pb bits is inexact (cinx).  CTA tile
// 32 k x 32 j: lane = column (coalesced loads along n), each thread four
// consecutive k packed into one 32-bit word per modulus; shared rows padded to
// 9 words so the lanes' stores hit distinct banks.
// binary32 B elements that do not fit pb bits at the column's scale 2^sh (or
// underflow it): list (k, what the rounding dropped) so that the
// reconstruction adds A[i, k] x it back.  The scaled value is exact in
// binary64 and B' is its nearest integer, ties to even, as the limbs'.  Out of
// line: a narrow-range B never gets here.
static __device__ __noinline__ void list_inexact(float c0, float c1, float c2, float c3, int sh, int kbase,
                                                 int* __restrict__ cnt, int* __restrict__ lk,
                                                 double* __restrict__ lr) {
  const float c[4] = {c0, c1, c2, c3};
  const double sc = pow2d(sh);
  for (int u = 0; u < 4; ++u) {
    const double xd = __dmul_rn((double)c[u], sc);
    const double rem = __dsub_rn(xd, rint(xd));
    if (rem != 0.0) {
      const int slot = atomicAdd(cnt, 1);
      if (slot < kMaxInx) {
        lk[slot] = kbase + u;
        lr[slot] = rem;
      }
    }
  }
}

template <int NC, int NMOD>
__global__ void __launch_bounds__(256, 4) k_res_cols(const float* __restrict__ b, int64_t n, int64_t ldb, int64_t k,
                                                   int64_t kp, int64_t np, int pb, const int* __restrict__ e,
                                                   int8_t* __restrict__ out, float* __restrict__ bt,
                                                   int* __restrict__ cinx, int* __restrict__ clk,
                                                   double* __restrict__ clr) {
  __shared__ unsigned dg[NMOD][kSlab][kSlab / 4 + 1];  // [t][j][k / 4]
  __shared__ float tv[kSlab][kSlab * NC + 1];          // [j][k * NC + c]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps x 4 k each
  const int64_t k0 = (int64_t)blockIdx.y * kSlab, j0 = (int64_t)blockIdx.x * kSlab;
  const int64_t j = j0 + tx;
  float sa = 1.0f, sb = 1.0f;
  if (j < n) scale_pair(pb, e[j], sa, sb);
  float c[NC][4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int kk = ty * 4 + u;
    const int64_t gk = k0 + kk;
    bool fin = gk < k && j < n;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      c[q][u] = fin ? b[(gk * ldb + j) * NC + q] : 0.0f;
      tv[tx][kk * NC + q] = c[q][u];
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) fin = fin && isfinite(c[q][u]);
    if (!fin)
#pragma unroll
      for (int q = 0; q < NC; ++q) c[q][u] = 0.0f;
  }
  // a binary32 B keeps pb = 48 bits (crt_plan): four 12-bit limbs; an MC B up to 73: six
  constexpr int NL = NC == 1 ? 4 : 6;
  float2 l01[6], l23[6];
  int inexact;
  {
    const float a0[2] = {c[0][0], c[0][1]}, a1[2] = {c[NC - 1][0], c[NC - 1][1]};
    const float b0[2] = {c[0][2], c[0][3]}, b1[2] = {c[NC - 1][2], c[NC - 1][3]};
    inexact = limbs_pair<NC, NL>(a0, a1, sa, sb, l01) + limbs_pair<NC, NL>(b0, b1, sa, sb, l23);
  }
  const int l0i[4] = {limb_int(l01[0].x), limb_int(l01[0].y), limb_int(l23[0].x), limb_int(l23[0].y)};
  if (inexact && j < n) {
    if constexpr (NC == 1) {
      list_inexact(c[0][0], c[0][1], c[0][2], c[0][3], pb - e[j], (int)(k0 + ty * 4), cinx + j, clk + j * kMaxInx,
                   clr + j * kMaxInx);
    } else {
      atomicAdd(cinx + j, inexact);
    }
  }
  unsigned wd[NMOD];
  residue_words<NMOD, 0, NL>(l01, l23, l0i, wd);
#pragma unroll
  for (int t = 0; t < NMOD; ++t) dg[t][tx][ty] = wd[t];
  __syncthreads();
  // residue rows: thread (jj = tid / 8, part = tid % 8) writes 4 bytes of
  // column j0 + jj's 32-k run in every plane (the planes a 32-bit word offset
  // apart: one address add per store) and the same four k of the transposed
  // binary32 copy (one 16-byte store when the run is whole and aligned)
  const int jj = threadIdx.x >> 3, part = threadIdx.x & 7;
  const int64_t gj = j0 + jj;
  if (gj >= n) return;
  unsigned* dst = reinterpret_cast<unsigned*>(out + gj * kp + k0 + part * 4);
  if ((uint64_t)NMOD * (uint64_t)np * (uint64_t)kp < (uint64_t(1) << 33)) {
    const unsigned pw = (unsigned)((np * kp) >> 2);  // plane stride in words
#pragma unroll
    for (int t = 0; t < NMOD; ++t) dst[(unsigned)t * pw] = dg[t][jj][part];
  } else {
#pragma unroll
    for (int t = 0; t < NMOD; ++t) dst[(int64_t)t * ((np * kp) >> 2)] = dg[t][jj][part];
  }
  const int64_t gk = k0 + part * 4;
  float* bo = bt + (gj * k + gk) * NC;
  const float* tr = &tv[jj][part * 4 * NC];
  if (gk + 4 <= k && (reinterpret_cast<uintptr_t>(bo) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < NC; ++q)
      reinterpret_cast<float4*>(bo)[q] = make_float4(tr[4 * q], tr[4 * q + 1], tr[4 * q + 2], tr[4 * q + 3]);
  } else {
    for (int u = 0; u < 4 * NC; ++u)
      if (gk + u / NC < k) bo[u] = tr[u];
  }
}

// ulp exponent of a binary32 (subnormals: -149); a nonzero c with
// ulp_exp(c) + s >= 0 is an integer after scaling by 2^s
__device__ __forceinline__ int ulp_exp(float c) {
  const int eb = (__float_as_int(c) >> 23) & 0xff;
  return (eb > 0 ? eb : 1) - 150;
}

// row exponents of A (rows x k, NC comps): warp per row, max of |c0| + |c1|;
// flags nf[r]: bit 0 a non-finite element, bit 1 some c0 + c1 is not one
// binary64, bit 2 (NC = 2) some nonzero c0 is not an integer at the scale
// 2^(p - e) (then both components may round: 1 unit per element instead of
// 1/2 in the error bound)
// rth[r] = cb (sum_k |A'_rk| bound): the sum of |c0| + |c1| rounded up, at the
// scale 2^(p - e), plus half a unit per element for the roundings
template <int NC>
__global__ void __launch_bounds__(256) k_rowexp(const float* __restrict__ a, int64_t rows, int64_t k, int p,
                                                 int* __restrict__ e, int* __restrict__ nf, double cb,
                                                 float* __restrict__ rth) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double m = 0.0;
  float sum = 0.0f;  // binary32, every add rounded up (the FMA pipe is idle here): an upper bound
  bool bad = false, split = false;
  int umin = 1 << 20;
  for (int64_t t = lane; t < k; t += 32) {  // (unrolling by eight measured slower: 34 -> 36 us)
    double hi, lo, mag;
    load_pair<NC>(a + (r * k + t) * NC, hi, lo, mag);
    bad |= !isfinite(mag);
    split |= lo != 0.0;
    m = fmax(m, mag);
    const float c0 = a[(r * k + t) * NC];
    sum = __fadd_ru(sum, NC == 2 ? __fadd_ru(fabsf(c0), fabsf(a[(r * k + t) * NC + NC - 1])) : fabsf(c0));
    if (NC == 2 && c0 != 0.0f) umin = min(umin, ulp_exp(c0));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    sum = __fadd_ru(sum, __shfl_xor_sync(0xffffffffu, sum, off));
    umin = min(umin, __shfl_xor_sync(0xffffffffu, umin, off));
  }
  bad = __any_sync(0xffffffffu, bad);
  split = __any_sync(0xffffffffu, split);
  if (lane == 0) {
    const int ex = exp_above_d(m);
    e[r] = ex;
    rth[r] = __double2float_ru(__dmul_ru(__fma_ru((double)sum, pow2d(p - ex), 0.5 * (double)k), cb));
    nf[r] = (bad ? 1 : 0) | (split ? 2 : 0) | (NC == 2 && umin + p - ex < 0 ? 4 : 0);
  }
}

// column maxima of B (k x n, NC comps, row stride ldb elements): slabs of 64
// rows, atomicMax on the binary64 bit pattern (monotone for non-negative
// values; cm starts at 0); cu = the column's least ulp exponent of a nonzero
// c0 (NC = 2; starts at INT_MAX)
template <int NC>
__global__ void __launch_bounds__(256) k_colmax(const float* __restrict__ b, int64_t k, int64_t n, int64_t ldb,
                                                 unsigned long long* __restrict__ cm, int* __restrict__ nf,
                                                 int* __restrict__ cu, float* __restrict__ csum) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t t0 = (int64_t)blockIdx.y * 64, t1 = t0 + 64 < k ? t0 + 64 : k;
  double m = 0.0;
  float sum = 0.0f;  // as k_rowexp's
  bool bad = false, split = false;
  int umin = 1 << 20;
  for (int64_t t = t0; t < t1; ++t) {  // (unrolling by eight measured slower: 17 -> 28 us)
    double hi, lo, mag;
    load_pair<NC>(b + (t * ldb + j) * NC, hi, lo, mag);
    bad |= !isfinite(mag);
    split |= lo != 0.0;
    m = fmax(m, mag);
    const float c0 = b[(t * ldb + j) * NC];
    sum = __fadd_ru(sum, NC == 2 ? __fadd_ru(fabsf(c0), fabsf(b[(t * ldb + j) * NC + NC - 1])) : fabsf(c0));
    if (NC == 2 && c0 != 0.0f) umin = min(umin, ulp_exp(c0));
  }
  if (m > 0.0) atomicMax(cm + j, (unsigned long long)__double_as_longlong(m));
  if (sum > 0.0f) atomicAdd(csum + j, sum);  // slab sums rounded up; the atomic adds to nearest (k_colexp pads)
  if (NC == 2 && umin < (1 << 20)) atomicMin(cu + j, umin);
  // bit 0: a non-finite element; bit 1: some c0 + c1 is not one binary64
  if (bad || split) atomicOr(nf + j, (bad ? 1 : 0) | (split ? 2 : 0));
}

// column exponents; flag bit 2 (MC B) as k_rowexp's at the scale 2^(p - e)
// cth[j] = ca (sum_k |B'_kj| bound) as k_rowexp's rth (the 2^-13 covers the
// round-to-nearest binary32 atomic adds of at most 2^10 slab sums)
__global__ void __launch_bounds__(256) k_colexp(const unsigned long long* __restrict__ cm, int64_t n, int p,
                                                 const int* __restrict__ cu, int* __restrict__ e,
                                                 int* __restrict__ nf, const float* __restrict__ csum, int64_t k,
                                                 double ca, float* __restrict__ cth) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int ex = exp_above_d(__longlong_as_double((long long)cm[j]));
  e[j] = ex;
  cth[j] = __double2float_ru(__dmul_ru(__fma_ru(__dmul_ru((double)csum[j], 1.0 + 0x1p-13), pow2d(p - ex), 0.5 * (double)k), ca));
  if (cu && cu[j] + p - ex < 0) nf[j] |= 4;
}

// binary32 B, after the residues have counted each column's inexact elements:
// a listed column (1 .. kMaxInx of them) gets 1.3 units per element (A's
// rounding against the part added back, an underflowed scaled value) and a
// negative sign, which tells k_crt8 to apply its list; a column with more
// than the list holds gets an infinite threshold (all of it falls back)
__global__ void __launch_bounds__(256) k_colfin(const int* __restrict__ cinx, int64_t n, float unit,
                                                 float* __restrict__ cth) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int c = cinx[j];
  if (c > kMaxInx) cth[j] = INFINITY;
  else if (c > 0) cth[j] = -__fadd_ru(cth[j], __fmul_ru(unit, (float)c));
}

// Optional fused epilogue of an MC-MLP layer (mc_linear_op, autodiff.hpp:265-
// 268, then Tape::relu): z = the product's two components, r = add_mcn(z,
// bias[i]) (mc_ops.hpp:440-446; bias is MC nc=2 per output row), h =
// approx(r); h and act = relu ? max(h, 0) : h are written instead of z.
struct Epilogue {
  const float* bias = nullptr;  // (m, 2); null: write the product's components
  float* h = nullptr;
  float* act = nullptr;  // optional
  int relu = 0;
};

__device__ __forceinline__ void emit(const double (&v)[2], int64_t i, int64_t j, float* out, int64_t ldo,
                                     const Epilogue& ep) {
  if (!ep.bias) {
    split_out<float, 2, 2>(v, out + (i * ldo + j) * 2);
    return;
  }
  float z[2], b[2], r[2];
  split_out<float, 2, 2>(v, z);
  b[0] = ep.bias[i * 2];
  b[1] = ep.bias[i * 2 + 1];
  // certified shortcut first (mcf_g2.cuh), then the register path, then the literal one
  if (!g2::add<g2::QF32>(z[0], z[1], b[0], b[1], r[0], r[1]) && !fast::add<PB32, 2>(z, b, r))
    lit::add<PB32>(z, 2, b, 2, r, 2);
  const float hv = fast::approx<PB32, 2>(r);
  ep.h[i * ldo + j] = hv;
  if (ep.act) ep.act[i * ldo + j] = ep.relu ? (hv > 0.0f ? hv : 0.0f) : hv;  // Tape::relu, autodiff.hpp:134
}

// fallback thresholds in units of Y = C' / 2^(L-96): 2^50 x the per-output
// error bound.  The roundings are bounded with the operands' own magnitude
// sums, not K times the largest element: A's rounding of row i against column
// j costs at most 0.51 sum_k |B'_kj| (cth[j], from the column sums of
// k_colmax), B's at most 0.51 sum_k |A'_ik| (rth[i], k_rowexp); each doubles
// for a row / MC column whose leading components are not integers at the
// scale (flag bit 2: both components round).  A binary32 B rounds only its
// counted inexact elements: k_crt8 adds their dropped parts back (CORRECTED;
// the 1.3 units left per element are already in cth, k_colfin), the int32-plane
// kernel k_crt charges the smaller of inexact * count and rth[i].  Operands
// with a wide dynamic range (config 0's 2^U(-8,8) magnitudes, heavy tails)
// have sums far below K maxima, and far fewer outputs fall back.
struct Thresholds {
  float base, inexact;    // base: the product of two roundings (K 1.1 units) + the CRT tail
  const float* cth;
  const float* rth;
  int mcb;                // B is MC (both operands round every element)
  // binary32, every operation rounded up; the caller compares with |Y| rounded down.
  // CORRECTED: the dropped parts of the inexact elements have been added back
  // (k_crt8); what is left per element -- A's rounding against it (<= 0.26) and an
  // underflowed scaled value (far below a unit) -- is already in ca (k_colfin)
  template <bool CORRECTED = false>
  __device__ __forceinline__ float at(int rowflags, int colflags, int inx, float ca, float rb) const {
    float t = __fadd_ru(base, (rowflags & 4) ? __fadd_ru(ca, ca) : ca);
    if (mcb) t = __fadd_ru(t, (colflags & 4) ? __fadd_ru(rb, rb) : rb);
    else if (!CORRECTED && inx) t = __fadd_ru(t, fminf(__fmul_ru(inexact, (float)inx), rb));
    return t;
  }
};

// C mod m_t (symmetric, |r| <= m_t / 2 + 1/2) of an int32 GEMM sum C (|C| <=
// K 2^14): C = ch 2^14 + cl (cl balanced), s = ch (2^14 mod m_t) + cl is an
// exact binary32 integer (|s| < 2^21 for K <= 2^14; below 2^24 for K < 2^17
// with BIG, which reduces twice), then one rounded quotient as in res_bits.
template <bool BIG>
__device__ __forceinline__ float mod_c(int c, int t) {
  const int cl = ((c + 8192) & 16383) - 8192, ch = (c - cl) >> 14;
  const float fl = __fsub_rn(__int_as_float(cl + 0x4B400000), kMagic);
  const float fh = __fsub_rn(__int_as_float(ch + 0x4B400000), kMagic);
  float s = __fmaf_rn(fh, c_c14[t], fl);
  if constexpr (BIG) {
    const float q0 = __fsub_rn(__fmaf_rn(s, c_inv[t], kMagic), kMagic);
    s = __fmaf_rn(-q0, c_mod[t], s);  // |s| <= 2 m
  }
  const float q = __fsub_rn(__fmaf_rn(s, c_inv[t], kMagic), kMagic);
  return __fmaf_rn(-q, c_mod[t], s);
}

// CRT reconstruction of C' from the NMOD int32 GEMM planes cq[t][i][np]
// (C' mod m_t), scaled back, split into two binary32 components written with
// row stride ldo; ill-conditioned / non-finite outputs are listed per row
// (rlist[i * n + slot] = j, rcnt[i] entries) for the fallback.
//   T_j = sum_t r_t w_tj  (|T_j| <= 22 128 2^11 < 2^22.5: exact binary32 sums)
//   q   = rint((T_0 + T_1 2^-12) 2^(L-12) / M)   (error < 2^-10; |C'/M| <= 1/4)
//   D_j = T_j - q M_j     (exact, |D_j| < 2^23.5)
//   Y   = sum_j D_j 2^(12 (7 - j)) = C' / 2^(L-96) + tail (binary64 Horner:
//         partial sums < 2^53 exact while the later terms can still cancel them)
// Four consecutive columns per thread (16-byte plane loads; np % 16 == 0).
template <int NMOD, bool BIG>
__global__ void __launch_bounds__(256) k_crt(const int* __restrict__ cq, int64_t m, int64_t n, int64_t np,
                                             const int* __restrict__ ea, const int* __restrict__ eb,
                                             const int* __restrict__ rnf, const int* __restrict__ cnf,
                                             const int* __restrict__ cinx, Thresholds th, int sexp,
                                             float* __restrict__ out, int64_t ldo, int* __restrict__ rlist,
                                             int* __restrict__ rcnt, Epilogue ep) {
  const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (j0 >= n) return;
  const int64_t plane = m * np;
  int fj[4], cfj[4], inx[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    fj[u] = j0 + u < n ? eb[j0 + u] : 0;
    cfj[u] = j0 + u < n ? cnf[j0 + u] : 0;
    inx[u] = cinx && j0 + u < n ? cinx[j0 + u] : 0;
  }
  for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
    const int64_t off = i * np + j0;
    float T[4][kSlices];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < kSlices; ++j) T[u][j] = 0.0f;
#pragma unroll
    for (int t = 0; t < NMOD; ++t) {
      const int4 v = __ldcs(reinterpret_cast<const int4*>(cq + t * plane + off));
      const int c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // m = 256: the balanced low byte
        const float r = t == 0 ? __fsub_rn(__int_as_float((((c[u] + 128) & 255) - 128) + 0x4B400000), kMagic)
                               : mod_c<BIG>(c[u], t);
#pragma unroll
        for (int j = 0; j < kSlices; ++j) T[u][j] = __fmaf_rn(r, c_crt[NMOD].w[t][j], T[u][j]);
      }
    }
    const int ei = ea[i], fi = rnf[i];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u;
      if (j >= n) break;
      const float u0 = __fmaf_rn(T[u][1], 0x1p-12f, T[u][0]);
      const float q = __fsub_rn(__fmaf_rn(u0, c_crt[NMOD].cq, kMagic), kMagic);
      double y = (double)__fmaf_rn(-q, c_crt[NMOD].mh[0], T[u][0]);
#pragma unroll
      for (int s = 1; s < kSlices; ++s) y = __fma_rn(y, 4096.0, (double)__fmaf_rn(-q, c_crt[NMOD].mh[s], T[u][s]));
      if (((fi | cfj[u]) & 1) || !(__double2float_rd(fabs(y)) >= th.at(fi, cfj[u], inx[u], fabsf(th.cth[j0 + u]), th.rth[i]))) {
        rlist[i * n + atomicAdd(rcnt + i, 1)] = (int)j;
        continue;
      }
      const double v[2] = {__dmul_rn(y, pow2d(sexp + ei + fj[u])), 0.0};
      emit(v, i, j, out, ldo, ep);
    }
  }
}


// k_crt on residues the tcgen05 GEMM's epilogue already reduced (int8 planes
// rq[t][i][ldr], tc_gemm.cu).  One row per thread-block row: thread =
// (row i, four columns), no loop over rows, so the 17 independent 32-bit
// plane loads of many rows are in flight per SM (the r02b capture of the
// row-looping version was latency-bound: 0.94 eligible warps per scheduler);
// the slice sums are packed FFMA2 over column pairs with the weights as
// scalar operands; the two components of the four outputs leave as two
// 16-byte stores.
// sum over a column's listed inexact elements of A[i, k] x (what B's rounding
// dropped); out of line: no column of a narrow-range B lists any
static __device__ __noinline__ double inexact_corr(const float* __restrict__ arow, int nca,
                                                   const int* __restrict__ lk, const double* __restrict__ lr,
                                                   int cnt) {
  double corr = 0.0;
  for (int sl = 0; sl < cnt; ++sl) {
    const float* ap = arow + (int64_t)lk[sl] * nca;
    const double av = nca == 2 ? __dadd_rn((double)ap[0], (double)ap[1]) : (double)ap[0];
    corr = __fma_rn(isfinite(av) ? av : 0.0, lr[sl], corr);
  }
  return corr;
}

#ifndef MCF_CRT8_CTAS
#define MCF_CRT8_CTAS 4
#endif
template <int NMOD>
__global__ void __launch_bounds__(256, MCF_CRT8_CTAS) k_crt8(const int8_t* __restrict__ rq, int64_t m, int64_t n, int64_t ldr,
                                                 const int* __restrict__ ea, const int* __restrict__ eb,
                                                 const int* __restrict__ rnf, const int* __restrict__ cnf,
                                                 const int* __restrict__ cinx, Thresholds th, int sexp,
                                                 float* __restrict__ out, int64_t ldo, int* __restrict__ rlist,
                                                 int* __restrict__ rcnt, Epilogue ep, const float* __restrict__ a,
                                                 int nca, int64_t k, const int* __restrict__ clk,
                                                 const double* __restrict__ clr, double ycorr) {
  const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t i = blockIdx.y;
  if (j0 >= n) return;
  const int64_t plane = m * ldr, off = i * ldr + j0;
  unsigned wv[NMOD];
  const unsigned* rw = reinterpret_cast<const unsigned*>(rq + off);
  if ((uint64_t)NMOD * (uint64_t)plane < (uint64_t(1) << 33)) {  // word offsets of the planes fit 32 bits
    const unsigned pw = (unsigned)(plane >> 2);
#pragma unroll
    for (int t = 0; t < NMOD; ++t) wv[t] = __ldcs(rw + (unsigned)t * pw);
  } else {
#pragma unroll
    for (int t = 0; t < NMOD; ++t) wv[t] = __ldcs(rw + (int64_t)t * (plane >> 2));
  }
  float2 T[2][kSlices];  // [column pair][slice] = (column 2p, column 2p + 1)
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < kSlices; ++j) T[h][j] = make_float2(0.0f, 0.0f);
  const float2 off2 = make_float2(-(kMagic + 128.0f), -(kMagic + 128.0f));
#pragma unroll
  for (int t = 0; t < NMOD; ++t) {
    // byte u of the word is r + 128 after flipping its top bit; one PRMT puts
    // it under kMagic's upper bytes (the float kMagic + 128 + r), one FADD2
    // per pair takes the offset off (exact)
    const unsigned x = wv[t] ^ 0x80808080u;
    const float2 r01 = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(x, 0x4B400000u, 0x7650)),
                                              __uint_as_float(__byte_perm(x, 0x4B400000u, 0x7651))), off2);
    const float2 r23 = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(x, 0x4B400000u, 0x7652)),
                                              __uint_as_float(__byte_perm(x, 0x4B400000u, 0x7653))), off2);
#pragma unroll
    for (int j = 0; j < kSlices; ++j) {
      const float c = c_crt[NMOD].w[t][j];
      T[0][j] = __ffma2_rn(r01, make_float2(c, c), T[0][j]);
      T[1][j] = __ffma2_rn(r23, make_float2(c, c), T[1][j]);
    }
  }
  const int ei = ea[i], fi = rnf[i];
  const float rthi = th.rth[i];
  float res[4][2];
  bool done[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t j = j0 + u;
    done[u] = false;
    res[u][0] = res[u][1] = 0.0f;
    if (j >= n) continue;
    float Tu[kSlices];
#pragma unroll
    for (int sl = 0; sl < kSlices; ++sl) Tu[sl] = (u & 1) ? T[u >> 1][sl].y : T[u >> 1][sl].x;
    const float u0 = __fmaf_rn(Tu[1], 0x1p-12f, Tu[0]);
    const float q = __fsub_rn(__fmaf_rn(u0, c_crt[NMOD].cq, kMagic), kMagic);
    double y = (double)__fmaf_rn(-q, c_crt[NMOD].mh[0], Tu[0]);
#pragma unroll
    for (int sl = 1; sl < kSlices; ++sl) y = __fma_rn(y, 4096.0, (double)__fmaf_rn(-q, c_crt[NMOD].mh[sl], Tu[sl]));
    const int fc = cnf[j];
    float tc = th.cth[j];
    if (tc < 0.0f) {
      // the column lists inexact elements (k_colfin marks it by the sign): add
      // A[i, k] x (what B's rounding dropped) back, in units of Y (ycorr =
      // 2^(pa + 96 - L); binary64 is ample: the terms are below 2^-45 of the
      // bound's scale)
      y = __fma_rn(inexact_corr(a + i * k * nca, nca, clk + j * kMaxInx, clr + j * kMaxInx, cinx[j]),
                   __dmul_rn(ycorr, pow2d(-ei)), y);
      tc = -tc;
    }
    if (((fi | fc) & 1) || !(__double2float_rd(fabs(y)) >= th.template at<true>(fi, fc, 0, tc, rthi))) {
      rlist[i * n + atomicAdd(rcnt + i, 1)] = (int)j;
      done[u] = true;  // the fallback writes it
      continue;
    }
    const double yv = __dmul_rn(y, pow2d(sexp + ei + eb[j]));
    if (ep.bias) {
      const double v[2] = {yv, 0.0};
      emit(v, i, j, out, ldo, ep);
      done[u] = true;
    } else {
      // the greedy split of a binary64 (split_out of (yv, 0) without the
      // double-double steps): c0 = RN32(yv), c1 = RN32(yv - c0), the
      // difference exact
      res[u][0] = __double2float_rn(yv);
      res[u][1] = __double2float_rn(__dsub_rn(yv, (double)res[u][0]));
    }
  }
  if (ep.bias) return;
  float* o = out + (i * ldo + j0) * 2;
  if (j0 + 3 < n && !(done[0] | done[1] | done[2] | done[3]) && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
    reinterpret_cast<float4*>(o)[0] = make_float4(res[0][0], res[0][1], res[1][0], res[1][1]);
    reinterpret_cast<float4*>(o)[1] = make_float4(res[2][0], res[2][1], res[3][0], res[3][1]);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u < n && !done[u]) {
        o[2 * u] = res[u][0];
        o[2 * u + 1] = res[u][1];
      }
  }
}

// the listed outputs: a CTA per row.  The CTA stages its row of A in shared
// memory (SMEM; rows too long for it read A through L1).  A row lists few
// outputs (config 2: 3.6 on average), so each listed output's k range is cut
// into G segments (G a power of two with cnt G <= 8 items, spread over the
// CTA's warps; G = 1 when the row
// lists 5 or more) and every warp takes one (output, segment) item: more
// loads in flight per SM, which is what bounds this latency-bound kernel.
// Each lane streams its k's of the column with eight loads in flight.
// A row whose every c0 + c1 is one binary64 is staged as those sums (same
// bytes; three FP64-pipe instructions per k fewer in the loops: config 2's
// launch 123.7 -> 112.4 us under ncu on B200, cold caches).
// Products of binary32 components are exact in binary64; each lane keeps
// eight double-doubles (k = lane + 32 (8 r + u) goes to accumulator u: two_sum
// into S, errors into C), merged in a fixed order, across the lanes by an xor
// butterfly, and across the segments in segment order through shared memory:
// deterministic (G depends only on the row's own list).
template <int NCA, int NCB, bool SMEM>
__global__ void __launch_bounds__(256) k_fallback(const float* __restrict__ a, const float* __restrict__ bt,
                                                  int64_t n, int64_t k, const int* __restrict__ rlist,
                                                  const int* __restrict__ rcnt, const int* __restrict__ rnf,
                                                  const int* __restrict__ cnf, float* __restrict__ out,
                                                  int64_t ldo, Epilogue ep) {
  extern __shared__ __align__(16) float arow[];
  __shared__ double2 part[8][8];
  const int64_t i = blockIdx.x;
  const int cnt = rcnt[i];
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const float* ag = a + i * k * NCA;
  // every c0 + c1 of the row one binary64 (and B single-component): one
  // two_prod per k instead of a two_sum per component product
  const bool rpair = NCA == 2 && !(rnf[i] & 2);
  // such a row is staged as its binary64 sums c0 + c1 (exact; same bytes)
  const bool dstage = SMEM && rpair;
  double* ad = reinterpret_cast<double*>(arow);
  if constexpr (SMEM) {
    // 16-byte loads, eight in flight per thread before the stores
    const int64_t nf = k * NCA;
    if ((reinterpret_cast<uintptr_t>(ag) & 15) == 0) {
      const int64_t n4 = nf / 4;
      const float4* a4 = reinterpret_cast<const float4*>(ag);
      float4* s4 = reinterpret_cast<float4*>(arow);
      for (int64_t t0 = threadIdx.x; t0 < n4; t0 += 8 * blockDim.x) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t0 + u * blockDim.x < n4) v[u] = __ldg(a4 + t0 + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t0 + u * blockDim.x < n4) {
            if (dstage)
              reinterpret_cast<double2*>(arow)[t0 + u * blockDim.x] =
                  make_double2(__dadd_rn((double)v[u].x, (double)v[u].y), __dadd_rn((double)v[u].z, (double)v[u].w));
            else
              s4[t0 + u * blockDim.x] = v[u];
          }
      }
      if (dstage) {
        for (int64_t t = n4 * 2 + threadIdx.x; t < k; t += blockDim.x)
          ad[t] = __dadd_rn((double)ag[2 * t], (double)ag[2 * t + 1]);
      } else {
        for (int64_t t = n4 * 4 + threadIdx.x; t < nf; t += blockDim.x) arow[t] = ag[t];
      }
    } else if (dstage) {
      for (int64_t t = threadIdx.x; t < k; t += blockDim.x) ad[t] = __dadd_rn((double)ag[2 * t], (double)ag[2 * t + 1]);
    } else {
      for (int64_t t = threadIdx.x; t < nf; t += blockDim.x) arow[t] = ag[t];
    }
    __syncthreads();
  }
  const float* ar = SMEM ? arow : ag;
  constexpr int U = 8;
  // segments per output: cnt * G <= 8 items (taken by the nw warps in turn; G
  // depends only on cnt, so the result does not depend on nw), k split on 32 U boundaries
  const int G = cnt >= 5 ? 1 : cnt >= 3 ? 2 : cnt == 2 ? 4 : 8;
  const int64_t seg = ((k + G - 1) / G + 32 * U - 1) / (32 * U) * (32 * U);
  for (int w = warp; w < cnt * G; w += nw) {
    const int o = w / G, g = w - o * G;
    const int64_t j = rlist[i * n + o];
    const float* br = bt + j * k * NCB;
    // every c0 + c1 of the row (and of the column, for an MC B) one binary64:
    // one two_prod per k (exact: <= 53 x 53 bits) instead of a two_sum per
    // component product
    const bool pair = rpair && (NCB == 1 || !(cnf[j] & 2));
    const int64_t kb = g * seg, ke = k < kb + seg ? k : kb + seg;
    double S8[U], C8[U];
#pragma unroll
    for (int u = 0; u < U; ++u) S8[u] = C8[u] = 0.0;
    // binary32 B, pair rows, 16-byte aligned column with k % 4 == 0: four k
    // per lane per load (k = 4 lane + 128 (8 r + u) + q -> accumulator u), so
    // a warp keeps 4 KiB of B in flight
    const bool vec = NCB == 1 && NCA == 2 && SMEM && pair && (k & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(br) & 15) == 0;
    // MC B (nc = 2, every c0 + c1 of the column one binary64): two k per
    // 16-byte load (k = 2 lane + 64 (8 r + u) + q -> accumulator u)
    const bool vec2 = NCB == 2 && NCA == 2 && SMEM && pair && (k & 1) == 0 &&
                      (reinterpret_cast<uintptr_t>(br) & 15) == 0;
    if (vec2) {
      for (int64_t t0 = kb + 2 * lane; t0 < ke; t0 += 64 * U) {
        float4 bq[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          bq[u] = t0 + 64 * u < ke ? __ldg(reinterpret_cast<const float4*>(br + (t0 + 64 * u) * NCB))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t t = t0 + 64 * u;
          if (t >= ke) break;
          const double2 a01 = *reinterpret_cast<const double2*>(ad + t);
          const double av[2] = {a01.x, a01.y};
          const float bvq[4] = {bq[u].x, bq[u].y, bq[u].z, bq[u].w};
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double v = av[q];
            const double bb = __dadd_rn((double)bvq[2 * q], (double)bvq[2 * q + 1]);  // exact (pair column)
            const double p = __dmul_rn(v, bb), pe = __fma_rn(v, bb, -p);
            double e;
            dsum(S8[u], p, S8[u], e);
            C8[u] = __dadd_rn(C8[u], __dadd_rn(e, pe));
          }
        }
      }
    }
    if (vec) {
      for (int64_t t0 = kb + 4 * lane; t0 < ke; t0 += 128 * U) {
        float4 bq[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          bq[u] = t0 + 128 * u < ke ? __ldg(reinterpret_cast<const float4*>(br + t0 + 128 * u))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t t = t0 + 128 * u;
          if (t >= ke) break;
          const double2 a01 = *reinterpret_cast<const double2*>(ad + t);
          const double2 a23 = *reinterpret_cast<const double2*>(ad + t + 2);
          const double av[4] = {a01.x, a01.y, a23.x, a23.y};
          const float bvq[4] = {bq[u].x, bq[u].y, bq[u].z, bq[u].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double v = av[q];
            const double bb = (double)bvq[q];
            const double p = __dmul_rn(v, bb), pe = __fma_rn(v, bb, -p);
            double e;
            dsum(S8[u], p, S8[u], e);
            C8[u] = __dadd_rn(C8[u], __dadd_rn(e, pe));
          }
        }
      }
    }
    for (int64_t t0 = kb + lane; !vec && !vec2 && t0 < ke; t0 += 32 * U) {
      float bv[U][NCB];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) bv[u][cb] = t0 + 32 * u < ke ? br[(t0 + 32 * u) * NCB + cb] : 0.0f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t t = t0 + 32 * u;
        if (t >= ke) break;
        if (pair) {
          const double v = dstage ? ad[t] : __dadd_rn((double)ar[t * 2], (double)ar[t * 2 + 1]);  // exact
          const double bb = NCB == 1 ? (double)bv[u][0] : __dadd_rn((double)bv[u][0], (double)bv[u][NCB - 1]);
          const double p = __dmul_rn(v, bb), pe = __fma_rn(v, bb, -p);  // v b = p + pe exactly
          double e;
          dsum(S8[u], p, S8[u], e);
          C8[u] = __dadd_rn(C8[u], __dadd_rn(e, pe));
        } else if (dstage) {
          // staged row, multi-component column: v b_cb = p + pe exactly per component
          const double v = ad[t];
#pragma unroll
          for (int cb = 0; cb < NCB; ++cb) {
            const double bb = (double)bv[u][cb];
            const double p = __dmul_rn(v, bb), pe = __fma_rn(v, bb, -p);
            double e;
            dsum(S8[u], p, S8[u], e);
            C8[u] = __dadd_rn(C8[u], __dadd_rn(e, pe));
          }
        } else {
#pragma unroll
          for (int ca = 0; ca < NCA; ++ca)
#pragma unroll
            for (int cb = 0; cb < NCB; ++cb) {
              const double p = __dmul_rn((double)ar[t * NCA + ca], (double)bv[u][cb]);
              double e;
              dsum(S8[u], p, S8[u], e);
              C8[u] = __dadd_rn(C8[u], e);
            }
        }
      }
    }
    double S = S8[0], C = C8[0];
#pragma unroll
    for (int u = 1; u < U; ++u) {
      double e;
      dsum(S, S8[u], S, e);
      C = __dadd_rn(__dadd_rn(C, C8[u]), e);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oS = __shfl_xor_sync(0xffffffffu, S, off), oC = __shfl_xor_sync(0xffffffffu, C, off);
      double e;
      dsum(S, oS, S, e);
      C = __dadd_rn(__dadd_rn(C, oC), e);
    }
    if (G == 1) {
      if (lane == 0) {
        const double v[2] = {S, C};
        emit(v, i, j, out, ldo, ep);
      }
    } else if (lane == 0) {
      part[o][g] = make_double2(S, C);
    }
  }
  if (G > 1) {
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int o = threadIdx.x;
      double S = part[o][0].x, C = part[o][0].y;
      for (int g = 1; g < G; ++g) {
        double e;
        dsum(S, part[o][g].x, S, e);
        C = __dadd_rn(__dadd_rn(C, part[o][g].y), e);
      }
      const double v[2] = {S, C};
      emit(v, i, rlist[i * n + o], out, ldo, ep);
    }
  }
}

template <int NCA, int NCB>
mcf_status launch_fallback(const float* x, const float* bt, int64_t m, int64_t n, int64_t k, const int* rlist,
                           const int* rcnt, const int* rnf, const int* cnf, float* out, int64_t ldo,
                           const Epilogue& ep, cudaStream_t s) {
  const std::size_t sm = (std::size_t)k * NCA * sizeof(float);
  constexpr std::size_t kMaxSmem = 200u << 10;
  if (sm <= kMaxSmem) {
    const mcf_status ast =
        mcfr::ensure_smem_attr<k_fallback<NCA, NCB, true>>((int)kMaxSmem, "mm_fast: cannot reserve shared memory");
    if (ast != MCF_OK) return ast;
    // 128-thread CTAs (four per SM at 126 registers) while four rows fit in
    // shared memory: one CTA's staging overlaps another's B streaming; config
    // 2's launch 112 -> 98 us under ncu (cold; 256 and 64 threads both 111-115
    // us, r01m).  Longer rows keep 256 threads, so the SM's warp count does
    // not halve when shared memory allows fewer CTAs.
    const int thr = sm <= (48u << 10) ? 128 : 256;
    k_fallback<NCA, NCB, true><<<(unsigned)m, thr, sm, s>>>(x, bt, n, k, rlist, rcnt, rnf, cnf, out, ldo, ep);
  } else {
    k_fallback<NCA, NCB, false><<<(unsigned)m, 256, 0, s>>>(x, bt, n, k, rlist, rcnt, rnf, cnf, out, ldo, ep);
  }
  mcfr::note_launch();
  return mcfr::check_launch("mm_fast fallback kernel");
}



// ---- cuBLASLt int8 GEMMs ------------------------------------------------------------------

// matmul descriptor, layouts and heuristic algorithm of one (shape, batch)
// key: built once and reused (read-only after creation)
struct LtPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulAlgo_t algo{};
};
struct Lt {
  cublasLtHandle_t h = nullptr;
  std::size_t ws_bytes = 0;
  std::map<cudaStream_t, void*> ws_by_stream;  // GEMMs may run concurrently on several streams
  std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t, int, int64_t, int64_t>, LtPlan> plans;
};
std::mutex g_lt_mu;
std::map<int, Lt> g_lt;

mcf_status lt_fail(const char* what, int code) {
  return mcfr::fail(MCF_ERR_CUDA, std::string("mm_fast int8 GEMM: ") + what + " (status " + std::to_string(code) + ")");
}

// C_b (rows_c x cols_c, col-major, ld rows_c, int32; C_b = C + b rows_c
// cols_c) = A_b^T B_b for b < batch, with A_b: kd x rows_c int8 col-major (ld
// lda, A_b = A + b sa), B_b: kd x cols_c int8 col-major (ld ldb, B + b sb).
// MCF_ERR_UNSUPPORTED (no message) when cuBLASLt has no algorithm for the shape.
mcf_status gemm_s8(const int8_t* A, int64_t lda, int64_t sa, const int8_t* B, int64_t ldb, int64_t sb, int* C,
                   int64_t rows_c, int64_t cols_c, int64_t kd, int batch, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  const LtPlan* pl = nullptr;
  cublasLtHandle_t h = nullptr;
  void* wss = nullptr;
  std::size_t ws_bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g_lt_mu);
    Lt& lt = g_lt[dev];
    if (!lt.h) {
      const cublasStatus_t st = cublasLtCreate(&lt.h);
      if (st != CUBLAS_STATUS_SUCCESS) return lt_fail("cublasLtCreate", st);
      lt.ws_bytes = 64u << 20;
    }
    const auto key = std::make_tuple(rows_c, cols_c, kd, lda, ldb, batch, sa, sb);
    auto it = lt.plans.find(key);
    if (it == lt.plans.end()) {
      LtPlan p;
      cublasStatus_t st = cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32I, CUDA_R_32I);
      const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
      if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
      if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
      if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatrixLayoutCreate(&p.la, CUDA_R_8I, kd, rows_c, lda);
      if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatrixLayoutCreate(&p.lb, CUDA_R_8I, kd, cols_c, ldb);
      if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatrixLayoutCreate(&p.lc, CUDA_R_32I, rows_c, cols_c, rows_c);
      if (batch > 1) {
        const int32_t bc = batch;
        const int64_t sc = rows_c * cols_c;
        for (auto* l : {p.la, p.lb, p.lc})
          if (st == CUBLAS_STATUS_SUCCESS)
            st = cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
        if (st == CUBLAS_STATUS_SUCCESS)
          st = cublasLtMatrixLayoutSetAttribute(p.la, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa));
        if (st == CUBLAS_STATUS_SUCCESS)
          st = cublasLtMatrixLayoutSetAttribute(p.lb, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sb, sizeof(sb));
        if (st == CUBLAS_STATUS_SUCCESS)
          st = cublasLtMatrixLayoutSetAttribute(p.lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc));
      }
      int found = 0;
      cublasLtMatmulHeuristicResult_t res{};
      if (st == CUBLAS_STATUS_SUCCESS) {
        cublasLtMatmulPreference_t pref = nullptr;
        cublasLtMatmulPreferenceCreate(&pref);
        cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &lt.ws_bytes,
                                             sizeof(lt.ws_bytes));
        st = cublasLtMatmulAlgoGetHeuristic(lt.h, p.op, p.la, p.lb, p.lc, p.lc, pref, 1, &res, &found);
        cublasLtMatmulPreferenceDestroy(pref);
      }
      if (st != CUBLAS_STATUS_SUCCESS || found == 0) {
        if (p.lc) cublasLtMatrixLayoutDestroy(p.lc);
        if (p.lb) cublasLtMatrixLayoutDestroy(p.lb);
        if (p.la) cublasLtMatrixLayoutDestroy(p.la);
        if (p.op) cublasLtMatmulDescDestroy(p.op);
        return MCF_ERR_UNSUPPORTED;  // caller runs the FP64-pipe kernel instead
      }
      p.algo = res.algo;
      it = lt.plans.emplace(key, p).first;
    }
    pl = &it->second;  // std::map nodes are stable
    h = lt.h;
    void*& w = lt.ws_by_stream[s];
    if (!w && cudaMalloc(&w, lt.ws_bytes) != cudaSuccess) {
      w = nullptr;
      return lt_fail("workspace", 0);
    }
    wss = w;
    ws_bytes = lt.ws_bytes;
  }
  const int32_t alpha = 1, beta = 0;
  const cublasStatus_t st = cublasLtMatmul(h, pl->op, &alpha, A, pl->la, B, pl->lb, &beta, C, pl->lc, C, pl->lc,
                                           &pl->algo, wss, ws_bytes, s);
  if (st != CUBLAS_STATUS_SUCCESS) return lt_fail("cublasLtMatmul", st);
  mcfr::note_launch();
  return MCF_OK;
}
mcf_status gemm_s8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int* C, int64_t rows_c, int64_t cols_c,
                   int64_t kd, cudaStream_t s) {
  return gemm_s8(A, lda, 0, B, ldb, 0, C, rows_c, cols_c, kd, 1, s);
}

// per-(device, stream) workspace for the residue planes and partial products
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, std::pair<void*, std::size_t>> g_ws;

char* oz_workspace(std::size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& slot = g_ws[{dev, s}];
  if (slot.second < bytes) {
    if (slot.first) {
      cudaStreamSynchronize(s);
      cudaFree(slot.first);
    }
    slot = {nullptr, 0};
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    slot = {p, bytes};
  }
  return static_cast<char*>(slot.first);
}

std::size_t al(std::size_t b) { return (b + 255) & ~std::size_t(255); }
int64_t pad16(int64_t v) { return (v + 15) / 16 * 16; }
int64_t pad32(int64_t v) { return (v + 31) / 32 * 32; }

}  // namespace

// Prepared B operand (a block of n columns of a k x ldb matrix): residue
// planes, column exponents, non-finite flags and the transposed binary32
// copy.  Built once; shared by every row chunk of A.
struct PreparedB {
  const int8_t* planes = nullptr;  // [plan.n][np][kp]
  const float* bt = nullptr;
  const int* eb = nullptr;
  const int* cnf = nullptr;
  const int* cinx = nullptr;  // per column: elements not exact in pb bits (binary32 B)
  const float* cth = nullptr;   // per column: fallback-threshold term of A's rounding (Thresholds)
  const int* clk = nullptr;     // [n][kMaxInx] k of the listed inexact elements (binary32 B)
  const double* clr = nullptr;  // [n][kMaxInx] what their rounding dropped, in units of B'
  int64_t k = 0, kp = 0, n = 0, np = 0;  // np: n padded to 16 (int8 GEMM alignment)
  int ncb = 1;
  CrtPlan plan{};
};

std::size_t b_bytes(int64_t k, int64_t n, int ncb) {
  const CrtPlan pl = crt_plan(k, ncb);
  return al(pl.n * pad16(n) * pad32(k)) + al(n * k * ncb * 4) + al(n * 4) * 4 + al(n * 8) * 3 +
         al(n * kMaxInx * 4) + al(n * kMaxInx * 8);
}

#define OZ_NMOD_SWITCH(N, ...)                         \
  switch (N) {                                         \
    case 16: { constexpr int NM = 16; __VA_ARGS__; } break; \
    case 17: { constexpr int NM = 17; __VA_ARGS__; } break; \
    case 18: { constexpr int NM = 18; __VA_ARGS__; } break; \
    case 19: { constexpr int NM = 19; __VA_ARGS__; } break; \
    case 20: { constexpr int NM = 20; __VA_ARGS__; } break; \
    case 21: { constexpr int NM = 21; __VA_ARGS__; } break; \
    default: { constexpr int NM = 22; __VA_ARGS__; } break; \
  }

// one unit of C' in units of Y = C' / 2^(L - 96), times the 2^50 of the fallback
// test (the thresholds are 2^50 x the error bound) and a rounding allowance
double threshold_unit(int nmod) {
  return std::ldexp(1.0, kYShift - host_crt().tab[nmod].L) * 1.0001 * std::ldexp(1.0, 50);
}

mcf_status prepare_b(const float* w, int ncb, int64_t k, int64_t n, int64_t ldb, char* buf, PreparedB& pb,
                     cudaStream_t s) {
  mcf_status st = upload_crt_tables();
  if (st != MCF_OK) return st;
  const CrtPlan pl = crt_plan(k, ncb);
  const int64_t np = pad16(n), kp = pad32(k);
  int8_t* planes = reinterpret_cast<int8_t*>(buf);
  buf += al(pl.n * np * kp);
  if (np > n)
    for (int t = 0; t < pl.n; ++t)
      if (cudaMemsetAsync(planes + (t * np + n) * kp, 0, (np - n) * kp, s) != cudaSuccess)
        return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the padding columns");
  float* bt = reinterpret_cast<float*>(buf);
  buf += al(n * k * ncb * 4);
  int* eb = reinterpret_cast<int*>(buf);
  buf += al(n * 4);
  int* cu = reinterpret_cast<int*>(buf);
  buf += al(n * 4);
  // zero-initialised arrays, contiguous: one memset
  char* z0 = buf;
  int* cnf = reinterpret_cast<int*>(buf);
  buf += al(n * 4);
  int* cinx = reinterpret_cast<int*>(buf);
  buf += al(n * 4);
  unsigned long long* cm = reinterpret_cast<unsigned long long*>(buf);
  buf += al(n * 8);
  float* csum = reinterpret_cast<float*>(buf);
  buf += al(n * 8);
  float* cth = reinterpret_cast<float*>(buf);  // read four columns at a time: n * 8 bytes hold the padded n
  buf += al(n * 8);
  const std::size_t zbytes = (std::size_t)(buf - z0);
  int* clk = reinterpret_cast<int*>(buf);
  buf += al(n * kMaxInx * 4);
  double* clr = reinterpret_cast<double*>(buf);
  if (cudaMemsetAsync(z0, 0, zbytes, s) != cudaSuccess || cudaMemsetAsync(cu, 0x7f, n * 4, s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the column maxima");
  const dim3 gm((unsigned)((n + 255) / 256), (unsigned)((k + 63) / 64));
  if (ncb == 2) k_colmax<2><<<gm, 256, 0, s>>>(w, k, n, ldb, cm, cnf, cu, csum);
  else k_colmax<1><<<gm, 256, 0, s>>>(w, k, n, ldb, cm, cnf, cu, csum);
  k_colexp<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cm, n, pl.pb, ncb == 2 ? cu : nullptr, eb, cnf, csum, k,
                                                        0.51 * threshold_unit(pl.n), cth);
  const dim3 gs((unsigned)((n + kSlab - 1) / kSlab), (unsigned)(kp / kSlab));
  OZ_NMOD_SWITCH(pl.n, if (ncb == 2) k_res_cols<2, NM><<<gs, 256, 0, s>>>(w, n, ldb, k, kp, np, pl.pb, eb, planes, bt, cinx, clk, clr);
                 else k_res_cols<1, NM><<<gs, 256, 0, s>>>(w, n, ldb, k, kp, np, pl.pb, eb, planes, bt, cinx, clk, clr));
  if (ncb == 1) {
    k_colfin<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cinx, n, std::nextafterf((float)(1.3 * threshold_unit(pl.n)), INFINITY), cth);
    mcfr::note_launch();
  }
  for (int i = 0; i < 3; ++i) mcfr::note_launch();
  pb = PreparedB{planes, bt, eb, cnf, ncb == 1 ? cinx : nullptr, cth, clk, clr, k, kp, n, np, ncb, pl};
  return mcfr::check_launch("mm_fast B residue kernels");
}

std::size_t rows_bytes(int64_t m, int64_t k, int64_t n, int ncb) {
  const CrtPlan pl = crt_plan(k, ncb);
  return al(pl.n * m * pad32(k)) + al((int64_t)pl.n * m * pad16(n) * 4) + al(m * pad16(n) * 4) + al(m * 4) * 3 + al(m * 8);
}

// workspace layout of one row block (see rows_bytes)
struct RowsWs {
  int8_t* planes;
  int* cq;
  int* rlist;
  int* ea;
  int* rnf;
  int* rcnt;
  float* rth;  // per row: fallback-threshold term of B's rounding (Thresholds)
};
RowsWs rows_ws(char* buf, int64_t m, int64_t kp, int64_t np, int nmod) {
  RowsWs w;
  w.planes = reinterpret_cast<int8_t*>(buf);
  buf += al(nmod * m * kp);
  w.cq = reinterpret_cast<int*>(buf);
  buf += al((int64_t)nmod * m * np * 4);
  w.rlist = reinterpret_cast<int*>(buf);
  buf += al(m * (np > 0 ? np : 1) * 4);
  w.ea = reinterpret_cast<int*>(buf);
  buf += al(m * 4);
  w.rnf = reinterpret_cast<int*>(buf);
  buf += al(m * 4);
  w.rcnt = reinterpret_cast<int*>(buf);
  buf += al(m * 4);
  w.rth = reinterpret_cast<float*>(buf);
  return w;
}

// A's row exponents and residue planes (independent of B: may run
// concurrently with prepare_b on another stream)
mcf_status a_residues(const float* x, int nca, int64_t m, int64_t k, const CrtPlan& pl, const RowsWs& w,
                      cudaStream_t s) {
  mcf_status st = upload_crt_tables();
  if (st != MCF_OK) return st;
  if (cudaMemsetAsync(w.rcnt, 0, m * sizeof(int), s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the fallback counters");
  const int64_t kp = pad32(k);
  const unsigned gr = (unsigned)((m + 7) / 8);
  const double cb = 0.51 * threshold_unit(pl.n);
  if (nca == 2) k_rowexp<2><<<gr, 256, 0, s>>>(x, m, k, pl.pa, w.ea, w.rnf, cb, w.rth);
  else k_rowexp<1><<<gr, 256, 0, s>>>(x, m, k, pl.pa, w.ea, w.rnf, cb, w.rth);
  const int64_t gx = (kp / 4 + 255) / 256;  // ~8 CTAs per SM in all, rows strided over y
  const dim3 gsl((unsigned)gx, (unsigned)std::max<int64_t>(1, std::min<int64_t>(m, mcfr::sm_count() * 8 / gx)));
  OZ_NMOD_SWITCH(pl.n, if (nca == 2) k_res_rows<2, NM><<<gsl, 256, 0, s>>>(x, m, k, kp, pl.pa, w.ea, w.planes);
                 else k_res_rows<1, NM><<<gsl, 256, 0, s>>>(x, m, k, kp, pl.pa, w.ea, w.planes));  mcfr::note_launch();
  mcfr::note_launch();
  return mcfr::check_launch("mm_fast A residue kernels");
}

mcf_status rows_products(const float* x, int nca, int64_t m, const PreparedB& pb, float* out, int64_t ldo,
                         const RowsWs& w, cudaStream_t s, cudaEvent_t* ev, const Epilogue& ep,
                         cudaStream_t cs = nullptr, cudaEvent_t gemm_done = nullptr);

// out (m x n x 2 binary32, row stride ldo elements) = A (m x k x nca) . B for
// a prepared B.  ev (optional, 4 events): recorded before the A residues,
// before the GEMMs, after the GEMMs and at the end (phase timing).
mcf_status rows(const float* x, int nca, int64_t m, const PreparedB& pb, float* out, int64_t ldo, char* buf,
                cudaStream_t s, cudaEvent_t* ev = nullptr, const Epilogue& ep = Epilogue{}) {
  const RowsWs w = rows_ws(buf, m, pb.kp, pb.np, pb.plan.n);
  if (ev) cudaEventRecord(ev[0], s);
  const mcf_status st = a_residues(x, nca, m, pb.k, pb.plan, w, s);
  if (st != MCF_OK) return st;
  return rows_products(x, nca, m, pb, out, ldo, w, s, ev, ep);
}

// the GEMMs, reconstruction and fallback of a row block whose A residues are
// done.  With a second stream cs (and an event), the reconstruction and the
// fallback are enqueued there after the GEMM: they then run concurrently with
// whatever the caller puts on s next (the next row block's GEMM).
mcf_status rows_products(const float* x, int nca, int64_t m, const PreparedB& pb, float* out, int64_t ldo,
                         const RowsWs& w, cudaStream_t s, cudaEvent_t* ev, const Epilogue& ep, cudaStream_t cs,
                         cudaEvent_t gemm_done) {
  const CrtPlan pl = pb.plan;
  const int64_t k = pb.k, kp = pb.kp, n = pb.n, np = pb.np;
  if (ev) cudaEventRecord(ev[1], s);
  // The residue GEMMs: by default the hand-written tcgen05 kernel
  // (tc_gemm.cu), whose epilogue reduces each int32 sum modulo its modulus and
  // writes int8 residues (planes [t][m][np]); MCF_OZ_GEMM=cublaslt runs one
  // strided-batched cuBLASLt GEMM writing the int32 sums instead (kept for
  // A/B measurement): C_t (np x m col-major = m x np row-major).
  static const bool use_lt = [] {
    const char* e = getenv("MCF_OZ_GEMM");
    return e && std::string(e) == "cublaslt";
  }();
  mcf_status st;
  if (use_lt) {
    st = gemm_s8(pb.planes, kp, np * kp, w.planes, kp, m * kp, w.cq, np, m, kp, pl.n, s);
  } else {
    st = mcfr::tc_gemm_s8(w.planes, pb.planes, w.cq, m, n, kp, pl.n, np, kModuli, s, np);
    if (st == MCF_ERR_UNSUPPORTED) st = mcfr::fail(MCF_ERR_CUDA, "mm_fast: the tcgen05 residue GEMM cannot run this shape");
  }
  if (st != MCF_OK) return st;
  if (ev) cudaEventRecord(ev[2], s);
  if (cs && gemm_done) {
    cudaEventRecord(gemm_done, s);
    cudaStreamWaitEvent(cs, gemm_done, 0);
    s = cs;
  }
  // error bound per output in C' units (2^-(pa+pb) scaled): A's rounding
  // (<= 0.51 per element) against the column's |B'| sum (pb.cth), B's against
  // the row's |A'| sum (w.rth; for a binary32 B only its counted inexact
  // elements, each <= 0.51 2^(pa-1)), their product (K 1.1 units covers it),
  // and the CRT slices' tail (<= 2^12 units of 2^(L - 96)).  The fallback
  // threshold is 2^50 times it, in units of Y = C' / 2^(L-96).
  const int L = host_crt().tab[pl.n].L;
  const double yu = threshold_unit(pl.n);
  Thresholds th;
  const auto up = [](double v) { return std::nextafterf((float)v, INFINITY); };  // binary32, rounded up
  th.base = up((double)k * 1.1 * yu + 4096.0 * 1.0001 * std::ldexp(1.0, 50));
  th.inexact = up(0.51 * std::ldexp(1.0, pl.pa - 1) * yu);
  th.cth = pb.cth;
  th.rth = w.rth;
  th.mcb = pb.ncb == 2;
  const int sexp = L - kYShift - pl.pa - pl.pb;
  const int64_t gcx = (n + 1023) / 1024;
  const dim3 gc((unsigned)gcx, (unsigned)std::max<int64_t>(1, std::min<int64_t>(m, mcfr::sm_count() * 8 / gcx)));
  const bool big = k > 16384;
  if (!use_lt) {
    const dim3 gc8((unsigned)((n + 1023) / 1024), (unsigned)m);
    OZ_NMOD_SWITCH(pl.n, k_crt8<NM><<<gc8, 256, 0, s>>>(reinterpret_cast<const int8_t*>(w.cq), m, n, np, w.ea, pb.eb,
                                                       w.rnf, pb.cnf, pb.cinx, th, sexp, out, ldo,
                                                       w.rlist, w.rcnt, ep, x, nca, k, pb.clk, pb.clr,
                                                       std::ldexp(1.0, pl.pa + kYShift - L)));
  } else
  OZ_NMOD_SWITCH(pl.n,
                 if (big) k_crt<NM, true><<<gc, 256, 0, s>>>(w.cq, m, n, np, w.ea, pb.eb, w.rnf, pb.cnf, pb.cinx, th,
                                                             sexp, out, ldo, w.rlist, w.rcnt, ep);
                 else k_crt<NM, false><<<gc, 256, 0, s>>>(w.cq, m, n, np, w.ea, pb.eb, w.rnf, pb.cnf, pb.cinx, th,
                                                          sexp, out, ldo, w.rlist, w.rcnt, ep));
  mcfr::note_launch();
  if (nca == 2 && pb.ncb == 2) st = launch_fallback<2, 2>(x, pb.bt, m, n, k, w.rlist, w.rcnt, w.rnf, pb.cnf, out, ldo, ep, s);
  else if (nca == 2) st = launch_fallback<2, 1>(x, pb.bt, m, n, k, w.rlist, w.rcnt, w.rnf, pb.cnf, out, ldo, ep, s);
  else if (pb.ncb == 2) st = launch_fallback<1, 2>(x, pb.bt, m, n, k, w.rlist, w.rcnt, w.rnf, pb.cnf, out, ldo, ep, s);
  else st = launch_fallback<1, 1>(x, pb.bt, m, n, k, w.rlist, w.rcnt, w.rnf, pb.cnf, out, ldo, ep, s);
  if (st != MCF_OK) return st;
  if (ev) cudaEventRecord(ev[3], s);
  return mcfr::check_launch("mm_fast reconstruction kernels");
}

// ---- binary32 x binary32 -> binary32 GEMM on the int8 tensor cores ---------------------
//
// Plan FAST's MLP backward products (dW = G A^T, dA = approx(W)^T G, the
// reference's plain binary32 matmul2d, autodiff.hpp:280-296) with the same
// digit scheme at binary32 accuracy: each row of op(A) / column of op(B) is
// scaled by a power of two 2^e > 2 max|x| and rounded to X = rint(x 2^(31-e))
// (|X| < 2^30, truncation <= 2^-32 in scaled units), cut into four balanced
// base-256 digits (d0 in [-64, 64]); diagonals q = s + t <= 3 (10 int8
// GEMM-equivalents, one GEMM per diagonal over the concatenated planes,
// exact int32 sums for K < 32768); the dropped pairs and truncations leave
// <= 2^-30 per product in scaled units, i.e. about 2^-26 |a|max |b|max:
// below a binary32 FFMA GEMM's error bound (K 2^-24 sum |a||b|).
// T = ((S0 256 + S1) 256 + S2) 256 + S3 is exact in binary64 (< 2^50 for
// K < 32768) and C = RN32(T 2^(ea + eb - 38)).  A row / column holding Inf
// or NaN makes its outputs NaN.

constexpr int kD4 = 4;

// max |x| bits per k-contiguous row (element (r, k) at p[r ld + k]): a CTA per
// row, 16-byte loads when the row is 16-byte aligned
__global__ void __launch_bounds__(256) k_f32_rowmax(const float* __restrict__ p, int64_t rows, int64_t k, int64_t ld,
                                                    unsigned* __restrict__ mx) {
  __shared__ unsigned part[8];
  const int64_t r = blockIdx.x;
  unsigned m0 = 0, m1 = 0, m2 = 0, m3 = 0;
  const float* pr = p + r * ld;
  int64_t t = 0;
  if ((reinterpret_cast<uintptr_t>(pr) & 15) == 0) {
    const uint4* p4 = reinterpret_cast<const uint4*>(pr);
    const int64_t k4 = k / 4;
    for (int64_t q = threadIdx.x; q < k4; q += blockDim.x) {
      const uint4 v = __ldg(p4 + q);
      m0 = max(m0, v.x & 0x7fffffffu);
      m1 = max(m1, v.y & 0x7fffffffu);
      m2 = max(m2, v.z & 0x7fffffffu);
      m3 = max(m3, v.w & 0x7fffffffu);
    }
    t = k4 * 4;
  }
  for (int64_t u = t + threadIdx.x; u < k; u += blockDim.x) m0 = max(m0, __float_as_uint(pr[u]) & 0x7fffffffu);
  unsigned m = max(max(m0, m1), max(m2, m3));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned a = part[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = max(a, part[w]);
    mx[r] = a;
  }
}

// max |x| bits per column of a k-strided operand (element (k, c) at p[k ld + c]),
// slabs of 64 k, atomicMax (mx cleared first)
__global__ void __launch_bounds__(256) k_f32_colmax(const float* __restrict__ p, int64_t k, int64_t cols, int64_t ld,
                                                    unsigned* __restrict__ mx) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int64_t t0 = (int64_t)blockIdx.y * 64, t1 = t0 + 64 < k ? t0 + 64 : k;
  unsigned m = 0;
  for (int64_t t = t0; t < t1; ++t) m = max(m, __float_as_uint(p[t * ld + c]) & 0x7fffffffu);
  if (m) atomicMax(mx + c, m);
}

// scale exponent from the max bits: 2^e > 2 max (0 for an all-zero line)
__device__ __forceinline__ int f32_scale_exp(unsigned mbits) {
  return mbits == 0 ? 0 : ilogbf(__uint_as_float(mbits)) + 2;
}

// four balanced digits of one element, packed little-endian per plane
__device__ __forceinline__ void f32_digits(float x, int e, int (&d)[kD4]) {
  int v = __double2int_rn(__dmul_rn((double)x, __longlong_as_double((long long)(1023 + 31 - e) << 52)));
#pragma unroll
  for (int s = kD4 - 1; s >= 1; --s) {
    const int t = ((v + 128) & 255) - 128;
    d[s] = t;
    v = (v - t) >> 8;
  }
  d[0] = v;
}

// digit planes of a k-contiguous operand: byte [r][pos(s) kp + k], pos(s) = s
// (REV = false, the A side) or kD4 - 1 - s (REV, the B side); zero for k >= K
template <bool REV>
__global__ void __launch_bounds__(256) k_f32_dig_rows(const float* __restrict__ p, int64_t rows, int64_t k,
                                                      int64_t ld, int64_t kp, const unsigned* __restrict__ mx,
                                                      int8_t* __restrict__ out) {
  const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k0 >= kp) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const unsigned mb = mx[r];
    const int e = f32_scale_exp(mb);
    const bool ok = mb < 0x7f800000u;
    unsigned packed[kD4] = {0u, 0u, 0u, 0u};
    const float* pr = p + r * ld;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (k0 + u >= k || !ok) break;
      int d[kD4];
      f32_digits(pr[k0 + u], e, d);
#pragma unroll
      for (int s = 0; s < kD4; ++s) packed[s] |= ((unsigned)(d[s] & 0xff)) << (8 * u);
    }
    int8_t* row = out + r * kD4 * kp + k0;
#pragma unroll
    for (int s = 0; s < kD4; ++s) *reinterpret_cast<unsigned*>(row + (REV ? kD4 - 1 - s : s) * kp) = packed[s];
  }
}

// digit planes of a k-strided operand (element (k, c) at p[k ld + c]) as rows
// per column c: 32 k x 32 c tiles transposed through shared memory
template <bool REV>
__global__ void __launch_bounds__(256) k_f32_dig_cols(const float* __restrict__ p, int64_t k, int64_t cols,
                                                      int64_t ld, int64_t kp, const unsigned* __restrict__ mx,
                                                      int8_t* __restrict__ out) {
  __shared__ unsigned dg[kD4][kSlab][kSlab / 4 + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)blockIdx.y * kSlab, c0 = (int64_t)blockIdx.x * kSlab;
  const int64_t c = c0 + tx;
  const unsigned mb = c < cols ? mx[c] : 0u;
  const int e = f32_scale_exp(mb);
  const bool ok = mb < 0x7f800000u;
  unsigned packed[kD4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t gk = k0 + ty * 4 + u;
    if (gk < k && c < cols && ok) {
      int d[kD4];
      f32_digits(p[gk * ld + c], e, d);
#pragma unroll
      for (int s = 0; s < kD4; ++s) packed[s] |= ((unsigned)(d[s] & 0xff)) << (8 * u);
    }
  }
#pragma unroll
  for (int s = 0; s < kD4; ++s) dg[s][tx][ty] = packed[s];
  __syncthreads();
  const int jj = threadIdx.x >> 3, part = threadIdx.x & 7;
  const int64_t gc = c0 + jj;
  if (gc < cols && k0 + part * 4 < kp) {
    int8_t* dst = out + gc * kD4 * kp + k0 + part * 4;
#pragma unroll
    for (int s = 0; s < kD4; ++s) *reinterpret_cast<unsigned*>(dst + (REV ? kD4 - 1 - s : s) * kp) = dg[s][jj][part];
  }
}

// C[i, j] (row-major, ldc) = RN32(T 2^(ea_i + eb_j - 38)), optional ReLU mask;
// four consecutive columns per thread (16-byte plane loads: np % 16 == 0)
__global__ void __launch_bounds__(256) k_f32_comb(const int* __restrict__ cq, int64_t m, int64_t n, int64_t np,
                                                  const unsigned* __restrict__ amx, const unsigned* __restrict__ bmx,
                                                  float* __restrict__ c, int64_t ldc, const float* __restrict__ mask) {
  const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (j0 >= n) return;
  const int64_t plane = m * np;
  unsigned bm[4];
  int eb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    bm[u] = j0 + u < n ? bmx[j0 + u] : 0u;
    eb[u] = f32_scale_exp(bm[u]);
  }
  const bool vec = j0 + 3 < n && (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0 &&
                   (!mask || (reinterpret_cast<uintptr_t>(mask) & 15) == 0);
  for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
    const int64_t o = i * np + j0;
    const int4 s0 = __ldcs(reinterpret_cast<const int4*>(cq + o));
    const int4 s1 = __ldcs(reinterpret_cast<const int4*>(cq + plane + o));
    const int4 s2 = __ldcs(reinterpret_cast<const int4*>(cq + 2 * plane + o));
    const int4 s3 = __ldcs(reinterpret_cast<const int4*>(cq + 3 * plane + o));
    const int a0[4] = {s0.x, s0.y, s0.z, s0.w}, a1[4] = {s1.x, s1.y, s1.z, s1.w};
    const int a2[4] = {s2.x, s2.y, s2.z, s2.w}, a3[4] = {s3.x, s3.y, s3.z, s3.w};
    const unsigned am = amx[i];
    const int ea = f32_scale_exp(am);
    float v[4], mk[4] = {1.f, 1.f, 1.f, 1.f};
    if (mask) {
      if (vec) {
        const float4 q = *reinterpret_cast<const float4*>(mask + i * ldc + j0);
        mk[0] = q.x, mk[1] = q.y, mk[2] = q.z, mk[3] = q.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) mk[u] = j0 + u < n ? mask[i * ldc + j0 + u] : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double t = __fma_rn(__fma_rn(__fma_rn((double)a0[u], 256.0, (double)a1[u]), 256.0, (double)a2[u]), 256.0,
                                (double)a3[u]);
      v[u] = __double2float_rn(__dmul_rn(t, pow2d(ea + eb[u] - 38)));
      if (am >= 0x7f800000u || bm[u] >= 0x7f800000u) v[u] = __int_as_float(0x7fffffff);
      if (!(mk[u] > 0.0f)) v[u] = 0.0f;
    }
    if (vec) {
      *reinterpret_cast<float4*>(c + i * ldc + j0) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < n) c[i * ldc + j0 + u] = v[u];
    }
  }
}

// ---- binary16 MC x MC (nc <= 3) on the int8 tensor cores ---------------------------------
//
// Config 4's binary16 variant.  Every binary16 value is a multiple of 2^-24
// below 2^16, so an element's components sum exactly in binary64 (<= 42
// bits).  That value is scaled per row of A / column of B (2^e > 2 max),
// rounded to X = rint(v 2^(39-e)) (|X| < 2^38, truncation <= 2^-40 in scaled
// units) and cut into five balanced base-256 digits; diagonals q = s + t <= 4
// (15 int8 GEMM-equivalents, exact int32 sums for K < 26214), the dropped
// pairs leave < 2^-37 per product (scaled): far inside the 4x-of-recipe-B
// contract (recipe B's own error is ~2^-10 median at this format).  The
// five diagonal sums combine exactly in int64 (< 2^59), go to a
// double-double and are split greedily into nc binary16 components.

constexpr int kD5 = 5;

template <int NC>
__device__ __forceinline__ double b16_val(const __half* p) {
  double v = (double)__half2float(p[0]);
#pragma unroll
  for (int c = 1; c < NC; ++c) v = __dadd_rn(v, (double)__half2float(p[c]));  // exact
  return v;
}

template <int NC>
__global__ void __launch_bounds__(256) k_b16_rowmax(const __half* __restrict__ x, int64_t k,
                                                    unsigned long long* __restrict__ mx) {
  __shared__ unsigned long long part[8];
  const int64_t r = blockIdx.x;
  unsigned long long m = 0;
  for (int64_t t = threadIdx.x; t < k; t += blockDim.x)
    m = max(m, (unsigned long long)__double_as_longlong(fabs(b16_val<NC>(x + (r * k + t) * NC))));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, part[w]);
    mx[r] = max(part[0], m);
  }
}

template <int NC>
__global__ void __launch_bounds__(256) k_b16_colmax(const __half* __restrict__ y, int64_t k, int64_t n,
                                                    unsigned long long* __restrict__ mx) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t t0 = (int64_t)blockIdx.y * 64, t1 = t0 + 64 < k ? t0 + 64 : k;
  unsigned long long m = 0;
  for (int64_t t = t0; t < t1; ++t)
    m = max(m, (unsigned long long)__double_as_longlong(fabs(b16_val<NC>(y + (t * n + j) * NC))));
  if (m) atomicMax(mx + j, m);
}

__device__ __forceinline__ int b16_scale_exp(unsigned long long mbits) {
  return mbits == 0 ? 0 : ilogb(__longlong_as_double((long long)mbits)) + 2;
}

__device__ __forceinline__ void b16_digits(double v, int e, int (&d)[kD5]) {
  long long x = __double2ll_rn(__dmul_rn(v, __longlong_as_double((long long)(1023 + 39 - e) << 52)));
#pragma unroll
  for (int s = kD5 - 1; s >= 1; --s) {
    const long long t = ((x + 128) & 255) - 128;
    d[s] = (int)t;
    x = (x - t) >> 8;
  }
  d[0] = (int)x;
}

// A (m x k x NC) rows -> planes [i][s kp + kk]
template <int NC>
__global__ void __launch_bounds__(256) k_b16_dig_rows(const __half* __restrict__ x, int64_t rows, int64_t k,
                                                      int64_t kp, const unsigned long long* __restrict__ mx,
                                                      int8_t* __restrict__ out) {
  const int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k0 >= kp) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const unsigned long long mb = mx[r];
    const int e = b16_scale_exp(mb);
    const bool ok = mb < 0x7ff0000000000000ull;
    unsigned packed[kD5] = {0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (k0 + u >= k || !ok) break;
      int d[kD5];
      b16_digits(b16_val<NC>(x + (r * k + k0 + u) * NC), e, d);
#pragma unroll
      for (int s = 0; s < kD5; ++s) packed[s] |= ((unsigned)(d[s] & 0xff)) << (8 * u);
    }
    int8_t* row = out + r * kD5 * kp + k0;
#pragma unroll
    for (int s = 0; s < kD5; ++s) *reinterpret_cast<unsigned*>(row + s * kp) = packed[s];
  }
}

// B (k x n x NC) columns -> planes [j][(kD5 - 1 - t) kp + kk] (32 x 32 tiles)
template <int NC>
__global__ void __launch_bounds__(256) k_b16_dig_cols(const __half* __restrict__ y, int64_t k, int64_t n,
                                                      int64_t kp, const unsigned long long* __restrict__ mx,
                                                      int8_t* __restrict__ out) {
  __shared__ unsigned dg[kD5][kSlab][kSlab / 4 + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)blockIdx.y * kSlab, c0 = (int64_t)blockIdx.x * kSlab;
  const int64_t c = c0 + tx;
  const unsigned long long mb = c < n ? mx[c] : 0ull;
  const int e = b16_scale_exp(mb);
  const bool ok = mb < 0x7ff0000000000000ull;
  unsigned packed[kD5] = {0u, 0u, 0u, 0u, 0u};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t gk = k0 + ty * 4 + u;
    if (gk < k && c < n && ok) {
      int d[kD5];
      b16_digits(b16_val<NC>(y + (gk * n + c) * NC), e, d);
#pragma unroll
      for (int s = 0; s < kD5; ++s) packed[s] |= ((unsigned)(d[s] & 0xff)) << (8 * u);
    }
  }
#pragma unroll
  for (int s = 0; s < kD5; ++s) dg[s][tx][ty] = packed[s];
  __syncthreads();
  const int jj = threadIdx.x >> 3, part = threadIdx.x & 7;
  const int64_t gc = c0 + jj;
  if (gc < n && k0 + part * 4 < kp) {
    int8_t* dst = out + gc * kD5 * kp + k0 + part * 4;
#pragma unroll
    for (int s = 0; s < kD5; ++s) *reinterpret_cast<unsigned*>(dst + (kD5 - 1 - s) * kp) = dg[s][jj][part];
  }
}

// out[i, j, :] (binary16, NC comps) from T' = sum_q S_q 256^(4 - q) (int64,
// exact), value = T' 2^(ea + eb - 46), greedy split of the double-double
template <int NC>
__global__ void __launch_bounds__(256) k_b16_comb(const int* __restrict__ cq, int64_t m, int64_t n, int64_t np,
                                                  const unsigned long long* __restrict__ amx,
                                                  const unsigned long long* __restrict__ bmx,
                                                  __half* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t plane = m * np;
  const unsigned long long bm = bmx[j];
  const int eb = b16_scale_exp(bm);
  for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
    const int64_t o = i * np + j;
    long long t = cq[o];
#pragma unroll
    for (int q = 1; q < kD5; ++q) t = t * 256 + cq[q * plane + o];
    const unsigned long long am = amx[i];
    const double sc = pow2d(b16_scale_exp(am) + eb - 46);
    const double hi = __ll2double_rn(t);
    const double lo = __ll2double_rn(t - (long long)hi);  // exact: |t - hi| <= 2^10
    double r = __dadd_rn(__dmul_rn(hi, sc), __dmul_rn(lo, sc));
    double rl = __dsub_rn(__dmul_rn(lo, sc), __dsub_rn(r, __dmul_rn(hi, sc)));
    const bool bad = am >= 0x7ff0000000000000ull || bm >= 0x7ff0000000000000ull;
    __half* oe = out + (i * n + j) * NC;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const __half h = __double2half(r);
      const double hv = (double)__half2float(h);
      oe[c] = bad ? __float2half(__int_as_float(0x7fffffff)) : h;
      const double nr = __dadd_rn(__dsub_rn(r, hv), rl);  // r - hv exact when h is finite
      rl = __dsub_rn(rl, __dsub_rn(nr, __dsub_rn(r, hv)));
      r = isfinite(hv) ? nr : 0.0;
    }
  }
}

}  // namespace oz
}  // namespace mcfg

namespace mcfr {

bool ozaki_supported(int64_t m, int64_t k, int64_t n) {
  // K <= 65536: the reconstruction's residue sums stay exact binary32 integers
  return m > 0 && n > 0 && k > 0 && k <= 65536 && m * n < (int64_t(1) << 31) && mcfg::oz::crt_plan(k, 2).n > 0 &&
         mcfg::oz::crt_plan(k, 1).n > 0;
}

// The one-call product, optionally pipelined over row blocks of A (MCF_OZ_PIPE).  B's residues run on
// the caller's stream s while the first block's A residues run on a side
// stream; then, per block c, s waits for its A residues and runs its residue
// GEMM, and the block's reconstruction + fallback go to a third stream.  The
// later blocks' A residues (issued once B's are done) and the earlier blocks'
// reconstructions run concurrently with the GEMM of the block in between:
// the GEMM keeps one CTA per SM busy on the tensor cores and TMA, and these
// FMA-pipe kernels fill the SMs' remaining warp slots.  Row blocks are
// multiples of 256 (the CTA-pair tile); products under 1024 rows run as one
// block.  Results are those of the unpipelined product bit for bit (every
// output depends on its own row and column only).
// row blocks of the one-call product: count nb, rows per block rb, and the
// workspace bytes (B's planes + nb row-block workspaces)
static std::size_t pipe_geometry(int64_t m, int64_t k, int64_t n, int ncb, int& nb, int64_t& rb) {
  using namespace mcfg::oz;
  static const int blocks_env = [] {
    // row blocks (1: no pipelining, the default).  Measured on B200 (r02,
    // config 2): 1 block 1.308 ms, 2 blocks 1.329, 4 blocks 1.355, 6 blocks
    // 1.388 -- the residue and reconstruction kernels do not hide under the
    // GEMM (both are FMA-pipe / issue heavy and the GEMM's epilogue needs the
    // same pipes), and the shorter GEMMs lose their last-wave tails.  Retried
    // with room for co-residency (a 5- or 6-stage GEMM ring, residue grids of
    // 2-4 CTAs per SM): 2 blocks 1.33, 4 blocks 1.36, 6 blocks 1.40 against
    // 1.31 -- the GEMM already runs at the power-capped clock (1.55 GHz), so
    // work added beside it slows it by as much as it hides.
    const char* e = getenv("MCF_OZ_PIPE");
    return e ? std::max(1, std::min(6, atoi(e))) : 1;
  }();
  nb = m >= 1024 ? blocks_env : 1;
  rb = (m + nb - 1) / nb;
  rb = (rb + 255) / 256 * 256;
  nb = (int)((m + rb - 1) / rb);
  return al(b_bytes(k, n, ncb)) + nb * al(rows_bytes(rb, k, n, ncb));
}

static mcf_status pipelined(const float* x, int nca, const float* w, int ncb, int64_t m, int64_t k, int64_t n,
                            float* out, int64_t ldo, const mcfg::oz::Epilogue& ep0, cudaStream_t s) {
  using namespace mcfg::oz;
  int nb;
  int64_t rb;
  const std::size_t total = pipe_geometry(m, k, n, ncb, nb, rb);
  const CrtPlan pl = crt_plan(k, ncb);
  const std::size_t bb = al(b_bytes(k, n, ncb)), rbytes = al(rows_bytes(rb, k, n, ncb));
  char* ws = oz_workspace(total, s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the residue-plane workspace");
  cudaStream_t as = side_stream(12), cs = side_stream(13);
  cudaEvent_t fork = tl_event(0), bdone = tl_event(1);
  cudaEventRecord(fork, s);
  cudaStreamWaitEvent(as, fork, 0);
  cudaStreamWaitEvent(cs, fork, 0);
  std::vector<RowsWs> rws(nb);
  mcf_status st = MCF_OK;
  // block 0's A residues alongside B's
  for (int c = 0; c < nb; ++c) {
    const int64_t r0 = c * rb, rows_c = std::min<int64_t>(rb, m - r0);
    rws[c] = rows_ws(ws + bb + c * rbytes, rows_c, pad32(k), pad16(n), pl.n);
  }
  st = a_residues(x, nca, std::min<int64_t>(rb, m), k, pl, rws[0], as);
  cudaEvent_t adone[16];
  adone[0] = tl_event(2);
  cudaEventRecord(adone[0], as);
  PreparedB pb;
  if (st == MCF_OK) st = prepare_b(w, ncb, k, n, n, ws, pb, s);
  cudaEventRecord(bdone, s);
  cudaStreamWaitEvent(as, bdone, 0);
  // the other blocks' A residues after B's: they then share the SMs with the
  // GEMMs, not with B's residues (which gate the first GEMM)
  for (int c = 1; c < nb && st == MCF_OK; ++c) {
    const int64_t r0 = c * rb, rows_c = std::min<int64_t>(rb, m - r0);
    st = a_residues(x + r0 * k * nca, nca, rows_c, k, pl, rws[c], as);
    adone[c] = tl_event(2 + c);
    cudaEventRecord(adone[c], as);
  }
  for (int c = 0; c < nb && st == MCF_OK; ++c) {
    const int64_t r0 = c * rb, rows_c = std::min<int64_t>(rb, m - r0);
    cudaStreamWaitEvent(s, adone[c], 0);
    Epilogue ep = ep0;
    if (ep.bias) {
      ep.bias += r0 * 2;
      ep.h += r0 * ldo;
      if (ep.act) ep.act += r0 * ldo;
    }
    st = rows_products(x + r0 * k * nca, nca, rows_c, pb, ep.bias ? nullptr : out + r0 * ldo * 2, ldo, rws[c], s,
                       nullptr, ep, nb > 1 ? cs : nullptr, nb > 1 ? tl_event(8 + c) : nullptr);
  }
  if (nb > 1) {
    cudaEvent_t join = tl_event(14);
    cudaEventRecord(join, cs);
    cudaStreamWaitEvent(s, join, 0);
  }
  return st;
}

// one-call MC(nc=2, binary32) x T / MC(nc=2) product on the INT8 tensor cores
mcf_status mm_ozaki(const float* x, int nca, const float* w, int ncb, int64_t m, int64_t k, int64_t n, float* out,
                    cudaStream_t s) {
  return pipelined(x, nca, w, ncb, m, k, n, out, n, mcfg::oz::Epilogue{}, s);
}

// MC-MLP layer forward on the tensor-core path with the bias / approx / ReLU
// epilogue fused into the reconstruction: h = approx(add_mcn(W . A, bias)),
// act = relu(h); the MC product itself is never written
mcf_status mm_ozaki_bias_act(const float* w, const float* a, int64_t m, int64_t k, int64_t n, const float* bias,
                             int relu, float* h, float* act, cudaStream_t s) {
  using namespace mcfg::oz;
  if (m < 64 || !ozaki_supported(m, k, n)) return MCF_ERR_UNSUPPORTED;
  Epilogue ep;
  ep.bias = bias;
  ep.h = h;
  ep.act = act;
  ep.relu = relu;
  return pipelined(w, 2, a, 1, m, k, n, nullptr, n, ep, s);
}

// host-side introspection of the CRT scheme (no device needed): the plan of a
// K-long product and the constants of an n-moduli reconstruction
int ozaki_crt_info(int64_t k, int ncb, int* n, int* pa, int* pb) {
  const mcfg::oz::CrtPlan pl = mcfg::oz::crt_plan(k, ncb);
  if (n) *n = pl.n;
  if (pa) *pa = pl.pa;
  if (pb) *pb = pl.pb;
  return pl.n;
}
int ozaki_crt_table(int n, int* moduli, float* w, float* mh, float* cq, int* bits) {
  using namespace mcfg::oz;
  if (n < 1 || n > kMaxMod) return 0;
  const HostCrt& h = host_crt();
  for (int t = 0; t < n; ++t) {
    if (moduli) moduli[t] = kModuli[t];
    for (int j = 0; j < kSlices; ++j)
      if (w) w[t * kSlices + j] = h.tab[n].w[t][j];
  }
  for (int j = 0; j < kSlices; ++j)
    if (mh) mh[j] = h.tab[n].mh[j];
  if (cq) *cq = h.tab[n].cq;
  if (bits) *bits = h.tab[n].L;
  return kSlices;
}

// moduli of a K = 4096 MC x T product (ABI compatibility: mcf_fast_tc_digits)
int ozaki_digits() { return mcfg::oz::crt_plan(4096, 1).n; }

// int8 GEMMs (M x N x K each) per product: one per modulus
int ozaki_gemm_equivalents(int ncb, int64_t k) { return mcfg::oz::crt_plan(k, ncb).n; }

// one product with phase timing: ms[0] B residues, ms[1] A residues, ms[2] the
// int8 GEMMs, ms[3] reconstruction + fallback; *fallback = listed outputs
// grows the stream's residue-plane workspace to what an m x k x n product
// with an ncb-component B needs (so that the product itself allocates nothing)
mcf_status ozaki_reserve(int64_t m, int64_t k, int64_t n, int ncb, cudaStream_t s) {
  using namespace mcfg::oz;
  if (!ozaki_supported(m, k, n) || (ncb != 1 && ncb != 2))
    return fail(MCF_ERR_UNSUPPORTED, "mm_fast: shape outside the tensor-core path");
  int nb;
  int64_t rb;
  if (!oz_workspace(pipe_geometry(m, k, n, ncb, nb, rb), s))
    return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the residue-plane workspace");
  return upload_crt_tables();
}

mcf_status ozaki_phases(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out, double* ms,
                        int64_t* fallback, cudaStream_t s) {
  using namespace mcfg::oz;
  if (!ozaki_supported(m, k, n)) return fail(MCF_ERR_UNSUPPORTED, "mm_fast: shape outside the tensor-core path");
  const std::size_t bb = al(b_bytes(k, n, 1));
  char* ws = oz_workspace(bb + al(rows_bytes(m, k, n, 1)), s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the residue-plane workspace");
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  cudaEventRecord(ev[4], s);
  PreparedB pb;
  mcf_status st = prepare_b(w, 1, k, n, n, ws, pb, s);
  if (st == MCF_OK) st = rows(x, 2, m, pb, out, n, ws + bb, s, ev);
  if (st == MCF_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(MCF_ERR_CUDA, "mm_fast: sync");
  if (st == MCF_OK) {
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[4], ev[0]);
    ms[0] = t;
    for (int i = 0; i < 3; ++i) {
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      ms[i + 1] = t;
    }
    const RowsWs rw = rows_ws(ws + bb, m, pb.kp, pb.np, pb.plan.n);
    std::vector<int> rc(m);
    cudaMemcpy(rc.data(), rw.rcnt, m * sizeof(int), cudaMemcpyDeviceToHost);
    int64_t c = 0;
    for (int v : rc) c += v;
    *fallback = c;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return st;
}

// Host-buffer MC(nc=2, binary32) x T on the tensor-core path, pipelined in
// two dimensions: B is sent and prepared in column blocks (each block is
// independent: per-column scaling), A in row chunks; the copy stream sends B
// block 0, A chunk 0, the remaining B blocks, then the remaining A chunks, so
// the first (chunk, block) product starts after two pieces instead of all of
// B.  Products alternate between two compute streams (each with its own
// workspace region); each product's D2H copy (a strided 2-D copy) runs on the
// copy-out stream as soon as it is done.
mcf_status ozaki_host(const float* hx, const float* hw, int64_t m, int64_t k, int64_t n, float* hout, float* dx,
                      float* dw, float* dout, cudaStream_t cin, const cudaStream_t comp[2], cudaStream_t cout) {
  using namespace mcfg::oz;
  if (!ozaki_supported(m, k, n)) return MCF_ERR_UNSUPPORTED;
  static const int64_t chunk_env = [] {
    const char* e = getenv("MCF_OZ_CHUNK");  // tuning knob: rows per chunk
    return e ? atoll(e) : 0LL;
  }();
  static const int64_t blocks_env = [] {
    const char* e = getenv("MCF_OZ_BLOCKS");  // tuning knob: column blocks of B
    return e ? atoll(e) : 0LL;
  }();
  // measured at config 2: 512-row chunks (4.99 ms) beat 256 (6.7), 768 (5.3), 1024 (5.2)
  const int64_t rc = std::min<int64_t>(m, chunk_env > 0 ? chunk_env : std::max<int64_t>(512, (m + 7) / 8));
  const int nch = (int)((m + rc - 1) / rc);
  const int64_t nbk = blocks_env > 0 ? blocks_env : 1;  // measured: column blocks do not pay at config 2
  const int64_t bw = pad16((n + nbk - 1) / nbk);
  const int nb = (int)((n + bw - 1) / bw);
  const std::size_t bb = al(b_bytes(k, bw, 1)), rb = al(rows_bytes(rc, k, bw, 1));
  char* ws = oz_workspace(nb * al(bb) + 2 * rb, comp[0]);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the residue-plane workspace");
  std::vector<cudaEvent_t> evb(nb, nullptr), evp(nb, nullptr), eva(nch, nullptr), evt(nch * nb, nullptr);
  std::vector<cudaEvent_t*> all;
  for (auto* v : {&evb, &evp, &eva, &evt})
    for (auto& e : *v) all.push_back(&e);
  for (auto* e : all)
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess)
      return fail(MCF_ERR_CUDA, "mm_fast: cannot create pipeline events");
  auto done = [&](mcf_status st) {
    for (auto* e : all)
      if (*e) cudaEventDestroy(*e);
    return st;
  };
  auto cu = [&](cudaError_t e, const char* what) {
    return e == cudaSuccess ? MCF_OK : fail(MCF_ERR_CUDA, std::string("mm_mcn pipeline: ") + what + ": " +
                                                              cudaGetErrorString(e));
  };
#define OZ_TRY(expr)                   \
  do {                                 \
    const mcf_status _s = (expr);      \
    if (_s != MCF_OK) return done(_s); \
  } while (0)
  std::vector<PreparedB> pb(nb);
  auto send_b = [&](int b) -> mcf_status {
    const int64_t j0 = b * bw, w = std::min<int64_t>(bw, n - j0);
    mcf_status st = cu(cudaMemcpy2DAsync(dw + j0, n * sizeof(float), hw + j0, n * sizeof(float), w * sizeof(float), k,
                                         cudaMemcpyHostToDevice, cin), "H2D w");
    if (st == MCF_OK) st = cu(cudaEventRecord(evb[b], cin), "event");
    cudaStream_t ps = comp[b & 1];
    if (st == MCF_OK) st = cu(cudaStreamWaitEvent(ps, evb[b], 0), "wait");
    if (st == MCF_OK) st = prepare_b(dw + j0, 1, k, w, n, ws + b * al(bb), pb[b], ps);
    if (st == MCF_OK) st = cu(cudaEventRecord(evp[b], ps), "event");
    return st;
  };
  auto send_a = [&](int c) -> mcf_status {
    const int64_t r0 = c * rc, rows_c = std::min<int64_t>(rc, m - r0);
    mcf_status st = cu(cudaMemcpyAsync(dx + r0 * k * 2, hx + r0 * k * 2, rows_c * k * 2 * sizeof(float),
                                       cudaMemcpyHostToDevice, cin), "H2D x");
    if (st == MCF_OK) st = cu(cudaEventRecord(eva[c], cin), "event");
    return st;
  };
  int task = 0;
  auto product = [&](int c, int b) -> mcf_status {
    const int64_t r0 = c * rc, rows_c = std::min<int64_t>(rc, m - r0);
    const int64_t j0 = b * bw, w = std::min<int64_t>(bw, n - j0);
    cudaStream_t cs = comp[task & 1];
    char* region = ws + nb * al(bb) + (task & 1) * rb;
    ++task;
    mcf_status st = cu(cudaStreamWaitEvent(cs, eva[c], 0), "wait");
    if (st == MCF_OK) st = cu(cudaStreamWaitEvent(cs, evp[b], 0), "wait");
    if (st == MCF_OK) st = rows(dx + r0 * k * 2, 2, rows_c, pb[b], dout + (r0 * n + j0) * 2, n, region, cs);
    cudaEvent_t et = evt[c * nb + b];
    if (st == MCF_OK) st = cu(cudaEventRecord(et, cs), "event");
    if (st == MCF_OK) st = cu(cudaStreamWaitEvent(cout, et, 0), "wait");
    if (st == MCF_OK)
      st = cu(cudaMemcpy2DAsync(hout + (r0 * n + j0) * 2, n * 2 * sizeof(float), dout + (r0 * n + j0) * 2,
                                n * 2 * sizeof(float), w * 2 * sizeof(float), rows_c, cudaMemcpyDeviceToHost,
                                cout), "D2H out");
    return st;
  };
  OZ_TRY(send_b(0));
  OZ_TRY(send_a(0));
  OZ_TRY(product(0, 0));
  for (int b = 1; b < nb; ++b) {
    OZ_TRY(send_b(b));
    OZ_TRY(product(0, b));
  }
  for (int c = 1; c < nch; ++c) {
    OZ_TRY(send_a(c));
    for (int b = 0; b < nb; ++b) OZ_TRY(product(c, b));
  }
#undef OZ_TRY
  return done(cu(cudaStreamSynchronize(cout), "sync"));
}


// Independent int8 GEMMs of one product spread over up to four streams
// forked from s and joined back (same rule as rows_products: short products
// use up to four, full-size ones two for wave-tail filling).
struct GemmFork {
  cudaStream_t st[4];
  int ns = 1, next = 0;
  cudaEvent_t fork = nullptr;
  cudaStream_t base;
  GemmFork(cudaStream_t s, int64_t rows_c, int64_t cols_c) : base(s) {
    const int64_t tiles = ((rows_c + 255) / 256) * ((cols_c + 255) / 256);
    const int sms = mcfr::sm_count();
    ns = 3 * tiles > sms ? 2 : (int)std::max<int64_t>(1, std::min<int64_t>(4, sms / std::max<int64_t>(tiles, 1)));
    for (auto& x : st) x = s;
    if (ns > 1) {
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      cudaEventRecord(fork, s);
      for (int i = 1; i < ns; ++i) {
        st[i] = mcfr::side_stream(12 + i);
        cudaStreamWaitEvent(st[i], fork, 0);
      }
    }
  }
  cudaStream_t take() { return st[next++ % ns]; }
  void join() {
    if (!fork) return;
    for (int i = 1; i < ns; ++i) {
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, st[i]);
      cudaStreamWaitEvent(base, j, 0);
      cudaEventDestroy(j);
    }
    cudaEventDestroy(fork);
    fork = nullptr;
  }
  ~GemmFork() { join(); }
};

// C (m x n, row-major, ldc) = op(A) op(B) in binary32 through four-digit int8
// products (see k_f32_comb above); MCF_ERR_UNSUPPORTED for shapes it does not
// take (the caller runs the FFMA GEMM).  op(A) = A (m x k, lda) or A^T (A
// stored k x m); op(B) = B (k x n, ldb) or B^T (B stored n x k).
mcf_status gemm_f32_i8(int trans_a, int trans_b, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                       int64_t ldc, int64_t m, int64_t n, int64_t k, const float* mask, cudaStream_t s) {
  using namespace mcfg::oz;
  if (m < 64 || n < 64 || k < 64 || k > 32640 || m * n >= (int64_t(1) << 31)) return MCF_ERR_UNSUPPORTED;
  // K padded to the tcgen05 GEMM's 128-byte K block (a diagonal's operand is
  // a run of whole planes: its last block must not reach the next plane)
  const int64_t kp = (k + 127) / 128 * 128, np = pad16(n);
  const std::size_t ba = al(m * kD4 * kp), bb = al(np * kD4 * kp), bq = al(4 * m * np * 4);
  char* ws = oz_workspace(ba + bb + bq + al(m * 4) + al(np * 4), s);
  if (!ws) return fail(MCF_ERR_CUDA, "gemm_f32: cannot allocate the digit-plane workspace");
  int8_t* ap = reinterpret_cast<int8_t*>(ws);
  int8_t* bp = reinterpret_cast<int8_t*>(ws + ba);
  int* cq = reinterpret_cast<int*>(ws + ba + bb);
  unsigned* amx = reinterpret_cast<unsigned*>(ws + ba + bb + bq);
  unsigned* bmx = reinterpret_cast<unsigned*>(ws + ba + bb + bq + al(m * 4));
  if (cudaMemsetAsync(amx, 0, al(m * 4) + al(np * 4), s) != cudaSuccess) return fail(MCF_ERR_CUDA, "gemm_f32: memset");
  // padding k (kp > k) and padding columns (np > n) must read as zero digits
  if (np > n && cudaMemsetAsync(bp + n * kD4 * kp, 0, (np - n) * kD4 * kp, s) != cudaSuccess)
    return fail(MCF_ERR_CUDA, "gemm_f32: memset");
  const int sms = mcfr::sm_count();
  // op(A): rows m along k
  if (!trans_a) {
    k_f32_rowmax<<<(unsigned)m, 256, 0, s>>>(a, m, k, lda, amx);
    const int64_t gx = (kp / 4 + 255) / 256;
    k_f32_dig_rows<false><<<dim3((unsigned)gx, (unsigned)std::min<int64_t>(m, sms * 8 / gx + 1)), 256, 0, s>>>(
        a, m, k, lda, kp, amx, ap);
  } else {
    k_f32_colmax<<<dim3((unsigned)((m + 255) / 256), (unsigned)((k + 63) / 64)), 256, 0, s>>>(a, k, m, lda, amx);
    k_f32_dig_cols<false><<<dim3((unsigned)((m + kSlab - 1) / kSlab), (unsigned)(kp / kSlab)), 256, 0, s>>>(
        a, k, m, lda, kp, amx, ap);
  }
  // op(B): columns n along k
  if (trans_b) {
    k_f32_rowmax<<<(unsigned)n, 256, 0, s>>>(b, n, k, ldb, bmx);
    const int64_t gx = (kp / 4 + 255) / 256;
    k_f32_dig_rows<true><<<dim3((unsigned)gx, (unsigned)std::min<int64_t>(n, sms * 8 / gx + 1)), 256, 0, s>>>(
        b, n, k, ldb, kp, bmx, bp);
  } else {
    k_f32_colmax<<<dim3((unsigned)((n + 255) / 256), (unsigned)((k + 63) / 64)), 256, 0, s>>>(b, k, n, ldb, bmx);
    k_f32_dig_cols<true><<<dim3((unsigned)((n + kSlab - 1) / kSlab), (unsigned)(kp / kSlab)), 256, 0, s>>>(
        b, k, n, ldb, kp, bmx, bp);
  }
  for (int i = 0; i < 4; ++i) mcfr::note_launch();
  mcf_status st = mcfr::check_launch("gemm_f32 digit kernels");
  if (st != MCF_OK) return st;
  // diagonal q: A planes s = 0 .. q (ascending) against B planes t = q .. 0
  // (stored reversed at kD4 - 1 - t: ascending positions), pairs (q - t, t):
  // all four diagonals in one launch of the tcgen05 GEMM (MCF_OZ_GEMM=cublaslt:
  // one cuBLASLt GEMM per diagonal)
  static const bool use_lt = [] {
    const char* e = getenv("MCF_OZ_GEMM");
    return e && std::string(e) == "cublaslt";
  }();
  if (!use_lt) {
    int ka[kD4], kb[kD4], kd[kD4];
    for (int q = 0; q < kD4; ++q) {
      ka[q] = 0;
      kb[q] = (int)((kD4 - 1 - q) * kp);
      kd[q] = (int)((q + 1) * kp);
    }
    st = mcfr::tc_gemm_s8_seg(ap, kD4 * kp, bp, kD4 * kp, cq, m, n, np, kD4, ka, kb, kd, np, s);
  } else {
    GemmFork gf(s, np, m);
    for (int q = 0; q < kD4 && st == MCF_OK; ++q) {
      const int th = q, tl = 0;  // pairs (q - t, t), t = 0 .. q (all within four digits)
      const int8_t* bq = bp + (int64_t)(kD4 - 1 - th) * kp;
      const int8_t* aq = ap + (int64_t)(q - th) * kp;
      st = gemm_s8(bq, kD4 * kp, aq, kD4 * kp, cq + (int64_t)q * m * np, np, m, (int64_t)(th - tl + 1) * kp,
                   gf.take());
    }
  }
  if (st != MCF_OK) return st;
  const int64_t gcx = (n + 1023) / 1024;
  k_f32_comb<<<dim3((unsigned)gcx, (unsigned)std::min<int64_t>(m, sms * 8 / gcx + 1)), 256, 0, s>>>(
      cq, m, n, np, amx, bmx, c, ldc, mask);
  mcfr::note_launch();
  return mcfr::check_launch("gemm_f32 combine kernel");
}


// MC binary16 (nc <= 3) x MC binary16 through five-digit int8 products;
// MCF_ERR_UNSUPPORTED outside its shapes (the caller runs the FP64 path)
mcf_status mm_b16_i8(const void* x, const void* y, int nc, int64_t m, int64_t k, int64_t n, void* out,
                     cudaStream_t s) {
  using namespace mcfg::oz;
  if (nc < 1 || nc > 3 || m < 64 || n < 64 || k < 64 || k >= 26000 || m * n >= (int64_t(1) << 31))
    return MCF_ERR_UNSUPPORTED;
  const int64_t kp = (k + 127) / 128 * 128, np = pad16(n);  // whole 128-byte K blocks per plane
  const std::size_t ba = al(m * kD5 * kp), bb = al(np * kD5 * kp), bq = al((int64_t)kD5 * m * np * 4);
  char* ws = oz_workspace(ba + bb + bq + al(m * 8) + al(np * 8), s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_mcmc: cannot allocate the digit-plane workspace");
  int8_t* ap = reinterpret_cast<int8_t*>(ws);
  int8_t* bp = reinterpret_cast<int8_t*>(ws + ba);
  int* cq = reinterpret_cast<int*>(ws + ba + bb);
  auto* amx = reinterpret_cast<unsigned long long*>(ws + ba + bb + bq);
  auto* bmx = reinterpret_cast<unsigned long long*>(ws + ba + bb + bq + al(m * 8));
  if (cudaMemsetAsync(amx, 0, al(m * 8) + al(np * 8), s) != cudaSuccess ||
      (np > n && cudaMemsetAsync(bp + n * kD5 * kp, 0, (np - n) * kD5 * kp, s) != cudaSuccess))
    return fail(MCF_ERR_CUDA, "mm_mcmc: memset");
  const __half* xh = static_cast<const __half*>(x);
  const __half* yh = static_cast<const __half*>(y);
  const int sms = mcfr::sm_count();
  const int64_t gx = (kp / 4 + 255) / 256;
  const dim3 gdr((unsigned)gx, (unsigned)std::min<int64_t>(m, sms * 8 / gx + 1));
  const dim3 gcm((unsigned)((n + 255) / 256), (unsigned)((k + 63) / 64));
  const dim3 gdc((unsigned)((n + kSlab - 1) / kSlab), (unsigned)(kp / kSlab));
  switch (nc) {
#define B16_PREP(NC)                                                           \
  case NC:                                                                     \
    k_b16_rowmax<NC><<<(unsigned)m, 256, 0, s>>>(xh, k, amx);                  \
    k_b16_dig_rows<NC><<<gdr, 256, 0, s>>>(xh, m, k, kp, amx, ap);             \
    k_b16_colmax<NC><<<gcm, 256, 0, s>>>(yh, k, n, bmx);                       \
    k_b16_dig_cols<NC><<<gdc, 256, 0, s>>>(yh, k, n, kp, bmx, bp);             \
    break;
    B16_PREP(1)
    B16_PREP(2)
    B16_PREP(3)
#undef B16_PREP
  }
  for (int i = 0; i < 4; ++i) mcfr::note_launch();
  mcf_status st = mcfr::check_launch("mm_mcmc binary16 digit kernels");
  static const bool use_lt = [] {
    const char* e = getenv("MCF_OZ_GEMM");
    return e && std::string(e) == "cublaslt";
  }();
  if (st == MCF_OK && !use_lt) {
    // the five diagonals in one tcgen05 launch (A planes 0..q against B planes q..0)
    int ka[kD5], kb[kD5], kd[kD5];
    for (int q = 0; q < kD5; ++q) {
      ka[q] = 0;
      kb[q] = (int)((kD5 - 1 - q) * kp);
      kd[q] = (int)((q + 1) * kp);
    }
    st = mcfr::tc_gemm_s8_seg(ap, kD5 * kp, bp, kD5 * kp, cq, m, n, np, kD5, ka, kb, kd, np, s);
  } else if (st == MCF_OK) {
    GemmFork gf(s, np, m);
    for (int q = 0; q < kD5 && st == MCF_OK; ++q)
      st = gemm_s8(bp + (int64_t)(kD5 - 1 - q) * kp, kD5 * kp, ap, kD5 * kp, cq + (int64_t)q * m * np, np, m,
                   (int64_t)(q + 1) * kp, gf.take());
  }
  if (st != MCF_OK) return st;
  const dim3 gc((unsigned)((n + 255) / 256), (unsigned)std::min<int64_t>(m, sms * 8 / ((n + 255) / 256) + 1));
  __half* oh = static_cast<__half*>(out);
  if (nc == 1) k_b16_comb<1><<<gc, 256, 0, s>>>(cq, m, n, np, amx, bmx, oh);
  else if (nc == 2) k_b16_comb<2><<<gc, 256, 0, s>>>(cq, m, n, np, amx, bmx, oh);
  else k_b16_comb<3><<<gc, 256, 0, s>>>(cq, m, n, np, amx, bmx, oh);
  mcfr::note_launch();
  return mcfr::check_launch("mm_mcmc binary16 combine kernel");
}

}  // namespace mcfr
