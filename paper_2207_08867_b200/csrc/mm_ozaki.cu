// mm_ozaki.cu -- MCF_FAST MC contractions on the INT8 tensor cores.
//
// The reference's mm_mcn (linalg.hpp:138-157) accumulates every output in MC
// arithmetic; its error is set by the nc-component result (2^-51.7
// median / 2^-49.1 max at nc=2 fp32).  On B200 the fastest exact arithmetic
// for a GEMM is the INT8 tensor core (int32 accumulation is exact), so the
// product is computed as an error-free integer splitting (Ozaki scheme):
//
//   * every row i of A is scaled by 2^-ea[i] and every column j of B by
//     2^-eb[j] (powers of two, exact) so all values lie in (-1, 1);
//   * each scaled value v = c0 + c1 (exact binary64 pair) becomes kS signed
//     digits d_s in [-64, 64] with weights 2^(-6-7s) (round to nearest, the
//     remainder carried exactly), |v - sum| <= 2^(-7 kS) (1 + 2^-50);
//   * for each diagonal q = s + t < kS one int8 GEMM with the digit planes
//     concatenated along K gives C_q = sum_{s+t=q} A_s B_t exactly in int32
//     ((q+1) Kp 64^2 < 2^31 for Kp <= 50000);
//   * C = sum_q C_q 2^(-12-7q) is formed exactly in double-double, scaled
//     back and split greedily into the nc output components.
//
// Error per product <= (kS + 1.1) 2^(-7 kS) (scaled units), so per output
// <= K (kS + 1.1) 2^(-7 kS).  Outputs whose magnitude is not at least 2^51
// times that bound (cancellation; rows or columns holding Inf/NaN) are put on
// a work list and recomputed by a warp each in double-double from the fp32
// operands, so every output has relative error <= 2^-51 before the final
// split -- the same bound the reference's own nc=2 result representation sets.
//
// The int8 GEMMs are plain library GEMMs (cuBLASLt IMMA, TN, int32 out); the
// digit extraction, the transposes, the recombination + split and the
// cancellation fallback are this file's kernels.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "mcf_accum.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace oz {
namespace {

constexpr int kS = 10;             // digits per operand
constexpr int kSlab = 32;          // transpose tile of the column slicer
constexpr int64_t kMaxKp = 50000;  // int32 headroom: kS * Kp * 64 * 64 < 2^31

__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// 2^e > m (m >= 0 finite), 0 for m == 0 or non-finite (those rows / columns
// go to the fallback list)
__device__ __forceinline__ int exp_above_d(double m) { return m > 0.0 && isfinite(m) ? ilogb(m) + 1 : 0; }

// kS signed digits of hi + lo (|hi + lo| < 1): digit s has weight 2^(-6-7s)
__device__ __forceinline__ void digits(double hi, double lo, int (&d)[kS]) {
  double h = __dmul_rn(hi, 64.0), l = __dmul_rn(lo, 64.0);
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    const double a = rint(h);
    d[s] = (int)a;
    double sh, sl;
    dsum(__dsub_rn(h, a), l, sh, sl);
    h = __dmul_rn(sh, 128.0);
    l = __dmul_rn(sl, 128.0);
  }
}

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

// row exponents of A (rows x k, NC comps): warp per row, max of |c0| + |c1|
template <int NC>
__global__ void __launch_bounds__(256) k_rowexp(const float* __restrict__ a, int64_t rows, int64_t k,
                                                 int* __restrict__ e, int* __restrict__ nf) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double m = 0.0;
  bool bad = false;
  for (int64_t t = lane; t < k; t += 32) {
    double hi, lo, mag;
    load_pair<NC>(a + (r * k + t) * NC, hi, lo, mag);
    bad |= !isfinite(mag);
    m = fmax(m, mag);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    e[r] = exp_above_d(m);
    nf[r] = bad ? 1 : 0;
  }
}

// column maxima of B (k x n, NC comps): slabs of 64 rows, atomicMax on the
// binary64 bit pattern (monotone for non-negative values; cm starts at 0)
template <int NC>
__global__ void __launch_bounds__(256) k_colmax(const float* __restrict__ b, int64_t k, int64_t n,
                                                 unsigned long long* __restrict__ cm, int* __restrict__ nf) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t t0 = (int64_t)blockIdx.y * 64, t1 = t0 + 64 < k ? t0 + 64 : k;
  double m = 0.0;
  bool bad = false;
  for (int64_t t = t0; t < t1; ++t) {
    double hi, lo, mag;
    load_pair<NC>(b + (t * n + j) * NC, hi, lo, mag);
    bad |= !isfinite(mag);
    m = fmax(m, mag);
  }
  if (m > 0.0) atomicMax(cm + j, (unsigned long long)__double_as_longlong(m));
  if (bad) nf[j] = 1;
}

__global__ void __launch_bounds__(256) k_colexp(const unsigned long long* __restrict__ cm, int64_t n,
                                                 int* __restrict__ e) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) e[j] = exp_above_d(__longlong_as_double((long long)cm[j]));
}

// A (rows x k, NC comps) -> digit planes, row-major rows of kS * kp bytes:
// out[i, s * kp + k] = digit s of A[i, k] 2^-e[i]; zero for k >= K.
// Each thread makes 4 consecutive k (one 32-bit store per digit).
template <int NC>
__global__ void __launch_bounds__(256) k_slice_rows(const float* __restrict__ a, int64_t rows, int64_t k, int64_t kp,
                                                     const int* __restrict__ e, int8_t* __restrict__ out) {
  const int64_t q4 = kp / 4;
  const int64_t total = rows * q4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int64_t i = q / q4, k0 = (q % q4) * 4;
    const double sc = pow2d(-e[i]);
    unsigned packed[kS];
#pragma unroll
    for (int s = 0; s < kS; ++s) packed[s] = 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (k0 + u >= k) break;
      double hi, lo, mag;
      load_pair<NC>(a + (i * k + k0 + u) * NC, hi, lo, mag);
      int d[kS];
      if (isfinite(mag)) {
        digits(__dmul_rn(hi, sc), __dmul_rn(lo, sc), d);
      } else {
#pragma unroll
        for (int s = 0; s < kS; ++s) d[s] = 0;
      }
#pragma unroll
      for (int s = 0; s < kS; ++s) packed[s] |= ((unsigned)(d[s] & 0xff)) << (8 * u);
    }
    int8_t* row = out + i * (kS * kp) + k0;
#pragma unroll
    for (int s = 0; s < kS; ++s) *reinterpret_cast<unsigned*>(row + s * kp) = packed[s];
  }
}

// B (k x n, NC comps, row-major) -> digit planes transposed, rows of kS * kp
// bytes per column j with the planes in reverse order,
//   out[j, (kS - 1 - t) * kp + k] = digit t of B[k, j] 2^-e[j],
// so the diagonal-q operand (planes q, q-1, .., 0) is one contiguous run; and
// bt[j, k, :] = B[k, j, :] (binary32, for the fallback list).
template <int NC>
__global__ void __launch_bounds__(256) k_slice_cols(const float* __restrict__ b, int64_t k, int64_t n, int64_t kp,
                                                     const int* __restrict__ e, int8_t* __restrict__ out,
                                                     float* __restrict__ bt) {
  __shared__ __align__(16) int8_t dg[kS][kSlab][kSlab];  // [t][j][k]
  __shared__ float tv[kSlab][kSlab * NC + 1];             // [j][k * NC + c]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  const int64_t k0 = (int64_t)blockIdx.y * kSlab, j0 = (int64_t)blockIdx.x * kSlab;
  const int64_t j = j0 + tx;
  const double sc = j < n ? pow2d(-e[j]) : 1.0;
#pragma unroll
  for (int r = 0; r < kSlab / 8; ++r) {
    const int kk = ty + 8 * r;
    const int64_t gk = k0 + kk;
    int d[kS];
#pragma unroll
    for (int s = 0; s < kS; ++s) d[s] = 0;
    if (gk < k && j < n) {
      double hi, lo, mag;
      load_pair<NC>(b + (gk * n + j) * NC, hi, lo, mag);
#pragma unroll
      for (int c = 0; c < NC; ++c) tv[tx][kk * NC + c] = b[(gk * n + j) * NC + c];
      if (isfinite(mag)) digits(__dmul_rn(hi, sc), __dmul_rn(lo, sc), d);
    }
#pragma unroll
    for (int s = 0; s < kS; ++s) dg[s][tx][kk] = (int8_t)d[s];
  }
  __syncthreads();
  // digit rows: kS * 32 rows (t, jj) of 32 bytes; 8 threads x 4 bytes per row
  for (int w = threadIdx.x; w < kS * kSlab * 8; w += blockDim.x) {
    const int row = w / 8, part = w % 8;
    const int t = row / kSlab, jj = row % kSlab;
    const int64_t gj = j0 + jj;
    if (gj >= n || k0 + part * 4 >= kp) continue;
    *reinterpret_cast<unsigned*>(out + gj * (kS * kp) + (kS - 1 - t) * kp + k0 + part * 4) =
        *reinterpret_cast<const unsigned*>(&dg[t][jj][part * 4]);
  }
  // transposed binary32 copy
  for (int w = threadIdx.x; w < kSlab * kSlab * NC; w += blockDim.x) {
    const int jj = w / (kSlab * NC), rest = w % (kSlab * NC);
    const int kk = rest / NC;
    const int64_t gj = j0 + jj, gk = k0 + kk;
    if (gj < n && gk < k) bt[(gj * k + gk) * NC + rest % NC] = tv[jj][rest];
  }
}

// C = sum_q C_q 2^(-12-7q) (exact double-double), scaled back, split into
// two binary32 components; ill-conditioned / non-finite outputs are listed
// for the fallback instead.
__global__ void __launch_bounds__(256) k_combine(const int* __restrict__ cq, int64_t m, int64_t n, int64_t ldc,
                                                 const int* __restrict__ ea, const int* __restrict__ eb,
                                                 const int* __restrict__ rnf, const int* __restrict__ cnf,
                                                 double thr, float* __restrict__ out, int* __restrict__ list,
                                                 int* __restrict__ count) {
  const int64_t mn = m * n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < mn; x += stride) {
    const int64_t i = x / n, j = x % n;
    double hi = 0.0, lo = 0.0;
#pragma unroll
    for (int q = kS - 1; q >= 0; --q) {
      const double t = __dmul_rn((double)cq[q * m * ldc + i * ldc + j], pow2d(-12 - 7 * q));
      double s, err;
      dsum(hi, t, s, err);
      hi = s;
      lo = __dadd_rn(lo, err);
    }
    double s2, e2;
    dsum(hi, lo, s2, e2);
    if (rnf[i] | cnf[j] || !(fabs(s2) >= thr)) {
      list[atomicAdd(count, 1)] = (int)x;
      continue;
    }
    const double sc = pow2d(ea[i] + eb[j]);
    const double v[2] = {__dmul_rn(s2, sc), __dmul_rn(e2, sc)};
    split_out<float, 2, 2>(v, out + x * 2);
  }
}

// the listed outputs, a warp each: products of binary32 components are exact
// in binary64; each lane keeps a double-double (two_sum into S, errors into
// C), lanes merge by an xor butterfly (the same value on every lane)
template <int NCA, int NCB>
__global__ void __launch_bounds__(256) k_fallback(const float* __restrict__ a, const float* __restrict__ bt,
                                                  int64_t n, int64_t k, const int* __restrict__ list,
                                                  const int* __restrict__ count, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int cnt = *count;
  for (int64_t w = gw; w < cnt; w += nw) {
    const int64_t x = list[w];
    const int64_t i = x / n, j = x % n;
    const float* ar = a + i * k * NCA;
    const float* br = bt + j * k * NCB;
    double S = 0.0, C = 0.0;
    for (int64_t t = lane; t < k; t += 32) {
#pragma unroll
      for (int ca = 0; ca < NCA; ++ca)
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) {
          const double p = __dmul_rn((double)ar[t * NCA + ca], (double)br[t * NCB + cb]);
          double e;
          dsum(S, p, S, e);
          C = __dadd_rn(C, e);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oS = __shfl_xor_sync(0xffffffffu, S, off), oC = __shfl_xor_sync(0xffffffffu, C, off);
      double e;
      dsum(S, oS, S, e);
      C = __dadd_rn(__dadd_rn(C, oC), e);
    }
    if (lane == 0) {
      const double v[2] = {S, C};
      split_out<float, 2, 2>(v, out + x * 2);
    }
  }
}

// ---- cuBLASLt int8 GEMMs ------------------------------------------------------------------

struct Lt {
  cublasLtHandle_t h = nullptr;
  void* ws = nullptr;
  std::size_t ws_bytes = 0;
  std::map<std::tuple<int64_t, int64_t, int64_t, int64_t>, cublasLtMatmulAlgo_t> algos;
};
std::mutex g_lt_mu;
std::map<int, Lt> g_lt;

mcf_status lt_fail(const char* what, int code) {
  return mcfr::fail(MCF_ERR_CUDA, std::string("mm_fast int8 GEMM: ") + what + " (status " + std::to_string(code) + ")");
}

// C (rows_c x cols_c, col-major, ld rows_c, int32) = opA^T(A) . B, with
// A: kd x rows_c int8 col-major (ld lda), B: kd x cols_c int8 col-major (ld ldb)
mcf_status gemm_s8(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int* C, int64_t rows_c,
                   int64_t cols_c, int64_t kd, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_lt_mu);
  Lt& lt = g_lt[dev];
  if (!lt.h) {
    const cublasStatus_t st = cublasLtCreate(&lt.h);
    if (st != CUBLAS_STATUS_SUCCESS) return lt_fail("cublasLtCreate", st);
    lt.ws_bytes = 64u << 20;
    if (cudaMalloc(&lt.ws, lt.ws_bytes) != cudaSuccess) return lt_fail("workspace", 0);
  }
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasStatus_t st = cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I);
  const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
  if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
  if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, kd, rows_c, lda);
  if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, kd, cols_c, ldb);
  if (st == CUBLAS_STATUS_SUCCESS) st = cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, rows_c, cols_c, rows_c);
  auto cleanup = [&]() {
    if (lc) cublasLtMatrixLayoutDestroy(lc);
    if (lb) cublasLtMatrixLayoutDestroy(lb);
    if (la) cublasLtMatrixLayoutDestroy(la);
    if (op) cublasLtMatmulDescDestroy(op);
  };
  if (st != CUBLAS_STATUS_SUCCESS) {
    cleanup();
    return lt_fail("descriptors", st);
  }
  const auto key = std::make_tuple(rows_c, cols_c, kd, lda);
  auto it = lt.algos.find(key);
  if (it == lt.algos.end()) {
    cublasLtMatmulPreference_t pref = nullptr;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &lt.ws_bytes,
                                         sizeof(lt.ws_bytes));
    cublasLtMatmulHeuristicResult_t res{};
    int found = 0;
    st = cublasLtMatmulAlgoGetHeuristic(lt.h, op, la, lb, lc, lc, pref, 1, &res, &found);
    cublasLtMatmulPreferenceDestroy(pref);
    if (st != CUBLAS_STATUS_SUCCESS || found == 0) {
      cleanup();
      return MCF_ERR_UNSUPPORTED;  // caller runs the FP64-pipe kernel instead
    }
    it = lt.algos.emplace(key, res.algo).first;
  }
  const int32_t alpha = 1, beta = 0;
  st = cublasLtMatmul(lt.h, op, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &it->second, lt.ws, lt.ws_bytes, s);
  cleanup();
  if (st != CUBLAS_STATUS_SUCCESS) return lt_fail("cublasLtMatmul", st);
  mcfr::note_launch();
  return MCF_OK;
}

// per-(device, stream) workspace for the digit planes and partial products
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

}  // namespace

// Prepared B operand: digit planes, column exponents, non-finite flags and
// the transposed binary32 copy.  Built once; shared by row chunks of A.
struct PreparedB {
  const int8_t* planes = nullptr;
  const float* bt = nullptr;
  const int* eb = nullptr;
  const int* cnf = nullptr;
  int64_t k = 0, kp = 0, n = 0, np = 0;  // np: n padded to 16 (int8 GEMM alignment)
  int ncb = 1;
};

int64_t pad16(int64_t v) { return (v + 15) / 16 * 16; }

std::size_t b_bytes(int64_t k, int64_t n, int ncb) {
  const int64_t kp = pad16(k), np = pad16(n);
  return al(np * kS * kp) + al(n * k * ncb * 4) + al(n * 4) * 2 + al(n * 8);
}

mcf_status prepare_b(const float* w, int ncb, int64_t k, int64_t n, char* buf, PreparedB& pb, cudaStream_t s) {
  const int64_t kp = pad16(k), np = pad16(n);
  int8_t* planes = reinterpret_cast<int8_t*>(buf);
  buf += al(np * kS * kp);
  if (np > n && cudaMemsetAsync(planes + n * kS * kp, 0, (np - n) * kS * kp, s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the padding columns");
  float* bt = reinterpret_cast<float*>(buf);
  buf += al(n * k * ncb * 4);
  int* eb = reinterpret_cast<int*>(buf);
  buf += al(n * 4);
  int* cnf = reinterpret_cast<int*>(buf);
  buf += al(n * 4);
  unsigned long long* cm = reinterpret_cast<unsigned long long*>(buf);
  if (cudaMemsetAsync(cnf, 0, n * 4, s) != cudaSuccess || cudaMemsetAsync(cm, 0, n * 8, s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the column maxima");
  const dim3 gm((unsigned)((n + 255) / 256), (unsigned)((k + 63) / 64));
  if (ncb == 2) k_colmax<2><<<gm, 256, 0, s>>>(w, k, n, cm, cnf);
  else k_colmax<1><<<gm, 256, 0, s>>>(w, k, n, cm, cnf);
  k_colexp<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cm, n, eb);
  const dim3 gs((unsigned)((n + kSlab - 1) / kSlab), (unsigned)((kp + kSlab - 1) / kSlab));
  if (ncb == 2) k_slice_cols<2><<<gs, 256, 0, s>>>(w, k, n, kp, eb, planes, bt);
  else k_slice_cols<1><<<gs, 256, 0, s>>>(w, k, n, kp, eb, planes, bt);
  for (int i = 0; i < 4; ++i) mcfr::note_launch();
  pb = PreparedB{planes, bt, eb, cnf, k, kp, n, np, ncb};
  return mcfr::check_launch("mm_fast B digit kernels");
}

std::size_t rows_bytes(int64_t m, int64_t k, int64_t n) {
  const int64_t kp = pad16(k), np = pad16(n);
  return al(m * kS * kp) + al((int64_t)kS * m * np * 4) + al(m * n * 4) + al(m * 4) * 2 + 256;
}

// out (m x n x 2 binary32) = A (m x k x nca) . B for a prepared B
// ev (optional, 4 events): recorded before the A digits, before the GEMMs,
// after the GEMMs and at the end (phase timing for the benchmark)
mcf_status rows(const float* x, int nca, int64_t m, const PreparedB& pb, float* out, char* buf, cudaStream_t s,
                cudaEvent_t* ev = nullptr) {
  const int64_t k = pb.k, kp = pb.kp, n = pb.n, np = pb.np;
  int8_t* planes = reinterpret_cast<int8_t*>(buf);
  buf += al(m * kS * kp);
  int* cq = reinterpret_cast<int*>(buf);
  buf += al((int64_t)kS * m * np * 4);
  int* list = reinterpret_cast<int*>(buf);
  buf += al(m * n * 4);
  int* ea = reinterpret_cast<int*>(buf);
  buf += al(m * 4);
  int* rnf = reinterpret_cast<int*>(buf);
  buf += al(m * 4);
  int* count = reinterpret_cast<int*>(buf);
  if (ev) cudaEventRecord(ev[0], s);
  if (cudaMemsetAsync(count, 0, sizeof(int), s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mm_fast: cannot clear the fallback counter");
  const unsigned gr = (unsigned)((m + 7) / 8);
  if (nca == 2) k_rowexp<2><<<gr, 256, 0, s>>>(x, m, k, ea, rnf);
  else k_rowexp<1><<<gr, 256, 0, s>>>(x, m, k, ea, rnf);
  const int gsl = mcfr::grid_for(m * (kp / 4), 256, 8);
  if (nca == 2) k_slice_rows<2><<<gsl, 256, 0, s>>>(x, m, k, kp, ea, planes);
  else k_slice_rows<1><<<gsl, 256, 0, s>>>(x, m, k, kp, ea, planes);
  mcfr::note_launch();
  mcfr::note_launch();
  mcf_status st = mcfr::check_launch("mm_fast A digit kernels");
  if (st != MCF_OK) return st;
  // diagonal q: A planes 0..q (the first (q+1) kp bytes of each row) against
  // B planes q..0 (the last (q+1) kp bytes of each column row); C_q is
  // produced as an n x m column-major = m x n row-major int32 matrix
  if (ev) cudaEventRecord(ev[1], s);
  for (int q = 0; q < kS; ++q) {
    st = gemm_s8(pb.planes + (int64_t)(kS - 1 - q) * kp, kS * kp, planes, kS * kp, cq + (int64_t)q * m * np, np, m,
                 (int64_t)(q + 1) * kp, s);
    if (st != MCF_OK) return st;
  }
  if (ev) cudaEventRecord(ev[2], s);
  // fallback threshold (scaled units): 2^51 K (kS + 1.1) 2^(-7 kS)
  const double thr = ldexp((double)k * (kS + 1.1), 51 - 7 * kS);
  k_combine<<<mcfr::grid_for(m * n, 256, 8), 256, 0, s>>>(cq, m, n, np, ea, pb.eb, rnf, pb.cnf, thr, out, list, count);
  mcfr::note_launch();
  const int gf = mcfr::sm_count() * 8;
  if (nca == 2 && pb.ncb == 2) k_fallback<2, 2><<<gf, 256, 0, s>>>(x, pb.bt, n, k, list, count, out);
  else if (nca == 2) k_fallback<2, 1><<<gf, 256, 0, s>>>(x, pb.bt, n, k, list, count, out);
  else if (pb.ncb == 2) k_fallback<1, 2><<<gf, 256, 0, s>>>(x, pb.bt, n, k, list, count, out);
  else k_fallback<1, 1><<<gf, 256, 0, s>>>(x, pb.bt, n, k, list, count, out);
  mcfr::note_launch();
  if (ev) cudaEventRecord(ev[3], s);
  return mcfr::check_launch("mm_fast combine kernels");
}

}  // namespace oz
}  // namespace mcfg

namespace mcfr {

bool ozaki_supported(int64_t m, int64_t k, int64_t n) {
  return m > 0 && n > 0 && k > 0 && (k + 15) / 16 * 16 <= mcfg::oz::kMaxKp && m * n < (int64_t(1) << 31);
}

// one-call MC(nc=2, binary32) x T / MC(nc=2) product on the INT8 tensor cores
mcf_status mm_ozaki(const float* x, int nca, const float* w, int ncb, int64_t m, int64_t k, int64_t n, float* out,
                    cudaStream_t s) {
  using namespace mcfg::oz;
  const std::size_t bb = b_bytes(k, n, ncb);
  char* ws = oz_workspace(bb + rows_bytes(m, k, n), s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the digit-plane workspace");
  PreparedB pb;
  mcf_status st = prepare_b(w, ncb, k, n, ws, pb, s);
  if (st != MCF_OK) return st;
  return rows(x, nca, m, pb, out, ws + bb, s);
}

int ozaki_digits() { return mcfg::oz::kS; }

// one product with phase timing: ms[0] B digits, ms[1] A digits, ms[2] the
// int8 GEMMs, ms[3] recombination + fallback; *fallback = listed outputs
mcf_status ozaki_phases(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out, double* ms,
                        int64_t* fallback, cudaStream_t s) {
  using namespace mcfg::oz;
  if (!ozaki_supported(m, k, n)) return fail(MCF_ERR_UNSUPPORTED, "mm_fast: shape outside the tensor-core path");
  const std::size_t bb = b_bytes(k, n, 1);
  char* ws = oz_workspace(bb + rows_bytes(m, k, n), s);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the digit-plane workspace");
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  cudaEventRecord(ev[4], s);
  PreparedB pb;
  mcf_status st = prepare_b(w, 1, k, n, ws, pb, s);
  if (st == MCF_OK) st = rows(x, 2, m, pb, out, ws + bb, s, ev);
  if (st == MCF_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(MCF_ERR_CUDA, "mm_fast: sync");
  if (st == MCF_OK) {
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[4], ev[0]);
    ms[0] = t;
    for (int i = 0; i < 3; ++i) {
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      ms[i + 1] = t;
    }
    // the fallback counter sits at the end of the rows region
    const int64_t kp = pad16(k), np = pad16(n);
    const char* cnt = ws + bb + al(m * kS * kp) + al((int64_t)kS * m * np * 4) + al(m * n * 4) + al(m * 4) * 2;
    int c = 0;
    cudaMemcpy(&c, cnt, sizeof(int), cudaMemcpyDeviceToHost);
    *fallback = c;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return st;
}

}  // namespace mcfr

namespace mcfr {

// Host-buffer MC(nc=2, binary32) x T on the tensor-core path, pipelined over
// row chunks: B is copied and prepared once; chunk c's H2D copy (cin), digit
// planes + GEMMs + combine (comp[c % 2], each with its own workspace region)
// and D2H copy (cout) overlap the neighbouring chunks.
mcf_status ozaki_host(const float* hx, const float* hw, int64_t m, int64_t k, int64_t n, float* hout, float* dx,
                      float* dw, float* dout, cudaStream_t cin, const cudaStream_t comp[2], cudaStream_t cout) {
  using namespace mcfg::oz;
  if (!ozaki_supported(m, k, n)) return MCF_ERR_UNSUPPORTED;
  const int64_t rc = std::min<int64_t>(m, std::max<int64_t>(1024, (m + 3) / 4));
  const int nch = (int)((m + rc - 1) / rc);
  const std::size_t bb = b_bytes(k, n, 1), rb = rows_bytes(rc, k, n);
  char* ws = oz_workspace(bb + 2 * rb, comp[0]);
  if (!ws) return fail(MCF_ERR_CUDA, "mm_fast: cannot allocate the digit-plane workspace");
  std::vector<cudaEvent_t> ev(2 * nch + 2, nullptr);
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return fail(MCF_ERR_CUDA, "mm_fast: cannot create pipeline events");
  auto done = [&](mcf_status st) {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
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
  OZ_TRY(cu(cudaMemcpyAsync(dw, hw, k * n * sizeof(float), cudaMemcpyHostToDevice, cin), "H2D w"));
  OZ_TRY(cu(cudaEventRecord(ev[0], cin), "event"));
  OZ_TRY(cu(cudaStreamWaitEvent(comp[0], ev[0], 0), "wait"));
  PreparedB pb;
  OZ_TRY(prepare_b(dw, 1, k, n, ws, pb, comp[0]));
  OZ_TRY(cu(cudaEventRecord(ev[1], comp[0]), "event"));
  OZ_TRY(cu(cudaStreamWaitEvent(comp[1], ev[1], 0), "wait"));
  for (int c = 0; c < nch; ++c) {
    const int64_t r0 = c * rc, rows_c = std::min<int64_t>(rc, m - r0);
    cudaStream_t cs = comp[c & 1];
    cudaEvent_t ex = ev[2 + 2 * c], em = ev[3 + 2 * c];
    OZ_TRY(cu(cudaMemcpyAsync(dx + r0 * k * 2, hx + r0 * k * 2, rows_c * k * 2 * sizeof(float),
                              cudaMemcpyHostToDevice, cin), "H2D x"));
    OZ_TRY(cu(cudaEventRecord(ex, cin), "event"));
    OZ_TRY(cu(cudaStreamWaitEvent(cs, ex, 0), "wait"));
    OZ_TRY(rows(dx + r0 * k * 2, 2, rows_c, pb, dout + r0 * n * 2, ws + bb + (c & 1) * rb, cs));
    OZ_TRY(cu(cudaEventRecord(em, cs), "event"));
    OZ_TRY(cu(cudaStreamWaitEvent(cout, em, 0), "wait"));
    OZ_TRY(cu(cudaMemcpyAsync(hout + r0 * n * 2, dout + r0 * n * 2, rows_c * n * 2 * sizeof(float),
                              cudaMemcpyDeviceToHost, cout), "D2H out"));
  }
#undef OZ_TRY
  return done(cu(cudaStreamSynchronize(cout), "sync"));
}

}  // namespace mcfr
