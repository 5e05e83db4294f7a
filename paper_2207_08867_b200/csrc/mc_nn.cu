// mc_nn.cu -- MC activations, the direct callers of the elementwise operators
// (SURVEY 8f, next row 1):
//   mc_relu_op forward  (autodiff.hpp:340-350): every component of an element
//     is zeroed where approx() <= 0;
//   mc_softmax          (autodiff.hpp:383-413): per slice along the axis
//     m = max approx() (std::max from -inf, in order), e = exp_mcn(grow_expn(x,
//     -m)), denominator = add_kernel fold of e from zeros in order, result =
//     div_mcn(e, denominator).
// Built from the literal per-element kernels (mcf_lit.cuh), so every
// precision and component count is bit-identical to the reference (exp:
// correctly rounded, as in exp_mcn).  The slice reductions (max, the add fold)
// keep the reference's order: one thread per slice; the elementwise stages
// run one thread per element.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "mcf_lit.cuh"
#include "mcf_prec.cuh"
#include "mcf_runtime.h"

namespace mcfg {
namespace {

template <class P>
using RT = typename P::rt;
template <class P>
using ST = typename P::st;

template <class P>
__device__ __forceinline__ void load(const ST<P>* x, int64_t e, int nc, RT<P>* a) {
  for (int c = 0; c < nc; ++c) a[c] = P::ld(x[e * nc + c]);
}
template <class P>
__device__ __forceinline__ void store(ST<P>* x, int64_t e, int nc, const RT<P>* a) {
  for (int c = 0; c < nc; ++c) x[e * nc + c] = P::sv(a[c]);
}

template <class P>
__global__ void __launch_bounds__(256) k_relu(const ST<P>* __restrict__ x, int nc, ST<P>* __restrict__ out,
                                              int64_t numel) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += stride) {
    RT<P> a[lit::kMaxNc];
    load<P>(x, e, nc, a);
    if (lit::approx<P>(a, nc) <= RT<P>(0))
      for (int c = 0; c < nc; ++c) a[c] = RT<P>(0);
    store<P>(out, e, nc, a);
  }
}

// slice s = (ob, ib) of the (outer, n, inner) view; element k of it
__device__ __forceinline__ int64_t elem(int64_t s, int64_t k, int64_t n, int64_t inner) {
  return ((s / inner) * n + k) * inner + s % inner;
}

template <class P>
__global__ void __launch_bounds__(128) k_sm_max(const ST<P>* __restrict__ x, int nc, int64_t slices, int64_t n,
                                                int64_t inner, double* __restrict__ neg_max) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= slices) return;
  RT<P> m = RT<P>(-INFINITY);
  for (int64_t k = 0; k < n; ++k) {
    RT<P> a[lit::kMaxNc];
    load<P>(x, elem(s, k, n, inner), nc, a);
    const RT<P> ax = lit::approx<P>(a, nc);
    if (m < ax) m = ax;  // std::max(m, ax)
  }
  neg_max[s] = -P::to_d(m);
}

// e = exp_mcn(grow_expn(x, -m)) for every element
template <class P>
__global__ void __launch_bounds__(256) k_sm_exp(const ST<P>* __restrict__ x, int nc, int64_t numel, int64_t n,
                                                int64_t inner, const double* __restrict__ neg_max,
                                                ST<P>* __restrict__ e_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += stride) {
    const int64_t s = (e / (n * inner)) * inner + e % inner;
    RT<P> a[lit::kMaxNc], g[lit::kMaxNc], ee[lit::kMaxNc];
    load<P>(x, e, nc, a);
    lit::grow<P>(a, nc, P::rd(neg_max[s]), g);
    lit::exp<P>(g, nc, ee);
    store<P>(e_out, e, nc, ee);
  }
}

// denominator of each slice: add_kernel fold from zeros, in order
template <class P>
__global__ void __launch_bounds__(128) k_sm_den(const ST<P>* __restrict__ ev, int nc, int64_t slices, int64_t n,
                                                int64_t inner, ST<P>* __restrict__ den) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= slices) return;
  RT<P> acc[lit::kMaxNc], ee[lit::kMaxNc];
  for (int c = 0; c < nc; ++c) acc[c] = RT<P>(0);
  for (int64_t k = 0; k < n; ++k) {
    load<P>(ev, elem(s, k, n, inner), nc, ee);
    lit::add<P>(acc, nc, ee, nc, acc, nc);
  }
  store<P>(den, s, nc, acc);
}

template <class P>
__global__ void __launch_bounds__(256) k_sm_div(ST<P>* __restrict__ ev, int nc, int64_t numel, int64_t n,
                                                int64_t inner, const ST<P>* __restrict__ den) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < numel; e += stride) {
    const int64_t s = (e / (n * inner)) * inner + e % inner;
    RT<P> ee[lit::kMaxNc], d[lit::kMaxNc], o[lit::kMaxNc];
    load<P>(ev, e, nc, ee);
    load<P>(den, s, nc, d);
    lit::div<P>(ee, d, nc, o);
    store<P>(ev, e, nc, o);
  }
}

template <class P>
mcf_status relu_prec(const void* x, int nc, void* out, int64_t numel, cudaStream_t s) {
  k_relu<P><<<mcfr::grid_for(numel, 256, 8), 256, 0, s>>>(static_cast<const ST<P>*>(x), nc,
                                                          static_cast<ST<P>*>(out), numel);
  mcfr::note_launch();
  return mcfr::check_launch("mc_relu kernel");
}

template <class P>
mcf_status softmax_prec(const void* xv, int nc, int64_t outer, int64_t n, int64_t inner, void* outv,
                        cudaStream_t s) {
  const ST<P>* x = static_cast<const ST<P>*>(xv);
  ST<P>* out = static_cast<ST<P>*>(outv);
  const int64_t slices = outer * inner, numel = slices * n;
  double* neg_max = nullptr;
  ST<P>* den = nullptr;
  if (cudaMallocAsync(&neg_max, slices * sizeof(double), s) != cudaSuccess ||
      cudaMallocAsync(&den, slices * nc * sizeof(ST<P>), s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mc_softmax: cannot allocate the slice buffers");
  const unsigned gs = (unsigned)((slices + 127) / 128);
  const int ge = mcfr::grid_for(numel, 256, 8);
  k_sm_max<P><<<gs, 128, 0, s>>>(x, nc, slices, n, inner, neg_max);
  k_sm_exp<P><<<ge, 256, 0, s>>>(x, nc, numel, n, inner, neg_max, out);
  k_sm_den<P><<<gs, 128, 0, s>>>(out, nc, slices, n, inner, den);
  k_sm_div<P><<<ge, 256, 0, s>>>(out, nc, numel, n, inner, den);
  for (int i = 0; i < 4; ++i) mcfr::note_launch();
  cudaFreeAsync(neg_max, s);
  cudaFreeAsync(den, s);
  return mcfr::check_launch("mc_softmax kernels");
}

}  // namespace
}  // namespace mcfg

namespace {
// this translation unit's copy of the device exp table (mcf_exp.cuh keeps the
// table per translation unit; lit::exp reads this one)
std::mutex g_tab_mu;
bool g_tab_done[64];
mcf_status ensure_tables_here() {
  const mcf_status st = mcfr::ensure_device_tables();  // stack limit + elementwise copy
  if (st != MCF_OK) return st;
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) d = 0;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (g_tab_done[d]) return MCF_OK;
  double tab[4096];
  mcfr::exp2_table(tab);
  if (cudaMemcpyToSymbol(mcfg::g_exp_tab, tab, sizeof(tab)) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot upload the exp table (mc_nn)");
  g_tab_done[d] = true;
  return MCF_OK;
}
}  // namespace

extern "C" {

mcf_status mcf_mc_relu(mcf_prec p, const void* x, int nc, void* out, int64_t numel, mcf_stream s) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_relu: unknown precision");
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (numel < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_relu: negative element count");
  if (numel == 0) return MCF_OK;
  const mcf_status st = mcfr::ensure_device_tables();
  if (st != MCF_OK) return st;
  switch (p) {
    case MCF_B16: return mcfg::relu_prec<mcfg::PB16>(x, nc, out, numel, s);
    case MCF_B32: return mcfg::relu_prec<mcfg::PB32>(x, nc, out, numel, s);
    default: return mcfg::relu_prec<mcfg::PB64>(x, nc, out, numel, s);
  }
}

mcf_status mcf_mc_softmax(mcf_prec p, const void* x, int nc, int64_t outer, int64_t n, int64_t inner, void* out,
                          mcf_stream s) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_softmax: unknown precision");
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (outer < 0 || n < 0 || inner < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_softmax: negative dimension");
  if (outer * n * inner == 0) return MCF_OK;
  const mcf_status st = ensure_tables_here();
  if (st != MCF_OK) return st;
  switch (p) {
    case MCF_B16: return mcfg::softmax_prec<mcfg::PB16>(x, nc, outer, n, inner, out, s);
    case MCF_B32: return mcfg::softmax_prec<mcfg::PB32>(x, nc, outer, n, inner, out, s);
    default: return mcfg::softmax_prec<mcfg::PB64>(x, nc, outer, n, inner, out, s);
  }
}

}  // extern "C"
