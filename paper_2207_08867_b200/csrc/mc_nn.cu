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
#include <type_traits>

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

// ---- hyperbolic half-space distances (hyperbolic.hpp:160-226; 8f next row 4) ------

template <class P>
__device__ __forceinline__ double max_finite() {
  if constexpr (std::is_same<P, PB16>::value) return 65504.0;
  else if constexpr (std::is_same<P, PB32>::value) return 3.4028234663852886e38;
  else return 1.7976931348623157e308;
}

// one pair per thread: the fused add / square / add fold over the
// coordinates, the canonical-order height product, scale, div, grow, approx
// (halfspace_arg, hyperbolic.hpp:183-212), then arcosh_guarded (:160-170)
template <class P>
__global__ void __launch_bounds__(128) k_halfspace(const ST<P>* __restrict__ table, int nc, int64_t n,
                                                   int64_t dim, const int64_t* __restrict__ us,
                                                   const int64_t* __restrict__ vs, int64_t npairs,
                                                   double* __restrict__ arg_out, double* __restrict__ dist_out,
                                                   int* __restrict__ domain) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npairs) return;
  const int64_t u = us[p], v = vs[p];
  if (u < 0 || u >= n || v < 0 || v >= n) {
    arg_out[p] = __longlong_as_double(0x7ff8000000000000LL);
    if (dist_out) dist_out[p] = arg_out[p];
    return;
  }
  using R = RT<P>;
  R xu[lit::kMaxNc], xv[lit::kMaxNc], neg[lit::kMaxNc], diff[lit::kMaxNc], sq[lit::kMaxNc], s[lit::kMaxNc];
  R hu[lit::kMaxNc], hv[lit::kMaxNc], hprod[lit::kMaxNc], den[lit::kMaxNc], t[lit::kMaxNc], arg[lit::kMaxNc];
  for (int i = 0; i < nc; ++i) s[i] = R(0);
  for (int64_t c = 0; c < dim; ++c) {
    load<P>(table, u * dim + c, nc, xu);
    load<P>(table, v * dim + c, nc, xv);
    for (int i = 0; i < nc; ++i) neg[i] = -xv[i];
    lit::add<P>(xu, nc, neg, nc, diff, nc);
    lit::square<P>(diff, nc, sq);
    lit::add<P>(s, nc, sq, nc, s, nc);
  }
  load<P>(table, u * dim + dim - 1, nc, hu);
  load<P>(table, v * dim + dim - 1, nc, hv);
  bool swap = false;  // comps_less(hv, hu), hyperbolic.hpp:174-179
  for (int i = 0; i < nc; ++i)
    if (hv[i] != hu[i]) {
      swap = hv[i] < hu[i];
      break;
    }
  lit::mul_fast<P>(swap ? hv : hu, swap ? hu : hv, nc, hprod);
  lit::scale<P>(hprod, nc, R(2), den, nc);
  lit::div<P>(s, den, nc, t);
  lit::grow<P>(t, nc, R(1), arg);
  const double a0 = P::to_d(lit::approx<P>(arg, nc));
  arg_out[p] = a0;
  // halfspace_distance's domain (hyperbolic.hpp:219-224): both heights, as
  // their approx values, strictly positive; otherwise NaN and the flag
  const double hua = P::to_d(lit::approx<P>(hu, nc)), hva = P::to_d(lit::approx<P>(hv, nc));
  if (dist_out && !(hua > 0.0 && hva > 0.0)) {
    dist_out[p] = __longlong_as_double(0x7ff8000000000000LL);
    if (domain) atomicOr(domain, 1);
    return;
  }
  if (dist_out) {
    double a = a0 < 1.0 ? 1.0 : a0;
    if (a > max_finite<P>()) a = max_finite<P>();
    double d;
    if (a <= 1.0 + 1e-12) {
      d = sqrt(2.0 * (a - 1.0));
    } else {
      const double inv = 1.0 / a;
      d = log(a) + log1p(sqrt((1.0 - inv) * (1.0 + inv)));
    }
    dist_out[p] = P::to_d(P::rd(d));
  }
}

template <class P>
mcf_status halfspace_prec(const void* table, int nc, int64_t n, int64_t dim, const int64_t* u, const int64_t* v,
                          int64_t npairs, double* arg, double* dist, cudaStream_t s, int* domain = nullptr) {
  k_halfspace<P><<<(unsigned)((npairs + 127) / 128), 128, 0, s>>>(static_cast<const ST<P>*>(table), nc, n, dim, u, v,
                                                                 npairs, arg, dist, domain);
  mcfr::note_launch();
  return mcfr::check_launch("halfspace kernel");
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

// halfspace_arg for pairs (u[p], v[p]) of an (n, dim) MC table (hyperbolic.hpp:
// 183-212): arg[p] bit-identical to the reference; dist[p] (optional) =
// arcosh_guarded (:160-170) of it, binary64 log / log1p on the device (within
// four units of P's last place of the host libm result).  Out-of-range indices
// give NaN.
mcf_status mcf_halfspace_arg(mcf_prec p, const void* table, int nc, int64_t n, int64_t dim, const int64_t* u,
                             const int64_t* v, int64_t npairs, double* arg, double* dist, mcf_stream s) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "halfspace_arg: unknown precision");
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (n < 0 || dim < 1 || npairs < 0)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "halfspace_distance: table rank");
  if (npairs == 0) return MCF_OK;
  const mcf_status st = mcfr::ensure_device_tables();
  if (st != MCF_OK) return st;
  switch (p) {
    case MCF_B16: return mcfg::halfspace_prec<mcfg::PB16>(table, nc, n, dim, u, v, npairs, arg, dist, s);
    case MCF_B32: return mcfg::halfspace_prec<mcfg::PB32>(table, nc, n, dim, u, v, npairs, arg, dist, s);
    default: return mcfg::halfspace_prec<mcfg::PB64>(table, nc, n, dim, u, v, npairs, arg, dist, s);
  }
}

// halfspace_distance (hyperbolic.hpp:214-226) for pairs, synchronously, with
// the reference's domain check: a pair whose height (last coordinate, as its
// approx value) is not strictly positive makes the call fail with
// MCF_ERR_DOMAIN, "halfspace_distance: nonpositive height" (std::domain_error
// in the reference); arg (optional) as mcf_halfspace_arg.
mcf_status mcf_halfspace_distance(mcf_prec p, const void* table, int nc, int64_t n, int64_t dim, const int64_t* u,
                                  const int64_t* v, int64_t npairs, double* arg, double* dist, mcf_stream s) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "halfspace_distance: unknown precision");
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (n < 0 || dim < 1 || npairs < 0 || !dist)
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "halfspace_distance: table rank");
  if (npairs == 0) return MCF_OK;
  mcf_status st = mcfr::ensure_device_tables();
  if (st != MCF_OK) return st;
  // arg scratch when the caller wants only distances; the domain flag after it
  char* ws = static_cast<char*>(mcfr::workspace((arg ? 0 : npairs * sizeof(double)) + 256, 7));
  if (!ws) return mcfr::fail(MCF_ERR_CUDA, "halfspace_distance: cannot allocate the workspace");
  int* flag = reinterpret_cast<int*>(ws);
  double* a = arg ? arg : reinterpret_cast<double*>(ws + 256);
  if (cudaMemsetAsync(flag, 0, sizeof(int), s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "halfspace_distance: memset");
  switch (p) {
    case MCF_B16: st = mcfg::halfspace_prec<mcfg::PB16>(table, nc, n, dim, u, v, npairs, a, dist, s, flag); break;
    case MCF_B32: st = mcfg::halfspace_prec<mcfg::PB32>(table, nc, n, dim, u, v, npairs, a, dist, s, flag); break;
    default: st = mcfg::halfspace_prec<mcfg::PB64>(table, nc, n, dim, u, v, npairs, a, dist, s, flag);
  }
  if (st != MCF_OK) return st;
  int h = 0;
  if (cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return mcfr::fail(MCF_ERR_CUDA, "halfspace_distance: sync");
  if (h) return mcfr::fail(MCF_ERR_DOMAIN, "halfspace_distance: nonpositive height");
  return MCF_OK;
}

}  // extern "C"
