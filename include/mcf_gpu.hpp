// mcf_gpu.hpp -- the reference's operator API, served by the B200 library.
//
// Drop-in for the MCF operator layer of the reference
// (proj/include/mcfloat/mc_ops.hpp and linalg.hpp): the same function names,
// argument types (mcf::MCTensor<P>, mcf::NdArray, mcf::ReductionPlan) and
// exceptions, in namespace mcf::gpu.  Include it after the reference headers
// (it uses the reference's own value types and validation helpers) and link
// libmcf_b200.so; INTEGRATION.md shows the two-line switch.
//
// Values cross the boundary exactly: a component of MCTensor<P> is a binary64
// holding a P value, converted to/from P's storage without rounding
// (B16 through the reference's own to_bits/from_bits, precision.hpp:128-161).
// Results of the elementwise operators are bit-identical to the reference's;
// contractions use the reference order by default (bit-identical) and the
// FP64-pipe plan when plan.strategy is kFast (see mcf_gpu.h).
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "mcf_gpu.h"
#include "mcfloat/autodiff.hpp"
#include "mcfloat/linalg.hpp"
#include "mcfloat/mc_ops.hpp"

namespace mcf {
namespace gpu {

// ReductionPlan extension: the GPU-order plan (mcf_gpu.h MCF_FAST)
inline constexpr int kFastPlan = MCF_FAST;

namespace detail {

template <class P>
struct Store;
template <>
struct Store<B16> {
  using T = std::uint16_t;
  static constexpr mcf_prec kPrec = MCF_B16;
  static T put(double v) { return B16::to_bits(v); }
  static double get(T b) { return B16::from_bits(b); }
};
template <>
struct Store<B32> {
  using T = float;
  static constexpr mcf_prec kPrec = MCF_B32;
  static T put(double v) { return static_cast<float>(v); }
  static double get(T b) { return b; }
};
template <>
struct Store<B64> {
  using T = double;
  static constexpr mcf_prec kPrec = MCF_B64;
  static T put(double v) { return v; }
  static double get(T b) { return b; }
};

template <class P>
std::vector<typename Store<P>::T> pack(const std::vector<double>& v) {
  std::vector<typename Store<P>::T> out(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = Store<P>::put(v[i]);
  return out;
}

template <class P>
void unpack(const std::vector<typename Store<P>::T>& s, std::vector<double>& v) {
  v.resize(s.size());
  for (std::size_t i = 0; i < s.size(); ++i) v[i] = Store<P>::get(s[i]);
}

// status -> the reference's exception types and messages
inline void check(mcf_status st) {
  if (st == MCF_OK) return;
  const std::string msg = mcf_last_error();
  if (st == MCF_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == MCF_ERR_UNSUPPORTED) throw unsupported_operation(msg);
  throw std::runtime_error("mcf gpu: " + msg);
}

// working-precision operand rounded into P (the reference rounds v where it
// reads it, e.g. div_n's P::round(v[e % vn]) at mc_ops.hpp:502)
template <class P>
std::vector<typename Store<P>::T> pack_wp(const NdArray& v) {
  std::vector<typename Store<P>::T> out(v.numel());
  for (std::size_t i = 0; i < v.numel(); ++i) out[i] = Store<P>::put(P::round(v[i]));
  return out;
}

template <class P>
MCTensor<P> elementwise(const char* op, const MCTensor<P>* x, const MCTensor<P>* y,
                        const NdArray* v, Shape shape, int out_nc) {
  using S = Store<P>;
  std::vector<typename S::T> xs, ys, vs;
  if (x) xs = pack<P>(x->raw());
  if (y) ys = pack<P>(y->raw());
  if (v) vs = pack_wp<P>(*v);
  const std::size_t numel = shape_numel(shape);
  std::vector<typename S::T> os(numel * out_nc);
  check(mcf_h_elementwise(op, S::kPrec, x ? xs.data() : nullptr, x ? x->nc() : 0,
                          y ? ys.data() : nullptr, y ? y->nc() : 0, v ? vs.data() : nullptr,
                          v ? static_cast<int64_t>(v->numel()) : 1, os.data(),
                          static_cast<int64_t>(numel)));
  MCTensor<P> out(std::move(shape), out_nc);
  unpack<P>(os, out.raw());
  return out;
}

}  // namespace detail

// ---- EFT array forms (eft.hpp:89-111) ------------------------------------------

// s[i] + e[i] == a[i] + b[i] exactly, s[i] = fl(a[i] + b[i]) (two_sum, eft.hpp:31-38)
template <class P>
void two_sum(const std::vector<double>& a, const std::vector<double>& b, std::vector<double>& s,
             std::vector<double>& e) {
  using S = detail::Store<P>;
  const auto as = detail::pack<P>(a), bs = detail::pack<P>(b);
  std::vector<typename S::T> ss(a.size()), es(a.size());
  detail::check(mcf_h_eft(0, S::kPrec, as.data(), bs.data(), ss.data(), es.data(), (int64_t)a.size()));
  detail::unpack<P>(ss, s);
  detail::unpack<P>(es, e);
}

// p[i] + e[i] == a[i] b[i] exactly, p[i] = fl(a[i] b[i]) (two_prod, eft.hpp:75-86)
template <class P>
void two_prod(const std::vector<double>& a, const std::vector<double>& b, std::vector<double>& p,
              std::vector<double>& e) {
  using S = detail::Store<P>;
  const auto as = detail::pack<P>(a), bs = detail::pack<P>(b);
  std::vector<typename S::T> ps(a.size()), es(a.size());
  detail::check(mcf_h_eft(1, S::kPrec, as.data(), bs.data(), ps.data(), es.data(), (int64_t)a.size()));
  detail::unpack<P>(ps, p);
  detail::unpack<P>(es, e);
}

// ---- renormalization (mc_ops.hpp:338-359) ---------------------------------------

namespace detail {
template <class P>
MCTensor<P> renorm(int kind, const MCTensor<P>& h, int r_nc) {
  using S = Store<P>;
  mcf::detail::check_nc_limit(h.nc());
  mcf::detail::check_nc_limit(r_nc);
  const auto hs = pack<P>(h.raw());
  std::vector<typename S::T> os(h.numel() * r_nc);
  check(mcf_h_renorm(kind, S::kPrec, hs.data(), h.nc(), os.data(), r_nc, (int64_t)h.numel()));
  MCTensor<P> out(h.shape(), r_nc);
  unpack<P>(os, out.raw());
  return out;
}
}  // namespace detail

template <class P>
MCTensor<P> renormalize(const MCTensor<P>& h, int r_nc) {  // mc_ops.hpp:338-348
  return detail::renorm<P>(0, h, r_nc);
}

template <class P>
MCTensor<P> simple_renorm(const MCTensor<P>& h, int r_nc) {  // mc_ops.hpp:350-359
  return detail::renorm<P>(1, h, r_nc);
}

// ---- elementwise operators (mc_ops.hpp:338-507) -------------------------------

template <class P>
MCTensor<P> grow_expn(const MCTensor<P>& x, const NdArray& v) {  // mc_ops.hpp:384-394
  mcf::detail::check_nc_limit(x.nc());
  mcf::detail::check_suffix_broadcast(x.shape(), v.shape(), "grow_expn");
  return detail::elementwise<P>("grow_expn", &x, nullptr, &v, x.shape(), x.nc());
}

template <class P>
MCTensor<P> scaling_n(const MCTensor<P>& x, const NdArray& v, bool expanded = false) {
  mcf::detail::check_nc_limit(x.nc());  // mc_ops.hpp:398-410
  mcf::detail::check_suffix_broadcast(x.shape(), v.shape(), "scaling_n");
  const int onc = expanded ? x.nc() + 1 : x.nc();
  mcf::detail::check_nc_limit(onc);
  return detail::elementwise<P>(expanded ? "scaling_n_expanded" : "scaling_n", &x, nullptr, &v,
                                x.shape(), onc);
}

template <class P>
MCTensor<P> div_n(const NdArray& v, const MCTensor<P>& y) {  // mc_ops.hpp:494-507
  mcf::detail::check_nc_limit(y.nc());
  mcf::detail::check_suffix_broadcast(y.shape(), v.shape(), "div_n");
  return detail::elementwise<P>("div_n", nullptr, &y, &v, y.shape(), y.nc());
}

#define MCF_GPU_BINARY(name)                                                             \
  template <class P>                                                                     \
  MCTensor<P> name(const MCTensor<P>& x, const MCTensor<P>& y) {                         \
    check_shapes_equal(x.shape(), y.shape(), #name);                                     \
    const int nc = x.nc() > y.nc() ? x.nc() : y.nc();                                    \
    mcf::detail::check_nc_limit(nc);                                                     \
    return detail::elementwise<P>(#name, &x, &y, nullptr, x.shape(), nc);                \
  }
MCF_GPU_BINARY(add_mcn)       // mc_ops.hpp:440-446
MCF_GPU_BINARY(div_mcn)       // mc_ops.hpp:448-454
MCF_GPU_BINARY(mul_mcn)       // mc_ops.hpp:456-462
MCF_GPU_BINARY(mul_mcn_slow)  // mc_ops.hpp:464-470
#undef MCF_GPU_BINARY

template <class P>
MCTensor<P> square_mcn(const MCTensor<P>& x) {  // mc_ops.hpp:472-480
  mcf::detail::check_nc_limit(x.nc());
  return detail::elementwise<P>("square_mcn", &x, nullptr, nullptr, x.shape(), x.nc());
}

template <class P>
MCTensor<P> exp_mcn(const MCTensor<P>& x) {  // mc_ops.hpp:482-490 (correctly rounded exp)
  mcf::detail::check_nc_limit(x.nc());
  return detail::elementwise<P>("exp_mcn", &x, nullptr, nullptr, x.shape(), x.nc());
}

template <class P>
MCTensor<P> negate(const MCTensor<P>& x) {  // mc_ops.hpp:376-381
  return detail::elementwise<P>("negate", &x, nullptr, nullptr, x.shape(), x.nc());
}

// ---- MC activations (autodiff.hpp) ------------------------------------------------

// the value mc_relu_op (autodiff.hpp:340-350) puts on the tape: components
// zeroed where approx() <= 0
template <class P>
MCTensor<P> mc_relu(const MCTensor<P>& x) {
  mcf::detail::check_nc_limit(x.nc());
  return detail::elementwise<P>("mc_relu", &x, nullptr, nullptr, x.shape(), x.nc());
}

// mc_softmax (autodiff.hpp:383-413), same rank / axis rules and message
template <class P>
MCTensor<P> mc_softmax(const MCTensor<P>& x, int axis = -1) {
  std::size_t outer, n, inner;
  mcf::detail::softmax_axis_dims(x, axis, outer, n, inner);
  mcf::detail::check_nc_limit(x.nc());
  using S = detail::Store<P>;
  const auto xs = detail::pack<P>(x.raw());
  std::vector<typename S::T> os(xs.size());
  detail::check(mcf_h_mc_softmax(S::kPrec, xs.data(), x.nc(), static_cast<int64_t>(outer), static_cast<int64_t>(n),
                                 static_cast<int64_t>(inner), os.data()));
  MCTensor<P> out(x.shape(), x.nc());
  detail::unpack<P>(os, out.raw());
  return out;
}

// ---- contractions (linalg.hpp) ---------------------------------------------------

namespace detail {
inline int strategy_of(const ReductionPlan& plan) {
  return plan.strategy == ReduceStrategy::kPairwiseTree ? MCF_PAIRWISE_TREE : MCF_SEQUENTIAL;
}

template <class P>
MCTensor<P> bmm(const MCTensor<P>& x, const NdArray& w, std::size_t batch, std::size_t m,
                std::size_t k, std::size_t n, bool w_batched, Shape out_shape, int strategy) {
  using S = Store<P>;
  mcf::detail::check_nc_limit(x.nc() + 1);
  const auto xs = pack<P>(x.raw());
  const auto ws = pack_wp<P>(w);
  std::vector<typename S::T> os(batch * m * n * x.nc());
  check(mcf_h_bmm_mcn(S::kPrec, xs.data(), x.nc(), ws.data(), batch, m, k, n, w_batched ? 1 : 0,
                      os.data(), strategy));
  MCTensor<P> out(std::move(out_shape), x.nc());
  unpack<P>(os, out.raw());
  return out;
}
}  // namespace detail

template <class P>
MCTensor<P> mm_mcn(const MCTensor<P>& x, const NdArray& w, const ReductionPlan& plan = {}) {
  mcf::detail::require_rank(x.shape(), 2, "mm_mcn");  // linalg.hpp:138-157
  mcf::detail::require_rank(w.shape(), 2, "mm_mcn");
  if (x.dim(1) != w.dim(0))
    throw std::invalid_argument("mm_mcn: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                shape_str(w.shape()));
  return detail::bmm<P>(x, w, 1, x.dim(0), x.dim(1), w.dim(1), false, Shape{x.dim(0), w.dim(1)},
                        detail::strategy_of(plan));
}

// GPU-order plan (MCF_FAST: INT8 tensor-core splitting where supported, else the FP64 pipe), same shapes and checks as mm_mcn
template <class P>
MCTensor<P> mm_mcn_fast(const MCTensor<P>& x, const NdArray& w) {
  mcf::detail::require_rank(x.shape(), 2, "mm_mcn");
  mcf::detail::require_rank(w.shape(), 2, "mm_mcn");
  if (x.dim(1) != w.dim(0))
    throw std::invalid_argument("mm_mcn: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                shape_str(w.shape()));
  return detail::bmm<P>(x, w, 1, x.dim(0), x.dim(1), w.dim(1), false, Shape{x.dim(0), w.dim(1)},
                        MCF_FAST);
}

// linalg.hpp:159-166: MC x MC stays refused on the drop-in overload
template <class P>
MCTensor<P> mm_mcn(const MCTensor<P>&, const MCTensor<P>&, const ReductionPlan& = {}) {
  detail::check(mcf_mm_mcn_mcmc_refusal());
  return {};
}

template <class P>
MCTensor<P> dot_mcn(const MCTensor<P>& x, const NdArray& v, const ReductionPlan& plan = {}) {
  mcf::detail::require_rank(x.shape(), 1, "dot_mcn");  // linalg.hpp:103-116
  mcf::detail::require_rank(v.shape(), 1, "dot_mcn");
  if (x.dim(0) != v.dim(0))
    throw std::invalid_argument("dot_mcn: length mismatch " + shape_str(x.shape()) + " vs " +
                                shape_str(v.shape()));
  return detail::bmm<P>(x, v, 1, 1, x.dim(0), 1, false, Shape{}, detail::strategy_of(plan));
}

template <class P>
MCTensor<P> mv_mcn(const MCTensor<P>& x, const NdArray& v, const ReductionPlan& plan = {}) {
  mcf::detail::require_rank(x.shape(), 2, "mv_mcn");  // linalg.hpp:119-135
  mcf::detail::require_rank(v.shape(), 1, "mv_mcn");
  if (x.dim(1) != v.dim(0))
    throw std::invalid_argument("mv_mcn: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                shape_str(v.shape()));
  return detail::bmm<P>(x, v, 1, x.dim(0), x.dim(1), 1, false, Shape{x.dim(0)},
                        detail::strategy_of(plan));
}

template <class P>
MCTensor<P> bmm_mcn(const MCTensor<P>& x, const NdArray& w, const ReductionPlan& plan = {}) {
  mcf::detail::require_rank(x.shape(), 3, "bmm_mcn");  // linalg.hpp:205-216
  mcf::detail::require_rank(w.shape(), 3, "bmm_mcn");
  if (x.dim(0) != w.dim(0) || x.dim(2) != w.dim(1))
    throw std::invalid_argument("bmm_mcn: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                shape_str(w.shape()));
  return detail::bmm<P>(x, w, x.dim(0), x.dim(1), x.dim(2), w.dim(2), true,
                        Shape{x.dim(0), x.dim(1), w.dim(2)}, detail::strategy_of(plan));
}

template <class P>
MCTensor<P> mm4d_mcn(const MCTensor<P>& x, const NdArray& w, const ReductionPlan& plan = {}) {
  mcf::detail::require_rank(x.shape(), 4, "mm4d_mcn");  // linalg.hpp:218-231
  mcf::detail::require_rank(w.shape(), 4, "mm4d_mcn");
  if (x.dim(0) != w.dim(0) || x.dim(1) != w.dim(1) || x.dim(3) != w.dim(2))
    throw std::invalid_argument("mm4d_mcn: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                shape_str(w.shape()));
  return detail::bmm<P>(x, w, x.dim(0) * x.dim(1), x.dim(2), x.dim(3), w.dim(3), true,
                        Shape{x.dim(0), x.dim(1), x.dim(2), w.dim(3)}, detail::strategy_of(plan));
}

// linalg.hpp:233-253: beta bias + alpha (x . w); the factors rounded into P
// and applied through ScalingN, the bias broadcast over the product's leading
// rows, the sum through add_mcn -- each step on the GPU
template <class P>
MCTensor<P> addmm_mcn(const MCTensor<P>& bias, const MCTensor<P>& x, const NdArray& w, double alpha = 1.0,
                      double beta = 1.0, const ReductionPlan& plan = {}) {
  MCTensor<P> prod = gpu::mm_mcn(x, w, plan);
  if (alpha != 1.0) prod = gpu::scaling_n(prod, NdArray::scalar(P::round(alpha)));
  MCTensor<P> sb = beta != 1.0 ? gpu::scaling_n(bias, NdArray::scalar(P::round(beta))) : bias;
  if (sb.shape() == prod.shape()) return gpu::add_mcn(sb, prod);
  mcf::detail::check_suffix_broadcast(prod.shape(), sb.shape(), "addmm_mcn");
  MCTensor<P> expanded(prod.shape(), sb.nc());
  const std::size_t bn = sb.numel();
  for (std::size_t e = 0; e < prod.numel(); ++e)
    for (int c = 0; c < sb.nc(); ++c) expanded.comps(e)[c] = sb.comps(e % bn)[c];
  return gpu::add_mcn(expanded, prod);
}

// linalg.hpp:255-299: rank dispatch; a rank-2 w broadcasts over x's batch axes
template <class P>
MCTensor<P> matmul_mcn(const MCTensor<P>& x, const NdArray& w, const ReductionPlan& plan = {}) {
  const int rx = x.rank(), rw = w.rank();
  const auto bad = [&] {
    return std::invalid_argument("matmul_mcn: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                 shape_str(w.shape()));
  };
  if (rx == 1 && rw == 1) return gpu::dot_mcn(x, w, plan);
  if (rx == 2 && rw == 1) return gpu::mv_mcn(x, w, plan);
  if (rx == 1 && rw == 2) {
    if (x.dim(0) != w.dim(0)) throw bad();
    return detail::bmm<P>(x, w, 1, 1, x.dim(0), w.dim(1), false, Shape{w.dim(1)}, detail::strategy_of(plan));
  }
  if (rx == 2 && rw == 2) return gpu::mm_mcn(x, w, plan);
  if (rx == 3 && rw == 3) return gpu::bmm_mcn(x, w, plan);
  if (rx == 3 && rw == 2) {
    if (x.dim(2) != w.dim(0)) throw bad();
    return detail::bmm<P>(x, w, x.dim(0), x.dim(1), x.dim(2), w.dim(1), false,
                          Shape{x.dim(0), x.dim(1), w.dim(1)}, detail::strategy_of(plan));
  }
  if (rx == 4 && rw == 4) return gpu::mm4d_mcn(x, w, plan);
  if (rx == 4 && rw == 2) {
    if (x.dim(3) != w.dim(0)) throw bad();
    return detail::bmm<P>(x, w, x.dim(0) * x.dim(1), x.dim(2), x.dim(3), w.dim(1), false,
                          Shape{x.dim(0), x.dim(1), x.dim(2), w.dim(1)}, detail::strategy_of(plan));
  }
  throw std::invalid_argument("matmul_mcn: unsupported rank pair for shapes " + shape_str(x.shape()) + " and " +
                              shape_str(w.shape()));
}

// linalg.hpp:301-315: component-preserving 2-D transpose
template <class P>
MCTensor<P> mc_transpose2d(const MCTensor<P>& x) {
  using S = detail::Store<P>;
  mcf::detail::require_rank(x.shape(), 2, "mc_transpose2d");
  const auto xs = detail::pack<P>(x.raw());
  std::vector<typename S::T> os(xs.size());
  detail::check(mcf_h_mc_transpose2d(S::kPrec, xs.data(), x.nc(), x.dim(0), x.dim(1), os.data()));
  MCTensor<P> out(Shape{x.dim(1), x.dim(0)}, x.nc());
  detail::unpack<P>(os, out.raw());
  return out;
}

// NEW: MC x MC product (SURVEY 8c recipe B by default; strategy MCF_FAST for
// the FP64-pipe kernel)
template <class P>
MCTensor<P> mm_mcmc(const MCTensor<P>& x, const MCTensor<P>& y, int strategy = MCF_SEQUENTIAL) {
  using S = detail::Store<P>;
  mcf::detail::require_rank(x.shape(), 2, "mm_mcmc");
  mcf::detail::require_rank(y.shape(), 2, "mm_mcmc");
  if (x.dim(1) != y.dim(0) || x.nc() != y.nc())
    throw std::invalid_argument("mm_mcmc: incompatible shapes " + shape_str(x.shape()) + " vs " +
                                shape_str(y.shape()));
  const auto xs = detail::pack<P>(x.raw());
  const auto ys = detail::pack<P>(y.raw());
  std::vector<typename S::T> os(x.dim(0) * y.dim(1) * x.nc());
  detail::check(mcf_h_mm_mcmc(S::kPrec, xs.data(), ys.data(), x.nc(), x.dim(0), x.dim(1), y.dim(1),
                              os.data(), strategy));
  MCTensor<P> out(Shape{x.dim(0), y.dim(1)}, x.nc());
  detail::unpack<P>(os, out.raw());
  return out;
}

}  // namespace gpu
}  // namespace mcf
