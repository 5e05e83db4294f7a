// ref_shim.cpp -- the reference implementation behind the oracle's C interface.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no MCF algorithm of its own:
// every mcfref_* entry converts the caller's arrays into the reference's value
// types (mcf::MCTensor<P>, mcf::NdArray) and calls the reference's public
// operator (or, for the MC x MC "recipe B" restatement, composes the
// reference's own detail kernels).  It is compiled from the reference headers
// where they lie (/root/reference/proj/include, unmodified) with the
// reference's FP flags by oracle/Makefile into oracle/_ref/libmcf_ref.so.
// That directory is git-ignored; the .so travels to the GPU box so bench.py
// can time the reference's CPU path there.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mcf_oracle.h"
#include "mcfloat/autodiff.hpp"
#include "mcfloat/hyperbolic.hpp"
#include "mcfloat/linalg.hpp"
#include "mcfloat/mc_ops.hpp"
#include "mcfloat/nn.hpp"
#include "mcfloat/optim.hpp"
#include "mcfloat/serialize.hpp"

namespace {

using mcf::MCTensor;
using mcf::NdArray;
using mcf::Shape;

template <class P>
struct Store;
template <>
struct Store<mcf::B16> {
  using T = std::uint16_t;
  static double get(T v) { return mcf::B16::from_bits(v); }
  static T put(double v) { return mcf::B16::to_bits(mcf::B16::round(v)); }
};
template <>
struct Store<mcf::B32> {
  using T = float;
  static double get(T v) { return v; }
  static T put(double v) { return static_cast<float>(v); }
};
template <>
struct Store<mcf::B64> {
  using T = double;
  static double get(T v) { return v; }
  static T put(double v) { return v; }
};

template <class P>
MCTensor<P> to_mct(const void* p, std::int64_t off, std::int64_t numel, int nc, Shape shape = {}) {
  using S = Store<P>;
  const auto* src = static_cast<const typename S::T*>(p) + off * nc;
  MCTensor<P> t(shape.empty() ? Shape{static_cast<std::size_t>(numel)} : shape, nc);
  for (std::int64_t i = 0; i < numel * nc; ++i) t.raw()[i] = S::get(src[i]);
  return t;
}

template <class P>
NdArray to_nd(const void* p, std::int64_t off, std::int64_t numel, Shape shape = {}) {
  using S = Store<P>;
  const auto* src = static_cast<const typename S::T*>(p) + off;
  NdArray a(shape.empty() ? Shape{static_cast<std::size_t>(numel)} : shape);
  for (std::int64_t i = 0; i < numel; ++i) a[i] = S::get(src[i]);
  return a;
}

template <class P>
void from_vec(const std::vector<double>& v, void* p, std::int64_t off) {
  using S = Store<P>;
  auto* dst = static_cast<typename S::T*>(p) + off;
  for (std::size_t i = 0; i < v.size(); ++i) dst[i] = S::put(v[i]);
}

template <class F>
int with_prec(int prec, F&& f) {
  try {
    switch (prec) {
      case MCFO_B16: f.template operator()<mcf::B16>(); return 0;
      case MCFO_B32: f.template operator()<mcf::B32>(); return 0;
      case MCFO_B64: f.template operator()<mcf::B64>(); return 0;
      default: return 1;
    }
  } catch (const std::exception&) {
    return 1;
  }
}

// Recipe B: the reference refuses MC x MC products
// (linalg.hpp:159-166), so the oracle composes them from the reference's own
// kernels: term = mul_mcn_slow's term set renormalized to nc+1, sequential
// add_kernel at nc+1, one final renorm to nc.
template <class P>
void recipe_b(const double* const* xs, const double* const* ys, int nc, std::int64_t len,
              double* out) {
  using namespace mcf;
  using namespace mcf::detail;
  if (len == 0) {
    for (int i = 0; i < nc; ++i) out[i] = 0.0;
    return;
  }
  if (nc == 1) {
    double acc = 0.0;
    for (std::int64_t k = 0; k < len; ++k) acc = fl_add<P>(acc, fl_mul<P>(xs[k][0], ys[k][0]));
    out[0] = acc;
    return;
  }
  auto term = [&](std::int64_t k, double* t) {
    double h[kStage];
    int m = 0;
    for (int i = 0; i < nc; ++i)
      for (int j = 0; i + j < nc; ++j) {
        const auto [p, e] = two_prod<P>(xs[k][i], ys[k][j]);
        h[m++] = p;
        h[m++] = e;
      }
    for (int i = 1; i < nc; ++i) h[m++] = fl_mul<P>(xs[k][i], ys[k][nc - i]);
    renorm_kernel<P>(h, m, t, nc + 1);
  };
  double acc[kMaxNc + 1], t[kMaxNc + 1];
  term(0, acc);
  for (std::int64_t k = 1; k < len; ++k) {
    term(k, t);
    add_kernel<P>(acc, nc + 1, t, nc + 1, acc, nc + 1);
  }
  renorm_kernel<P>(acc, nc + 1, out, nc);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

template <class F>
void run_threads(int threads, std::int64_t total, F&& f) {
  if (threads < 1) threads = 1;
  if (threads == 1 || total < threads) {
    f(0, total);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const std::int64_t lo = total * t / threads, hi = total * (t + 1) / threads;
    pool.emplace_back([&, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int mcfref_two_sum(int prec, const void* a, const void* b, void* s, void* e, std::int64_t n) {
  return with_prec(prec, [&]<class P>() {
    const NdArray A = to_nd<P>(a, 0, n), B = to_nd<P>(b, 0, n);
    std::vector<double> S, E;
    mcf::two_sum<P>(A.vec(), B.vec(), S, E);
    from_vec<P>(S, s, 0);
    from_vec<P>(E, e, 0);
  });
}

int mcfref_two_prod(int prec, const void* a, const void* b, void* p, void* e, std::int64_t n,
                    int use_fma) {
  return with_prec(prec, [&]<class P>() {
    const NdArray A = to_nd<P>(a, 0, n), B = to_nd<P>(b, 0, n);
    std::vector<double> Pv, E;
    const bool saved = mcf::fma_enabled().load();
    mcf::fma_enabled().store(use_fma != 0);
    mcf::two_prod<P>(A.vec(), B.vec(), Pv, E);
    mcf::fma_enabled().store(saved);
    from_vec<P>(Pv, p, 0);
    from_vec<P>(E, e, 0);
  });
}

int mcfref_renormalize(int prec, const void* h, int nc, void* out, int r_nc, std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::renormalize(to_mct<P>(h, 0, numel, nc), r_nc).raw(), out, 0);
  });
}

int mcfref_simple_renorm(int prec, const void* h, int nc, void* out, int r_nc,
                         std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::simple_renorm(to_mct<P>(h, 0, numel, nc), r_nc).raw(), out, 0);
  });
}

int mcfref_approx(int prec, const void* x, int nc, void* out, std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(to_mct<P>(x, 0, numel, nc).approx().vec(), out, 0);
  });
}

int mcfref_negate(int prec, const void* x, int nc, void* out, std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::negate(to_mct<P>(x, 0, numel, nc)).raw(), out, 0);
  });
}

int mcfref_grow_expn(int prec, const void* x, int nc, const void* v, std::int64_t vn, void* out,
                     std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::grow_expn(to_mct<P>(x, 0, numel, nc), to_nd<P>(v, 0, vn)).raw(), out, 0);
  });
}

int mcfref_scaling_n(int prec, const void* x, int nc, const void* v, std::int64_t vn,
                     int expanded, void* out, std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(
        mcf::scaling_n(to_mct<P>(x, 0, numel, nc), to_nd<P>(v, 0, vn), expanded != 0).raw(),
        out, 0);
  });
}

int mcfref_div_n(int prec, const void* v, std::int64_t vn, const void* y, int nc, void* out,
                 std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::div_n(to_nd<P>(v, 0, vn), to_mct<P>(y, 0, numel, nc)).raw(), out, 0);
  });
}

#define MCFREF_BINARY(name)                                                                 \
  int mcfref_##name(int prec, const void* x, int ncx, const void* y, int ncy, void* out,    \
                    std::int64_t numel) {                                                   \
    return with_prec(prec, [&]<class P>() {                                                 \
      from_vec<P>(mcf::name(to_mct<P>(x, 0, numel, ncx), to_mct<P>(y, 0, numel, ncy)).raw(), \
                  out, 0);                                                                  \
    });                                                                                     \
  }
MCFREF_BINARY(add_mcn)
MCFREF_BINARY(div_mcn)
MCFREF_BINARY(mul_mcn)
MCFREF_BINARY(mul_mcn_slow)

int mcfref_square_mcn(int prec, const void* x, int nc, void* out, std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::square_mcn(to_mct<P>(x, 0, numel, nc)).raw(), out, 0);
  });
}

int mcfref_exp_mcn(int prec, const void* x, int nc, void* out, std::int64_t numel,
                   int exp_mode) {
  if (exp_mode != MCFO_EXP_LIBM) return 1;  // the reference only has libm exp
  return with_prec(prec, [&]<class P>() {
    from_vec<P>(mcf::exp_mcn(to_mct<P>(x, 0, numel, nc)).raw(), out, 0);
  });
}

int mcfref_bmm_mcn(int prec, const void* x, int nc, const void* w, std::int64_t batch,
                   std::int64_t m, std::int64_t k, std::int64_t n, int w_batched, void* out,
                   int strategy, int leaf_arity) {
  return with_prec(prec, [&]<class P>() {
    const mcf::ReductionPlan plan{strategy == MCFO_PAIRWISE_TREE
                                      ? mcf::ReduceStrategy::kPairwiseTree
                                      : mcf::ReduceStrategy::kSequential,
                                  leaf_arity};
    const auto B = static_cast<std::size_t>(batch), M = static_cast<std::size_t>(m),
               K = static_cast<std::size_t>(k), N = static_cast<std::size_t>(n);
    const MCTensor<P> X = to_mct<P>(x, 0, batch * m * k, nc, Shape{B, M, K});
    if (w_batched) {
      const NdArray W = to_nd<P>(w, 0, batch * k * n, Shape{B, K, N});
      from_vec<P>(mcf::bmm_mcn(X, W, plan).raw(), out, 0);
    } else {
      const NdArray W = to_nd<P>(w, 0, k * n, Shape{K, N});
      from_vec<P>(mcf::matmul_mcn(X, W, plan).raw(), out, 0);  // rank 3/2 dispatch
    }
  });
}

int mcfref_mm_mcn_sampled(int prec, const void* x, int nc, const void* w, std::int64_t m,
                          std::int64_t k, std::int64_t n, const std::int64_t* rows,
                          const std::int64_t* cols, std::int64_t nsamp, void* out) {
  (void)m;
  return with_prec(prec, [&]<class P>() {
    // each sample is mm_mcn of one row against one column (1 x k times k x 1)
    const auto K = static_cast<std::size_t>(k);
    for (std::int64_t s = 0; s < nsamp; ++s) {
      const MCTensor<P> row = to_mct<P>(x, rows[s] * k, k, nc, Shape{1, K});
      NdArray col(Shape{K, 1});
      for (std::int64_t kk = 0; kk < k; ++kk)
        col[kk] = Store<P>::get(static_cast<const typename Store<P>::T*>(w)[kk * n + cols[s]]);
      from_vec<P>(mcf::mm_mcn(row, col).raw(), out, s * nc);
    }
  });
}

int mcfref_dot_mcmc(int prec, const void* x, const void* y, int nc, std::int64_t batch,
                    std::int64_t k, void* out) {
  return with_prec(prec, [&]<class P>() {
    const MCTensor<P> X = to_mct<P>(x, 0, batch * k, nc), Y = to_mct<P>(y, 0, batch * k, nc);
    std::vector<const double*> xs(k), ys(k);
    std::vector<double> o(nc);
    for (std::int64_t b = 0; b < batch; ++b) {
      for (std::int64_t kk = 0; kk < k; ++kk) {
        xs[kk] = X.comps(b * k + kk);
        ys[kk] = Y.comps(b * k + kk);
      }
      recipe_b<P>(xs.data(), ys.data(), nc, k, o.data());
      from_vec<P>(o, out, b * nc);
    }
  });
}

int mcfref_mm_mcmc_sampled(int prec, const void* x, const void* y, int nc, std::int64_t m,
                           std::int64_t k, std::int64_t n, const std::int64_t* rows,
                           const std::int64_t* cols, std::int64_t nsamp, void* out) {
  (void)m;
  return with_prec(prec, [&]<class P>() {
    std::vector<const double*> xs(k), ys(k);
    std::vector<double> o(nc);
    for (std::int64_t s = 0; s < nsamp; ++s) {
      const MCTensor<P> X = to_mct<P>(x, rows[s] * k, k, nc);
      MCTensor<P> Y(Shape{static_cast<std::size_t>(k)}, nc);
      for (std::int64_t kk = 0; kk < k; ++kk)
        for (int c = 0; c < nc; ++c)
          Y.comps(kk)[c] = Store<P>::get(
              static_cast<const typename Store<P>::T*>(y)[(kk * n + cols[s]) * nc + c]);
      for (std::int64_t kk = 0; kk < k; ++kk) {
        xs[kk] = X.comps(kk);
        ys[kk] = Y.comps(kk);
      }
      recipe_b<P>(xs.data(), ys.data(), nc, k, o.data());
      from_vec<P>(o, out, s * nc);
    }
  });
}

int mcfref_matmul2d(int prec, const void* a, const void* b, std::int64_t m, std::int64_t k,
                    std::int64_t n, void* out) {
  return with_prec(prec, [&]<class P>() {
    const auto M = static_cast<std::size_t>(m), K = static_cast<std::size_t>(k),
               N = static_cast<std::size_t>(n);
    from_vec<P>(mcf::matmul2d<P>(to_nd<P>(a, 0, m * k, Shape{M, K}),
                                 to_nd<P>(b, 0, k * n, Shape{K, N}))
                    .vec(),
                out, 0);
  });
}

// mc_relu_op (autodiff.hpp:340-350) through the reference's tape: an MC
// parameter leaf, the op, its MC value
int mcfref_mc_relu(int prec, const void* x, int nc, void* out, std::int64_t numel) {
  return with_prec(prec, [&]<class P>() {
    MCTensor<P> p = to_mct<P>(x, 0, numel, nc);
    mcf::Tape<P> tape;
    const auto a = tape.mc_param(p);
    const auto r = mcf::mc_relu_op(tape, a);
    from_vec<P>(tape.mc_value(r).raw(), out, 0);
  });
}

// mc_softmax (autodiff.hpp:383-413): the (outer, n, inner) view as the
// reference's rank-1 / rank-2 tensor and axis
int mcfref_mc_softmax(int prec, const void* x, int nc, std::int64_t outer, std::int64_t n, std::int64_t inner,
                      void* out, int exp_mode) {
  if (exp_mode != MCFO_EXP_LIBM) return 1;
  if (outer != 1 && inner != 1) return 1;  // the reference takes rank 1 / 2 only
  return with_prec(prec, [&]<class P>() {
    const auto O = static_cast<std::size_t>(outer), N = static_cast<std::size_t>(n),
               I = static_cast<std::size_t>(inner);
    Shape shape = inner == 1 ? (outer == 1 ? Shape{N} : Shape{O, N}) : Shape{N, I};
    const int axis = inner == 1 ? -1 : 0;
    from_vec<P>(mcf::mc_softmax(to_mct<P>(x, 0, outer * n * inner, nc, shape), axis).raw(), out, 0);
  });
}

// mct_to_json (serialize.hpp:40-54) dumped as write_json_file does (indent 2);
// returns the string length, or -1 if it does not fit
std::int64_t mcfref_mct_to_json(int prec, const void* x, int nc, const std::int64_t* shape, int rank, char* buf,
                                std::int64_t cap) {
  std::int64_t len = -1;
  with_prec(prec, [&]<class P>() {
    Shape sh;
    std::int64_t numel = 1;
    for (int d = 0; d < rank; ++d) {
      sh.push_back(static_cast<std::size_t>(shape[d]));
      numel *= shape[d];
    }
    const std::string s = mcf::mct_to_json(to_mct<P>(x, 0, numel, nc, sh)).dump(2);
    if (static_cast<std::int64_t>(s.size()) < cap) {
      std::memcpy(buf, s.data(), s.size());
      buf[s.size()] = 0;
      len = static_cast<std::int64_t>(s.size());
    }
  });
  return len;
}

int mcfref_halfspace_arg(int prec, const void* table, int nc, std::int64_t n, std::int64_t dim,
                         const std::int64_t* u, const std::int64_t* v, std::int64_t npairs, double* out) {
  return with_prec(prec, [&]<class P>() {
    const auto t = to_mct<P>(table, 0, n * dim, nc, Shape{static_cast<std::size_t>(n), static_cast<std::size_t>(dim)});
    for (std::int64_t p = 0; p < npairs; ++p)
      out[p] = mcf::halfspace_arg(t, static_cast<std::size_t>(u[p]), static_cast<std::size_t>(v[p]),
                                  static_cast<std::size_t>(dim));
  });
}

// ---- timing entry points (bench.py cpu_baseline / --impl reference) ----------

double mcfref_time_elementwise(const char* op, int prec, const void* x, int nc, const void* y,
                               const void* v, std::int64_t numel, int threads, int reps,
                               void* out) {
  const std::string name(op);
  double elapsed = -1.0;
  with_prec(prec, [&]<class P>() {
    if (threads < 1) threads = 1;
    struct Slice {
      std::int64_t lo, hi;
      MCTensor<P> x, y;
      NdArray v;
      std::vector<double> res;
    };
    std::vector<Slice> slices(threads);
    // inputs are converted to the reference's value types outside the timed region
    for (int t = 0; t < threads; ++t) {
      Slice& s = slices[t];
      s.lo = numel * t / threads;
      s.hi = numel * (t + 1) / threads;
      const std::int64_t len = s.hi - s.lo;
      if (x) s.x = to_mct<P>(x, s.lo, len, nc);
      if (y) s.y = to_mct<P>(y, s.lo, len, nc);
      if (v) s.v = to_nd<P>(v, s.lo, len);
    }
    auto body = [&](Slice& s) {
      MCTensor<P> r;
      if (name == "grow_expn") r = mcf::grow_expn(s.x, s.v);
      else if (name == "scaling_n") r = mcf::scaling_n(s.x, s.v);
      else if (name == "div_n") r = mcf::div_n(s.v, s.y);
      else if (name == "add_mcn") r = mcf::add_mcn(s.x, s.y);
      else if (name == "mul_mcn") r = mcf::mul_mcn(s.x, s.y);
      else if (name == "mul_mcn_slow") r = mcf::mul_mcn_slow(s.x, s.y);
      else if (name == "div_mcn") r = mcf::div_mcn(s.x, s.y);
      else if (name == "exp_mcn") r = mcf::exp_mcn(s.x);
      else if (name == "square_mcn") r = mcf::square_mcn(s.x);
      else throw std::invalid_argument("unknown op " + name);
      s.res = std::move(r.raw());
    };
    const double t0 = now_s();
    for (int rep = 0; rep < reps; ++rep) {
      if (threads == 1) {
        body(slices[0]);
      } else {
        std::vector<std::thread> pool;
        for (auto& s : slices) pool.emplace_back([&body, &s] { body(s); });
        for (auto& th : pool) th.join();
      }
    }
    elapsed = now_s() - t0;
    if (out)
      for (auto& s : slices) from_vec<P>(s.res, out, s.lo * nc);
  });
  return elapsed;
}

double mcfref_time_mm_rows(int prec, const void* x, int nc, const void* w, std::int64_t rows,
                           std::int64_t k, std::int64_t n, int threads, void* out) {
  double elapsed = -1.0;
  with_prec(prec, [&]<class P>() {
    const auto K = static_cast<std::size_t>(k), N = static_cast<std::size_t>(n);
    const NdArray W = to_nd<P>(w, 0, k * n, Shape{K, N});
    if (threads < 1) threads = 1;
    std::vector<MCTensor<P>> xs(threads), res(threads);
    std::vector<std::int64_t> lo(threads), hi(threads);
    for (int t = 0; t < threads; ++t) {
      lo[t] = rows * t / threads;
      hi[t] = rows * (t + 1) / threads;
      xs[t] = to_mct<P>(x, lo[t] * k, (hi[t] - lo[t]) * k, nc,
                        Shape{static_cast<std::size_t>(hi[t] - lo[t]), K});
    }
    const double t0 = now_s();
    run_threads(threads, threads, [&](std::int64_t a, std::int64_t b) {
      for (std::int64_t t = a; t < b; ++t)
        if (hi[t] > lo[t]) res[t] = mcf::mm_mcn(xs[t], W);
    });
    elapsed = now_s() - t0;
    if (out)
      for (int t = 0; t < threads; ++t)
        if (hi[t] > lo[t]) from_vec<P>(res[t].raw(), out, lo[t] * n * nc);
  });
  return elapsed;
}

double mcfref_time_dot_mcmc(int prec, const void* x, const void* y, int nc, std::int64_t batch,
                            std::int64_t k, int threads, void* out) {
  double elapsed = -1.0;
  with_prec(prec, [&]<class P>() {
    const MCTensor<P> X = to_mct<P>(x, 0, batch * k, nc), Y = to_mct<P>(y, 0, batch * k, nc);
    std::vector<double> o(batch * nc);
    const double t0 = now_s();
    run_threads(threads, batch, [&](std::int64_t a, std::int64_t b) {
      std::vector<const double*> xs(k), ys(k);
      for (std::int64_t d = a; d < b; ++d) {
        for (std::int64_t kk = 0; kk < k; ++kk) {
          xs[kk] = X.comps(d * k + kk);
          ys[kk] = Y.comps(d * k + kk);
        }
        recipe_b<P>(xs.data(), ys.data(), nc, k, o.data() + d * nc);
      }
    });
    elapsed = now_s() - t0;
    if (out) from_vec<P>(o, out, 0);
  });
  return elapsed;
}

// MC-MLP training with the reference's own modules (config 3 oracle):
// MCSequential of MCLinear(+bias) and ReLULayer (nn.hpp:49-92,132-136,162-201),
// cross_entropy_loss (autodiff.hpp:541-582), Tape::backward (:209-228) and
// MCSGD (optim.hpp:34-77, momentum 0).  params: for each layer l the weight
// (dims[l+1] x dims[l] x nc) then the bias (dims[l+1] x nc), binary32
// components; X (n x dims[0]) binary32; losses[s] = loss before update s.
int mcfref_mlp_train(const int* dims, int nlayers, int nc, const float* params, const float* X,
                     const int* labels, int64_t n, int steps, double lr, float* losses,
                     float* params_out) {
  using P = mcf::B32;
  try {
    mcf::Rng rng(1);
    mcf::MCSequential<P> model;
    std::vector<mcf::MCLinear<P>*> lins;
    for (int l = 0; l < nlayers; ++l) {
      auto lin = std::make_unique<mcf::MCLinear<P>>(dims[l], dims[l + 1], true, nc, rng);
      lins.push_back(lin.get());
      model.add(std::move(lin));
      if (l + 1 < nlayers) model.add(std::make_unique<mcf::ReLULayer<P>>());
    }
    const float* p = params;
    for (auto* lin : lins) {
      for (auto& v : lin->weight().raw()) v = *p++;
      for (auto& v : lin->bias()->raw()) v = *p++;
    }
    NdArray x(Shape{static_cast<std::size_t>(n), static_cast<std::size_t>(dims[0])});
    for (std::size_t i = 0; i < x.numel(); ++i) x[i] = X[i];
    const std::vector<int> lab(labels, labels + n);
    mcf::MCSGD<P> opt(model.parameters(), {lr, 0.0, false});
    for (int s = 0; s < steps; ++s) {
      mcf::Tape<P> tape;
      const mcf::Var in = tape.leaf(x);
      const mcf::Var logits = model.forward(tape, in);
      const mcf::Var loss = mcf::cross_entropy_loss(tape, logits, lab);
      losses[s] = static_cast<float>(tape.value(loss)[0]);
      tape.backward(loss);
      opt.step();
      model.zero_grad();
    }
    float* q = params_out;
    for (auto* lin : lins) {
      for (double v : lin->weight().raw()) *q++ = static_cast<float>(v);
      for (double v : lin->bias()->raw()) *q++ = static_cast<float>(v);
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}


// the reference's own generator (rng.hpp:13-65): the bench's reference arm
// draws its inputs here, so it never loads the product library
void mcfref_rng_uniform(std::uint64_t seed, std::int64_t n, double* out) {
  mcf::Rng g(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = g.uniform();
}
void mcfref_rng_normal(std::uint64_t seed, std::int64_t n, double* out) {
  mcf::Rng g(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = g.normal();
}
void mcfref_rng_below(std::uint64_t seed, std::uint64_t bound, std::int64_t n, std::uint64_t* out) {
  mcf::Rng g(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = g.below(bound);
}

// checkpoint_to_json (nn.hpp:207-214) of the reference's MC-MLP (MCSequential
// of MCLinear + ReLU, as mcfref_mlp_train builds it) holding `params`, dumped
// as write_json_file does; returns the length or -1 if it does not fit
std::int64_t mcfref_mlp_checkpoint(const int* dims, int nlayers, int nc, const float* params, char* buf,
                                   std::int64_t cap) {
  using P = mcf::B32;
  try {
    mcf::Rng rng(1);
    mcf::MCSequential<P> model;
    std::vector<mcf::MCLinear<P>*> lins;
    for (int l = 0; l < nlayers; ++l) {
      auto lin = std::make_unique<mcf::MCLinear<P>>(dims[l], dims[l + 1], true, nc, rng);
      lins.push_back(lin.get());
      model.add(std::move(lin));
      if (l + 1 < nlayers) model.add(std::make_unique<mcf::ReLULayer<P>>());
    }
    const float* p = params;
    for (auto* lin : lins) {
      for (auto& v : lin->weight().raw()) v = *p++;
      for (auto& v : lin->bias()->raw()) v = *p++;
    }
    const std::string s = mcf::checkpoint_to_json(model).dump(2);
    if (static_cast<std::int64_t>(s.size()) >= cap) return -1;
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
    return static_cast<std::int64_t>(s.size());
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
