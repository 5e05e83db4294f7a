// shim_check.cpp -- the drop-in C++ API (include/mcf_gpu.hpp) against the
// reference itself: every mcf::gpu:: operator must return exactly the
// reference's mcf:: result (raw component doubles compared bitwise) on
// seeded inputs, and raise the same exception types.  Built by oracle/Makefile
// (it needs the reference headers) into oracle/_ref/shim_check; run on the GPU
// box by tests/test_gpu_shim.py.
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "mcf_gpu.hpp"
#include "mcfloat/rng.hpp"

using namespace mcf;

static int g_fail = 0;

template <class P>
static MCTensor<P> random_mct(Rng& rng, std::size_t n, int nc) {
  MCTensor<P> t(Shape{n}, nc);
  for (std::size_t e = 0; e < n; ++e) {
    const double v = rng.uniform(-1.0, 1.0) * std::exp2(rng.uniform(-6.0, 6.0));
    detail::expansion_of_double<P>(v, t.comps(e), nc);
  }
  return t;
}

template <class P>
static NdArray random_wp(Rng& rng, Shape s) {
  NdArray a(s);
  for (std::size_t i = 0; i < a.numel(); ++i) a[i] = P::round(rng.uniform(-1.0, 1.0) * std::exp2(rng.uniform(-4.0, 4.0)));
  return a;
}

template <class P>
static void same(const MCTensor<P>& got, const MCTensor<P>& want, const char* what) {
  bool ok = got.raw().size() == want.raw().size() && got.shape() == want.shape();
  for (std::size_t i = 0; ok && i < got.raw().size(); ++i) {
    const double a = got.raw()[i], b = want.raw()[i];
    ok = std::bit_cast<std::uint64_t>(a) == std::bit_cast<std::uint64_t>(b) || (std::isnan(a) && std::isnan(b));
  }
  std::printf("%-40s %s %s\n", what, P::name, ok ? "ok" : "MISMATCH");
  if (!ok) ++g_fail;
}

template <class P>
static void run(int nc) {
  Rng rng(700 + nc);
  const std::size_t n = 4097;
  const auto x = random_mct<P>(rng, n, nc), y = random_mct<P>(rng, n, nc);
  auto yd = y;
  for (std::size_t e = 0; e < n; ++e) {
    const double shifted = y.comps(e)[0] + std::copysign(0.5, y.comps(e)[0]);
    detail::expansion_of_double<P>(shifted, yd.comps(e), nc);
  }
  const NdArray v = random_wp<P>(rng, Shape{n});
  const NdArray s = NdArray::scalar(P::round(1.75));
  char buf[64];
  auto tag = [&](const char* op) {
    std::snprintf(buf, sizeof buf, "%s nc=%d", op, nc);
    return buf;
  };
  same(gpu::grow_expn(x, v), grow_expn(x, v), tag("grow_expn"));
  same(gpu::grow_expn(x, s), grow_expn(x, s), tag("grow_expn scalar"));
  same(gpu::scaling_n(x, v), scaling_n(x, v), tag("scaling_n"));
  if (nc < 8) same(gpu::scaling_n(x, v, true), scaling_n(x, v, true), tag("scaling_n expanded"));
  same(gpu::div_n(v, yd), div_n(v, yd), tag("div_n"));
  same(gpu::add_mcn(x, y), add_mcn(x, y), tag("add_mcn"));
  same(gpu::div_mcn(x, yd), div_mcn(x, yd), tag("div_mcn"));
  same(gpu::mul_mcn(x, y), mul_mcn(x, y), tag("mul_mcn"));
  same(gpu::mul_mcn_slow(x, y), mul_mcn_slow(x, y), tag("mul_mcn_slow"));
  same(gpu::square_mcn(x), square_mcn(x), tag("square_mcn"));
  same(gpu::negate(x), negate(x), tag("negate"));
  {
    // mc_relu_op's value, through the reference's tape
    MCTensor<P> px = x;
    Tape<P> tape;
    const auto r = mc_relu_op(tape, tape.mc_param(px));
    same(gpu::mc_relu(x), tape.mc_value(r), tag("mc_relu"));
    // mc_softmax: the GPU's exp is correctly rounded, the reference's is libm:
    // compare the evaluated values (the expansions may differ in the last bit
    // of a component where libm's exp is not correctly rounded)
    MCTensor<P> a(Shape{6, 9}, nc);
    for (std::size_t e = 0; e < a.numel(); ++e)
      detail::expansion_of_double<P>(rng.uniform(-3.0, 3.0), a.comps(e), nc);
    for (int axis : {-1, 0}) {
      const NdArray g = gpu::mc_softmax(a, axis).approx(), w = mc_softmax(a, axis).approx();
      double worst = 0;
      for (std::size_t i = 0; i < g.numel(); ++i) worst = std::fmax(worst, std::fabs(g[i] - w[i]) / std::fabs(w[i]));
      const bool ok = worst <= std::ldexp(1.0, -P::significand_bits + 2);
      std::printf("%-40s %s %s\n", tag(axis < 0 ? "mc_softmax axis -1" : "mc_softmax axis 0"), P::name,
                  ok ? "ok" : "MISMATCH");
      g_fail += ok ? 0 : 1;
    }
  }
  if (nc < 8) {
    MCTensor<P> a(Shape{19, 33}, nc);
    for (std::size_t e = 0; e < a.numel(); ++e)
      detail::expansion_of_double<P>(rng.uniform(-2.0, 2.0), a.comps(e), nc);
    const NdArray w = random_wp<P>(rng, Shape{33, 7});
    same(gpu::mm_mcn(a, w), mm_mcn(a, w), tag("mm_mcn (reference order)"));
    const NdArray vv = random_wp<P>(rng, Shape{33});
    same(gpu::mv_mcn(a, vv), mv_mcn(a, vv), tag("mv_mcn"));
    const ReductionPlan tree{ReduceStrategy::kPairwiseTree, 2};
    same(gpu::mm_mcn(a, w, tree), mm_mcn(a, w, tree), tag("mm_mcn (pairwise tree)"));
    bool threw = false;
    try {
      gpu::mm_mcn(a, a);
    } catch (const unsupported_operation&) {
      threw = true;
    }
    std::printf("%-40s %s %s\n", tag("mm_mcn MC x MC refused"), P::name, threw ? "ok" : "MISMATCH");
    g_fail += threw ? 0 : 1;
    threw = false;
    try {
      gpu::mm_mcn(a, NdArray(Shape{3, 2}));
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()).find("(19,33)") != std::string::npos;
    }
    std::printf("%-40s %s %s\n", tag("mm_mcn shape error message"), P::name, threw ? "ok" : "MISMATCH");
    g_fail += threw ? 0 : 1;
    // the remaining linalg.hpp entry points, and the rank dispatcher against
    // both the reference and the specialised GPU operators (T/test_linalg.cpp:220-257)
    MCTensor<P> x4(Shape{2, 3, 5, 6}, nc), x3(Shape{3, 5, 6}, nc), x1(Shape{6}, nc);
    for (auto* t : {&x4, &x3, &x1})
      for (std::size_t e = 0; e < t->numel(); ++e)
        detail::expansion_of_double<P>(rng.uniform(-2.0, 2.0), t->comps(e), nc);
    const NdArray w4 = random_wp<P>(rng, Shape{2, 3, 6, 4}), w3 = random_wp<P>(rng, Shape{3, 6, 4});
    const NdArray w2 = random_wp<P>(rng, Shape{6, 4}), w1 = random_wp<P>(rng, Shape{6});
    same(gpu::mm4d_mcn(x4, w4), mm4d_mcn(x4, w4), tag("mm4d_mcn"));
    same(gpu::matmul_mcn(x4, w4), mm4d_mcn(x4, w4), tag("matmul_mcn 4x4 == mm4d"));
    same(gpu::matmul_mcn(x4, w4), gpu::mm4d_mcn(x4, w4), tag("matmul_mcn 4x4 == gpu mm4d"));
    same(gpu::matmul_mcn(x4, w2), matmul_mcn(x4, w2), tag("matmul_mcn 4x2"));
    same(gpu::matmul_mcn(x3, w3), bmm_mcn(x3, w3), tag("matmul_mcn 3x3 == bmm"));
    same(gpu::matmul_mcn(x3, w2), matmul_mcn(x3, w2), tag("matmul_mcn 3x2"));
    const MCTensor<P> x2 = mc_transpose2d(mc_transpose2d(gpu::mc_transpose2d(a)));
    same(gpu::matmul_mcn(x1, w2), matmul_mcn(x1, w2), tag("matmul_mcn 1x2"));
    same(gpu::matmul_mcn(x1, w1), dot_mcn(x1, w1), tag("matmul_mcn 1x1 == dot"));
    same(gpu::matmul_mcn(a, w), gpu::mm_mcn(a, w), tag("matmul_mcn 2x2 == gpu mm"));
    same(gpu::matmul_mcn(a, vv), mv_mcn(a, vv), tag("matmul_mcn 2x1 == mv"));
    same(gpu::mc_transpose2d(a), mc_transpose2d(a), tag("mc_transpose2d"));
    same(x2, mc_transpose2d(a), tag("mc_transpose2d (thrice)"));
    threw = false;
    try {
      gpu::matmul_mcn(x3, NdArray(Shape{5, 2}));
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()).find("(3,5,6)") != std::string::npos;
    }
    std::printf("%-40s %s %s\n", tag("matmul_mcn shape error message"), P::name, threw ? "ok" : "MISMATCH");
    g_fail += threw ? 0 : 1;
    // addmm: alpha / beta through ScalingN, bias broadcast over the rows
    MCTensor<P> bias_full(Shape{19, 7}, nc), bias_row(Shape{7}, nc);
    for (auto* t : {&bias_full, &bias_row})
      for (std::size_t e = 0; e < t->numel(); ++e)
        detail::expansion_of_double<P>(rng.uniform(-1.0, 1.0), t->comps(e), nc);
    same(gpu::addmm_mcn(bias_full, a, w), addmm_mcn(bias_full, a, w), tag("addmm_mcn"));
    same(gpu::addmm_mcn(bias_row, a, w, 0.75, -1.5), addmm_mcn(bias_row, a, w, 0.75, -1.5),
         tag("addmm_mcn alpha beta broadcast"));
    // EFT arrays and renormalization of raw expansions
    std::vector<double> av(333), bv(333);
    for (std::size_t i = 0; i < av.size(); ++i) {
      av[i] = P::round(rng.uniform(-1.0, 1.0) * std::exp2(rng.uniform(-20.0, 20.0)));
      bv[i] = P::round(rng.uniform(-1.0, 1.0) * std::exp2(rng.uniform(-20.0, 20.0)));
    }
    for (int k = 0; k < 2; ++k) {
      std::vector<double> gs, ge, rs, re;
      if (k == 0) {
        gpu::two_sum<P>(av, bv, gs, ge);
        two_sum<P>(av, bv, rs, re);
      } else {
        gpu::two_prod<P>(av, bv, gs, ge);
        two_prod<P>(av, bv, rs, re);
      }
      MCTensor<P> g(Shape{av.size()}, 2), r(Shape{av.size()}, 2);
      for (std::size_t i = 0; i < av.size(); ++i) {
        g.comps(i)[0] = gs[i], g.comps(i)[1] = ge[i];
        r.comps(i)[0] = rs[i], r.comps(i)[1] = re[i];
      }
      same(g, r, tag(k == 0 ? "two_sum (array form)" : "two_prod (array form)"));
    }
    MCTensor<P> raw(Shape{257}, nc + 1);  // unnormalised expansions: any order, zeros, overlaps
    for (std::size_t e = 0; e < raw.numel(); ++e)
      for (int c = 0; c <= nc; ++c)
        raw.comps(e)[c] = (e + c) % 5 == 0 ? 0.0 : P::round(rng.uniform(-1.0, 1.0) * std::exp2(rng.uniform(-30.0, 2.0)));
    for (int rn : {1, nc, nc + 1}) {
      std::snprintf(buf, sizeof buf, "renormalize nc=%d->%d", nc + 1, rn);
      same(gpu::renormalize(raw, rn), renormalize(raw, rn), buf);
      std::snprintf(buf, sizeof buf, "simple_renorm nc=%d->%d", nc + 1, rn);
      same(gpu::simple_renorm(raw, rn), simple_renorm(raw, rn), buf);
    }
  }
}

int main() {
  for (int nc : {1, 2, 3, 4, 8}) {
    run<B32>(nc);
    run<B16>(nc);
    run<B64>(nc);
  }
  bool threw = false;
  try {
    gpu::square_mcn(MCTensor<B32>(Shape{1}, 9));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  std::printf("nc limit enforced: %s\n", threw ? "ok" : "MISMATCH");
  g_fail += threw ? 0 : 1;
  std::printf("%s: %d failures\n", g_fail ? "FAIL" : "PASS", g_fail);
  return g_fail ? 1 : 0;
}
