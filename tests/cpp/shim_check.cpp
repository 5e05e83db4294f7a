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
