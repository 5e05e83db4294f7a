// g2_verify.cpp -- checks the certified nc = 2 shortcuts (csrc/mcf_g2.cuh)
// against the reference's own algorithms in an emulated binary format with p
// significand bits and unbounded exponent (TEST TOOL, not product code).
//
// The reference's algorithms are restated below generically (renorm_kernel
// with its pass cap, scale_raw, add_kernel, div_kernel, mul_fast_kernel,
// square_kernel: mc_ops.hpp:41-282).  For small p every compressed operand
// pair in a window of exponents is enumerated; for p = 24 operands are
// sampled like config 0.  For each case it records
//   * whether any renorm inside the reference op reached its pass cap
//     without being compressed (the certification argument assumes not),
//   * whether the shortcut accepted, and if so whether it equals the
//     reference bit for bit (including the sign of zeros).
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp tools/g2_verify.cpp -o /tmp/g2v
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include <omp.h>

#include "../paper_2207_08867_b200/csrc/mcf_g2.cuh"
#include "../paper_2207_08867_b200/csrc/mcf_w2.cuh"

static int P = 24;  // significand bits of the emulated format

// round to nearest even at P bits, unbounded exponent (exact for the double
// results used here: double rounding is innocuous for p <= 25)
static double rn(double x) {
  if (x == 0 || !std::isfinite(x)) return x;
  int e;
  const double m = std::frexp(x, &e);
  return std::ldexp(std::nearbyint(std::ldexp(m, P)), e - P);
}

struct QE {
  using T = double;
  using B = bool;
  static T c(double v) { return v; }
  static T neg(T a) { return -a; }
  static T sel(B m, T a, T b) { return m ? a : b; }
  static B eq(T a, T b) { return a == b; }
  static B lt(T a, T b) { return a < b; }
  static B ge(T a, T b) { return a >= b; }
  static T add(T a, T b) { return rn(a + b); }
  static T sub(T a, T b) { return rn(a - b); }
  static T mul(T a, T b) { return rn(a * b); }
  static T div(T a, T b) { return rn(a / b); }
  static T fma(T a, T b, T c) { return rn(a * b + c); }  // a*b exact for p <= 26
  static T abs(T a) { return std::fabs(a); }
  static bool finite(T a) { return std::isfinite(a); }
  static bool big(T a) { return a != 0; }  // no underflow in the emulation
  static T canon(T a) { return a + 0.0; }
  // the device construction: 2^floor(log2(RN(|t| (1 - 2^-p)))) * 2^-p, i.e.
  // ulp(t)/2, or ulp(t)/4 when |t| is a power of two
  static T hb(T t) { return hbd(t, 0.0, false); }
  static T hbd(T t, T d, bool dir = true) {
    if (t == 0 || !std::isfinite(t)) return t == 0 ? 0 : INFINITY;
    const bool away = dir && (std::signbit(d) == std::signbit(t));
    const double u = rn(std::fabs(t) * (away ? 1.0 : 1.0 - std::ldexp(1.0, -P)));
    int e;
    std::frexp(u, &e);
    return std::ldexp(1.0, e - 1 - P);
  }
  static T ulpb(T w) { return std::fabs(w) * std::ldexp(1.0, -P); }
  static T shrink(T h) { return rn(h * (1.0 - std::ldexp(1.0, -(P - 2)))); }
};

// wide format of the mcf_w2.cuh tier: 2 P + 5 significand bits (53 for P = 24,
// where the emulation is the host's own binary64 arithmetic)
static int WB() { return 2 * P + 5; }
static double rnw(double x) {
  if (WB() >= 53 || x == 0 || !std::isfinite(x)) return x;
  int e;
  const double m = std::frexp(x, &e);
  return std::ldexp(std::nearbyint(std::ldexp(m, WB())), e - WB());
}
static uint64_t wmant(double t) {  // the W-bit significand of a wide value as an integer
  if (t == 0) return 0;
  int e;
  return (uint64_t)std::ldexp(std::frexp(std::fabs(t), &e), WB());
}
static int g_lg1 = 10;    // div_core1's margin (log2 units); G2_LG1 lowers it to probe the bound's slack
static bool g_only1 = false;  // G2_ONLY1: only the one-digit rows
struct VE {
  using N = double;
  using W = double;
  static W c(double v) { return v; }
  static W two(int k) { return std::ldexp(1.0, k); }
  static W tol_rcp() { return std::ldexp(1.0, -(WB() - 3)); }
  static W wide(N x) { return x; }
  static N narrow(W x) { return x; }
  static N canon(N x) { return x + 0.0; }
  static W neg(W a) { return -a; }
  static W abs(W a) { return std::fabs(a); }
  static W add(W a, W b) { return rnw(a + b); }
  static W sub(W a, W b) { return rnw(a - b); }
  static W mul(W a, W b) { return rnw(a * b); }
  static W fma(W a, W b, W c) { return WB() >= 53 ? std::fma(a, b, c) : rnw(a * b + c); }
  static bool eq(W a, W b) { return a == b; }
  static bool ge(W a, W b) { return a >= b; }
  static bool le(W a, W b) { return a <= b; }
  static W rcp_seed(W y) { return rnw((1.0 / y) * (1.0 + std::ldexp(1.0, -16))); }
  static int lg1() { return g_lg1; }
  static constexpr int kP_dummy = 0;
  struct KP { operator int() const { return P; } };
  static constexpr KP kP{};
  static bool in_window(N a) { return std::fabs(a) >= std::ldexp(1.0, -40) && std::fabs(a) <= std::ldexp(1.0, 40); }
  static bool below_window(N a) { return std::fabs(a) <= std::ldexp(1.0, 40); }
  static bool lead_window(N a) { return std::fabs(a) >= std::ldexp(1.0, -30) && std::fabs(a) <= std::ldexp(1.0, 40); }
  static bool tail_window(N a) { return a == 0.0 || std::fabs(a) >= std::ldexp(1.0, -60); }
  static W rnpe(W t) { return rn(t); }
  static W rnp(W t) {  // ties away from zero, as the device's pattern rounding
    if (t == 0 || !std::isfinite(t)) return t;
    int e;
    const double m = std::frexp(std::fabs(t), &e);
    return std::copysign(std::ldexp(std::floor(std::ldexp(m, P) + 0.5), e - P), t);
  }
  // the device declines L - mid in [-m, 3 m) (one mask test): a superset of
  // this symmetric margin, which keeps more accepted cases to check here
  static W rnpm(W t, int m, bool& ok) {
    ok &= away(t, m);
    return rnp(t);
  }
  static W rnpv(W t, W ref, int lg, bool& ok) {  // as the device: distance to the nearest midpoint of t's grid
    const W o = rnp(t);
    if (t == 0 || !std::isfinite(t)) { ok = false; return o; }
    const double half = std::ldexp(1.0, std::ilogb(t) - P);
    ok &= sub(half, std::fabs(sub(t, o))) > mul(std::fabs(ref), std::ldexp(1.0, lg - (WB() - 1)));
    return o;
  }
  static bool away(W t, int m) {
    const int64_t L = (int64_t)(wmant(t) & ((1ull << (WB() - P)) - 1)), mid = 1ll << (WB() - P - 1);
    return std::llabs(L - mid) > m;
  }
  static bool span2p(W t) { return (wmant(t) & ((1ull << (WB() - 2 * P)) - 1)) == 0; }
};

// ---- the reference, restated generically (mc_ops.hpp) ----------------------
static bool g_cap = false;  // a renorm ended at its pass cap uncompressed

struct TS { double s, e; };
static TS two_sum(double a, double b) {
  const double s = rn(a + b), bv = rn(s - a), av = rn(s - bv);
  return {s, rn(rn(a - av) + rn(b - bv))};
}
static TS two_prod(double a, double b) {
  const double p = rn(a * b);
  return {p, rn(a * b - p)};
}
static bool is_compressed(const double* h, int n) {
  for (int i = 0; i + 1 < n; ++i)
    if (rn(h[i] + h[i + 1]) != h[i]) return false;
  return true;
}
static void renorm(const double* in, int n, double* out, int r_nc) {  // mc_ops.hpp:68-92
  double h[64];
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (in[i] != 0.0) h[m++] = in[i];
  if (m > 1) {
    for (int i = 1; i < m; ++i) {  // stable insertion sort by decreasing magnitude
      const double v = h[i];
      int j = i - 1;
      while (j >= 0 && std::fabs(h[j]) < std::fabs(v)) {
        h[j + 1] = h[j];
        --j;
      }
      h[j + 1] = v;
    }
    int pass = 0;
    for (; pass < m + 4 && !is_compressed(h, m); ++pass) {
      for (int i = m - 2; i >= 0; --i) {
        const TS r = two_sum(h[i], h[i + 1]);
        h[i] = r.s;
        h[i + 1] = r.e;
      }
      int k = 0;
      for (int i = 0; i < m; ++i)
        if (h[i] != 0.0) h[k++] = h[i];
      m = k;
      if (m <= 1) break;
    }
    if (m > 1 && !is_compressed(h, m)) g_cap = true;
  }
  for (int i = 0; i < r_nc; ++i) out[i] = i < m ? h[i] : 0.0;
}
static int scale_raw(const double* x, int nc, double v, double* out) {  // :143-158
  TS qp = two_prod(x[nc - 1], v);
  double q = qp.s;
  out[0] = qp.e;
  int k = 1;
  for (int i = nc - 2; i >= 0; --i) {
    const TS t = two_prod(x[i], v);
    const TS s1 = two_sum(q, t.e);
    out[k++] = s1.e;
    const TS s2 = two_sum(t.s, s1.s);
    out[k++] = s2.e;
    q = s2.s;
  }
  out[k++] = q;
  return k;
}
static void ref_scale(const double* x, double v, double* out) {
  double st[16];
  const int m = scale_raw(x, 2, v, st);
  renorm(st, m, out, 2);
}
static void ref_grow(const double* x, double v, double* out) {  // mc_ops.hpp:118-138, nc = 2
  double h[3];
  double q = v;
  for (int k = 2; k >= 1; --k) {
    const TS r = two_sum(x[k - 1], q);
    q = r.s;
    h[k] = r.e;
  }
  h[0] = q;
  double c[3];
  int m = 0;
  for (int i = 0; i < 3; ++i)
    if (h[i] != 0.0) c[m++] = h[i];
  if (is_compressed(c, m)) {
    for (int i = 0; i < 2; ++i) out[i] = i < m ? c[i] : 0.0;
  } else {
    renorm(h, 3, out, 2);
  }
}
static void ref_add(const double* x, const double* y, double* out) {  // :173-184
  double h[8];
  int i = 0, j = 0, k = 0;
  while (i < 2 && j < 2) h[k++] = std::fabs(x[i]) >= std::fabs(y[j]) ? x[i++] : y[j++];
  while (i < 2) h[k++] = x[i++];
  while (j < 2) h[k++] = y[j++];
  renorm(h, k, out, 2);
}
static void ref_div(const double* x, const double* y, double* out) {  // :188-207
  double q[3] = {0, 0, 0}, r[2] = {x[0], x[1]}, sc[2], st[16];
  for (int d = 0;; ++d) {
    q[d] = rn(r[0] / y[0]);
    if (d == 2) break;
    const int m = scale_raw(y, 2, -q[d], st);
    renorm(st, m, sc, 2);
    ref_add(r, sc, r);
  }
  renorm(q, 3, out, 2);
}
static void ref_mul(const double* x, const double* y, double* out) {  // :216-230
  if (rn(y[1] + y[0]) == 0.0 || rn(x[1] + x[0]) == 0.0) {
    out[0] = out[1] = 0.0;
    return;
  }
  const double one[2] = {1.0, 0.0};
  double rec[2];
  ref_div(one, y, rec);
  ref_div(x, rec, out);
}
static void ref_mul_slow(const double* x, const double* y, double* out) {  // :234-251, nc = 2
  double h[8];
  int m = 0;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; i + j < 2; ++j) {
      const TS t = two_prod(x[i], y[j]);
      h[m++] = t.s;
      h[m++] = t.e;
    }
  h[m++] = rn(x[1] * y[1]);
  renorm(h, m, out, 2);
}
static void ref_square(const double* x, double* out) {  // :256-282
  double h[8];
  int m = 0;
  for (int i = 0; i < 2; ++i)
    for (int j = i; i + j < 2; ++j) {
      const TS t = two_prod(x[i], x[j]);
      h[m++] = i == j ? t.s : 2.0 * t.s;
      h[m++] = i == j ? t.e : 2.0 * t.e;
    }
  h[m++] = rn(x[1] * x[1]);
  renorm(h, m, out, 2);
}

// ---- comparison ----------------------------------------------------------------
struct Stat {
  const char* name;
  long long n = 0, acc = 0, bad = 0, cap = 0;
};
static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

template <class F, class G>
static void check(Stat& st, F ref, G fast, const char* what) {
  if (g_only1 && st.name[1] != '1' && st.name[2] != 'm') return;
  double ro[2], fo[2];
  g_cap = false;
  ref(ro);
  const bool cap = g_cap;
  const bool ok = fast(fo);
#pragma omp atomic
  st.n++;
  if (cap) {
#pragma omp atomic
    st.cap++;
  }
  if (ok) {
#pragma omp atomic
    st.acc++;
    if (!same(ro[0], fo[0]) || !same(ro[1], fo[1])) {
      long long b;
#pragma omp atomic capture
      b = ++st.bad;
      if (b <= 5)
#pragma omp critical
        printf("  MISMATCH %s %s: ref (%.17g, %.17g) fast (%.17g, %.17g)\n", st.name, what, ro[0], ro[1],
               fo[0], fo[1]);
    }
  }
}

static void report(const Stat& s) {
  printf("p=%2d %-7s cases %11lld  accepted %6.3f%%  mismatches %lld  cap-hits %lld\n", P, s.name, s.n,
         s.n ? 100.0 * s.acc / s.n : 0.0, s.bad, s.cap);
}

// compressed pairs (x0, x1), x0 in +-[1,2) on the p-bit grid, x1 = 0 or
// +-m 2^k with k in [-(p+1+K), -(p-1)], filtered by the reference predicate
static std::vector<std::pair<double, double>> pairs(int K, int mstep) {
  std::vector<std::pair<double, double>> v;
  const int M = 1 << (P - 1);
  for (int s0 = -1; s0 <= 1; s0 += 2)
    for (int a = 0; a < M; a += 1) {
      const double x0 = s0 * std::ldexp(M + a, -(P - 1));
      v.push_back({x0, 0.0});
      for (int k = -(P - 1); k >= -(P + 1 + K); --k)
        for (int s1 = -1; s1 <= 1; s1 += 2)
          for (int b = 0; b < M; b += mstep) {
            const double x1 = s1 * std::ldexp(M + b, k - (P - 1));
            if (rn(x0 + x1) == x0) v.push_back({x0, x1});
          }
    }
  return v;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "small";
  if (getenv("G2_LG1")) g_lg1 = atoi(getenv("G2_LG1"));
  g_only1 = getenv("G2_ONLY1") != nullptr;
  using namespace mcfg;
  if (!strcmp(mode, "small")) {
    const int p = argc > 2 ? atoi(argv[2]) : 5;
    const int K = argc > 3 ? atoi(argv[3]) : 6;
    P = p;
    auto X = pairs(K, 1);
    const int M = 1 << (P - 1);
    printf("p=%d: %zu compressed pairs\n", P, X.size());
    Stat ss{"scale"}, sq{"square"}, sd{"div"}, sm{"mul"}, sa{"add"}, sg{"grow"}, wd{"w2div"}, wm{"w2mul"}, ws{"w2scale"}, od{"w1div"}, om{"w1mul"}, wl{"w2mslow"}, wq{"w2msq"};
#pragma omp parallel for schedule(dynamic, 16)
    for (long long i = 0; i < (long long)X.size(); ++i) {
      const double x[2] = {X[i].first, X[i].second};
      check(sq, [&](double* o) { ref_square(x, o); },
            [&](double* o) { return g2::square<QE>(x[0], x[1], o[0], o[1]); }, "sq");
      check(wq, [&](double* o) { ref_square(x, o); },
            [&](double* o) { return w2::square<VE>(x[0], x[1], true, o[0], o[1]); }, "sq");
      for (int a = 0; a < M; ++a) {  // div_n: a single-component numerator over x as divisor
        const double vn[2] = {std::ldexp(M + a, -(P - 1)), 0.0};
        check(sd, [&](double* o) { ref_div(vn, x, o); },
              [&](double* o) { return g2::div<QE, true>(vn[0], vn[1], x[0], x[1], o[0], o[1]); }, "divn");
        check(wd, [&](double* o) { ref_div(vn, x, o); },
              [&](double* o) { return w2::div<VE, true>(vn[0], vn[1], x[0], x[1], true, true, o[0], o[1]); }, "divn");
        check(od, [&](double* o) { ref_div(vn, x, o); },
              [&](double* o) { return w2::div<VE, true, true>(vn[0], vn[1], x[0], x[1], true, true, o[0], o[1]); }, "divn");
      }
      for (int s = -1; s <= 1; s += 2)
        for (int a = 0; a < M; ++a) {
          const double v = s * std::ldexp(M + a, -(P - 1));
          check(ss, [&](double* o) { ref_scale(x, v, o); },
                [&](double* o) { return g2::scale<QE>(x[0], x[1], v, o[0], o[1]); }, "sc");
          check(ws, [&](double* o) { ref_scale(x, v, o); },
                [&](double* o) { return w2::scale<VE>(x[0], x[1], v, true, o[0], o[1]); }, "sc");
          for (int sh = -(P + 3); sh <= 2; ++sh) {  // grow by values around every component
            const double vg = std::ldexp(v, sh);
            check(sg, [&](double* o) { ref_grow(x, vg, o); },
                  [&](double* o) { return g2::grow<QE>(x[0], x[1], vg, o[0], o[1]); }, "grow");
          }
        }
      for (size_t j = 0; j < X.size(); ++j) {
        const double y[2] = {X[j].first, X[j].second};
        check(sd, [&](double* o) { ref_div(x, y, o); },
              [&](double* o) { return g2::div<QE>(x[0], x[1], y[0], y[1], o[0], o[1]); }, "div");
        check(wd, [&](double* o) { ref_div(x, y, o); },
              [&](double* o) { return w2::div<VE, false>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "div");
        check(od, [&](double* o) { ref_div(x, y, o); },
              [&](double* o) { return w2::div<VE, false, true>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "div");
        check(wl, [&](double* o) { ref_mul_slow(x, y, o); },
              [&](double* o) { return w2::mul_slow<VE>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "mslow");
        for (int sh = -3; sh <= 3; sh += 3) {  // relative exponent of y
          const double ys[2] = {std::ldexp(y[0], sh), std::ldexp(y[1], sh)};
          check(sa, [&](double* o) { ref_add(x, ys, o); },
                [&](double* o) { return g2::add<QE>(x[0], x[1], ys[0], ys[1], o[0], o[1]); }, "add");
        }
        if ((i + j) % 3 == 0) {
          check(sm, [&](double* o) { ref_mul(x, y, o); },
                [&](double* o) { return g2::mul<QE>(x[0], x[1], y[0], y[1], o[0], o[1]); }, "mul");
          check(wm, [&](double* o) { ref_mul(x, y, o); },
                [&](double* o) { return w2::mul<VE>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "mul");
          check(om, [&](double* o) { ref_mul(x, y, o); },
                [&](double* o) { return w2::mul<VE, true>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "mul");
        }
      }
    }
    report(ss), report(sq), report(sd), report(sm), report(sa), report(sg), report(wd), report(wm), report(ws), report(od), report(om), report(wl), report(wq);
    return (ss.bad | sq.bad | sd.bad | sm.bad | sa.bad | sg.bad | wd.bad | wm.bad | ws.bad | od.bad | om.bad | wl.bad | wq.bad | ss.cap | sq.cap | sd.cap | sm.cap |
            sa.cap | sg.cap) ? 1 : 0;
  }
  // sampled, config-0 style operands: v = U(-1,1) 2^U(-8,8) split greedily into p-bit comps
  P = argc > 2 ? atoi(argv[2]) : 24;
  const long long N = argc > 3 ? atoll(argv[3]) : 2000000;
  Stat ss{"scale"}, sq{"square"}, sd{"div"}, sm{"mul"}, sa{"add"}, sg{"grow"}, wd{"w2div"}, wm{"w2mul"}, ws{"w2scale"}, od{"w1div"}, om{"w1mul"}, wl{"w2mslow"}, wq{"w2msq"};
#pragma omp parallel
  {
    std::mt19937_64 g(1234 + 7919 * (unsigned long long)omp_get_thread_num());
    std::uniform_real_distribution<double> u(-1.0, 1.0), ue(-8.0, 8.0);
    auto draw = [&](double* x, bool divisor) {
      double v = u(g) * std::exp2(ue(g));
      if (divisor) v += v < 0 ? -0.5 : 0.5;
      x[0] = rn(v);
      x[1] = rn(v - x[0]);
    };
#pragma omp for schedule(static)
    for (long long i = 0; i < N; ++i) {
      double x[2], y[2], v2[2];
      draw(x, false), draw(y, true), draw(v2, false);
      const double v = v2[0];
      check(ss, [&](double* o) { ref_scale(x, v, o); },
            [&](double* o) { return g2::scale<QE>(x[0], x[1], v, o[0], o[1]); }, "sc");
      check(ws, [&](double* o) { ref_scale(x, v, o); },
            [&](double* o) { return w2::scale<VE>(x[0], x[1], v, true, o[0], o[1]); }, "sc");
      check(sq, [&](double* o) { ref_square(x, o); },
            [&](double* o) { return g2::square<QE>(x[0], x[1], o[0], o[1]); }, "sq");
      check(wq, [&](double* o) { ref_square(x, o); },
            [&](double* o) { return w2::square<VE>(x[0], x[1], true, o[0], o[1]); }, "sq");
      check(sd, [&](double* o) { ref_div(x, y, o); },
            [&](double* o) { return g2::div<QE>(x[0], x[1], y[0], y[1], o[0], o[1]); }, "div");
      const double vv[2] = {v2[0], 0.0};
      check(sd, [&](double* o) { ref_div(vv, y, o); },
            [&](double* o) { return g2::div<QE, true>(vv[0], vv[1], y[0], y[1], o[0], o[1]); }, "divn");
      check(sm, [&](double* o) { ref_mul(x, y, o); },
            [&](double* o) { return g2::mul<QE>(x[0], x[1], y[0], y[1], o[0], o[1]); }, "mul");
      check(wd, [&](double* o) { ref_div(x, y, o); },
            [&](double* o) { return w2::div<VE, false>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "div");
      check(od, [&](double* o) { ref_div(x, y, o); },
            [&](double* o) { return w2::div<VE, false, true>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "div");
      check(wd, [&](double* o) { ref_div(vv, y, o); },
            [&](double* o) { return w2::div<VE, true>(vv[0], vv[1], y[0], y[1], true, true, o[0], o[1]); }, "divn");
      check(od, [&](double* o) { ref_div(vv, y, o); },
            [&](double* o) { return w2::div<VE, true, true>(vv[0], vv[1], y[0], y[1], true, true, o[0], o[1]); }, "divn");
      check(wl, [&](double* o) { ref_mul_slow(x, y, o); },
            [&](double* o) { return w2::mul_slow<VE>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "mslow");
      check(wm, [&](double* o) { ref_mul(x, y, o); },
            [&](double* o) { return w2::mul<VE>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "mul");
      check(om, [&](double* o) { ref_mul(x, y, o); },
            [&](double* o) { return w2::mul<VE, true>(x[0], x[1], y[0], y[1], true, true, o[0], o[1]); }, "mul");
      check(sa, [&](double* o) { ref_add(x, y, o); },
            [&](double* o) { return g2::add<QE>(x[0], x[1], y[0], y[1], o[0], o[1]); }, "add");
      check(sg, [&](double* o) { ref_grow(x, v, o); },
            [&](double* o) { return g2::grow<QE>(x[0], x[1], v, o[0], o[1]); }, "grow");
      const double yn[2] = {-x[0], -x[1] * 0.5};  // near-cancelling sums
      check(sa, [&](double* o) { ref_add(x, yn, o); },
            [&](double* o) { return g2::add<QE>(x[0], x[1], yn[0], yn[1], o[0], o[1]); }, "add");
    }
  }
  report(ss), report(sq), report(sd), report(sm), report(sa), report(sg), report(wd), report(wm), report(ws), report(od), report(om), report(wl), report(wq);
  return (ss.bad | sq.bad | sd.bad | sm.bad | sa.bad | sg.bad | wd.bad | wm.bad | ws.bad | od.bad | om.bad | wl.bad | wq.bad | ss.cap | sq.cap | sd.cap | sm.cap |
          sa.cap | sg.cap) ? 1 : 0;
}
