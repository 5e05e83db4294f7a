/*
 * mcf_oracle.c -- plain-C restatement of the MCF operator hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see mcf_oracle.h).  This is the checker the GPU
 * path is compared against; it is never linked into the product library.
 *
 * The algorithms are restated from the reference's header-only C++ library
 * (/root/reference/proj/include/mcfloat, cited per function in
 * mcf_oracle_body.inc).  Where the reference emulates a narrow format by
 * computing in binary64 and rounding once, this restatement computes in the
 * native format (binary32 / binary64), or in binary32 followed by one
 * rounding to binary16; both are bit-identical to the reference because
 * double rounding is innocuous for + - * / at these widths
 * (precision.hpp:3-12), and the only fma use (two_prod) is exact.
 *
 * Pinned against the reference itself: tests/test_oracle_pin.py compares
 * every entry point bitwise with oracle/_ref (the reference compiled here),
 * and tests/golden/ holds fixtures generated from oracle/_ref.
 *
 * Build (see oracle/Makefile): gcc -O2 -ffp-contract=off -fno-fast-math
 * -- the reference's FP flags (proj/CMakeLists.txt:12-18).
 */
#include "mcf_oracle.h"

#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MCFO_MAXNC 8                           /* kMaxNc, mc_ops.hpp:27 */
#define MCFO_STAGE (4 * MCFO_MAXNC * MCFO_MAXNC) /* kStage, mc_ops.hpp:31 */

/* ---- binary16 helpers ----------------------------------------------------- */

double mcfo_round_b16(double x) {
  if (!isfinite(x) || x == 0.0) return x;
  const double a = fabs(x);
  if (a >= 65520.0) return copysign(INFINITY, x); /* halfway to 2^16 rounds up */
  int e2;
  (void)frexp(a, &e2);                     /* a in [2^(e2-1), 2^e2) */
  const int quantum = (e2 - 1 >= -14) ? (e2 - 1 - 10) : -24;
  const double r = nearbyint(ldexp(a, -quantum)); /* RN-even on the kept bits */
  return copysign(ldexp(r, quantum), x);
}

static inline float h16f(float x) { return (float)mcfo_round_b16((double)x); }

static inline float b16_dec(uint16_t b) {
  const int s = b >> 15, ex = (b >> 10) & 31, f = b & 1023;
  float m;
  if (ex == 31)
    m = f ? NAN : INFINITY;
  else if (ex == 0)
    m = ldexpf((float)f, -24);
  else
    m = ldexpf((float)(1024 + f), ex - 25);
  return s ? -m : m;
}

static inline uint16_t b16_enc(float x) {
  const uint16_t sign = signbit(x) ? 0x8000 : 0;
  if (isnan(x)) return sign | 0x7e00;
  if (isinf(x)) return sign | 0x7c00;
  const float a = fabsf(x);
  if (a == 0.0f) return sign;
  if (a >= 0x1p-14f) {
    int e2;
    (void)frexpf(a, &e2);
    const int unb = e2 - 1;
    const int mant = (int)ldexpf(a, 10 - unb) - 1024;
    return (uint16_t)(sign | ((unb + 15) << 10) | mant);
  }
  return (uint16_t)(sign | (int)ldexpf(a, 24));
}

/* ---- binary64 exponentials -------------------------------------------------- */

double mcfo_libm_exp(double x) { return exp(x); }

double mcfo_cr_exp(double x, int* ambiguous) {
  if (ambiguous) *ambiguous = 0;
  if (isnan(x)) return x + x;
  if (x > 710.0) return INFINITY;
  if (x < -746.0) return 0.0;
  const __float128 y = expq((__float128)x);
  const double d = (double)y; /* binary128 -> binary64 is correctly rounded */
  if (ambiguous && isfinite(d) && d > 0.0) {
    /* the rounding is decided unless y sits within the quad error of a midpoint */
    const __float128 tol = y * 0x1p-106Q;
    const __float128 up = ((__float128)d + (__float128)nextafter(d, INFINITY)) / 2;
    const __float128 dn = ((__float128)d + (__float128)nextafter(d, 0.0)) / 2;
    if (fabsq(y - up) <= tol || fabsq(y - dn) <= tol) *ambiguous = 1;
  }
  return d;
}

static double cr_exp_plain(double x) { return mcfo_cr_exp(x, NULL); }

/* ---- per-precision instantiations ----------------------------------------- */

#define FN(name) b32_##name
#define real float
#define ST float
#define LD(s) (s)
#define SV(r) (r)
#define ADD(a, b) ((float)((a) + (b)))
#define SUB(a, b) ((float)((a) - (b)))
#define MUL(a, b) ((float)((a) * (b)))
#define DIV(a, b) ((float)((a) / (b)))
#define FMA(a, b, c) fmaf((a), (b), (c))
#define RD(d) ((float)(d))
#define SIGBITS 24
#include "mcf_oracle_body.inc"
#undef FN
#undef real
#undef ST
#undef LD
#undef SV
#undef ADD
#undef SUB
#undef MUL
#undef DIV
#undef FMA
#undef RD
#undef SIGBITS

#define FN(name) b64_##name
#define real double
#define ST double
#define LD(s) (s)
#define SV(r) (r)
#define ADD(a, b) ((a) + (b))
#define SUB(a, b) ((a) - (b))
#define MUL(a, b) ((a) * (b))
#define DIV(a, b) ((a) / (b))
#define FMA(a, b, c) fma((a), (b), (c))
#define RD(d) (d)
#define SIGBITS 53
#include "mcf_oracle_body.inc"
#undef FN
#undef real
#undef ST
#undef LD
#undef SV
#undef ADD
#undef SUB
#undef MUL
#undef DIV
#undef FMA
#undef RD
#undef SIGBITS

#define FN(name) b16_##name
#define real float
#define ST uint16_t
#define LD(s) b16_dec(s)
#define SV(r) b16_enc(r)
#define ADD(a, b) h16f((a) + (b))
#define SUB(a, b) h16f((a) - (b))
#define MUL(a, b) h16f((a) * (b))
#define DIV(a, b) h16f((a) / (b))
#define FMA(a, b, c) h16f(fmaf((a), (b), (c)))
#define RD(d) ((float)mcfo_round_b16(d))
#define SIGBITS 11
#include "mcf_oracle_body.inc"

/* ---- dispatch --------------------------------------------------------------- */

#define BAD_NC(nc) ((nc) < 1 || (nc) > MCFO_MAXNC)
#define DISPATCH(prec, call16, call32, call64) \
  switch (prec) {                              \
    case MCFO_B16: call16; break;              \
    case MCFO_B32: call32; break;              \
    case MCFO_B64: call64; break;              \
    default: return 1;                         \
  }                                            \
  return 0

int mcfo_two_sum(int prec, const void* a, const void* b, void* s, void* e, int64_t n) {
  DISPATCH(prec, b16_op_two_sum(a, b, s, e, n), b32_op_two_sum(a, b, s, e, n),
           b64_op_two_sum(a, b, s, e, n));
}

int mcfo_two_prod(int prec, const void* a, const void* b, void* p, void* e, int64_t n,
                  int use_fma) {
  DISPATCH(prec, b16_op_two_prod(a, b, p, e, n, use_fma), b32_op_two_prod(a, b, p, e, n, use_fma),
           b64_op_two_prod(a, b, p, e, n, use_fma));
}

int mcfo_renormalize(int prec, const void* h, int nc, void* out, int r_nc, int64_t numel) {
  if (BAD_NC(nc) || BAD_NC(r_nc)) return 1;
  DISPATCH(prec, b16_op_renorm(h, nc, out, r_nc, numel, 0), b32_op_renorm(h, nc, out, r_nc, numel, 0),
           b64_op_renorm(h, nc, out, r_nc, numel, 0));
}

int mcfo_simple_renorm(int prec, const void* h, int nc, void* out, int r_nc, int64_t numel) {
  if (BAD_NC(nc) || BAD_NC(r_nc)) return 1;
  DISPATCH(prec, b16_op_renorm(h, nc, out, r_nc, numel, 1), b32_op_renorm(h, nc, out, r_nc, numel, 1),
           b64_op_renorm(h, nc, out, r_nc, numel, 1));
}

#define UNARY(opid, expf_)                                                             \
  DISPATCH(prec, b16_op_unary(opid, x, nc, out, numel, expf_),                         \
           b32_op_unary(opid, x, nc, out, numel, expf_),                               \
           b64_op_unary(opid, x, nc, out, numel, expf_))

int mcfo_approx(int prec, const void* x, int nc, void* out, int64_t numel) {
  if (BAD_NC(nc)) return 1;
  UNARY(0, exp);
}
int mcfo_negate(int prec, const void* x, int nc, void* out, int64_t numel) {
  if (nc < 1) return 1;
  UNARY(1, exp);
}
int mcfo_square_mcn(int prec, const void* x, int nc, void* out, int64_t numel) {
  if (BAD_NC(nc)) return 1;
  UNARY(2, exp);
}
int mcfo_exp_mcn(int prec, const void* x, int nc, void* out, int64_t numel, int exp_mode) {
  if (BAD_NC(nc)) return 1;
  if (exp_mode == MCFO_EXP_CR) {
    UNARY(3, cr_exp_plain);
  }
  UNARY(3, exp);
}

#define WITHV(opid, expanded)                                                          \
  DISPATCH(prec, b16_op_with_v(opid, x, nc, v, vn, expanded, out, numel),              \
           b32_op_with_v(opid, x, nc, v, vn, expanded, out, numel),                    \
           b64_op_with_v(opid, x, nc, v, vn, expanded, out, numel))

int mcfo_grow_expn(int prec, const void* x, int nc, const void* v, int64_t vn, void* out,
                   int64_t numel) {
  if (BAD_NC(nc) || vn < 1) return 1;
  WITHV(0, 0);
}
int mcfo_scaling_n(int prec, const void* x, int nc, const void* v, int64_t vn, int expanded,
                   void* out, int64_t numel) {
  if (BAD_NC(nc) || vn < 1 || (expanded && BAD_NC(nc + 1))) return 1;
  WITHV(1, expanded);
}
int mcfo_div_n(int prec, const void* v, int64_t vn, const void* y, int nc, void* out,
               int64_t numel) {
  const void* x = y;
  if (BAD_NC(nc) || vn < 1) return 1;
  WITHV(2, 0);
}

#define BINARY(opid)                                                                   \
  if (BAD_NC(ncx) || BAD_NC(ncy)) return 1;                                            \
  DISPATCH(prec, b16_binary(opid, x, ncx, y, ncy, out, numel),                         \
           b32_binary(opid, x, ncx, y, ncy, out, numel),                               \
           b64_binary(opid, x, ncx, y, ncy, out, numel))

int mcfo_add_mcn(int prec, const void* x, int ncx, const void* y, int ncy, void* out,
                 int64_t numel) {
  BINARY(0);
}
int mcfo_div_mcn(int prec, const void* x, int ncx, const void* y, int ncy, void* out,
                 int64_t numel) {
  BINARY(1);
}
int mcfo_mul_mcn(int prec, const void* x, int ncx, const void* y, int ncy, void* out,
                 int64_t numel) {
  BINARY(2);
}
int mcfo_mul_mcn_slow(int prec, const void* x, int ncx, const void* y, int ncy, void* out,
                      int64_t numel) {
  BINARY(3);
}

int mcfo_bmm_mcn(int prec, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                 int64_t k, int64_t n, int w_batched, void* out, int strategy, int leaf_arity) {
  if (BAD_NC(nc + 1)) return 1; /* linalg needs nc+1 <= kMaxNc (linalg.hpp:147) */
  DISPATCH(prec,
           b16_op_bmm(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf_arity),
           b32_op_bmm(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf_arity),
           b64_op_bmm(x, nc, w, batch, m, k, n, w_batched, out, strategy, leaf_arity));
}

int mcfo_mm_mcn_sampled(int prec, const void* x, int nc, const void* w, int64_t m, int64_t k,
                        int64_t n, const int64_t* rows, const int64_t* cols, int64_t nsamp,
                        void* out) {
  (void)m;
  if (BAD_NC(nc + 1)) return 1;
  DISPATCH(prec, b16_op_mm_sampled(x, nc, w, k, n, rows, cols, nsamp, out),
           b32_op_mm_sampled(x, nc, w, k, n, rows, cols, nsamp, out),
           b64_op_mm_sampled(x, nc, w, k, n, rows, cols, nsamp, out));
}

int mcfo_dot_mcmc(int prec, const void* x, const void* y, int nc, int64_t batch, int64_t k,
                  void* out) {
  if (BAD_NC(nc + 1)) return 1;
  DISPATCH(prec, b16_op_dot_mcmc(x, y, nc, batch, k, out), b32_op_dot_mcmc(x, y, nc, batch, k, out),
           b64_op_dot_mcmc(x, y, nc, batch, k, out));
}

int mcfo_mm_mcmc_sampled(int prec, const void* x, const void* y, int nc, int64_t m, int64_t k,
                         int64_t n, const int64_t* rows, const int64_t* cols, int64_t nsamp,
                         void* out) {
  (void)m;
  if (BAD_NC(nc + 1)) return 1;
  DISPATCH(prec, b16_op_mm_mcmc_sampled(x, y, nc, k, n, rows, cols, nsamp, out),
           b32_op_mm_mcmc_sampled(x, y, nc, k, n, rows, cols, nsamp, out),
           b64_op_mm_mcmc_sampled(x, y, nc, k, n, rows, cols, nsamp, out));
}

int mcfo_matmul2d(int prec, const void* a, const void* b, int64_t m, int64_t k, int64_t n,
                  void* out) {
  DISPATCH(prec, b16_op_matmul2d(a, b, m, k, n, out), b32_op_matmul2d(a, b, m, k, n, out),
           b64_op_matmul2d(a, b, m, k, n, out));
}

/* ---- binary128 truth ---------------------------------------------------------- */

static __float128 q_load(int prec, const void* p, int64_t i) {
  switch (prec) {
    case MCFO_B16: return (__float128)b16_dec(((const uint16_t*)p)[i]);
    case MCFO_B32: return (__float128)((const float*)p)[i];
    default: return (__float128)((const double*)p)[i];
  }
}

static double q_relerr(__float128 got, __float128 truth) {
  const __float128 d = fabsq(got - truth);
  return truth == 0 ? (double)d : (double)(d / fabsq(truth));
}

int mcfo_mc_relu(int prec, const void* x, int nc, void* out, int64_t numel) {
  if (BAD_NC(nc)) return 1;
  DISPATCH(prec, b16_op_relu(x, nc, out, numel), b32_op_relu(x, nc, out, numel), b64_op_relu(x, nc, out, numel));
}

int mcfo_mc_softmax(int prec, const void* x, int nc, int64_t outer, int64_t n, int64_t inner, void* out,
                    int exp_mode) {
  if (BAD_NC(nc) || outer < 0 || n < 0 || inner < 0) return 1;
  if (exp_mode == MCFO_EXP_CR) {
    DISPATCH(prec, b16_op_softmax(x, nc, outer, n, inner, out, cr_exp_plain),
             b32_op_softmax(x, nc, outer, n, inner, out, cr_exp_plain),
             b64_op_softmax(x, nc, outer, n, inner, out, cr_exp_plain));
  }
  DISPATCH(prec, b16_op_softmax(x, nc, outer, n, inner, out, exp), b32_op_softmax(x, nc, outer, n, inner, out, exp),
           b64_op_softmax(x, nc, outer, n, inner, out, exp));
}

int mcfo_halfspace_arg(int prec, const void* table, int nc, int64_t n, int64_t dim, const int64_t* u,
                       const int64_t* v, int64_t npairs, double* out) {
  if (BAD_NC(nc) || dim < 1) return 1;
  for (int64_t p = 0; p < npairs; ++p) {
    if (u[p] < 0 || u[p] >= n || v[p] < 0 || v[p] >= n) return 1;
    switch (prec) {
      case MCFO_B16: out[p] = b16_op_halfspace_arg(table, nc, dim, u[p], v[p]); break;
      case MCFO_B32: out[p] = b32_op_halfspace_arg(table, nc, dim, u[p], v[p]); break;
      case MCFO_B64: out[p] = b64_op_halfspace_arg(table, nc, dim, u[p], v[p]); break;
      default: return 1;
    }
  }
  return 0;
}

int mcfo_relerr_mm_mct(int prec, const void* x, int nc, const void* w, int64_t m, int64_t k,
                       int64_t n, const int64_t* rows, const int64_t* cols, int64_t nsamp,
                       const void* cand, int cand_nc, double* relerr) {
  (void)m;
  for (int64_t s = 0; s < nsamp; ++s) {
    __float128 t = 0;
    for (int64_t kk = 0; kk < k; ++kk) {
      const __float128 wv = q_load(prec, w, kk * n + cols[s]);
      for (int c = 0; c < nc; ++c) t += q_load(prec, x, (rows[s] * k + kk) * nc + c) * wv;
    }
    __float128 g = 0;
    for (int c = cand_nc - 1; c >= 0; --c) g += q_load(prec, cand, s * cand_nc + c);
    relerr[s] = q_relerr(g, t);
  }
  return 0;
}

int mcfo_relerr_mm_mcmc(int prec, const void* x, const void* y, int nc, int64_t m, int64_t k,
                        int64_t n, const int64_t* rows, const int64_t* cols, int64_t nsamp,
                        const void* cand, int cand_nc, double* relerr) {
  (void)m;
  for (int64_t s = 0; s < nsamp; ++s) {
    __float128 t = 0;
    for (int64_t kk = 0; kk < k; ++kk) {
      __float128 a = 0, b = 0;
      /* each product of two components is exact in binary128 */
      for (int c = 0; c < nc; ++c) {
        a = q_load(prec, x, (rows[s] * k + kk) * nc + c);
        for (int d = 0; d < nc; ++d) {
          b = q_load(prec, y, (kk * n + cols[s]) * nc + d);
          t += a * b;
        }
      }
    }
    __float128 g = 0;
    for (int c = cand_nc - 1; c >= 0; --c) g += q_load(prec, cand, s * cand_nc + c);
    relerr[s] = q_relerr(g, t);
  }
  return 0;
}
