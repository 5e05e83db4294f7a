/*
 * mcf_oracle.h -- CPU oracle for the MCF operator hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2207_08867_b200/) may include, link or call this.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs use it, and only as the checker.
 *
 * Two implementations export this interface:
 *   mcfo_*    oracle/mcf_oracle.c  -- plain-C restatement of the reference
 *             algorithms (each function cites the reference file:line it
 *             restates).  Built into oracle/libmcf_oracle.so.
 *   mcfref_*  oracle/ref_shim.cpp  -- the reference's own header-only C++
 *             (/root/reference/proj/include/mcfloat) compiled unmodified
 *             with the reference's FP flags, behind the same C signatures.
 *             Built into oracle/_ref/libmcf_ref.so (not in git history).
 *
 * Storage conventions are those of the device C-ABI (include/mcf_gpu.h):
 * MC tensors are (numel, nc) with the component index fastest; B16 values are
 * IEEE binary16 bit patterns (uint16), B32 floats, B64 doubles.
 */
#ifndef MCF_ORACLE_H
#define MCF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* precision tags: same values as mcf_prec in include/mcf_gpu.h */
enum { MCFO_B16 = 0, MCFO_B32 = 1, MCFO_B64 = 2 };
/* exp mode for exp_mcn: 0 = host libm exp (what the reference calls),
 * 1 = correctly rounded binary64 exp (what the GPU computes). */
enum { MCFO_EXP_LIBM = 0, MCFO_EXP_CR = 1 };
/* reduction strategies: linalg.hpp:23 */
enum { MCFO_SEQUENTIAL = 0, MCFO_PAIRWISE_TREE = 1 };

#define MCFO_DECL(pfx)                                                                   \
  int pfx##two_sum(int prec, const void* a, const void* b, void* s, void* e, int64_t n); \
  int pfx##two_prod(int prec, const void* a, const void* b, void* p, void* e, int64_t n, \
                    int use_fma);                                                        \
  int pfx##renormalize(int prec, const void* h, int nc, void* out, int r_nc,             \
                       int64_t numel);                                                   \
  int pfx##simple_renorm(int prec, const void* h, int nc, void* out, int r_nc,           \
                         int64_t numel);                                                 \
  int pfx##approx(int prec, const void* x, int nc, void* out, int64_t numel);            \
  int pfx##negate(int prec, const void* x, int nc, void* out, int64_t numel);            \
  int pfx##grow_expn(int prec, const void* x, int nc, const void* v, int64_t vn,         \
                     void* out, int64_t numel);                                          \
  int pfx##scaling_n(int prec, const void* x, int nc, const void* v, int64_t vn,         \
                     int expanded, void* out, int64_t numel);                            \
  int pfx##div_n(int prec, const void* v, int64_t vn, const void* y, int nc, void* out,  \
                 int64_t numel);                                                         \
  int pfx##add_mcn(int prec, const void* x, int ncx, const void* y, int ncy, void* out,  \
                   int64_t numel);                                                       \
  int pfx##div_mcn(int prec, const void* x, int ncx, const void* y, int ncy, void* out,  \
                   int64_t numel);                                                       \
  int pfx##mul_mcn(int prec, const void* x, int ncx, const void* y, int ncy, void* out,  \
                   int64_t numel);                                                       \
  int pfx##mul_mcn_slow(int prec, const void* x, int ncx, const void* y, int ncy,        \
                        void* out, int64_t numel);                                       \
  int pfx##square_mcn(int prec, const void* x, int nc, void* out, int64_t numel);        \
  int pfx##exp_mcn(int prec, const void* x, int nc, void* out, int64_t numel,            \
                   int exp_mode);                                                        \
  /* batched MC x Tensor product: out[b,i,j] = sum_k x[b,i,k] * w[b?,k,j]         */     \
  /* dot = (m=1,n=1), mv = (n=1), mm, bmm (w_batched=1), matmul 3/2 (w_batched=0) */     \
  int pfx##bmm_mcn(int prec, const void* x, int nc, const void* w, int64_t batch,        \
                   int64_t m, int64_t k, int64_t n, int w_batched, void* out,            \
                   int strategy, int leaf_arity);                                        \
  /* sampled outputs of the same product: rows[i], cols[i] (batch 1) */                  \
  int pfx##mm_mcn_sampled(int prec, const void* x, int nc, const void* w, int64_t m,     \
                          int64_t k, int64_t n, const int64_t* rows,                     \
                          const int64_t* cols, int64_t nsamp, void* out);                \
  /* MC x MC restatement "recipe B": per-output DotCore whose terms */      \
  /* are the mul_mcn_slow term set renormalized to nc+1.                        */      \
  int pfx##dot_mcmc(int prec, const void* x, const void* y, int nc, int64_t batch,       \
                    int64_t k, void* out);                                               \
  int pfx##mm_mcmc_sampled(int prec, const void* x, const void* y, int nc, int64_t m,    \
                           int64_t k, int64_t n, const int64_t* rows,                    \
                           const int64_t* cols, int64_t nsamp, void* out);               \
  /* plain working-precision matmul2d (ndarray.hpp:147-165) */                           \
  int pfx##matmul2d(int prec, const void* a, const void* b, int64_t m, int64_t k,        \
                    int64_t n, void* out);                                               \
  /* mc_relu_op forward (autodiff.hpp:340-350) */                                        \
  int pfx##mc_relu(int prec, const void* x, int nc, void* out, int64_t numel);           \
  /* mc_softmax (autodiff.hpp:383-413) over the middle index of (outer, n, inner) */     \
  int pfx##mc_softmax(int prec, const void* x, int nc, int64_t outer, int64_t n,         \
                      int64_t inner, void* out, int exp_mode);                           \
  /* halfspace_arg (hyperbolic.hpp:183-212) for pairs (u[p], v[p]) of an (n, dim) */     \
  /* MC table: the P value as a double per pair                                  */     \
  int pfx##halfspace_arg(int prec, const void* table, int nc, int64_t n, int64_t dim,    \
                         const int64_t* u, const int64_t* v, int64_t npairs, double* out);

MCFO_DECL(mcfo_)
MCFO_DECL(mcfref_)

/* ---- oracle-only helpers (mcf_oracle.c) ---------------------------------- */

/* binary64 exp: correctly rounded (quad evaluation + rounding-boundary check).
 * *ambiguous is set when the quad result could not decide the rounding. */
double mcfo_cr_exp(double x, int* ambiguous);
/* glibc exp, exported so tests can see which inputs differ from CR. */
double mcfo_libm_exp(double x);
/* round a binary64 to the nearest binary16 value (RN-even), as a double */
double mcfo_round_b16(double x);

/* Relative error |value(cand) - truth| / |truth| with the truth computed in
 * binary128 (exact products; 113-bit accumulation).  0 truth -> abs error. */
int mcfo_relerr_mm_mct(int prec, const void* x, int nc, const void* w, int64_t m,
                       int64_t k, int64_t n, const int64_t* rows, const int64_t* cols,
                       int64_t nsamp, const void* cand, int cand_nc, double* relerr);
int mcfo_relerr_mm_mcmc(int prec, const void* x, const void* y, int nc, int64_t m,
                        int64_t k, int64_t n, const int64_t* rows, const int64_t* cols,
                        int64_t nsamp, const void* cand, int cand_nc, double* relerr);

/* ---- reference-shim-only helpers (ref_shim.cpp) -------------------------- */

/* Times the reference's public operator `op` (a name such as "add_mcn") on
 * MCTensor<P> inputs prepared outside the timed region, split over `threads`
 * host threads on disjoint slices.  Returns seconds for `reps` repetitions;
 * writes the last result to out.  Negative return = error. */
double mcfref_time_elementwise(const char* op, int prec, const void* x, int nc,
                               const void* y, const void* v, int64_t numel,
                               int threads, int reps, void* out);
/* Times mm_mcn over `rows` full output rows (x rows [0,rows) of an m x k
 * operand) with the whole w; returns seconds for one pass. */
double mcfref_time_mm_rows(int prec, const void* x, int nc, const void* w, int64_t rows,
                           int64_t k, int64_t n, int threads, void* out);
/* Times the recipe-B MC x MC dot over `batch` dots of length k. */
double mcfref_time_dot_mcmc(int prec, const void* x, const void* y, int nc,
                            int64_t batch, int64_t k, int threads, void* out);
/* MC-MLP training with the reference's own MCSequential / MCLinear / ReLU /
 * cross_entropy_loss / Tape / MCSGD (binary32, momentum 0).  params holds,
 * per layer, W (dims[l+1] x dims[l] x nc) then b (dims[l+1] x nc). */
int mcfref_mlp_train(const int* dims, int nlayers, int nc, const float* params, const float* X,
                     const int* labels, int64_t n, int steps, double lr, float* losses,
                     float* params_out);

#ifdef __cplusplus
}
#endif
#endif /* MCF_ORACLE_H */
