/*
 * mcf_gpu.h -- C-ABI of the B200 MCF operator library (libmcf_b200.so).
 *
 * This is the drop-in boundary for the MCTensor operator layer of the
 * reference (/root/reference/proj/include/mcfloat).  The reference exposes a
 * header-only C++20 template API (namespace mcf) over host value types
 * MCTensor<P> / NdArray; each function below replaces one of those entry
 * points and is cited as  [replaces <file>:<line>].  include/mcf_gpu.hpp
 * re-exposes the reference's own signatures on top of this ABI.
 *
 * Conventions (all entry points):
 *  - MC tensors are (numel, nc) arrays with the component index fastest
 *    (mctensor.hpp:8-9); component storage is IEEE binary16 (uint16 bits),
 *    binary32 or binary64 according to `prec` (precision.hpp:84-162).  The
 *    reference stores the same values as exactly representable doubles.
 *  - Working-precision ("Tensor") operands are plain arrays of the same
 *    storage type.  `vn` is the operand's element count: 1 (scalar) or any
 *    count dividing numel for a trailing-suffix broadcast, read as
 *    v[e % vn] (mc_ops.hpp:14-15, 317-329, 391).
 *  - Pointers without the mcf_h_ prefix are DEVICE pointers; the call is
 *    asynchronous on `stream` (NULL = legacy default stream) and safe from
 *    several host threads on distinct streams.  The elementwise operators and
 *    the reference-order contractions allocate nothing.  The MCF_FAST
 *    contractions keep a workspace per (device, stream) -- residue planes, or
 *    widened binary64 operands -- that grows on first use or when a larger
 *    shape arrives (cudaMalloc; regrowing synchronizes that stream).  Call
 *    mcf_fast_mm_reserve first where a call must not allocate (stream
 *    capture, latency-critical loops).
 *    mcf_h_* entry points take HOST pointers, stage through the library's
 *    device workspace and return when the result is in host memory.
 *  - Results are bit-identical to the reference for every elementwise
 *    operator, every precision and 1 <= nc <= 8, including unordered or
 *    overlapping components, zeros and non-finite values.  The one
 *    documented difference: exp uses a correctly rounded binary64 exp where
 *    the reference calls the host libm ("Exp-MCN").
 *  - Contractions (dot/mv/mm) are within the reference's own error bound,
 *    not bitwise (the summation order is the GPU's); nc == 1 is bitwise the
 *    reference's plain left-to-right fl-MAC chain (linalg.hpp:47-53).
 *  - Return value: MCF_OK or an error code; mcf_last_error() returns the
 *    calling thread's last message, worded like the reference's exceptions
 *    (e.g. "MCTensor ops support 1 <= nc <= 8", mc_ops.hpp:35).
 */
#ifndef MCF_GPU_H
#define MCF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mcf_stream; /* == cudaStream_t */

typedef enum mcf_status {
  MCF_OK = 0,
  MCF_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  MCF_ERR_UNSUPPORTED = 2,      /* mcf::unsupported_operation (linalg.hpp:30-32) */
  MCF_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
  MCF_ERR_NO_DEVICE = 4,        /* library loaded without a usable B200 */
  MCF_ERR_DOMAIN = 5            /* std::domain_error in the reference (hyperbolic.hpp:222-223) */
} mcf_status;

typedef enum mcf_prec { MCF_B16 = 0, MCF_B32 = 1, MCF_B64 = 2 } mcf_prec; /* precision.hpp:209 */

typedef enum mcf_reduce { /* linalg.hpp:23 */
  MCF_SEQUENTIAL = 0,    /* reference order, bit-identical to the reference */
  MCF_PAIRWISE_TREE = 1, /* reference tree order, bit-identical */
  MCF_FAST = 2,          /* GPU order, within the reference's error bound: the
                            INT8 tensor-core splitting (mm_ozaki.cu) for binary32
                            nc=2 matrix products, else the compensated binary64
                            accumulation on the FP64 pipe */
  MCF_FAST_FP64 = 3      /* MCF_FAST restricted to the FP64-pipe kernels */
} mcf_reduce;

/* ---- library ------------------------------------------------------------- */
int mcf_abi_version(void);
const char* mcf_last_error(void);
/* kernels launched by this thread since the last reset (instrumentation) */
int64_t mcf_launch_count(void);
void mcf_reset_launch_count(void);
/* measured FMA instruction rates (lane-ops/s, whole GPU) of the FP64 and FP32
 * pipes on the current device: the roofline denominators of the contractions */
int mcf_probe_pipe_rates(double* fp64_ops_per_s, double* fp32_ops_per_s);

/* ---- error-free transforms, array forms  [replaces eft.hpp:89-111] -------- */
mcf_status mcf_two_sum(mcf_prec p, const void* a, const void* b, void* s, void* e, int64_t n,
                       mcf_stream stream);
mcf_status mcf_two_prod(mcf_prec p, const void* a, const void* b, void* prod, void* e,
                        int64_t n, mcf_stream stream);

/* ---- renormalization ------------------------------------------------------ */
/* [replaces mc_ops.hpp:339-348 renormalize] */
mcf_status mcf_renormalize(mcf_prec p, const void* h, int nc, void* out, int r_nc, int64_t numel,
                           mcf_stream stream);
/* [replaces mc_ops.hpp:350-359 simple_renorm] */
mcf_status mcf_simple_renorm(mcf_prec p, const void* h, int nc, void* out, int r_nc,
                             int64_t numel, mcf_stream stream);
/* [replaces mctensor.hpp:56-65 MCTensor::approx]  out: numel values */
mcf_status mcf_approx(mcf_prec p, const void* x, int nc, void* out, int64_t numel,
                      mcf_stream stream);
/* [replaces mc_ops.hpp:376-381 negate] */
mcf_status mcf_negate(mcf_prec p, const void* x, int nc, void* out, int64_t numel,
                      mcf_stream stream);

/* ---- elementwise MCF operators ------------------------------------------- */
/* [replaces mc_ops.hpp:384-394 grow_expn(MCTensor, NdArray)] */
mcf_status mcf_grow_expn(mcf_prec p, const void* x, int nc, const void* v, int64_t vn,
                         void* out, int64_t numel, mcf_stream stream);
/* [replaces mc_ops.hpp:398-410 scaling_n(MCTensor, NdArray, expanded)]
 * out has nc+1 components when expanded != 0 */
mcf_status mcf_scaling_n(mcf_prec p, const void* x, int nc, const void* v, int64_t vn,
                         int expanded, void* out, int64_t numel, mcf_stream stream);
/* [replaces mc_ops.hpp:494-507 div_n(NdArray, MCTensor)] */
mcf_status mcf_div_n(mcf_prec p, const void* v, int64_t vn, const void* y, int nc, void* out,
                     int64_t numel, mcf_stream stream);
/* binary ops pad mixed nc to max(ncx, ncy) [mc_ops.hpp:414-436]; out has that nc */
/* [replaces mc_ops.hpp:440-446 add_mcn] */
mcf_status mcf_add_mcn(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                       int64_t numel, mcf_stream stream);
/* [replaces mc_ops.hpp:448-454 div_mcn] */
mcf_status mcf_div_mcn(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                       int64_t numel, mcf_stream stream);
/* [replaces mc_ops.hpp:456-462 mul_mcn (fast: x / (1/y))] */
mcf_status mcf_mul_mcn(mcf_prec p, const void* x, int ncx, const void* y, int ncy, void* out,
                       int64_t numel, mcf_stream stream);
/* [replaces mc_ops.hpp:464-470 mul_mcn_slow] */
mcf_status mcf_mul_mcn_slow(mcf_prec p, const void* x, int ncx, const void* y, int ncy,
                            void* out, int64_t numel, mcf_stream stream);
/* [replaces mc_ops.hpp:472-480 square_mcn] */
mcf_status mcf_square_mcn(mcf_prec p, const void* x, int nc, void* out, int64_t numel,
                          mcf_stream stream);
/* [replaces mc_ops.hpp:482-490 exp_mcn] */
mcf_status mcf_exp_mcn(mcf_prec p, const void* x, int nc, void* out, int64_t numel,
                       mcf_stream stream);

/* ---- contractions, MC x Tensor  [replaces linalg.hpp:38-253] -------------- */
/* out[b,i,j,:] = sum_k x[b,i,k,:] * w[b',k,j], b' = b if w_batched else 0.
 * dot_mcn = (batch=1, m=1, n=1), mv_mcn = (n=1), mm_mcn = (batch=1),
 * bmm_mcn / mm4d_mcn = (w_batched=1), matmul_mcn 3/2 and 4/2 = (w_batched=0).
 * nc + 1 <= 8 (linalg.hpp:112,128,147,187).  strategy/leaf_arity mirror
 * ReductionPlan (linalg.hpp:25-28); nc == 1 with MCF_SEQUENTIAL is the plain
 * working-precision chain, bitwise.  For nc >= 2 the GPU carries an
 * extended accumulator in registers; results are within the reference's own
 * relative error (tests/test_gpu_linalg.py states the bound). */
mcf_status mcf_bmm_mcn(mcf_prec p, const void* x, int nc, const void* w, int64_t batch,
                       int64_t m, int64_t k, int64_t n, int w_batched, void* out,
                       int strategy, int leaf_arity, mcf_stream stream);
/* [replaces linalg.hpp:159-166 mm_mcn(MCTensor, MCTensor)]: always returns
 * MCF_ERR_UNSUPPORTED with the reference's message, like the reference. */
mcf_status mcf_mm_mcn_mcmc_refusal(void);
/* NEW capability (the reference refuses it): MC x MC products.
 * out[i,j,:] = sum_k x[i,k,:] * y[k,j,:].  strategy MCF_SEQUENTIAL runs SURVEY
 * 8c recipe B (bit-identical to the oracle's composition of reference
 * kernels); MCF_FAST the compensated binary64 accumulation. */
mcf_status mcf_mm_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t m, int64_t k,
                       int64_t n, void* out, int strategy, mcf_stream stream);
/* out[b,:] = sum_k x[b,k,:] * y[b,k,:]  (batched MC x MC dots) */
mcf_status mcf_dot_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t batch,
                        int64_t k, void* out, int strategy, mcf_stream stream);
/* MCF_FAST tensor-core scheme (mm_ozaki.cu): the binary32 nc=2 MC x T / MC x MC
 * contractions are exact integer products by Chinese remaindering over n
 * moduli (one int8 GEMM each).  mcf_fast_tc_digits: moduli of a K = 4096
 * MC x T product (kept for ABI compatibility). */
int mcf_fast_tc_digits(void);
/* int8 GEMMs (M x N x K each) of one tensor-core product of depth k whose
 * second operand has b_components components per element (1: Tensor, 2: MC). */
int mcf_fast_tc_gemm_equivalents(int b_components, int64_t k);
/* Host-only introspection (no device needed): the plan of a depth-k product
 * (moduli count, integer bits kept of A and of B); returns the moduli count
 * (0: k outside the scheme). */
int mcf_fast_tc_plan(int64_t k, int b_components, int* moduli, int* bits_a, int* bits_b);
/* The reconstruction constants of n moduli: moduli[n], w_slices[n * S] (the
 * symmetric CRT weights in S balanced 11-bit slices), m_slices[S] (the
 * modulus product M), q_scale = RN32(2^(L-11) / M), m_bits = L; returns S
 * (0 for n outside 1..22).  Null pointers are skipped. */
int mcf_fast_tc_crt_table(int n, int* moduli, float* w_slices, float* m_slices, float* q_scale, int* m_bits);
/* Grows `stream`'s tensor-core workspace (and uploads the CRT tables) for an
 * m x k x n binary32 nc=2 product with a b_components-component B, so that the
 * product itself allocates nothing.  MCF_ERR_UNSUPPORTED outside the scheme. */
mcf_status mcf_fast_mm_reserve(int64_t m, int64_t k, int64_t n, int b_components, mcf_stream stream);
/* Instrumentation: one MC(nc=2, binary32) x T product on the tensor-core
 * path with per-phase device times (phase_ms[4]: B residues, A residues, int8
 * GEMMs, reconstruction + fallback) and the number of outputs recomputed by
 * the fallback.  Synchronises the stream. */
mcf_status mcf_fast_mm_phases(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out,
                              double* phase_ms, int64_t* fallback_outputs, mcf_stream stream);
/* The hand-written tcgen05 int8 GEMM (tc_gemm.cu) behind the tensor-core
 * path, exposed for tests and probes: out_b = a_b . b_b^T for b < batch with
 * a: [batch][m][kp], b: [batch][n][kp] int8 (kp % 16 == 0), out: [batch][m][ldo]
 * int32 when moduli is null, else the symmetric int8 residues out_b mod
 * moduli[b] (moduli are those of mcf_fast_tc_crt_table, batch <= 32). */
mcf_status mcf_tc_gemm_s8(const void* a, const void* b, void* out, int64_t m, int64_t n, int64_t kp, int batch,
                          int64_t ldo, const int* moduli, mcf_stream stream);
/* mc_transpose2d (linalg.hpp:301-315): out (n, m, nc) = x (m, n, nc) transposed,
 * components kept in order (bit copy). */
mcf_status mcf_mc_transpose2d(mcf_prec p, const void* x, int nc, int64_t m, int64_t n, void* out,
                              mcf_stream stream);
/* FP64-pipe instructions per multiply-add of the MCF_FAST kernel for this
 * operand kind (mcmc = 0: MC x Tensor, 1: MC x MC); 0 = no fast kernel. */
int mcf_fast_ops_per_mad(int mcmc, mcf_prec p, int nc);

/* ---- MC-MLP step pieces (config 3; binary32 components) -------------------
 * Activations are feature-major (features x n).  Forward of one MCLinear is
 * mcf_bmm_mcn(W (out x in, MC), A_prev (in x n)) followed by
 * mcf_mlp_bias_act: h = approx(add_mcn(z, bias)), act = relu(h) or h
 * [replaces autodiff.hpp:255-276 mc_linear_op forward + :133-144 relu]. */
mcf_status mcf_mlp_bias_act(const float* z, int nc, const float* bias, int64_t out_dim, int64_t n,
                            int relu, float* h, float* act, mcf_stream stream);
/* One MCLinear forward + ReLU (mc_linear_op, autodiff.hpp:255-268; Tape::relu
 * :133-144): h = approx(add_mcn(W . A_prev, bias)), act = relu ? max(h, 0) : h
 * (act may be null).  Under MCF_FAST on the tensor-core shapes the bias /
 * approx / ReLU run in the product's recombination epilogue and z is unused;
 * otherwise z (out_dim x n x nc) receives the MC product. */
mcf_status mcf_mlp_linear_fwd(const float* w, int nc, const float* a_prev, int64_t out_dim, int64_t in_dim,
                              int64_t n, const float* bias, int relu, float* z, float* h, float* act, int strategy,
                              mcf_stream stream);
/* cross-entropy over logits (classes x n): per-sample terms, gradient
 * (softmax - onehot) / n_global, and (optionally) the left-to-right sum of the
 * terms [replaces autodiff.hpp:541-582]. */
mcf_status mcf_mlp_cross_entropy(const float* logits, const int* labels, int64_t classes, int64_t n,
                                 int64_t n_global, float* grad, float* terms, float* term_sum,
                                 mcf_stream stream);
/* the left-to-right binary32 sum of n loss terms (autodiff.hpp:572), alone:
 * lets a caller run it on a side stream, off the backward's critical path. */
mcf_status mcf_mlp_loss_sum(const float* terms, int64_t n, float* term_sum, mcf_stream stream);
/* C = op(A) op(B) in binary32 with the reduction index increasing, fl_mul then
 * fl_add (matmul2d, ndarray.hpp:147-165); relu_mask (optional, C's shape)
 * zeroes entries whose mask <= 0 (ReLU backward) [mc_linear_op backward,
 * autodiff.hpp:279-297]. */
mcf_status mcf_gemm_f32_ordered(int trans_a, int trans_b, const float* a, int64_t lda, const float* b,
                                int64_t ldb, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k,
                                const float* relu_mask, mcf_stream stream);
/* out[r] = sum_j g[r, j] in order (bias gradient, autodiff.hpp:287-292) */
mcf_status mcf_rowsum_f32_ordered(const float* g, int64_t rows, int64_t n, float* out,
                                  mcf_stream stream);
/* ---- MC activations (autodiff.hpp) ------------------- */
/* mc_relu_op forward (autodiff.hpp:340-350): the components of every element
 * whose approx() is <= 0 are zeroed; bit-identical. */
mcf_status mcf_mc_relu(mcf_prec p, const void* x, int nc, void* out, int64_t numel, mcf_stream stream);
/* mc_softmax (autodiff.hpp:383-413) over the middle index of an (outer, n,
 * inner) view of x (the reference's rank-1 / rank-2 tensor and axis: rows x
 * cols with axis -1 is (rows, cols, 1), axis 0 is (1, rows, cols)):
 * bit-identical, with the correctly rounded exp of exp_mcn. */
mcf_status mcf_mc_softmax(mcf_prec p, const void* x, int nc, int64_t outer, int64_t n, int64_t inner, void* out,
                          mcf_stream stream);

/* Hyperbolic half-space distances (hyperbolic.hpp:160-226):
 * for pairs (u[p], v[p]) of an (n, dim) MC embedding table, arg[p] =
 * halfspace_arg (the fused per-coordinate add / square / add fold, height
 * product, scale, div, grow, approx; bit-identical) and, if dist is not null,
 * dist[p] = arcosh_guarded(arg[p]) (device log/log1p: within four units in
 * the last place of P of the host libm result).  u, v, arg, dist: device arrays. */
mcf_status mcf_halfspace_arg(mcf_prec p, const void* table, int nc, int64_t n, int64_t dim, const int64_t* u,
                             const int64_t* v, int64_t npairs, double* arg, double* dist, mcf_stream stream);
/* halfspace_distance (hyperbolic.hpp:214-226), synchronous, with its domain
 * check: a non-positive height fails with MCF_ERR_DOMAIN; arg may be null. */
mcf_status mcf_halfspace_distance(mcf_prec p, const void* table, int nc, int64_t n, int64_t dim, const int64_t* u,
                                  const int64_t* v, int64_t npairs, double* arg, double* dist, mcf_stream stream);

/* host-buffer form of mcf_mc_softmax (mcf_h_elementwise takes "mc_relu") */
mcf_status mcf_h_mc_softmax(mcf_prec p, const void* x, int nc, int64_t outer, int64_t n, int64_t inner,
                            void* out);

/* Plan MCF_FAST versions of the two above (the reference-order plan needs
 * neither): FP32 GEMM in cuBLAS order (no TF32) with the same operands and
 * optional ReLU mask, and a tree-ordered row sum. */
mcf_status mcf_gemm_f32_fast(int trans_a, int trans_b, const float* a, int64_t lda, const float* b, int64_t ldb,
                             float* c, int64_t ldc, int64_t m, int64_t n, int64_t k, const float* relu_mask,
                             mcf_stream stream);
mcf_status mcf_rowsum_f32_fast(const float* g, int64_t rows, int64_t n, float* out, mcf_stream stream);
/* MC-SGD, momentum 0: w <- grow_expn(w, -lr * g) in place
 * [replaces optim.hpp:54-77 + mc_ops.hpp:509-513] */
mcf_status mcf_sgd_grow(float* w, int nc, const float* g, int64_t numel, float lr, mcf_stream stream);

/* ---- host-buffer entry points (blocking; the reference's calling model) --- */
/* op: "grow_expn" "scaling_n" "div_n" "add_mcn" "div_mcn" "mul_mcn"
 *     "mul_mcn_slow" "square_mcn" "exp_mcn" "negate" "approx".
 * x/y: MC operands (host), v: working-precision operand (host) or NULL.
 * Staged through pinned buffers in chunks so H2D, compute and D2H overlap. */
mcf_status mcf_h_elementwise(const char* op, mcf_prec p, const void* x, int ncx, const void* y,
                             int ncy, const void* v, int64_t vn, void* out, int64_t numel);
mcf_status mcf_h_bmm_mcn(mcf_prec p, const void* x, int nc, const void* w, int64_t batch,
                         int64_t m, int64_t k, int64_t n, int w_batched, void* out, int strategy);
mcf_status mcf_h_mm_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t m, int64_t k,
                         int64_t n, void* out, int strategy);
/* Host-buffer forms of renormalize / simple_renorm (kind 0 / 1,
 * mc_ops.hpp:338-359), the two_sum / two_prod array forms (kind 0 / 1,
 * eft.hpp:89-111) and mc_transpose2d (linalg.hpp:301-315); blocking. */
mcf_status mcf_h_renorm(int kind, mcf_prec p, const void* h, int nc, void* out, int r_nc, int64_t numel);
mcf_status mcf_h_eft(int kind, mcf_prec p, const void* a, const void* b, void* r, void* e, int64_t n);
mcf_status mcf_h_mc_transpose2d(mcf_prec p, const void* x, int nc, int64_t m, int64_t n, void* out);

/* ---- host input generation (mcf::Rng, rng.hpp:13-65) ----------------------- */
/* n draws of Rng(seed).uniform() (53-bit, [0,1)), bitwise the reference's */
void mcf_rng_uniform(uint64_t seed, int64_t n, double* out);
/* n draws of Rng(seed).normal() (Box-Muller with spare) */
void mcf_rng_normal(uint64_t seed, int64_t n, double* out);
/* n draws of Rng(seed).below(bound) */
void mcf_rng_below(uint64_t seed, uint64_t bound, int64_t n, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MCF_GPU_H */
