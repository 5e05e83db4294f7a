// hostapi.cu -- host-buffer entry points (the reference's calling model).
//
// The reference operates on host MCTensor<P> values.  mcf_h_* take host
// pointers, run the device kernels and return with the result in host
// memory.  Elementwise work is pipelined in chunks over three streams so the
// H2D copy of chunk c+1, the kernel on chunk c and the D2H copy of chunk c-1
// overlap (PCIe is full duplex).  Pinned caller buffers are copied directly;
// pageable ones go through the driver's staging.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "mcf_runtime.h"

namespace {

constexpr int kPipe = 3;

struct Op {
  const char* name;
  int kind;  // 0: x,v  1: x,y  2: x only  3: v,y (div_n)  4: approx  5: scaling expanded
};

const Op kOps[] = {{"grow_expn", 0}, {"scaling_n", 0},  {"div_n", 3},        {"add_mcn", 1},
                   {"div_mcn", 1},   {"mul_mcn", 1},    {"mul_mcn_slow", 1}, {"square_mcn", 2},
                   {"exp_mcn", 2},   {"negate", 2},     {"approx", 4},       {"scaling_n_expanded", 5},
                   {"mc_relu", 2}};

mcf_status run_chunk(const std::string& op, mcf_prec p, const void* x, int ncx, const void* y,
                     int ncy, const void* v, int64_t vn, void* out, int64_t n, cudaStream_t s) {
  if (op == "grow_expn") return mcf_grow_expn(p, x, ncx, v, vn, out, n, s);
  if (op == "scaling_n") return mcf_scaling_n(p, x, ncx, v, vn, 0, out, n, s);
  if (op == "scaling_n_expanded") return mcf_scaling_n(p, x, ncx, v, vn, 1, out, n, s);
  if (op == "div_n") return mcf_div_n(p, v, vn, y, ncy, out, n, s);
  if (op == "add_mcn") return mcf_add_mcn(p, x, ncx, y, ncy, out, n, s);
  if (op == "div_mcn") return mcf_div_mcn(p, x, ncx, y, ncy, out, n, s);
  if (op == "mul_mcn") return mcf_mul_mcn(p, x, ncx, y, ncy, out, n, s);
  if (op == "mul_mcn_slow") return mcf_mul_mcn_slow(p, x, ncx, y, ncy, out, n, s);
  if (op == "square_mcn") return mcf_square_mcn(p, x, ncx, out, n, s);
  if (op == "exp_mcn") return mcf_exp_mcn(p, x, ncx, out, n, s);
  if (op == "negate") return mcf_negate(p, x, ncx, out, n, s);
  if (op == "approx") return mcf_approx(p, x, ncx, out, n, s);
  if (op == "mc_relu") return mcf_mc_relu(p, x, ncx, out, n, s);
  return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mcf_h_elementwise: unknown operator " + op);
}

mcf_status cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return mcfr::fail(MCF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return MCF_OK;
}

#define TRY(expr)                 \
  do {                            \
    const mcf_status _s = (expr); \
    if (_s != MCF_OK) return _s;  \
  } while (0)

}  // namespace

extern "C" {

mcf_status mcf_h_elementwise(const char* op_c, mcf_prec p, const void* x, int ncx, const void* y,
                             int ncy, const void* v, int64_t vn, void* out, int64_t numel) {
  if (!op_c) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mcf_h_elementwise: null operator");
  const std::string op(op_c);
  const Op* spec = nullptr;
  for (const Op& o : kOps)
    if (op == o.name) spec = &o;
  if (!spec) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mcf_h_elementwise: unknown operator " + op);
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, op + ": unknown precision");
  if (numel < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, op + ": negative element count");
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    return mcfr::fail(MCF_ERR_NO_DEVICE, "mcf: no CUDA device");
  const bool has_x = spec->kind != 3, has_y = spec->kind == 1 || spec->kind == 3;
  const bool has_v = spec->kind == 0 || spec->kind == 3 || spec->kind == 5;
  if (has_x && mcfr::bad_nc(ncx)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (has_y && mcfr::bad_nc(ncy)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (has_v && (vn < 1 || (numel > 0 && numel % vn != 0)))
    return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, op + ": operand does not broadcast");
  if (numel == 0) return MCF_OK;

  const std::size_t es = mcfr::elem_bytes(p);
  const int onc = spec->kind == 4 ? 1
                  : spec->kind == 5 ? ncx + 1
                  : spec->kind == 1 ? std::max(ncx, ncy)
                  : spec->kind == 3 ? ncy
                                    : ncx;
  // chunk: whole periods of a broadcast operand, ~32 MiB of traffic per chunk
  const std::size_t per_elem = es * ((has_x ? ncx : 0) + (has_y ? ncy : 0) + onc + (has_v && vn == numel ? 1 : 0));
  int64_t chunk = std::max<int64_t>(1, (int64_t)((32u << 20) / per_elem));
  const bool v_full = has_v && vn == numel;
  if (has_v && !v_full && vn > 1) chunk = std::max<int64_t>(vn, chunk / vn * vn);
  chunk = std::min<int64_t>(chunk, numel);

  // device buffers per pipeline slot, plus one for a broadcast v
  const std::size_t bx = has_x ? chunk * ncx * es : 0, by = has_y ? chunk * ncy * es : 0;
  const std::size_t bv = has_v ? (v_full ? chunk * es : vn * es) : 0, bo = chunk * onc * es;
  auto align = [](std::size_t b) { return (b + 255) & ~std::size_t(255); };
  const std::size_t slot_bytes = align(bx) + align(by) + align(bv) + align(bo);
  cudaStream_t streams[kPipe];
  char* bufs[kPipe];
  for (int i = 0; i < kPipe; ++i) {
    bufs[i] = static_cast<char*>(mcfr::workspace(slot_bytes, i));
    if (!bufs[i]) return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot allocate device workspace");
    streams[i] = mcfr::side_stream(i);
  }
  // a broadcast v is uploaded once per slot buffer (small)
  if (has_v && !v_full) {
    for (int i = 0; i < kPipe; ++i)
      TRY(cuda_ok(cudaMemcpyAsync(bufs[i] + align(bx) + align(by), v, vn * es, cudaMemcpyHostToDevice, streams[i]),
                  "H2D v"));
  }
  const char* hx = static_cast<const char*>(x);
  const char* hy = static_cast<const char*>(y);
  const char* hv = static_cast<const char*>(v);
  char* ho = static_cast<char*>(out);
  int c = 0;
  for (int64_t e0 = 0; e0 < numel; e0 += chunk, ++c) {
    const int64_t n = std::min<int64_t>(chunk, numel - e0);
    const int slot = c % kPipe;
    cudaStream_t s = streams[slot];
    char* dx = bufs[slot];
    char* dy = dx + align(bx);
    char* dv = dy + align(by);
    char* dout = dv + align(bv);
    if (has_x) TRY(cuda_ok(cudaMemcpyAsync(dx, hx + e0 * ncx * es, n * ncx * es, cudaMemcpyHostToDevice, s), "H2D x"));
    if (has_y) TRY(cuda_ok(cudaMemcpyAsync(dy, hy + e0 * ncy * es, n * ncy * es, cudaMemcpyHostToDevice, s), "H2D y"));
    if (v_full) TRY(cuda_ok(cudaMemcpyAsync(dv, hv + e0 * es, n * es, cudaMemcpyHostToDevice, s), "H2D v"));
    TRY(run_chunk(op, p, dx, ncx, dy, ncy, dv, v_full ? n : vn, dout, n, s));
    TRY(cuda_ok(cudaMemcpyAsync(ho + e0 * onc * es, dout, n * onc * es, cudaMemcpyDeviceToHost, s), "D2H out"));
  }
  for (int i = 0; i < kPipe; ++i) TRY(cuda_ok(cudaStreamSynchronize(streams[i]), "sync"));
  return MCF_OK;
}

mcf_status mcf_h_bmm_mcn(mcf_prec p, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                         int64_t k, int64_t n, int w_batched, void* out, int strategy) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_mcn: unknown precision");
  if (mcfr::bad_nc(nc) || mcfr::bad_nc(nc + 1)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  const std::size_t es = mcfr::elem_bytes(p);
  const std::size_t bx = batch * m * k * nc * es, bw = (w_batched ? batch : 1) * k * n * es,
                    bo = batch * m * n * nc * es;
  auto align = [](std::size_t b) { return (b + 255) & ~std::size_t(255); };
  char* d = static_cast<char*>(mcfr::workspace(align(bx) + align(bw) + align(bo) + 256, 0));
  if (!d) return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot allocate device workspace");
  char *dx = d, *dw = d + align(bx), *dout = dw + align(bw);
  if ((strategy == MCF_FAST || strategy == MCF_FAST_FP64) && p == MCF_B32 && nc == 2 && batch == 1 &&
      m >= 1024 && k > 0 && mcfr::ensure_device_tables() == MCF_OK) {
    // the headline shape: row-chunked so the copies overlap the product
    const cudaStream_t comp[2] = {mcfr::side_stream(4), mcfr::side_stream(5)};
    auto pipe = strategy == MCF_FAST ? mcfr::ozaki_host : mcfr::mm_fast_mct_host;
    const mcf_status st = pipe(
        static_cast<const float*>(x), static_cast<const float*>(w), m, k, n, static_cast<float*>(out),
        reinterpret_cast<float*>(dx), reinterpret_cast<float*>(dw), reinterpret_cast<float*>(dout),
        mcfr::side_stream(3), comp, mcfr::side_stream(6));
    if (st != MCF_ERR_UNSUPPORTED) return st;
  }
  cudaStream_t s = mcfr::side_stream(0);
  if (bx) TRY(cuda_ok(cudaMemcpyAsync(dx, x, bx, cudaMemcpyHostToDevice, s), "H2D x"));
  if (bw) TRY(cuda_ok(cudaMemcpyAsync(dw, w, bw, cudaMemcpyHostToDevice, s), "H2D w"));
  TRY(mcf_bmm_mcn(p, dx, nc, dw, batch, m, k, n, w_batched, dout, strategy, 1, s));
  if (bo) TRY(cuda_ok(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, s), "D2H out"));
  return cuda_ok(cudaStreamSynchronize(s), "sync");
}

mcf_status mcf_h_mc_softmax(mcf_prec p, const void* x, int nc, int64_t outer, int64_t n, int64_t inner,
                            void* out) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_softmax: unknown precision");
  if (mcfr::bad_nc(nc)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  if (outer < 0 || n < 0 || inner < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_softmax: negative dimension");
  const std::size_t bytes = (std::size_t)outer * n * inner * nc * mcfr::elem_bytes(p);
  if (bytes == 0) return MCF_OK;
  char* d = static_cast<char*>(mcfr::workspace(2 * bytes + 512, 0));
  if (!d) return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot allocate device workspace");
  cudaStream_t s = mcfr::side_stream(0);
  char* dout = d + ((bytes + 255) & ~std::size_t(255));
  TRY(cuda_ok(cudaMemcpyAsync(d, x, bytes, cudaMemcpyHostToDevice, s), "H2D x"));
  TRY(mcf_mc_softmax(p, d, nc, outer, n, inner, dout, s));
  TRY(cuda_ok(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s), "D2H out"));
  return cuda_ok(cudaStreamSynchronize(s), "sync");
}

mcf_status mcf_h_mm_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t m, int64_t k,
                         int64_t n, void* out, int strategy) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mm_mcmc: unknown precision");
  if (mcfr::bad_nc(nc) || mcfr::bad_nc(nc + 1)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "MCTensor ops support 1 <= nc <= 8");
  const std::size_t es = mcfr::elem_bytes(p);
  const std::size_t bx = m * k * nc * es, by = k * n * nc * es, bo = m * n * nc * es;
  auto align = [](std::size_t b) { return (b + 255) & ~std::size_t(255); };
  char* d = static_cast<char*>(mcfr::workspace(align(bx) + align(by) + align(bo) + 256, 0));
  if (!d) return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot allocate device workspace");
  cudaStream_t s = mcfr::side_stream(0);
  char *dx = d, *dy = d + align(bx), *dout = dy + align(by);
  if (bx) TRY(cuda_ok(cudaMemcpyAsync(dx, x, bx, cudaMemcpyHostToDevice, s), "H2D x"));
  if (by) TRY(cuda_ok(cudaMemcpyAsync(dy, y, by, cudaMemcpyHostToDevice, s), "H2D y"));
  TRY(mcf_mm_mcmc(p, dx, dy, nc, m, k, n, dout, strategy, s));
  if (bo) TRY(cuda_ok(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, s), "D2H out"));
  return cuda_ok(cudaStreamSynchronize(s), "sync");
}


// ---- host-buffer forms of the remaining drop-in entry points -------------------
// (copy in, one device call on the library's stream, copy out; blocking)

namespace {
struct Staged {
  char* base = nullptr;
  std::size_t off = 0;
  char* take(std::size_t b) {
    char* p = base + off;
    off += (b + 255) & ~std::size_t(255);
    return p;
  }
};
mcf_status stage(std::size_t total, Staged& st) {
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    return mcfr::fail(MCF_ERR_NO_DEVICE, "mcf: no CUDA device");
  st.base = static_cast<char*>(mcfr::workspace(total + 4096, 0));
  if (!st.base) return mcfr::fail(MCF_ERR_CUDA, "mcf: cannot allocate device workspace");
  return MCF_OK;
}
}  // namespace

mcf_status mcf_h_renorm(int kind, mcf_prec p, const void* h, int nc, void* out, int r_nc, int64_t numel) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "renormalize: unknown precision");
  if (numel < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "renormalize: negative element count");
  const std::size_t es = mcfr::elem_bytes(p), bi = numel * nc * es, bo = numel * (r_nc > 0 ? r_nc : 0) * es;
  Staged st;
  TRY(stage(bi + bo + 512, st));
  cudaStream_t s = mcfr::side_stream(0);
  char *dh = st.take(bi), *dout = st.take(bo);
  if (bi) TRY(cuda_ok(cudaMemcpyAsync(dh, h, bi, cudaMemcpyHostToDevice, s), "H2D h"));
  TRY(kind == 0 ? mcf_renormalize(p, dh, nc, dout, r_nc, numel, s) : mcf_simple_renorm(p, dh, nc, dout, r_nc, numel, s));
  if (bo) TRY(cuda_ok(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, s), "D2H out"));
  return cuda_ok(cudaStreamSynchronize(s), "sync");
}

mcf_status mcf_h_eft(int kind, mcf_prec p, const void* a, const void* b, void* r, void* e, int64_t n) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "two_sum: unknown precision");
  if (n < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "two_sum: negative element count");
  const std::size_t bytes = n * mcfr::elem_bytes(p);
  Staged st;
  TRY(stage(4 * bytes + 1024, st));
  cudaStream_t s = mcfr::side_stream(0);
  char *da = st.take(bytes), *db = st.take(bytes), *dr = st.take(bytes), *de = st.take(bytes);
  if (bytes) {
    TRY(cuda_ok(cudaMemcpyAsync(da, a, bytes, cudaMemcpyHostToDevice, s), "H2D a"));
    TRY(cuda_ok(cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, s), "H2D b"));
  }
  TRY(kind == 0 ? mcf_two_sum(p, da, db, dr, de, n, s) : mcf_two_prod(p, da, db, dr, de, n, s));
  if (bytes) {
    TRY(cuda_ok(cudaMemcpyAsync(r, dr, bytes, cudaMemcpyDeviceToHost, s), "D2H"));
    TRY(cuda_ok(cudaMemcpyAsync(e, de, bytes, cudaMemcpyDeviceToHost, s), "D2H"));
  }
  return cuda_ok(cudaStreamSynchronize(s), "sync");
}

mcf_status mcf_h_mc_transpose2d(mcf_prec p, const void* x, int nc, int64_t m, int64_t n, void* out) {
  if (!mcfr::valid_prec(p)) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_transpose2d: unknown precision");
  if (m < 0 || n < 0) return mcfr::fail(MCF_ERR_INVALID_ARGUMENT, "mc_transpose2d: negative dimension");
  const std::size_t bytes = m * n * nc * mcfr::elem_bytes(p);
  Staged st;
  TRY(stage(2 * bytes + 512, st));
  cudaStream_t s = mcfr::side_stream(0);
  char *dx = st.take(bytes), *dout = st.take(bytes);
  if (bytes) TRY(cuda_ok(cudaMemcpyAsync(dx, x, bytes, cudaMemcpyHostToDevice, s), "H2D x"));
  TRY(mcf_mc_transpose2d(p, dx, nc, m, n, dout, s));
  if (bytes) TRY(cuda_ok(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s), "D2H out"));
  return cuda_ok(cudaStreamSynchronize(s), "sync");
}

}  // extern "C"
