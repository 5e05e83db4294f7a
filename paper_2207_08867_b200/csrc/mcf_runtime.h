// mcf_runtime.h -- host-side runtime shared by the library's translation units:
// error reporting (thread-local, reference-worded messages), launch
// accounting, grid sizing and the device workspace used by the mcf_h_* entry
// points.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <functional>
#include <string>

#include "../../include/mcf_gpu.h"

namespace mcfr {

mcf_status fail(mcf_status code, const std::string& msg);
inline mcf_status ok() { return MCF_OK; }
void note_launch();
// CUDA error after a launch -> MCF_ERR_CUDA with the runtime's message
mcf_status check_launch(const char* what);

int sm_count();
// fn() once per (device, tag), thread-safe (per-device kernel attributes and
// __constant__ tables: both are per-device state).  Tags: see kOnce* below.
void per_device_once(int tag, const std::function<void()>& fn);
enum : int { kOnceEwSmem = 0, kOnceMmSmem = 1, kOnceFallbackSmem = 2, kOnceCrtTables = 3, kOnceTcGemm = 4 };
// Raise a kernel's dynamic shared-memory limit on the current device once.
// The attribute is per device, so the flag is a per-kernel bitmask of
// devices (atomic: concurrent host threads may both set it, which is
// harmless; none launches before its own device's attribute is set).
template <auto Kern>
mcf_status ensure_smem_attr(int bytes, const char* what) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return MCF_OK;
  if (cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return fail(MCF_ERR_CUDA, what);
  done.fetch_or(bit, std::memory_order_release);
  return MCF_OK;
}
// grid for a grid-stride kernel: enough CTAs to fill every SM `per_sm` deep,
// never more than needed to cover `work_items` with `threads` each.
inline int grid_for(int64_t work_items, int threads, int per_sm) {
  const int64_t need = (work_items + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
  const int64_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

inline bool bad_nc(int nc) { return nc < 1 || nc > 8; }
inline std::size_t elem_bytes(mcf_prec p) {
  return p == MCF_B16 ? 2 : (p == MCF_B32 ? 4 : 8);
}
bool valid_prec(int p);

// binary128-computed 2^(j/2048), j < 2048, as (hi, lo) pairs (4096 doubles)
void exp2_table(double* out);

// per-device init of constant tables used by the elementwise kernels (and the
// stack limit the literal fallback path needs)
mcf_status ensure_device_tables();
// raise the per-thread device stack to at least `bytes` (recursive tree plan)
mcf_status ensure_stack(std::size_t bytes);

// MCF_FAST contraction kernels (mm_fast.cu, stream_fast.cu); each returns
// MCF_ERR_UNSUPPORTED without a message when it has no instantiation for the
// call, and the C-ABI then runs the reference-order kernel instead.
mcf_status mm_fast_mct(mcf_prec p, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                       int64_t k, int64_t n, int w_batched, void* out, cudaStream_t s, bool tc = true);
mcf_status mv_fast_mct(mcf_prec p, const void* x, int nc, const void* w, int64_t batch, int64_t m,
                       int64_t k, int w_batched, void* out, cudaStream_t s);
mcf_status mm_fast_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t m, int64_t k,
                        int64_t n, void* out, cudaStream_t s, bool tc = true);
mcf_status dot_fast_mcmc(mcf_prec p, const void* x, const void* y, int nc, int64_t batch, int64_t k,
                         void* out, cudaStream_t s);
int mm_fast_ops_per_mad(int mcmc, mcf_prec p, int nc);
// INT8 tensor-core (Ozaki) path of MCF_FAST (mm_ozaki.cu)
bool ozaki_supported(int64_t m, int64_t k, int64_t n);
mcf_status mm_ozaki(const float* x, int nca, const float* w, int ncb, int64_t m, int64_t k, int64_t n, float* out,
                    cudaStream_t s);
int ozaki_digits();
// MC binary16 (nc <= 3) x MC binary16 through five-digit int8 products (config 4's variant)
mcf_status mm_b16_i8(const void* x, const void* y, int nc, int64_t m, int64_t k, int64_t n, void* out,
                     cudaStream_t s);
// binary32 GEMM through four-digit int8 products (plan FAST's MLP backward)
mcf_status gemm_f32_i8(int trans_a, int trans_b, const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                       int64_t ldc, int64_t m, int64_t n, int64_t k, const float* mask, cudaStream_t s);
mcf_status mm_ozaki_bias_act(const float* w, const float* a, int64_t m, int64_t k, int64_t n, const float* bias,
                             int relu, float* h, float* act, cudaStream_t s);
int ozaki_gemm_equivalents(int ncb, int64_t k);
int ozaki_crt_info(int64_t k, int ncb, int* n, int* pa, int* pb);
int ozaki_crt_table(int n, int* moduli, float* w, float* mh, float* cq, int* bits);
// MC(nc=2, binary32) x T for m <= 16 rows in one FP64-pipe kernel (mm_skinny.cu)
mcf_status mm_skinny_mct(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out, cudaStream_t s);
mcf_status ozaki_reserve(int64_t m, int64_t k, int64_t n, int ncb, cudaStream_t s);
mcf_status ozaki_phases(const float* x, const float* w, int64_t m, int64_t k, int64_t n, float* out, double* ms,
                        int64_t* fallback, cudaStream_t s);
mcf_status ozaki_host(const float* hx, const float* hw, int64_t m, int64_t k, int64_t n, float* hout, float* dx,
                      float* dw, float* dout, cudaStream_t cin, const cudaStream_t comp[2], cudaStream_t cout);
// hand-written tcgen05 int8 GEMM (tc_gemm.cu): int32 products or residues
mcf_status tc_gemm_s8(const int8_t* a, const int8_t* b, void* out, int64_t m, int64_t n, int64_t kp, int batch,
                      int64_t ldo, const int* moduli, cudaStream_t s, int64_t b_rows = -1);
// the diagonal GEMMs of a digit-plane scheme in one tcgen05 launch (int32 out)
mcf_status tc_gemm_s8_seg(const int8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int* out, int64_t m, int64_t n,
                          int64_t b_rows, int nseg, const int* ka, const int* kb, const int* kd, int64_t ldo,
                          cudaStream_t s);
// host-buffer MC(nc=2, binary32) x T, pipelined over row chunks (hostapi.cu)
mcf_status mm_fast_mct_host(const float* hx, const float* hw, int64_t m, int64_t k, int64_t n, float* hout,
                            float* dx, float* dw, float* dout, cudaStream_t cin, const cudaStream_t comp[2],
                            cudaStream_t cout);

// device workspace for the host-buffer entry points (grows, per device)
void* workspace(std::size_t bytes, int slot);
cudaStream_t side_stream(int slot);
// reusable fork / join event, per host thread and device (slot < 16)
cudaEvent_t tl_event(int slot);
void* pinned(std::size_t bytes, int slot);

}  // namespace mcfr
