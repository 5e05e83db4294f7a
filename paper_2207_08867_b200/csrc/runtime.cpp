// runtime.cpp -- host runtime of libmcf_b200.so: errors, launch accounting,
// device workspace and streams for the host-buffer entry points, the
// binary128 table for the device exp, and the reference's Rng mappings.
#include <cuda_runtime.h>
#include <quadmath.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "mcf_runtime.h"

namespace mcfr {

namespace {
thread_local std::string t_err;
thread_local int64_t t_launches = 0;
std::mutex g_mu;

constexpr int kMaxDev = 64;
constexpr int kSlots = 24;
struct DevState {
  void* ws[kSlots] = {};
  std::size_t ws_bytes[kSlots] = {};
  void* pin[kSlots] = {};
  std::size_t pin_bytes[kSlots] = {};
  cudaStream_t streams[kSlots] = {};
  bool tables = false;
};
DevState g_dev[kMaxDev];

int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDev ? 0 : d;
}
}  // namespace

mcf_status fail(mcf_status code, const std::string& msg) {
  t_err = msg;
  return code;
}

void note_launch() { ++t_launches; }

mcf_status check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MCF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return MCF_OK;
}

int sm_count() {
  static int cached[kMaxDev] = {};
  const int d = cur_dev();
  if (!cached[d]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0) n = 148;
    cached[d] = n;
  }
  return cached[d];
}

bool valid_prec(int p) { return p == MCF_B16 || p == MCF_B32 || p == MCF_B64; }

void exp2_table(double* out) {
  for (int j = 0; j < 2048; ++j) {
    const __float128 t = exp2q((__float128)j / 2048);
    const double hi = (double)t;
    out[2 * j] = hi;
    out[2 * j + 1] = (double)(t - (__float128)hi);
  }
}

void* workspace(std::size_t bytes, int slot) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevState& s = g_dev[cur_dev()];
  if (s.ws_bytes[slot] < bytes) {
    if (s.ws[slot]) cudaFree(s.ws[slot]);
    s.ws[slot] = nullptr;
    s.ws_bytes[slot] = 0;
    if (cudaMalloc(&s.ws[slot], bytes) != cudaSuccess) return nullptr;
    s.ws_bytes[slot] = bytes;
  }
  return s.ws[slot];
}

void* pinned(std::size_t bytes, int slot) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevState& s = g_dev[cur_dev()];
  if (s.pin_bytes[slot] < bytes) {
    if (s.pin[slot]) cudaFreeHost(s.pin[slot]);
    s.pin[slot] = nullptr;
    s.pin_bytes[slot] = 0;
    if (cudaMallocHost(&s.pin[slot], bytes) != cudaSuccess) return nullptr;
    s.pin_bytes[slot] = bytes;
  }
  return s.pin[slot];
}

cudaStream_t side_stream(int slot) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevState& s = g_dev[cur_dev()];
  if (!s.streams[slot]) cudaStreamCreateWithFlags(&s.streams[slot], cudaStreamNonBlocking);
  return s.streams[slot];
}

// fn() exactly once per (device, tag); concurrent callers on the same device
// wait until it has finished (std::call_once)
namespace {
constexpr int kOnceTags = 16;
std::once_flag g_once[kMaxDev][kOnceTags];
}  // namespace
void per_device_once(int tag, const std::function<void()>& fn) {
  std::call_once(g_once[cur_dev()][tag % kOnceTags], fn);
}

// thread-local, per-device reusable fork/join events (disable-timing): a wait
// captures the event's state when it is enqueued, so re-recording the same
// event later on the same host thread is safe
cudaEvent_t tl_event(int slot) {
  constexpr int kEv = 16;
  thread_local cudaEvent_t ev[kMaxDev][kEv] = {};
  cudaEvent_t& e = ev[cur_dev()][slot % kEv];
  if (!e) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

mcf_status ensure_stack(std::size_t bytes) {
  std::size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitStackSize);
  if (cur >= bytes) return MCF_OK;
  if (cudaDeviceSetLimit(cudaLimitStackSize, bytes) != cudaSuccess)
    return fail(MCF_ERR_CUDA, "mcf: cannot raise the device stack limit");
  return MCF_OK;
}

}  // namespace mcfr

extern "C" {

int mcf_abi_version(void) { return 1; }
const char* mcf_last_error(void) { return mcfr::t_err.c_str(); }
int64_t mcf_launch_count(void) { return mcfr::t_launches; }
void mcf_reset_launch_count(void) { mcfr::t_launches = 0; }

// rng.hpp:20-25 -- 53 random bits scaled by 2^-53
void mcf_rng_uniform(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(g() >> 11) * 0x1p-53;
}

// rng.hpp:30-43 -- Box-Muller with a cached spare
void mcf_rng_normal(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 g(seed);
  auto uni = [&] { return static_cast<double>(g() >> 11) * 0x1p-53; };
  bool have = false;
  double spare = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (have) {
      have = false;
      out[i] = spare;
      continue;
    }
    double u1 = uni();
    while (u1 == 0.0) u1 = uni();
    const double u2 = uni();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(th);
    have = true;
    out[i] = r * std::cos(th);
  }
}

// rng.hpp:48-54 -- rejection sampling
void mcf_rng_below(uint64_t seed, uint64_t bound, int64_t n, uint64_t* out) {
  std::mt19937_64 g(seed);
  const uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % bound);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t v = g();
    while (v >= limit) v = g();
    out[i] = v % bound;
  }
}

}  // extern "C"
