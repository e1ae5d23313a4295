// Shared plumbing for the sm_100a RS kernels: status codes, the per-thread
// error message behind rs_last_error(), launch checks, double-double helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/rs_b200.h"

#include <atomic>
#include <mutex>
#include <string.h>
#include <vector>

namespace rsb {

extern thread_local char g_err[512];
extern std::atomic<int64_t> g_launches;

// Optional per-kernel CUDA-event timing (rs_prof_enable); off by default.
struct ProfRec {
  const char *name;
  cudaEvent_t a, b;
};
extern std::vector<ProfRec> g_prof;
extern std::vector<cudaEvent_t> g_prof_pool;  // recycled timing events
extern std::mutex g_prof_mu;
extern bool g_prof_on;

inline cudaEvent_t prof_event() {
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_pool.empty()) {
      cudaEvent_t e = g_prof_pool.back();
      g_prof_pool.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  cudaStream_t s;
  const char *name;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(cudaStream_t s_, const char *n_) : s(s_), name(n_) {
    if (!g_prof_on) return;
    a = prof_event();
    b = prof_event();
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(ProfRec{name, a, b});
  }
};

inline int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

inline int check_launch(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return RS_OK;
  if (e == cudaErrorMemoryAllocation)
    return fail(RS_ERR_CAPACITY, "%s: %s", what, cudaGetErrorString(e));
  return fail(RS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define RS_REQUIRE(cond, ...)                         \
  do {                                                \
    if (!(cond)) return ::rsb::fail(RS_ERR_DOMAIN, __VA_ARGS__); \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when the (function,
// device) has not been raised to `bytes` yet: the driver call costs
// microseconds on the launch-bound build path
inline cudaError_t smem_attr(const void *fn, int bytes) {
  static std::mutex mu;
  static std::vector<const void *> fns;
  static std::vector<int> devs, sizes;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t i = 0;
  for (; i < fns.size(); ++i)
    if (fns[i] == fn && devs[i] == dev) break;
  if (i < fns.size() && sizes[i] >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  if (i < fns.size()) {
    sizes[i] = bytes;
  } else {
    fns.push_back(fn);
    devs.push_back(dev);
    sizes.push_back(bytes);
  }
  return cudaSuccess;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// grid size for a grid-stride loop over `total` items with 256-thread blocks
inline unsigned grid_blocks(int64_t total, int threads = 256) {
  int64_t g = ceil_div(total, threads);
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return (unsigned)g;
}

// ---- double-double accumulation (Knuth TwoSum; no FMA contraction) -------
struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd dd_add_d(dd a, double b) {
  double s = __dadd_rn(a.hi, b);
  double bb = __dsub_rn(s, a.hi);
  double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  double lo = __dadd_rn(a.lo, err);
  double hi = __dadd_rn(s, lo);
  lo = __dsub_rn(lo, __dsub_rn(hi, s));
  return dd{hi, lo};
}

__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd r = dd_add_d(a, b.hi);
  return dd_add_d(r, b.lo);
}

}  // namespace rsb
