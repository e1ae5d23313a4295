// SM partitions for concurrent streams (green contexts).
//
// The RS step runs two chains at once: a throughput-bound one (short-range
// row builder + plane GEMM, thousands of CTAs) and a latency-bound one (Gram,
// eigen block, core: small dependent kernels).  Stream priorities alone do
// not keep SMs free for the latter -- the wide kernels fill every SM and the
// small kernels queue behind resident CTAs.  A green context confines the
// wide chain to a fixed SM subset; the remaining SMs stay available to the
// latency-bound chain (which, on an ordinary stream, may still use any SM).
// Runtime-API launches into the green stream work with the primary context
// current (probed on B200, driver 580).
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include "rs_common.cuh"

using namespace rsb;

namespace {
struct Partition {
  CUgreenCtx ctx = nullptr;
  CUstream stream = nullptr;
  int sms = 0;
};
std::mutex g_mu;
std::map<std::pair<int, int>, Partition> g_parts;  // (device, requested SMs)

int cu_fail(CUresult r, const char *what) {
  return fail(RS_ERR_CUDA, "%s: CUresult %d", what, (int)r);
}

// Driver entry points through the runtime (no link-time libcuda dependency,
// so the library still loads on machines without a driver).
struct Driver {
  decltype(&cuDeviceGet) DeviceGet = nullptr;
  decltype(&cuDeviceGetDevResource) DeviceGetDevResource = nullptr;
  decltype(&cuDevSmResourceSplitByCount) DevSmResourceSplitByCount = nullptr;
  decltype(&cuDevResourceGenerateDesc) DevResourceGenerateDesc = nullptr;
  decltype(&cuGreenCtxCreate) GreenCtxCreate = nullptr;
  decltype(&cuGreenCtxStreamCreate) GreenCtxStreamCreate = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char *name, F &fn) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver &driver() {
  static Driver d = [] {
    Driver x;
    x.ok = entry("cuDeviceGet", x.DeviceGet) &&
           entry("cuDeviceGetDevResource", x.DeviceGetDevResource) &&
           entry("cuDevSmResourceSplitByCount", x.DevSmResourceSplitByCount) &&
           entry("cuDevResourceGenerateDesc", x.DevResourceGenerateDesc) &&
           entry("cuGreenCtxCreate", x.GreenCtxCreate) &&
           entry("cuGreenCtxStreamCreate", x.GreenCtxStreamCreate);
    return x;
  }();
  return d;
}
}  // namespace

extern "C" {

/* A non-blocking stream whose kernels run on a fixed subset of >= `sms` SMs
 * of the current device (green context; created once per (device, sms) and
 * kept for the process).  *sms_out = the partition's SM count. */
int rs_partition_stream(int sms, int priority, void **stream_out, int *sms_out) {
  RS_REQUIRE(sms >= 1 && stream_out && sms_out, "rs_partition_stream: bad arguments");
  int dev_ord = 0;
  cudaGetDevice(&dev_ord);
  cudaFree(0);  // primary context initialised and current
  std::lock_guard<std::mutex> lock(g_mu);
  auto key = std::make_pair(dev_ord, sms);
  auto it = g_parts.find(key);
  if (it == g_parts.end()) {
    const Driver &D = driver();
    if (!D.ok) return fail(RS_ERR_UNSUPPORTED, "rs_partition_stream: green contexts unavailable");
    CUdevice dev;
    CUresult r = D.DeviceGet(&dev, dev_ord);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuDeviceGet");
    CUdevResource all, part, rest;
    if ((r = D.DeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM)) != CUDA_SUCCESS)
      return cu_fail(r, "cuDeviceGetDevResource");
    RS_REQUIRE((unsigned)sms <= all.sm.smCount, "rs_partition_stream: %d SMs > device %u", sms,
               all.sm.smCount);
    unsigned nb = 1;
    if ((r = D.DevSmResourceSplitByCount(&part, &nb, &all, &rest, 0, (unsigned)sms)) !=
        CUDA_SUCCESS)
      return cu_fail(r, "cuDevSmResourceSplitByCount");
    CUdevResourceDesc desc;
    if ((r = D.DevResourceGenerateDesc(&desc, &part, 1)) != CUDA_SUCCESS)
      return cu_fail(r, "cuDevResourceGenerateDesc");
    Partition p;
    if ((r = D.GreenCtxCreate(&p.ctx, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS)
      return cu_fail(r, "cuGreenCtxCreate");
    if ((r = D.GreenCtxStreamCreate(&p.stream, p.ctx, CU_STREAM_NON_BLOCKING, priority)) !=
        CUDA_SUCCESS)
      return cu_fail(r, "cuGreenCtxStreamCreate");
    p.sms = (int)part.sm.smCount;
    it = g_parts.emplace(key, p).first;
  }
  *stream_out = (void *)it->second.stream;
  *sms_out = it->second.sms;
  return RS_OK;
}

}  // extern "C"
