// Probe: can runtime-API kernels run in a green-context stream (SM partition)
// while the primary context stays current?  Reports the SMs each launch used.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k_smid(int *hits, int spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) atomicAdd(&hits[s], 1);
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *m; cuGetErrorString(r, &m); printf("%s -> %s\n", #x, m); return 1; } } while (0)

int main() {
  cudaFree(0);  // primary context current
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  CUdevResource part[1], rest;
  unsigned nb = 1;
  CK(cuDevSmResourceSplitByCount(part, &nb, &all, &rest, 0, 128));
  printf("split: groups=%u part=%u rest=%u\n", nb, part[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc desc;
  CK(cuDevResourceGenerateDesc(&desc, part, 1));
  CUgreenCtx g;
  CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream gs;
  CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
  int *hits;
  cudaMalloc(&hits, 256 * sizeof(int));
  cudaMemset(hits, 0, 256 * sizeof(int));
  cudaDeviceSynchronize();
  k_smid<<<1000, 128, 0, (cudaStream_t)gs>>>(hits, 20000);
  cudaError_t e = cudaGetLastError();
  printf("launch into green stream: %s\n", cudaGetErrorString(e));
  e = cudaStreamSynchronize((cudaStream_t)gs);
  printf("sync: %s\n", cudaGetErrorString(e));
  int h[256];
  cudaMemcpy(h, hits, sizeof(h), cudaMemcpyDeviceToHost);
  int used = 0, total = 0;
  for (int i = 0; i < 256; ++i) { if (h[i]) ++used; total += h[i]; }
  printf("green launch: %d SMs used, %d blocks\n", used, total);
  cudaMemset(hits, 0, 256 * sizeof(int));
  k_smid<<<1000, 128>>>(hits, 20000);
  cudaDeviceSynchronize();
  cudaMemcpy(h, hits, sizeof(h), cudaMemcpyDeviceToHost);
  used = 0; total = 0;
  for (int i = 0; i < 256; ++i) { if (h[i]) ++used; total += h[i]; }
  printf("default launch: %d SMs used, %d blocks\n", used, total);
  return 0;
}
