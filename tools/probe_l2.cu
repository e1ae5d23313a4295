// L2 read-bandwidth probe variants (diagnostic): 8- vs 16-byte loads, .cg
// (L1 bypass) vs .nc, a 32 MiB (L2-resident) buffer streamed by every CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_l2 tools/probe_l2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V, bool NC>
__global__ void __launch_bounds__(256) probe(const double *__restrict__ buf, long n, int iters,
                                             double *out) {
  double acc = 0.0;
  const long stride = (long)gridDim.x * blockDim.x * V;
  long start = ((long)blockIdx.x * blockDim.x + threadIdx.x) * V;
  for (int it = 0; it < iters; ++it) {
    for (long e = start; e < n; e += stride) {
      if (V == 1) {
        acc += NC ? __ldg(buf + e) : __ldcg(buf + e);
      } else {
        const double2 v = NC ? __ldg(reinterpret_cast<const double2 *>(buf + e))
                             : __ldcg(reinterpret_cast<const double2 *>(buf + e));
        acc += v.x + v.y;
      }
    }
    start = (start + 7919L * 32 * V) % stride;
  }
  if (acc == 1.2345e300) out[0] = acc;
}

template <int V, bool NC>
void run(const char *name, const double *buf, long n, double *out, int ctas_per_sm) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = 148 * ctas_per_sm;
  probe<V, NC><<<grid, 256>>>(buf, n, 5, out);
  cudaEventRecord(a);
  probe<V, NC><<<grid, 256>>>(buf, n, 100, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-24s ctas/SM %2d : %.2f TB/s\n", name, ctas_per_sm, n * 8.0 * 100 / (ms / 1e3) / 1e12);
}

int main() {
  const long n = (32L << 20) / 8;
  double *buf, *out;
  cudaMalloc(&buf, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, n * 8);
  for (int c : {4, 8}) {
    run<1, false>("8B ld.cg", buf, n, out, c);
    run<2, false>("16B ld.cg", buf, n, out, c);
    run<1, true>("8B ld.nc", buf, n, out, c);
    run<2, true>("16B ld.nc", buf, n, out, c);
  }
  // a 64 MiB buffer (both dies' L2 halves) and 16 MiB
  for (long mb : {16L, 64L, 96L}) {
    const long m = (mb << 20) / 8;
    double *b2;
    cudaMalloc(&b2, m * 8);
    cudaMemset(b2, 0, m * 8);
    char nm[64];
    snprintf(nm, sizeof nm, "8B ld.cg %ld MiB", mb);
    run<1, false>(nm, b2, m, out, 8);
    snprintf(nm, sizeof nm, "16B ld.cg %ld MiB", mb);
    run<2, false>(nm, b2, m, out, 8);
    cudaFree(b2);
  }
  return 0;
}
