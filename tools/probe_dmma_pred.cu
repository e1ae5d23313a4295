// Probe: does a predicated-off DMMA.8x8x4 still occupy the FP64 tensor pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_dmma_pred tools/probe_dmma_pred.cu
// Prints cycles per 16-DMMA step per warp for masks with 16 / 12 / 8 / 0 live DMMAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <bool BRANCH>
__global__ void __launch_bounds__(256, 2) k(const unsigned *mask, int steps, double *out, long long *cyc, int one) {
  double acc[2][8][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1.0, b = 0.5;
  const long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const unsigned live = __reduce_or_sync(0xffffffffu, mask[s & 63]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (live & (1u << j)) {
        if (BRANCH) {   // a loop of unknown trip count (= 1) cannot be if-converted: real branch
#pragma unroll 1
          for (int r = 0; r < one; ++r) {
            dmma(acc[0][j], a0, b);
            dmma(acc[1][j], a1, b);
          }
        } else {        // ptxas predicates the pair: @P DMMA
          dmma(acc[0][j], a0, b);
          dmma(acc[1][j], a1, b);
        }
      }
    }
  }
  const long long t1 = clock64();
  double sum = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) sum += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned *m; double *out; long long *cyc;
  cudaMalloc(&m, 64 * 4); cudaMalloc(&out, 296 * 256 * 8); cudaMalloc(&cyc, 296 * 8);
  const unsigned masks[] = {0xFFu, 0x3Fu, 0x0Fu, 0x01u, 0x00u};
  const int steps = 200000;
  for (int br = 0; br < 2; ++br)
  for (unsigned mk : masks) {
    unsigned h[64];
    for (int i = 0; i < 64; ++i) h[i] = mk;
    cudaMemcpy(m, h, sizeof h, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (br) k<true><<<296, 256>>>(m, steps, out, cyc, 1);
      else k<false><<<296, 256>>>(m, steps, out, cyc, 1);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long c[296]; cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
      if (rep) printf("%s mask %02x: %.3f ms, %.1f cycles per step per CTA (16 warps/SM: x%d live DMMAs per warp-step)\n",
                      br ? "branch   " : "predicate", mk, ms, (double)c[0] / steps, 2 * __builtin_popcount(mk));
    }
  }
  return 0;
}
