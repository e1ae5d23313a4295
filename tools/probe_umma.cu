// Microbenchmark: back-to-back tcgen05.mma kind::i8 (SS) issue rate vs N and
// the number of distinct accumulators; operands stay in shared memory.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw32(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)16 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int N, int NACC, bool SW128>
__global__ void k(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tbase;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint64_t da = SW128 ? desc_sw128(su32(sm)) : desc_sw32(su32(sm));
    const uint64_t db = SW128 ? desc_sw128(su32(sm + 16384)) : desc_sw32(su32(sm + 16384));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int a = 0; a < 16; ++a) {
        const uint32_t acc = tm + (a % NACC) * N;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(acc),
                     "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}\n" ::"r"(su32(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}
template <int N, int NACC, bool SW128>
void run(const char *name) {
  long long *d, h[148];
  cudaMalloc(&d, sizeof(h));
  auto kern = k<N, NACC, SW128>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 200;
  kern<<<148, 128, 64 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  kern<<<148, 128, 64 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-28s N=%3d acc=%d: %.1f clk/UMMA  (%s)\n", name, N, NACC, avg / (iters * 16.0),
         cudaGetErrorString(e));
}
int main() {
  run<64, 1, false>("sw32 one acc");
  run<64, 7, false>("sw32 7 acc");
  run<128, 1, false>("sw32 one acc");
  run<256, 1, false>("sw32 one acc");
  run<64, 1, true>("sw128 one acc");
  run<64, 7, true>("sw128 7 acc");
  run<128, 1, true>("sw128 one acc");
  run<256, 1, true>("sw128 one acc");
  return 0;
}
