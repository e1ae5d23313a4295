// tcgen05 (5th-gen tensor core) int8 GEMM building block for sm_100a.
//
// C_s32[M x N] (+)= A_s8[M x K] * B_s8[N x K]^T, both operands K-major.
// One CTA owns a 128 x BN output tile whose int32 accumulator lives in TMEM;
// a single elected thread issues tcgen05.mma.kind::i8 (UMMA 128 x BN x 32),
// operands are staged global -> shared with 16-byte cp.async into the
// canonical no-swizzle K-major core-matrix layout (8 rows x 16 bytes per core
// matrix), double buffered; MMA completion is tracked with tcgen05.commit on
// an mbarrier per stage; the epilogue reads TMEM with tcgen05.ld.
//
// This is the exact-integer engine of the Ozaki-split FP64 plane GEMM
// (rs_tc8_gemm_f64): fp64 operands are cut into 7-bit signed slices per row,
// slice products are exact in int32, and the fp64 result is recombined with
// power-of-two scales -- FP64 accuracy at int8 tensor-core throughput.
#include <stdint.h>

#include <algorithm>

#include "rs_common.cuh"

namespace rsb {
namespace tc8 {

constexpr int BM = 128;
constexpr int BK = 128;  // K bytes per stage = 4 UMMA_K steps of 32
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp16(uint32_t dst, const void *src, bool valid) {
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}

// Shared-memory matrix descriptor, K-major, no swizzle (bits per the sm_100
// UMMA SmemDescriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), base offset 0, lbo mode 0, layout SWIZZLE_NONE = 0).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor: c_format S32 (2) at [4,6), a/b format INT8 (1) at
// [7,10) / [10,13), K-major A/B, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
      smem_u32(bar)));
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// Stage a (rows x BK) int8 tile (row-major, leading dim ld bytes) into the
// canonical layout: core (m_c, k_c) at ((k_c * rows/8) + m_c) * 128 bytes.
template <int ROWS>
__device__ __forceinline__ void load_tile(uint8_t *s, const int8_t *g, int64_t ld, int64_t r0,
                                          int64_t rmax, int64_t k0, int64_t kmax) {
  constexpr int PIECES = ROWS * (BK / 16);
  for (int e = threadIdx.x; e < PIECES; e += THREADS) {
    const int r = e / (BK / 16), kc = e % (BK / 16);
    const int64_t gr = r0 + r, gk = k0 + kc * 16;
    const bool ok = gr < rmax && gk < kmax;
    const uint32_t dst = smem_u32(s + ((kc * (ROWS / 8) + (r >> 3)) * 128 + (r & 7) * 16));
    cp16(dst, ok ? (const void *)(g + gr * ld + gk) : (const void *)g, ok);
  }
}

// One 128 x BN tile: acc(TMEM) = sum over K of A B^T; write int32 C (ldc).
template <int BN>
__global__ void __launch_bounds__(THREADS)
    k_gemm_s8(const int8_t *__restrict__ A, int64_t lda, const int8_t *__restrict__ B, int64_t ldb,
              int32_t *__restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K) {
  constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK;
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *sA[2] = {smem, smem + A_BYTES + B_BYTES};
  uint8_t *sB[2] = {smem + A_BYTES, smem + 2 * A_BYTES + B_BYTES};
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc(BM, BN);

  const int64_t chunks = (K + BK - 1) / BK;
  uint32_t phase[2] = {0, 0};
  if (chunks > 0) {
    load_tile<BM>(sA[0], A, lda, m0, M, 0, K);
    load_tile<BN>(sB[0], B, ldb, n0, N, 0, K);
    asm volatile("cp.async.commit_group;\n");
  }
  for (int64_t c = 0; c < chunks; ++c) {
    const int st = (int)(c & 1);
    // prefetch the next chunk into the other stage once its MMAs retired
    if (c + 1 < chunks) {
      if (c >= 1) {
        mbar_wait(&bar[st ^ 1], phase[st ^ 1]);
        phase[st ^ 1] ^= 1;
      }
      load_tile<BM>(sA[st ^ 1], A, lda, m0, M, (c + 1) * BK, K);
      load_tile<BN>(sB[st ^ 1], B, ldb, n0, N, (c + 1) * BK, K);
      asm volatile("cp.async.commit_group;\n");
      asm volatile("cp.async.wait_group 1;\n");
    } else {
      asm volatile("cp.async.wait_group 0;\n");
    }
    // make this thread's cp.async writes visible to the tensor-core (async) proxy
    asm volatile("fence.proxy.async.shared::cta;\n");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t a0 = smem_u32(sA[st]), b0 = smem_u32(sB[st]);
#pragma unroll
      for (int kk = 0; kk < BK / 32; ++kk) {
        // K step of 32 bytes = 2 core matrices along K (LBO apart)
        const uint64_t da = make_desc(a0 + kk * 2 * (BM / 8) * 128, (BM / 8) * 128, 128);
        const uint64_t db = make_desc(b0 + kk * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
        umma_i8(tmem, da, db, idesc, (c > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&bar[st]);
    }
    __syncwarp();
  }
  // wait for the last chunk's MMAs (and the one before, if still pending)
  if (chunks >= 2) {
    const int st = (int)((chunks - 2) & 1);
    // the chunk before last was already waited on inside the loop only if a
    // further chunk followed; wait on both stages' final phases
    mbar_wait(&bar[st], phase[st]);
  }
  if (chunks >= 1) {
    const int st = (int)((chunks - 1) & 1);
    mbar_wait(&bar[st], phase[st]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // epilogue: warp w owns TMEM lanes (rows) 32w .. 32w+31
  const int64_t row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int j = 0; j < BN; j += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (row < M) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (n0 + j + u < N) C[row * ldc + n0 + j + u] = (int32_t)v[u];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

}  // namespace tc8
}  // namespace rsb

using namespace rsb;

extern "C" {

/* C (M x N, int32, ldc) = A (M x K int8, lda) * B (N x K int8, ldb)^T on
 * tcgen05 (kind::i8).  K multiple of 16, lda/ldb multiples of 16, 16-byte
 * aligned bases. */
int rs_tc8_gemm_s8(const int8_t *A, int64_t lda, const int8_t *B, int64_t ldb, int32_t *C,
                   int64_t ldc, int64_t M, int64_t N, int64_t K, void *stream) {
  RS_REQUIRE(M >= 1 && N >= 1 && K >= 16 && K % 16 == 0 && lda % 16 == 0 && ldb % 16 == 0 &&
                 lda >= K && ldb >= K && ldc >= N,
             "rs_tc8_gemm_s8: bad shape");
  constexpr int BN = 64;
  const size_t smem = 2 * (size_t)(tc8::BM + BN) * tc8::BK + 1024;
  cudaError_t e = cudaFuncSetAttribute((const void *)tc8::k_gemm_s8<BN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "tc8 smem: %s", cudaGetErrorString(e));
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, tc8::BM));
  tc8::k_gemm_s8<BN><<<grid, tc8::THREADS, smem, as_stream(stream)>>>(A, lda, B, ldb, C, ldc, M, N,
                                                                      K);
  return check_launch("rs_tc8_gemm_s8");
}

}  // extern "C"
