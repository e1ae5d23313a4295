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
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

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

// K-major SWIZZLE_64B descriptor: 64-byte rows, 8-row atoms of 512 B (SBO),
// LBO unused (1), layout type 4.  Chunk c of row r sits at c ^ ((r >> 1) & 3).
__device__ __forceinline__ uint64_t make_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
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

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes));
}

// 1-D bulk copy global -> shared, completion counted on `bar` (tx bytes)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
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


// ============================================ Ozaki-split FP64 GEMM (int8)
// X (fp64) = 2^e_row * sum_p d_p 2^(-6-7p), d_p in [-64, 64] (int8): the row
// scale e is the exponent of the row's max |x|; digit p is the rounded
// remainder after p digits.  C = A B^T in fp64 then is
//   C_ij = 2^(ea_i + eb_j - 12) * sum_t 2^(-7t) * sum_{p+q=t} (D^A_p D^B_q^T)_ij
// where every slice product is exact in int32 (|d| <= 64, K * 8 * 4096 < 2^31
// for K < 65536) and accumulates in its own TMEM accumulator t.  Terms with
// p + q >= S are dropped: relative error ~ K 2^(-7S) of 2^(ea_i + eb_j).
constexpr int OZ_BN = 64;   // output columns per CTA (S accumulators x 64 <= 512 TMEM cols)
constexpr int OZ_BK = 64;   // int8 columns per stage

// e[r] = exponent with max_k |X[r, k]| < 2^e (0 for an all-zero row); warp per row
// Used columns: `cols`, or r3p + (*nb) * G when the bucket count lives on the
// device (the plane-assembly operands are allocated for the upper bound).
__device__ __forceinline__ int64_t oz_cols(int64_t cols, const int32_t *nb, int64_t r3p, int64_t G) {
  if (!nb) return cols;
  const int64_t u = r3p + (int64_t)(*nb) * G;
  return u < cols ? u : cols;
}

__global__ void k_oz_rowexp(const double *__restrict__ X, int64_t rows, int64_t ld, int64_t cols0,
                            const int32_t *__restrict__ nb, int64_t r3p, int64_t G,
                            int *__restrict__ e) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= rows) return;
  const int64_t cols = oz_cols(cols0, nb, r3p, G);
  const double *x = X + r * ld;
  double m = 0.0;
  for (int64_t c = lane; c < cols; c += 32) m = fmax(m, fabs(x[c]));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) {
    int ex = 0;
    if (m > 0.0) frexp(m, &ex);
    e[r] = ex;
  }
}

// out[p][r][k] (slice stride sstride, row stride ldk) for k < ldk (zeros past
// cols); thread per (row, 16 columns), 16-byte stores per slice
template <int S>
__global__ void k_oz_slice(const double *__restrict__ X, int64_t rows, int64_t ld, int64_t cols0,
                           const int32_t *__restrict__ nb, int64_t r3p, int64_t G,
                           const int *__restrict__ e, int8_t *__restrict__ out, int64_t ldk,
                           int64_t sstride) {
  const int64_t groups = ldk / 16;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * groups) return;
  const int64_t r = t / groups, c0 = (t - r * groups) * 16;
  const int64_t cols = oz_cols(cols0, nb, r3p, G);
  if (c0 >= (cols + 63) / 64 * 64) return;  // never inside a K range
  const int ex = e[r];
  uint32_t w[S][4];
#pragma unroll
  for (int p = 0; p < S; ++p) w[p][0] = w[p][1] = w[p][2] = w[p][3] = 0u;
  const double *x = X + r * ld;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t c = c0 + j;
    double a = c < cols ? ldexp(x[c], 6 - ex) : 0.0;  // |a| < 64
#pragma unroll
    for (int p = 0; p < S; ++p) {
      const double d = rint(a);
      a = (a - d) * 128.0;
      const uint32_t b = (uint32_t)((int32_t)d & 0xff);
      w[p][j >> 2] |= b << (8 * (j & 3));
    }
  }
#pragma unroll
  for (int p = 0; p < S; ++p)
    *reinterpret_cast<uint4 *>(out + p * sstride + r * ldk + c0) =
        make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// Tiled form for the bulk-copy GEMM: per slice, (tile of `TR` rows) x
// (32-column step) blocks of TR*32 bytes, each already in the SWIZZLE_32B
// K-major shared-memory image (row r at r*32, 16-byte chunk c at
// c ^ ((r >> 2) & 1)).  Thread per (row, 16 columns), rows fastest; rows past
// `rows` (tile padding) are zero.
template <int S>
__global__ void k_oz_slice_t(const double *__restrict__ X, int64_t rows, int64_t rows_pad,
                             int64_t ld, int64_t cols0, const int32_t *__restrict__ nb,
                             int64_t r3p, int64_t G, const int *__restrict__ e,
                             int8_t *__restrict__ out, int TR, int64_t ksteps, int64_t sstride,
                             int64_t tstride) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows_pad * ksteps * 2) return;
  const int64_t r = t % rows_pad, g = t / rows_pad;
  const int64_t cols = oz_cols(cols0, nb, r3p, G);
  if (g * 16 >= (cols + 31) / 32 * 32) return;  // never inside a K range
  const int ex = r < rows ? e[r] : 0;
  uint32_t w[S][4];
#pragma unroll
  for (int p = 0; p < S; ++p) w[p][0] = w[p][1] = w[p][2] = w[p][3] = 0u;
  if (r < rows) {
    const double *x = X + r * ld + g * 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      double a = g * 16 + j < cols ? ldexp(x[j], 6 - ex) : 0.0;  // |a| < 64
#pragma unroll
      for (int p = 0; p < S; ++p) {
        const double d = rint(a);
        a = (a - d) * 128.0;
        w[p][j >> 2] |= ((uint32_t)((int32_t)d & 0xff)) << (8 * (j & 3));
      }
    }
  }
  const int64_t rt = r / TR, rr = r - rt * TR, ks = g >> 1, c = g & 1;
  // tstride: bytes between consecutive (row tile, K step) blocks of one slice (TR * 32
  // when a slice is contiguous, S * TR * 32 when the S slices of a block are interleaved)
  const int64_t off = (rt * ksteps + ks) * tstride + rr * 32 + ((c ^ ((rr >> 2) & 1)) << 4);
#pragma unroll
  for (int p = 0; p < S; ++p)
    *reinterpret_cast<uint4 *>(out + p * sstride + off) =
        make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// Row exponent and slices in one pass (the A-resident kernel's operands): 16 lanes per
// row, lane g reads the row's columns [16 g, 16 g + 16) -- a row is one contiguous,
// coalesced read, seen once -- the half-warp reduces the row's max |x| to the exponent,
// every lane cuts its 16 values into S digits and writes 16 bytes per slice into the
// tiled SWIZZLE_32B image (lanes 2 m, 2 m + 1 fill one 32-byte row of K step m).
// K <= 256 (16 lanes x 16 columns); rows past `rows` (tile padding) are zero.
template <int S>
__global__ void __launch_bounds__(256)
    k_oz_rowslice(const double *__restrict__ X, int64_t rows, int64_t rows_pad, int64_t ld,
                  int64_t cols, int *__restrict__ e, int8_t *__restrict__ out, int TR,
                  int64_t ksteps, int64_t sstride, int64_t tstride) {
  const int g = threadIdx.x & 15;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 4;
  if (r >= rows_pad) return;   // (whole half-warps leave together)
  const int64_t kcols = (cols + 31) / 32 * 32;   // K steps in use
  double x[16];
  double m = 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t c = g * 16 + j;
    x[j] = (r < rows && c < cols) ? X[r * ld + c] : 0.0;
    m = fmax(m, fabs(x[j]));
  }
#pragma unroll
  for (int o = 8; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o, 16));
  int ex = 0;
  if (m > 0.0) frexp(m, &ex);
  if (g == 0 && r < rows) e[r] = ex;
  if (g * 16 >= kcols) return;
  uint32_t w[S][4];
#pragma unroll
  for (int p = 0; p < S; ++p) w[p][0] = w[p][1] = w[p][2] = w[p][3] = 0u;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    double a = ldexp(x[j], 6 - ex);  // |a| < 64
#pragma unroll
    for (int p = 0; p < S; ++p) {
      const double d = rint(a);
      a = (a - d) * 128.0;
      w[p][j >> 2] |= ((uint32_t)((int32_t)d & 0xff)) << (8 * (j & 3));
    }
  }
  const int64_t rt = r / TR, rr = r - rt * TR, ks = g >> 1, c = g & 1;
  const int64_t off = (rt * ksteps + ks) * tstride + rr * 32 + ((c ^ ((rr >> 2) & 1)) << 4);
#pragma unroll
  for (int p = 0; p < S; ++p)
    *reinterpret_cast<uint4 *>(out + p * sstride + off) =
        make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// fp64-column ranges (nr per column tile) -> int8-slice ranges rounded out to
// multiples of 32 (the UMMA K step) and merged when they touch; columns added
// by the rounding hold zero operands for this tile (outside its band).
__global__ void k_oz_ranges(const int64_t *__restrict__ in, int nr, int64_t ntiles, int64_t ldk,
                            int64_t *__restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  int64_t lo_prev = -1, hi_prev = -1;
  int k = 0;
  for (int r = 0; r < nr; ++r) {
    int64_t lo = in[(t * nr + r) * 2], hi = in[(t * nr + r) * 2 + 1];
    if (hi <= lo) continue;
    lo = lo / 32 * 32;
    hi = (hi + 31) / 32 * 32;
    if (hi > ldk) hi = ldk;
    if (hi_prev >= 0 && lo <= hi_prev) {
      if (hi > hi_prev) hi_prev = hi;
      continue;
    }
    if (hi_prev >= 0) {
      out[(t * nr + k) * 2] = lo_prev;
      out[(t * nr + k) * 2 + 1] = hi_prev;
      ++k;
    }
    lo_prev = lo;
    hi_prev = hi;
  }
  if (hi_prev >= 0) {
    out[(t * nr + k) * 2] = lo_prev;
    out[(t * nr + k) * 2 + 1] = hi_prev;
    ++k;
  }
  for (; k < nr; ++k) out[(t * nr + k) * 2] = out[(t * nr + k) * 2 + 1] = 0;
}

template <int S>
struct OzCfg {
  // one stage = all S slices of a 32-column K step of the A (128 rows) and
  // B (64 rows) tiles, SWIZZLE_32B K-major (32-byte rows, 8-row atoms)
  static constexpr int A_SLICE = BM * 32, B_SLICE = OZ_BN * 32;
  static constexpr int STAGE = S * (A_SLICE + B_SLICE);
  static constexpr int NST = (220 * 1024) / STAGE < 8 ? (220 * 1024) / STAGE : 8;
  static constexpr int SMEM = NST * STAGE + 1024;
};

// K-major SWIZZLE_32B descriptor: 32-byte rows, 8-row atoms of 256 B (SBO),
// LBO unused (1), layout type 6.  Chunk c of row r sits at c ^ ((r >> 2) & 1).
__device__ __forceinline__ uint64_t make_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}

// C[m0.., n0..] (=, or += with ACC) = Ozaki product over this column tile's
// K ranges.  One CTA per 128 x 64 tile; S accumulators in TMEM.  Thread 0
// drives an NST-deep ring: per 32-column step it posts 2S bulk copies of
// pre-tiled, pre-swizzled slice blocks (one mbarrier, tx-counted), and once
// a step's operands landed issues its S(S+1)/2 slice MMAs round-robin over
// the accumulators and commits them to the step's "empty" barrier.
template <int S, bool ACC>
__global__ void __launch_bounds__(THREADS)
    k_oz_gemm(const int8_t *__restrict__ SA, int64_t sa_stride, const int8_t *__restrict__ SB,
              int64_t sb_stride, int64_t ksteps, const int *__restrict__ ea,
              const int *__restrict__ eb, const int64_t *__restrict__ ranges, int nr,
              double *__restrict__ C, int64_t ldc, int64_t M, int64_t N) {
  using Cfg = OzCfg<S>;
  constexpr int NST = Cfg::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[NST];
  __shared__ __align__(8) uint64_t empty[NST];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n0 = (int64_t)blockIdx.x * OZ_BN, m0 = (int64_t)blockIdx.y * BM;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc(BM, OZ_BN);

  // K steps: 32-column pieces of this tile's ranges (multiples of 32)
  const int64_t lo0 = ranges[(blockIdx.x * nr) * 2], hi0 = ranges[(blockIdx.x * nr) * 2 + 1];
  const int64_t n_first = hi0 > lo0 ? (hi0 - lo0) / 32 : 0;
  int64_t nsteps = n_first;
  for (int r = 1; r < nr; ++r) {
    const int64_t lo = ranges[(blockIdx.x * nr + r) * 2], hi = ranges[(blockIdx.x * nr + r) * 2 + 1];
    if (hi > lo) nsteps += (hi - lo) / 32;
  }
  if (threadIdx.x == 0 && nsteps > 0) {
    auto step_ks = [&](int64_t c) -> int64_t {
      if (c < n_first) return lo0 / 32 + c;
      c -= n_first;
      for (int r = 1; r < nr; ++r) {
        const int64_t lo = ranges[(blockIdx.x * nr + r) * 2],
                      hi = ranges[(blockIdx.x * nr + r) * 2 + 1];
        if (hi <= lo) continue;
        const int64_t cnt = (hi - lo) / 32;
        if (c < cnt) return lo / 32 + c;
        c -= cnt;
      }
      return 0;
    };
    const uint32_t sbase = smem_u32(smem);
    const int8_t *gA = SA + blockIdx.y * ksteps * (int64_t)Cfg::A_SLICE;
    const int8_t *gB = SB + blockIdx.x * ksteps * (int64_t)Cfg::B_SLICE;
    auto load = [&](int st, int64_t ks) {
      const uint32_t base = sbase + st * Cfg::STAGE;
      mbar_expect_tx(&full[st], (uint32_t)Cfg::STAGE);
#pragma unroll
      for (int p = 0; p < S; ++p) {
        bulk_g2s(base + p * Cfg::A_SLICE, gA + p * sa_stride + ks * Cfg::A_SLICE, Cfg::A_SLICE,
                 &full[st]);
        bulk_g2s(base + S * Cfg::A_SLICE + p * Cfg::B_SLICE, gB + p * sb_stride + ks * Cfg::B_SLICE,
                 Cfg::B_SLICE, &full[st]);
      }
    };
    uint32_t fph = 0, eph = 0;  // parity bits per stage
    for (int i = 0; i < NST && i < nsteps; ++i) load(i, step_ks(i));
    const uint64_t desc0 = make_desc_sw32(sbase);
    for (int64_t c = 0; c < nsteps; ++c) {
      const int st = (int)(c % NST);
      mbar_wait(&full[st], (fph >> st) & 1u);
      fph ^= 1u << st;
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint64_t ds = desc0 + (uint64_t)((st * Cfg::STAGE) >> 4);
#pragma unroll
      for (int j = 0; j < S; ++j) {
#pragma unroll
        for (int t = j; t < S; ++t) {
          const uint64_t da = ds + (uint64_t)((j * Cfg::A_SLICE) >> 4);
          const uint64_t db = ds + (uint64_t)((S * Cfg::A_SLICE + (t - j) * Cfg::B_SLICE) >> 4);
          umma_i8(tmem + t * OZ_BN, da, db, idesc, (c > 0 || j > 0) ? 1u : 0u);
        }
      }
      umma_commit(&empty[st]);
      // refill the stage of step c-1 with step c-1+NST once its MMAs retired
      if (c >= 1 && c - 1 + NST < nsteps) {
        const int sp = (int)((c - 1) % NST);
        mbar_wait(&empty[sp], (eph >> sp) & 1u);
        eph ^= 1u << sp;
        load(sp, step_ks(c - 1 + NST));
      }
    }
    // remaining MMA commits: steps max(0, nsteps-NST) .. nsteps-1
    for (int64_t c = nsteps - NST > 0 ? nsteps - NST : 0; c < nsteps; ++c) {
      const int sp = (int)(c % NST);
      mbar_wait(&empty[sp], (eph >> sp) & 1u);
      eph ^= 1u << sp;
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // epilogue: warp w owns rows 32w..32w+31 (TMEM lanes); Horner over the
  // accumulators t = S-1 .. 0, then the power-of-two row/column scale
  const int64_t row = m0 + warp * 32 + lane;
  const bool any = nsteps > 0;
  const int er = (row < M) ? ea[row] : 0;
#pragma unroll 1
  for (int j = 0; j < OZ_BN; j += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = 0.0;
#pragma unroll
    for (int t = S - 1; t >= 0; --t) {
      uint32_t a[8];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(t * OZ_BN + j);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]),
                     "=r"(a[6]), "=r"(a[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = fma(v[u], 0.0078125, (double)(int32_t)a[u]);
    }
    if (row < M) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t col = n0 + j + u;
        if (col < N) {
          const double val = any ? ldexp(v[u], er + eb[col] - 12) : 0.0;
          double *dst = C + row * ldc + col;
          if (ACC) *dst += val; else *dst = val;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------------
// A-resident, warp-specialised Ozaki GEMM for dense K <= 160 (the Tucker part
// of the grid at large ranks: C (M x N) (+)= A (M x K) B (N x K)^T, M = planes
// x n rows, N = n, K = r3).  One persistent CTA per SM:
//   warp 0 (one thread)  bulk-copies the S slices of a 128-row block of A into
//                        shared memory once (all K steps: S x 5 x 4 KB), then
//                        streams the B slices of every 64-column tile through
//                        a 4-stage ring (S x 2 KB per 32-column K step);
//   warp 1 (one thread)  issues tcgen05.mma kind::i8 (128 x 64 x 32) into TMEM;
//   warps 2-9            drain TMEM, recombine in fp64 and update C.
// TMEM holds S accumulators of 64 columns (one per diagonal p + q = t).  To
// overlap the drain with the tensor pipe the diagonals are split in two groups
// -- {0..4} (15 slice products per K step) and {5, 6} (13) -- each computed in
// its own pass over the tile's K steps: while the MMAs of one group run, the
// epilogue warps drain the other (group 0 into per-thread fp64 partials, group
// 1 on top, then one coalesced-by-row update of C).  int32 partial sums are
// merged pairwise in integers (a_t 2^7 + a_{t+1} fits 31 bits) before the
// conversion, so a C entry costs 4 conversions and 3 FMAs.
template <int S>
struct OzRes {
  static constexpr int BN = 64, G1 = 5;
  static constexpr int A_SLICE = BM * 32, B_SLICE = BN * 32;
  static constexpr int MAXSTEPS = 5;                      // K <= 160
  static constexpr int A_BYTES = S * MAXSTEPS * A_SLICE;  // 140 KB at S = 7
  static constexpr int B_STAGE = S * B_SLICE;
  static constexpr int NSTB = MAXSTEPS;                   // one stage per K step of the tile
  static constexpr int EPW = 16;                          // epilogue warps: 4 per TMEM lane quarter
  static constexpr int SMEM = A_BYTES + NSTB * B_STAGE + 1024;
  static constexpr int THREADS_RES = (2 + EPW) * 32;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(taddr));
}

// 16 TMEM lanes x 16 columns: thread T holds rows T/4 (v[0], v[1], v[4], v[5]) and T/4 + 8
// (v[2], v[3], v[6], v[7]), columns 2 (T%4) + {0, 1} (v[0..3]) and 8 + 2 (T%4) + {0, 1}
// (v[4..7]) -- the accumulator-fragment layout, so 4 lanes cover 64 contiguous bytes of C
__device__ __forceinline__ void tmem_ld_16x256b_x2(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(taddr));
}

// int32 -> double without the conversion pipe: 2^52 + 2^31 + a is exact
__device__ __forceinline__ double s32_to_f64(int32_t a) {
  return __hiloint2double(0x43300000, a ^ (int32_t)0x80000000) - 4503601774854144.0;
}

__device__ __forceinline__ double pow2_f64(int e) {   // 2^e, e in the normal range
  return __hiloint2double((e + 1023) << 20, 0);
}

template <int S>
__global__ void __launch_bounds__(OzRes<S>::THREADS_RES, 1)
    k_oz_res(const int8_t *__restrict__ SA, const int8_t *__restrict__ SB, int64_t ksteps, int nsteps, const int *__restrict__ ea,
             const int *__restrict__ eb, double *__restrict__ C, int64_t ldc, int64_t M,
             int64_t N, int accumulate) {
  using Cfg = OzRes<S>;
  constexpr int NSTB = Cfg::NSTB, G1 = Cfg::G1, BN = Cfg::BN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[NSTB], empty[NSTB], a_full, a_empty, acc_full[2],
      acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTB; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&a_full, 1);
    mbar_init(&a_empty, 1);
    for (int g = 0; g < 2; ++g) {
      mbar_init(&acc_full[g], 1);
      mbar_init(&acc_empty[g], Cfg::EPW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int64_t nrb = (M + BM - 1) / BM, ntn = (N + BN - 1) / BN;
  const uint32_t a_s = smem_u32(smem), b_s = a_s + Cfg::A_BYTES;
  // every CTA walks the column tiles from its own start: 148 CTAs on the same B block and
  // the same C columns at once hot-spot a few L2 slices
  const int64_t ct0 = ((int64_t)blockIdx.x * 5) % ntn;
  long long dbg_c0 = 0;
  unsigned long long dbg_t0 = 0;
  if ((accumulate >> 4) & 128) {
    dbg_c0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t0));
  }
  const int dbg = accumulate >> 4;   // RSB200_OZ_DBG (diagnostics): 1 no C update, 2 no TMEM drain, 4 no MMA, 8 MMAs wait for nothing, 16 no L2 prefetch of C
  accumulate &= 1;

  if (warp == 0) {
    if (lane == 0) {   // ---------------------------------------------- loader
      uint32_t it = 0, ra = 0;
      for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ra) {
        mbar_wait(&a_empty, (ra & 1u) ^ 1u);
        // A: [K step][slice] blocks of the row tile lie back to back (interleaved slices)
        mbar_expect_tx(&a_full, (uint32_t)(S * nsteps * Cfg::A_SLICE));
        for (int ks = 0; ks < nsteps; ++ks)
          bulk_g2s(a_s + ks * S * Cfg::A_SLICE,
                   SA + (rb * ksteps + ks) * (int64_t)(S * Cfg::A_SLICE),
                   (uint32_t)(S * Cfg::A_SLICE), &a_full);
        for (int64_t ci = 0; ci < ntn; ++ci) {
          const int64_t ct = (ct0 + ci) % ntn;
          // B: the S slices of a (column tile, K step) block lie back to back: one copy
          // (both passes of the tile read them from shared memory: stage = K step)
          const int8_t *gB = SB + ct * ksteps * (int64_t)Cfg::B_STAGE;
          for (int ks = 0; ks < nsteps; ++ks) {
            mbar_wait(&empty[ks], (it & 1u) ^ 1u);
            mbar_expect_tx(&full[ks], (uint32_t)Cfg::B_STAGE);
            bulk_g2s(b_s + ks * Cfg::B_STAGE, gB + ks * (int64_t)Cfg::B_STAGE,
                     (uint32_t)Cfg::B_STAGE, &full[ks]);
          }
          ++it;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {   // -------------------------------------------- MMA issuer
    // The whole warp walks the (warp-uniform) loops and waits; one elected lane issues.
    // With a single divergent thread the descriptor arithmetic ran on the vector
    // datapath plus register -> uniform-register moves: ~110 cycles per MMA against the
    // 48 the 128 x 64 x 32 MMA itself takes.
    const uint32_t idesc = make_idesc(BM, BN);
    const uint64_t da0 = make_desc_sw32(a_s), db0 = make_desc_sw32(b_s);
    uint32_t leader;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(leader));
    uint32_t ra = 0, ut = 0;
    long long w_a = 0, w_e0 = 0, w_e1 = 0, w_f = 0;   // (128) cycles spent waiting, by barrier
    const bool prof = dbg & 128;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ra) {
      long long tw = prof ? clock64() : 0;
      mbar_wait(&a_full, ra & 1u);
      if (prof) w_a += clock64() - tw;
      for (int64_t ct = 0; ct < ntn; ++ct, ++ut) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          tw = prof ? clock64() : 0;
          if (!(dbg & 8)) mbar_wait(&acc_empty[g], (ut & 1u) ^ 1u);   // (8: free-running MMAs)
          if (prof) (g ? w_e1 : w_e0) += clock64() - tw;
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          for (int ks = 0; ks < nsteps; ++ks) {
            if (g == 0 && !(dbg & 8)) {   // pass 2 finds the K step in place
              tw = prof ? clock64() : 0;
              mbar_wait(&full[ks], ut & 1u);
              if (prof) w_f += clock64() - tw;
              asm volatile("tcgen05.fence::after_thread_sync;\n");
            }
            const uint64_t dak = da0 + (uint64_t)((ks * S * Cfg::A_SLICE) >> 4);
            const uint64_t dbk = db0 + (uint64_t)((ks * Cfg::B_STAGE) >> 4);
            const uint32_t acc0 = ks > 0 ? 1u : 0u;
            if (leader && !(dbg & 4)) {
#pragma unroll
              for (int t = (g ? G1 : 0); t < (g ? S : G1); ++t) {
#pragma unroll
                for (int p = 0; p <= t; ++p)
                  umma_i8(tmem + t * BN, dak + (uint64_t)((p * Cfg::A_SLICE) >> 4),
                          dbk + (uint64_t)(((t - p) * Cfg::B_SLICE) >> 4), idesc, p > 0 ? 1u : acc0);
              }
            }
            if (leader && g == 1) umma_commit(&empty[ks]);   // the next tile's K step may land
            __syncwarp();
          }
          if (leader) umma_commit(&acc_full[g]);
          __syncwarp();
        }
      }
      if (leader) umma_commit(&a_empty);
      __syncwarp();
    }
    // measured at C5 (2.70 M cycles per launch of a 64-plane slab): A 40 K, acc_empty[0]
    // 423 K, acc_empty[1] 20 K, B full 118 K -- the rest is MMA issue, ~55 cycles per MMA
    // from one lane, about what the 128 x 64 x 32 MMA takes to execute: the warp is issue
    // bound and every wait delays the tensor pipe.  An issue form predicated inside the
    // instruction block (uniform control flow) measured slower (2.96 M cycles); 576
    // threads cap the kernel at 96 registers (104 already fail to launch), which is what
    // keeps the old values of C from being requested earlier.
    if (prof && blockIdx.x == 0 && leader)
      printf("k_oz_res MMA warp waits (cycles): A %lld, acc_empty0 %lld, acc_empty1 %lld, B full %lld\n",
             w_a, w_e0, w_e1, w_f);
  } else {             // --------------------------------------------- epilogue
    // 16 warps: warp -> (TMEM lane quarter, 16-column group).  tcgen05.ld 16x256b hands
    // thread T rows T/4 (+8) and column pairs 2 (T%4) (+8) of a 16 x 16 block, so the
    // update of C runs as 16-byte accesses, 8 rows x 64 contiguous bytes per instruction,
    // straight from registers.
    const int quarter = warp & 3, cg = (warp - 2) >> 2;
    const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(cg * 16);
    const int r4 = lane >> 2, c2 = 2 * (lane & 3);
    const bool vec = !(ldc & 1);
    uint32_t ut = 0;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
      const int64_t rbase = rb * BM + quarter * 32 + r4;   // rows rbase + {0, 8, 16, 24}
      int er[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) er[i] = rbase + 8 * i < M ? ea[rbase + 8 * i] : 0;
      for (int64_t ci = 0; ci < ntn; ++ci, ++ut) {
        const int64_t ct = (ct0 + ci) % ntn;
        const int64_t n0 = ct * BN + cg * 16 + c2;          // columns n0 + {0, 1, 8, 9}
        int ecol[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t col = n0 + (j & 1) + 8 * (j >> 1);
          ecol[j] = col < N ? eb[col] : 0;
        }
        if (accumulate && !(dbg & (1 | 32 | 16))) {   // old values of the block into L2 (no registers)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (rbase + 8 * i < M) {
              const double *src = C + (rbase + 8 * i) * ldc + n0;
              if (n0 < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
              if (n0 + 8 < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 8));
            }
        }
        // v[h][k]: k = register index of the 16x256b.x2 load of lanes 16 h .. 16 h + 15:
        // rows (2 h + ((k >> 1) & 1)), column j = (k & 1) + 2 (k >> 2)
        double v[2][8];
        mbar_wait(&acc_full[0], ut & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (dbg & 2) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int k = 0; k < 8; ++k) v[h][k] = 0.0;
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t th = tq + ((uint32_t)(16 * h) << 16);
            uint32_t x[8], y[8];
            tmem_ld_16x256b_x2(th + 0 * BN, x);
            tmem_ld_16x256b_x2(th + 1 * BN, y);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int k = 0; k < 8; ++k)
              v[h][k] = s32_to_f64((int32_t)x[k] * 128 + (int32_t)y[k]) * 0.0078125;
            tmem_ld_16x256b_x2(th + 2 * BN, x);
            tmem_ld_16x256b_x2(th + 3 * BN, y);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int k = 0; k < 8; ++k)
              v[h][k] = fma(s32_to_f64((int32_t)x[k] * 128 + (int32_t)y[k]), 0x1p-21, v[h][k]);
            tmem_ld_16x256b_x2(th + 4 * BN, x);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int k = 0; k < 8; ++k) v[h][k] = fma(s32_to_f64((int32_t)x[k]), 0x1p-28, v[h][k]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[0]);
        mbar_wait(&acc_full[1], ut & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (!(dbg & 2)) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t th = tq + ((uint32_t)(16 * h) << 16);
            uint32_t x[8], y[8];
            tmem_ld_16x256b_x2(th + 5 * BN, x);
            if (S > 6) tmem_ld_16x256b_x2(th + 6 * BN, y);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int k = 0; k < 8; ++k)
              v[h][k] = fma(s32_to_f64((int32_t)x[k] * 128 + (S > 6 ? (int32_t)y[k] : 0)), 0x1p-42,
                            v[h][k]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[1]);
        // C[row, col] (+)= v 2^(ea[row] + eb[col] - 12), v = sum_t acc_t 2^(-7 t); two rows
        // (one 16-lane half) at a time: 4 x 16 bytes of old values in flight per lane
        if (!(dbg & 1)) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double o[2][4];
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int64_t grow = rbase + 8 * (2 * h + ii);
#pragma unroll
              for (int jp = 0; jp < 2; ++jp) {
                const int64_t col = n0 + 8 * jp;
                o[ii][2 * jp] = o[ii][2 * jp + 1] = 0.0;
                if (accumulate && !(dbg & 32) && grow < M) {   // (32: store only)
                  const double *src = C + grow * ldc + col;
                  if (vec && col + 1 < N) {
                    const double2 t2 = __ldcs(reinterpret_cast<const double2 *>(src));
                    o[ii][2 * jp] = t2.x;
                    o[ii][2 * jp + 1] = t2.y;
                  } else {
                    if (col < N) o[ii][2 * jp] = __ldcs(src);
                    if (col + 1 < N) o[ii][2 * jp + 1] = __ldcs(src + 1);
                  }
                }
              }
            }
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int i = 2 * h + ii;
              const int64_t grow = rbase + 8 * i;
              if (grow >= M) continue;
#pragma unroll
              for (int jp = 0; jp < 2; ++jp) {
                const int64_t col = n0 + 8 * jp;
                double r[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  // (exponents beyond the normal range are clamped: no physical operand gets there)
                  const int x = min(max(er[i] + ecol[2 * jp + u] - 12, -1022), 1023);
                  r[u] = fma(v[h][u + 2 * ii + 4 * jp], pow2_f64(x), o[ii][2 * jp + u]);
                }
                double *dst = C + grow * ldc + col;
                if (dbg & 64) {   // (64: no stores (the values are still formed))
                  if (r[0] + r[1] == 1.2345e-300) dst[0] = r[1];
                } else if (vec && col + 1 < N) {
                  __stcs(reinterpret_cast<double2 *>(dst), make_double2(r[0], r[1]));
                } else {
                  if (col < N) __stcs(dst, r[0]);
                  if (col + 1 < N) __stcs(dst + 1, r[1]);
                }
              }
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if ((dbg & 128) && blockIdx.x == 0 && threadIdx.x == 0) {   // effective SM clock of this CTA
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    const long long c1 = clock64();
    printf("k_oz_res: %lld cycles in %llu ns = %.0f MHz\n", c1 - dbg_c0, t1 - dbg_t0,
           1e3 * (double)(c1 - dbg_c0) / (double)(t1 - dbg_t0));
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
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
  cudaError_t e = smem_attr((const void *)tc8::k_gemm_s8<BN>, (int)smem);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "tc8 smem: %s", cudaGetErrorString(e));
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, tc8::BM));
  tc8::k_gemm_s8<BN><<<grid, tc8::THREADS, smem, as_stream(stream)>>>(A, lda, B, ldb, C, ldc, M, N,
                                                                      K);
  return check_launch("rs_tc8_gemm_s8");
}


/* Ozaki-split FP64 GEMM workspace for C (M x N) = A (M x K) B (N x K)^T. */
int64_t rs_oz_workspace_bytes(int64_t M, int64_t N, int64_t K, int slices) {
  const int64_t ldk = round_up(std::max<int64_t>(K, 1), 64);
  return round_up(slices * (round_up(M, 128) + round_up(N, 64)) * ldk, 256) +
         round_up((M + N) * 4, 256) +
         round_up(ceil_div(N, tc8::OZ_BN) * 2 * (4 * 2 * 8), 256);  // ranges in + out
}

/* C (=, or += with accumulate) = A B^T in FP64 via `slices` int8 slices on
 * tcgen05 (slices in {6, 7, 8}).  ranges (optional, NULL = [0, K)): nr fp64
 * column ranges per 64-column tile of C (K columns outside them must hold
 * zero B entries for that tile). */
int rs_oz_gemm_cols(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, const int64_t *ranges, int nr,
                    int slices, int accumulate, void *work, int64_t work_bytes,
                    const int32_t *nb, int64_t r3p, int64_t G, void *stream, int phase);

int rs_oz_gemm(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
               int64_t M, int64_t N, int64_t K, const int64_t *ranges, int nr, int slices,
               int accumulate, void *work, int64_t work_bytes, void *stream) {
  return rs_oz_gemm_cols(A, lda, B, ldb, C, ldc, M, N, K, ranges, nr, slices, accumulate, work,
                         work_bytes, nullptr, 0, 0, stream, 3);
}

/* as rs_oz_gemm; with nb != NULL only the first r3p + (*nb) * G columns of A
 * and B are live (device-side count; the rest is never read).  phase: 1 = row
 * exponents and slices only (the operands' preparation), 2 = the GEMM on slices
 * prepared by an earlier call with the same arguments, 3 = both. */
int rs_oz_gemm_cols(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, const int64_t *ranges, int nr,
                    int slices, int accumulate, void *work, int64_t work_bytes,
                    const int32_t *nb, int64_t r3p, int64_t G, void *stream, int phase) {
  RS_REQUIRE(M >= 1 && N >= 1 && K >= 1 && lda >= K && ldb >= K && ldc >= N,
             "rs_oz_gemm: bad shape");
  RS_REQUIRE(slices >= 6 && slices <= 8, "rs_oz_gemm: slices must be 6..8");
  RS_REQUIRE(nr >= 1 && nr <= 4, "rs_oz_gemm: nr must be 1..4");
  if (work_bytes < rs_oz_workspace_bytes(M, N, K, slices))
    return fail(RS_ERR_CAPACITY, "rs_oz_gemm: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t ldk = round_up(K, 64), ksteps = ldk / 32;
  const int64_t Mp = round_up(M, 128), Np = round_up(N, 64);
  char *w = (char *)work;
  int8_t *SA = (int8_t *)w;
  int8_t *SB = SA + slices * Mp * ldk;
  int *ea = (int *)(w + round_up(slices * (Mp + Np) * ldk, 256));
  int *eb = ea + M;
  int64_t *rg = (int64_t *)((char *)ea + round_up((M + N) * 4, 256));
  int64_t *rin = rg + ceil_div(N, tc8::OZ_BN) * 4 * 2;  // 4 ranges x 2 per tile each
  const int64_t ntn = ceil_div(N, tc8::OZ_BN);
  int st;
  // dense K <= 160 (the Tucker part): the A-resident warp-specialised kernel
  // (RSB200_OZ_RES=0: the per-tile kernel below)
  static const bool res_on = [] {
    const char *e = getenv("RSB200_OZ_RES");
    return !(e && e[0] == '0');
  }();
  const bool res = res_on && !ranges && !nb && slices <= 7 &&
                   ceil_div(K, 32) <= tc8::OzRes<7>::MAXSTEPS;
  if ((phase & 1) && !res) {
    tc8::k_oz_rowexp<<<(unsigned)ceil_div(M * 32, 256), 256, 0, s>>>(A, M, lda, K, nb, r3p, G, ea);
    if ((st = check_launch("oz_rowexp A"))) return st;
    tc8::k_oz_rowexp<<<(unsigned)ceil_div(N * 32, 256), 256, 0, s>>>(B, N, ldb, K, nb, r3p, G, eb);
    if ((st = check_launch("oz_rowexp B"))) return st;
  }
  auto slice = [&](const double *X, int64_t rows, int64_t rows_pad, int TR, int64_t ld,
                   const int *e, int8_t *out, bool interleave) {
    const unsigned g = (unsigned)ceil_div(rows_pad * ksteps * 2, 256);
    // contiguous slices, or the S slices of every (row tile, K step) block back to back
    const int64_t ss = interleave ? (int64_t)TR * 32 : rows_pad * ldk;
    const int64_t ts = interleave ? (int64_t)slices * TR * 32 : (int64_t)TR * 32;
    switch (slices) {
      case 6:
        tc8::k_oz_slice_t<6><<<g, 256, 0, s>>>(X, rows, rows_pad, ld, K, nb, r3p, G, e, out, TR,
                                                ksteps, ss, ts);
        break;
      case 7:
        tc8::k_oz_slice_t<7><<<g, 256, 0, s>>>(X, rows, rows_pad, ld, K, nb, r3p, G, e, out, TR,
                                                ksteps, ss, ts);
        break;
      default:
        tc8::k_oz_slice_t<8><<<g, 256, 0, s>>>(X, rows, rows_pad, ld, K, nb, r3p, G, e, out, TR,
                                                ksteps, ss, ts);
        break;
    }
    return check_launch("oz_slice");
  };
  // exponent + slices of a dense operand in one pass, S slices of a block interleaved
  auto rowslice = [&](const double *X, int64_t rows, int64_t rows_pad, int TR, int64_t ld, int *e,
                      int8_t *out) {
    const unsigned g = (unsigned)ceil_div(rows_pad * 16, 256);
    const int64_t ss = (int64_t)TR * 32, ts = (int64_t)slices * TR * 32;
    if (slices == 6)
      tc8::k_oz_rowslice<6><<<g, 256, 0, s>>>(X, rows, rows_pad, ld, K, e, out, TR, ksteps, ss, ts);
    else
      tc8::k_oz_rowslice<7><<<g, 256, 0, s>>>(X, rows, rows_pad, ld, K, e, out, TR, ksteps, ss, ts);
    return check_launch("oz_rowslice");
  };
  if ((phase & 1) && res) {
    if ((st = rowslice(A, M, Mp, 128, lda, ea, SA))) return st;
    if ((st = rowslice(B, N, Np, 64, ldb, eb, SB))) return st;
  } else if (phase & 1) {
    if ((st = slice(A, M, Mp, 128, lda, ea, SA, res))) return st;
    if ((st = slice(B, N, Np, 64, ldb, eb, SB, res))) return st;
  }
  if (!(phase & 2)) return RS_OK;
  if (res) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int nsteps = (int)ceil_div(K, 32);
    const char *denv = getenv("RSB200_OZ_DBG");
    const int dbgv = denv ? atoi(denv) : 0;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(M, tc8::BM), sms);
    auto go = [&](auto kern, int smem, int threads) -> int {
      cudaError_t e = smem_attr((const void *)kern, smem);
      if (e != cudaSuccess) return fail(RS_ERR_CUDA, "oz smem: %s", cudaGetErrorString(e));
      kern<<<grid, threads, smem, s>>>(SA, SB, ksteps, nsteps, ea, eb, C, ldc,
                                       M, N, (accumulate ? 1 : 0) | (dbgv << 4));
      return check_launch("oz_res");
    };
    ProfScope ps(s, "oz_mma");
    return slices == 6 ? go(tc8::k_oz_res<6>, tc8::OzRes<6>::SMEM, tc8::OzRes<6>::THREADS_RES)
                       : go(tc8::k_oz_res<7>, tc8::OzRes<7>::SMEM, tc8::OzRes<7>::THREADS_RES);
  }
  const int64_t *use = ranges;
  if (!ranges) {  // one full range per tile
    std::vector<int64_t> h(ntn * nr * 2, 0);
    for (int64_t t = 0; t < ntn; ++t) { h[t * nr * 2] = 0; h[t * nr * 2 + 1] = K; }
    cudaMemcpyAsync(rin, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    use = rin;
  }
  tc8::k_oz_ranges<<<(unsigned)ceil_div(ntn, 128), 128, 0, s>>>(use, nr, ntn, ldk, rg);
  if ((st = check_launch("oz_ranges"))) return st;
  dim3 grid((unsigned)ntn, (unsigned)ceil_div(M, tc8::BM));
  auto go = [&](auto kern, int smem) -> int {
    cudaError_t e = smem_attr((const void *)kern, smem);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "oz smem: %s", cudaGetErrorString(e));
    kern<<<grid, tc8::THREADS, smem, s>>>(SA, Mp * ldk, SB, Np * ldk, ksteps, ea, eb, rg, nr, C,
                                          ldc, M, N);
    return check_launch("oz_gemm");
  };
  ProfScope ps(s, "oz_mma");
  if (slices == 6)
    return accumulate ? go(tc8::k_oz_gemm<6, true>, tc8::OzCfg<6>::SMEM)
                      : go(tc8::k_oz_gemm<6, false>, tc8::OzCfg<6>::SMEM);
  if (slices == 7)
    return accumulate ? go(tc8::k_oz_gemm<7, true>, tc8::OzCfg<7>::SMEM)
                      : go(tc8::k_oz_gemm<7, false>, tc8::OzCfg<7>::SMEM);
  return accumulate ? go(tc8::k_oz_gemm<8, true>, tc8::OzCfg<8>::SMEM)
                    : go(tc8::k_oz_gemm<8, false>, tc8::OzCfg<8>::SMEM);
}

}  // extern "C"
