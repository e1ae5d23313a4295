// FP64 tensor-core (DMMA) tiled NT-GEMM building blocks for sm_100a.
//
// sm_100a exposes no FP64 kind for tcgen05.mma, so double-precision tensor
// math is the warp-level mma.sync.m8n8k4.f64 (SASS: DMMA.8x8x4).  Operands
// are staged global->shared with 16-byte cp.async in a STAGES-deep ring, both
// operands K-contiguous ("NT": C = A * B^T), rows padded by 4 doubles so the
// (row = lane/4, k = lane%4) fragment reads are bank-conflict free.
#pragma once

#include "rs_common.cuh"

namespace rsb {

__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
  int bytes = valid ? 16 : 0;  // 0 => zero-fill, nothing read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BM_, int BN_, int WM_, int WN_, int STAGES_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, BK = 16, LDS = BK + 4;
  static constexpr int WM = WM_, WN = WN_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int STAGES = STAGES_;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int STAGE_DOUBLES = (BM + BN) * LDS;
  static constexpr int SMEM_BYTES = STAGE_DOUBLES * STAGES * 8;
};

template <class T>
struct Acc {
  double v[T::MT][T::NT][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < T::MT; ++i)
#pragma unroll
      for (int j = 0; j < T::NT; ++j) v[i][j][0] = v[i][j][1] = 0.0;
  }
};

// One BK-wide K chunk of both operand tiles -> shared memory.  Columns at or
// beyond k_hi and rows beyond M/N are zero-filled (k even, k_hi may be odd).
template <class T>
__device__ __forceinline__ void stage_load(double *s, const double *A, int64_t lda, int64_t m0,
                                           int64_t M, const double *B, int64_t ldb, int64_t n0,
                                           int64_t N, int64_t k, int64_t k_hi) {
  constexpr int CH = T::BK / 2;
  constexpr int TOTAL = (T::BM + T::BN) * CH;
#pragma unroll
  for (int c0 = 0; c0 < TOTAL; c0 += T::THREADS) {
    int c = c0 + threadIdx.x;
    if (TOTAL % T::THREADS != 0 && c >= TOTAL) break;
    int row = c / CH, ch = c % CH;
    int64_t kk = k + 2 * ch;
    bool kin = kk < k_hi;
    const double *src;
    bool ok;
    if (row < T::BM) {
      int64_t g = m0 + row;
      ok = kin && g < M;
      src = ok ? A + g * lda + kk : A;
    } else {
      int64_t g = n0 + (row - T::BM);
      ok = kin && g < N;
      src = ok ? B + g * ldb + kk : B;
    }
    // odd k_hi: the last pair reads one element and zero-fills the other
    const int bytes = ok ? (kk + 1 < k_hi ? 16 : 8) : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                     smem_addr(s + row * T::LDS + 2 * ch)),
                 "l"(src), "r"(bytes));
  }
}

template <class T>
__device__ __forceinline__ void stage_mma(const double *s, Acc<T> &acc, int wm0, int wn0, int gid,
                                          int tig) {
  const double *sA = s;
  const double *sB = s + T::BM * T::LDS;
#pragma unroll
  for (int kk = 0; kk < T::BK; kk += 4) {
    double a[T::MT], b[T::NT];
#pragma unroll
    for (int i = 0; i < T::MT; ++i) a[i] = sA[(wm0 + i * 8 + gid) * T::LDS + kk + tig];
#pragma unroll
    for (int j = 0; j < T::NT; ++j) b[j] = sB[(wn0 + j * 8 + gid) * T::LDS + kk + tig];
#pragma unroll
    for (int i = 0; i < T::MT; ++i)
#pragma unroll
      for (int j = 0; j < T::NT; ++j) dmma_884(acc.v[i][j], a[i], b[j]);
  }
}

// as stage_mma, only the first `kv` (<= BK, rounded up to 4) columns of the chunk
template <class T>
__device__ __forceinline__ void stage_mma_kv(const double *s, Acc<T> &acc, int wm0, int wn0,
                                             int gid, int tig, int kv) {
  const double *sA = s;
  const double *sB = s + T::BM * T::LDS;
#pragma unroll
  for (int kk = 0; kk < T::BK; kk += 4) {
    if (kk >= kv) break;  // uniform across the CTA
    double a[T::MT], b[T::NT];
#pragma unroll
    for (int i = 0; i < T::MT; ++i) a[i] = sA[(wm0 + i * 8 + gid) * T::LDS + kk + tig];
#pragma unroll
    for (int j = 0; j < T::NT; ++j) b[j] = sB[(wn0 + j * 8 + gid) * T::LDS + kk + tig];
#pragma unroll
    for (int i = 0; i < T::MT; ++i)
#pragma unroll
      for (int j = 0; j < T::NT; ++j) dmma_884(acc.v[i][j], a[i], b[j]);
  }
}

// acc += A[m0:m0+BM, k_lo:k_hi] * B[n0:n0+BN, k_lo:k_hi]^T, cp.async ring.
template <class T>
__device__ __forceinline__ void mainloop(double *smem, Acc<T> &acc, const double *A, int64_t lda,
                                         int64_t m0, int64_t M, const double *B, int64_t ldb,
                                         int64_t n0, int64_t N, int64_t k_lo, int64_t k_hi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / T::WARPS_N) * T::WM, wn0 = (warp % T::WARPS_N) * T::WN;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t chunks = (k_hi - k_lo + T::BK - 1) / T::BK;
  if (chunks <= 0) return;
#pragma unroll
  for (int s = 0; s < T::STAGES - 1; ++s) {
    if (s < chunks)
      stage_load<T>(smem + s * T::STAGE_DOUBLES, A, lda, m0, M, B, ldb, n0, N, k_lo + s * T::BK,
                    k_hi);
    cp_async_commit();
  }
  for (int64_t c = 0; c < chunks; ++c) {
    cp_async_wait<T::STAGES - 2>();
    __syncthreads();
    int64_t nx = c + T::STAGES - 1;
    if (nx < chunks)
      stage_load<T>(smem + (nx % T::STAGES) * T::STAGE_DOUBLES, A, lda, m0, M, B, ldb, n0, N,
                    k_lo + nx * T::BK, k_hi);
    cp_async_commit();
    stage_mma<T>(smem + (c % T::STAGES) * T::STAGE_DOUBLES, acc, wm0, wn0, gid, tig);
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Store the warp tiles of acc into C (row-major, ldc even), predicated on M/N.
template <class T, bool ACC = false>
__device__ __forceinline__ void store_tile(const Acc<T> &acc, double *C, int64_t ldc, int64_t m0,
                                           int64_t M, int64_t n0, int64_t N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / T::WARPS_N) * T::WM, wn0 = (warp % T::WARPS_N) * T::WN;
  const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int i = 0; i < T::MT; ++i) {
    int64_t r = m0 + wm0 + i * 8 + gid;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < T::NT; ++j) {
      int64_t c = n0 + wn0 + j * 8 + tig * 2;
      double *p = C + r * ldc + c;
      if (c + 1 < N && (ldc % 2 == 0)) {
        double2 v = make_double2(acc.v[i][j][0], acc.v[i][j][1]);
        if (ACC) {
          const double2 old = *reinterpret_cast<const double2 *>(p);
          v.x += old.x;
          v.y += old.y;
        }
        *reinterpret_cast<double2 *>(p) = v;
      } else {
        if (c < N) p[0] = ACC ? p[0] + acc.v[i][j][0] : acc.v[i][j][0];
        if (c + 1 < N) p[1] = ACC ? p[1] + acc.v[i][j][1] : acc.v[i][j][1];
      }
    }
  }
}

}  // namespace rsb
