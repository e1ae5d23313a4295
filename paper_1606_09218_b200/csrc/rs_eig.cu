// Top-b eigenpairs of small symmetric PSD Gram matrices (the per-mode
// eigen-truncation of rankred.py:90-96, 129-148) without cuSOLVER's
// latency-bound full syevd.
//
// The side-matrix Grams of the RS long part have exponentially decaying
// spectra (lambda_i / lambda_0 reaches the 1e-16 noise floor after a few
// dozen indices), so a block of b basis vectors captures everything above
// rounding: block subspace iteration Q <- orth(Q G) (q steps, CGS2
// orthonormalisation in one CTA per matrix), Rayleigh-Ritz T = Q G Q^T,
// parallel cyclic Jacobi on T in shared memory, Ritz vectors U = V^T Q,
// largest-|entry|-positive signs.  The host checks convergence with the
// returned Ritz values (and escalates b, see rankred.top_eig).
#include <math.h>

#include <algorithm>

#include "rs_common.cuh"
#include "rs_dmma.cuh"

namespace rsb {

__device__ __forceinline__ double hash_unit(uint64_t a, uint64_t b) {
  uint64_t x = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull);
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

// Qt[m][j][i] = pseudo-random start block (deterministic)
__global__ void k_eig_start(double *__restrict__ Qt, int nmat, int b, int64_t n, uint64_t seed) {
  const int64_t total = (int64_t)nmat * b * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    Qt[e] = hash_unit(seed, (uint64_t)e);
}

// One-sided (Hestenes) Jacobi on the b rows of Y (n each): plane rotations
// of row pairs until all rows are mutually orthogonal, then rows are
// normalised and sorted by norm (descending).  For Y = W G with W spanning
// the dominant invariant subspace of G this yields the eigenvectors of G as
// rows and the eigenvalues as row norms -- orthonormalisation, Rayleigh-Ritz
// and the small eigenproblem in one numerically stable step.  Warp per row
// pair (parallel round-robin ordering), rows in shared memory (b*n <= 27k).
constexpr int OJ_MAX_THREADS = 1024;

__global__ void __launch_bounds__(OJ_MAX_THREADS)
    k_ojac_rows(const double *__restrict__ Yall, int b, int64_t n, int64_t stride,
                double *__restrict__ Wall, double *__restrict__ sig_all, int max_sweeps) {
  extern __shared__ double sm[];
  double *nrm = sm;                    // b
  int *flag = (int *)(nrm + b);        // 1 (+pad)
  double *R = nrm + b + 2;             // b * n rows
  const double *Y = Yall + blockIdx.x * stride;
  double *W = Wall + blockIdx.x * stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int64_t e = threadIdx.x; e < (int64_t)b * n; e += blockDim.x) R[e] = Y[e];
  __syncthreads();
  const int half = b / 2;
  // rounding floor of a length-n dot product relative to |x||y| (de Rijk / Demmel-Veselic)
  const double tol = fmax(1e-15, 2.3e-16 * (double)n);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int round = 0; round < b - 1; ++round) {
      for (int i = warp; i < half; i += nwarps) {
        const int a0 = i, a1 = b - 1 - i;
        int p = a0 == 0 ? 0 : 1 + (a0 - 1 + round) % (b - 1);
        int q = a1 == 0 ? 0 : 1 + (a1 - 1 + round) % (b - 1);
        if (p > q) {
          int t = p;
          p = q;
          q = t;
        }
        double *rp = R + (int64_t)p * n, *rq = R + (int64_t)q * n;
        double aa = 0.0, bb = 0.0, gg = 0.0;
        for (int64_t e = lane; e < n; e += 32) {
          const double x = rp[e], y = rq[e];
          aa = fma(x, x, aa);
          bb = fma(y, y, bb);
          gg = fma(x, y, gg);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          aa += __shfl_xor_sync(0xffffffffu, aa, o);
          bb += __shfl_xor_sync(0xffffffffu, bb, o);
          gg += __shfl_xor_sync(0xffffffffu, gg, o);
        }
        if (gg != 0.0 && fabs(gg) > tol * sqrt(aa * bb)) {
          const double zeta = (bb - aa) / (2.0 * gg);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = rsqrt(1.0 + t * t), sn = c * t;
          for (int64_t e = lane; e < n; e += 32) {
            const double x = rp[e], y = rq[e];
            rp[e] = c * x - sn * y;
            rq[e] = sn * x + c * y;
          }
          if (lane == 0) *flag = 1;
        }
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  for (int i = warp; i < b; i += nwarps) {
    const double *ri = R + (int64_t)i * n;
    double ss = 0.0;
    for (int64_t e = lane; e < n; e += 32) ss = fma(ri[e], ri[e], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) nrm[i] = sqrt(ss);
  }
  __syncthreads();
  // rank rows by norm (descending, ties by index), scatter normalised rows
  double *sig = sig_all + (int64_t)blockIdx.x * b;
  __shared__ int dest[128];
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    int pos = 0;
    for (int j = 0; j < b; ++j) pos += (nrm[j] > nrm[i]) || (nrm[j] == nrm[i] && j < i);
    dest[i] = pos;
    sig[pos] = nrm[i];
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < (int64_t)b * n; e += blockDim.x) {
    const int i = (int)(e / n);
    const double inv = nrm[i] > 0.0 ? 1.0 / nrm[i] : 0.0;
    W[(int64_t)dest[i] * n + (e - (int64_t)i * n)] = R[e] * inv;
  }
}

// Largest-|entry| (first occurrence) of each row made positive; row per block.
__global__ void k_sign_rows(double *__restrict__ U, int64_t n) {
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  double *row = U + (int64_t)blockIdx.x * n;
  double best = -1.0;
  int64_t arg = 0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    double a = fabs(row[e]);
    if (a > best) {
      best = a;
      arg = e;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ob = __shfl_xor_sync(0xffffffffu, best, o);
    int64_t oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) {
      best = ob;
      arg = oa;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = arg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) {
        bv[0] = bv[w];
        bi[0] = bi[w];
      }
  }
  __syncthreads();
  const double sgn = row[bi[0]] < 0.0 ? -1.0 : 1.0;
  if (sgn < 0.0)
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) row[e] = -row[e];
}

// trace of each matrix (fixed order)
__global__ void k_trace(const double *__restrict__ G, int64_t n, double *__restrict__ tr) {
  if (threadIdx.x != 0) return;
  const double *g = G + (int64_t)blockIdx.x * n * n;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += g[i * n + i];
  tr[blockIdx.x] = s;
}

template <class T>
__global__ void __launch_bounds__(T::THREADS)
    k_gemm_nt_batched(const double *__restrict__ A, int64_t lda, int64_t sA,
                      const double *__restrict__ B, int64_t ldb, int64_t sB, double *__restrict__ C,
                      int64_t ldc, int64_t sC, int64_t M, int64_t N, int64_t K) {
  extern __shared__ __align__(16) double smem[];
  const int64_t n0 = (int64_t)blockIdx.x * T::BN;
  const int64_t m0 = (int64_t)blockIdx.y * T::BM;
  A += blockIdx.z * sA;
  B += blockIdx.z * sB;
  C += blockIdx.z * sC;
  Acc<T> acc;
  acc.zero();
  mainloop<T>(smem, acc, A, lda, m0, M, B, ldb, n0, N, 0, K);
  store_tile<T>(acc, C, ldc, m0, M, n0, N);
}

using TileEig = Tile<64, 64, 32, 32, 3>;

static int gemm_batched(const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb,
                        int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t M, int64_t N,
                        int64_t K, int nb, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute((const void *)k_gemm_nt_batched<TileEig>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       TileEig::SMEM_BYTES);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
  dim3 grid((unsigned)ceil_div(N, TileEig::BN), (unsigned)ceil_div(M, TileEig::BM), (unsigned)nb);
  k_gemm_nt_batched<TileEig><<<grid, TileEig::THREADS, TileEig::SMEM_BYTES, s>>>(
      A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K);
  return check_launch("eig gemm");
}

}  // namespace rsb

using namespace rsb;

extern "C" {

int64_t rs_topeig_workspace_bytes(int64_t nmat, int64_t n, int64_t b) {
  return 2 * nmat * b * n * 8 + 1024;  // Y, W
}

int rs_topeig(const double *G, int64_t nmat, int64_t n, int64_t b, int64_t iters, double *evals,
              double *U, double *trace, void *work, int64_t work_bytes, void *stream) {
  RS_REQUIRE(nmat >= 1 && n >= 2 && b >= 2 && b <= n && b % 2 == 0 && b <= 128 && iters >= 1,
             "rs_topeig: bad sizes (need 2 <= b <= min(n, 128), b even)");
  RS_REQUIRE(n % 2 == 0, "rs_topeig: n must be even");
  if (work_bytes < rs_topeig_workspace_bytes(nmat, n, b))
    return fail(RS_ERR_CAPACITY, "rs_topeig: workspace too small");
  const size_t need = (size_t)(b + 2 + b * n) * 8;
  if (need > 220 * 1024)
    return fail(RS_ERR_UNSUPPORTED, "rs_topeig: b*n = %lld exceeds the shared-memory block",
                (long long)(b * n));
  cudaStream_t s = as_stream(stream);
  double *Y = (double *)work;
  double *W = Y + nmat * b * n;
  int st;
  ProfScope ps(s, "topeig");
  k_eig_start<<<grid_blocks(nmat * b * n), 256, 0, s>>>(W, (int)nmat, (int)b, n, 12345);
  if ((st = check_launch("eig start"))) return st;
  cudaError_t e = cudaFuncSetAttribute((const void *)k_ojac_rows,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "ojac smem: %s", cudaGetErrorString(e));
  const int threads = (int)std::min<int64_t>(OJ_MAX_THREADS, 32 * (b / 2));
  for (int64_t it = 0; it < iters; ++it) {
    // Y = W G, then W <- orthonormal rows of Y (eigen-directions of G)
    if ((st = gemm_batched(W, n, b * n, G, n, n * n, Y, n, b * n, b, n, n, (int)nmat, s))) return st;
    double *dst = (it == iters - 1) ? U : W;
    k_ojac_rows<<<(unsigned)nmat, threads, need, s>>>(Y, (int)b, n, b * n, dst, evals, 40);
    if ((st = check_launch("ojac"))) return st;
  }
  k_sign_rows<<<(unsigned)(nmat * b), 256, 0, s>>>(U, n);
  if ((st = check_launch("sign"))) return st;
  k_trace<<<(unsigned)nmat, 32, 0, s>>>(G, n, trace);
  return check_launch("trace");
}

}  // extern "C"
