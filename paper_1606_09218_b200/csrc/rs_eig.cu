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
#include <stdlib.h>

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

constexpr int ORTH_THREADS = 256;

__device__ double block_sum(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;  // identical in every thread (fixed order)
}

// Orthonormalise the b rows of Q (n each) in place: classical Gram-Schmidt
// applied twice per vector ("twice is enough"); a vector that collapses is
// replaced by a fresh pseudo-random one.  One CTA per matrix.  With
// IN_SMEM the finished rows live in shared memory (n*b*8 bytes) and are
// written back at the end; otherwise they are read from global/L2.
template <bool IN_SMEM>
__global__ void __launch_bounds__(ORTH_THREADS)
    k_orth_rows(double *__restrict__ Qall, int b, int64_t n, int64_t stride, uint64_t seed) {
  extern __shared__ double sm[];
  double *v = sm;           // n
  double *coef = sm + n;    // b
  double *red = coef + b;   // 32
  double *Qs = red + 32;    // b*n when IN_SMEM
  double *Qg = Qall + blockIdx.x * stride;
  double *Q = IN_SMEM ? Qs : Qg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  if (IN_SMEM) {
    for (int64_t e = threadIdx.x; e < (int64_t)b * n; e += blockDim.x) Qs[e] = Qg[e];
    __syncthreads();
  }
  for (int i = 0; i < b; ++i) {
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) v[e] = Q[i * n + e];
    __syncthreads();
    double ss = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) ss += v[e] * v[e];
    double nrm0 = sqrt(block_sum(ss, red));
    double nrm = 0.0;
    for (int attempt = 0; attempt < 3; ++attempt) {
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = warp; j < i; j += nwarps) {
          const double *qj = Q + (int64_t)j * n;
          double d = 0.0;
          for (int64_t e = lane; e < n; e += 32) d = fma(qj[e], v[e], d);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (lane == 0) coef[j] = d;
        }
        __syncthreads();
        for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
          double a0 = v[e], a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int j = 0;
          for (; j + 4 <= i; j += 4) {
            a0 -= coef[j] * Q[(int64_t)j * n + e];
            a1 -= coef[j + 1] * Q[(int64_t)(j + 1) * n + e];
            a2 -= coef[j + 2] * Q[(int64_t)(j + 2) * n + e];
            a3 -= coef[j + 3] * Q[(int64_t)(j + 3) * n + e];
          }
          for (; j < i; ++j) a0 -= coef[j] * Q[(int64_t)j * n + e];
          v[e] = (a0 + a1) + (a2 + a3);
        }
        __syncthreads();
      }
      ss = 0.0;
      for (int64_t e = threadIdx.x; e < n; e += blockDim.x) ss += v[e] * v[e];
      nrm = sqrt(block_sum(ss, red));
      if (nrm > 1e-13 * nrm0 && nrm > 0.0) break;
      // breakdown: restart this vector from a fresh deterministic direction
      for (int64_t e = threadIdx.x; e < n; e += blockDim.x)
        v[e] = hash_unit(seed + 7919 * (attempt + 1), (uint64_t)(i * n + e));
      __syncthreads();
      ss = 0.0;
      for (int64_t e = threadIdx.x; e < n; e += blockDim.x) ss += v[e] * v[e];
      nrm0 = sqrt(block_sum(ss, red));
    }
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) Q[i * n + e] = v[e] * inv;
    __syncthreads();
  }
  if (IN_SMEM)
    for (int64_t e = threadIdx.x; e < (int64_t)b * n; e += blockDim.x) Qg[e] = Qs[e];
}

// CGS2 with the block in shared memory and the normalisation of row i-1
// folded into row i's first projection: row i is projected on the
// unnormalised v_{i-1} (coefficient (v_{i-1}.x)/|v_{i-1}|^2) while the same
// reduction pass yields |v_{i-1}|^2 and |x|^2, and v_{i-1} is scaled in the
// update phase -- 4 barriers per row instead of 10.  A collapsed row (norm
// <= 1e-13 of its input norm) is redone from pseudo-random directions exactly
// as in k_orth_rows (same seeds), then the current row restarts.
__device__ void orth_dots(const double *__restrict__ Qs, const double *__restrict__ x, int nd,
                          int i, int64_t n, double *__restrict__ coef) {
  // coef[j] = q_j . x (j < i); coef[i] = x . x; coef[i + 1] = q_{i-1} . q_{i-1} (nd = i + 2)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int j = warp; j < nd; j += nwarps) {
    const double *a = j < i ? Qs + (int64_t)j * n : (j == i ? x : Qs + (int64_t)(i - 1) * n);
    const double *c = j <= i ? x : a;
    double d = 0.0;
    for (int64_t e = lane; e < n; e += 32) d = fma(a[e], c[e], d);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) coef[j] = d;
  }
}

// rows < r normalised; row r regenerated from pseudo-random directions until
// it survives CGS2 (at most 3 attempts, as k_orth_rows), then normalised
__device__ void orth_row_redo(double *__restrict__ Qs, int r, int64_t n, uint64_t seed,
                              double *__restrict__ coef, double *__restrict__ red) {
  double *v = Qs + (int64_t)r * n;
  double nrm = 0.0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x)
      v[e] = hash_unit(seed + 7919 * (attempt + 1), (uint64_t)(r * n + e));
    __syncthreads();
    double ss = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) ss += v[e] * v[e];
    const double nrm0 = sqrt(block_sum(ss, red));
    for (int pass = 0; pass < 2; ++pass) {
      orth_dots(Qs, v, r, r, n, coef);
      __syncthreads();
      for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
        double a = v[e];
        for (int j = 0; j < r; ++j) a -= coef[j] * Qs[(int64_t)j * n + e];
        v[e] = a;
      }
      __syncthreads();
    }
    ss = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) ss += v[e] * v[e];
    nrm = sqrt(block_sum(ss, red));
    if (nrm > 1e-13 * nrm0 && nrm > 0.0) break;
  }
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) v[e] *= inv;
  __syncthreads();
}

// v[e] -= sum_{j < jn} coef[j] Q_j[e] for every e < n, with P threads per
// element (consecutive lanes) splitting the j sum and combining it by a fixed
// xor tree; with `pending`, row im1 (= i - 1, unnormalised) is also projected
// out with coefficient cprev and scaled by inv_prev in the same pass.
__device__ __forceinline__ void orth_update(double *__restrict__ Qs, double *__restrict__ v,
                                            const double *__restrict__ coef, int jn, int64_t n,
                                            int P, bool pending, int im1, double cprev,
                                            double inv_prev) {
  const int part = threadIdx.x & (P - 1);
  const int64_t stride = blockDim.x / P;
  for (int64_t eb = 0; eb < n; eb += stride) {  // uniform trip count: the shuffles stay converged
    const int64_t e = eb + threadIdx.x / P;
    const bool ok = e < n;
    double a0 = 0.0, a1 = 0.0;
    if (ok) {
      int j = part;
      for (; j + P < jn; j += 2 * P) {
        a0 -= coef[j] * Qs[(int64_t)j * n + e];
        a1 -= coef[j + P] * Qs[(int64_t)(j + P) * n + e];
      }
      if (j < jn) a0 -= coef[j] * Qs[(int64_t)j * n + e];
      if (part == 0) {
        if (pending) {
          double *qp = Qs + (int64_t)im1 * n + e;
          const double q = *qp;
          a1 -= cprev * q;
          *qp = q * inv_prev;
        }
        a0 += v[e];
      }
    }
    double a = a0 + a1;
    for (int o = 1; o < P; o <<= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (ok && part == 0) v[e] = a;
  }
}

__global__ void __launch_bounds__(1024)
    k_orth_rows_fused(double *__restrict__ Qall, int b, int64_t n, int64_t stride,
                      uint64_t seed) {
  extern __shared__ double sm[];
  double *coef = sm;            // b + 8
  double *red = coef + b + 8;   // 32
  double *Qs = red + 32;        // b * n
  double *Qg = Qall + blockIdx.x * stride;
  for (int64_t e = threadIdx.x; e < (int64_t)b * n; e += blockDim.x) Qs[e] = Qg[e];
  __syncthreads();
  // threads per element in the projection updates (power of two, <= 8)
  int P = 1;
  while (P < 8 && (int64_t)blockDim.x >= 2 * P * n) P <<= 1;
  bool pending = false;  // row i-1 orthogonalised but not yet normalised
  double nrm0_prev = 0.0;
  for (int i = 0; i < b; ++i) {
    double *v = Qs + (int64_t)i * n;
    orth_dots(Qs, v, pending ? i + 2 : i + 1, i, n, coef);
    __syncthreads();
    double cprev = 0.0, inv_prev = 1.0;
    if (pending) {
      const double pp = coef[i + 1], nprev = sqrt(pp);
      if (!(nprev > 1e-13 * nrm0_prev && nprev > 0.0)) {  // row i-1 collapsed (uniform)
        __syncthreads();
        orth_row_redo(Qs, i - 1, n, seed, coef, red);
        pending = false;
        --i;          // redo row i with row i-1 normalised
        continue;
      }
      cprev = coef[i - 1] / pp;
      inv_prev = 1.0 / nprev;
    }
    const double nrm0 = sqrt(coef[i]);
    const int jn = pending ? i - 1 : i;  // rows already normalised
    orth_update(Qs, v, coef, jn, n, P, pending, i - 1, cprev, inv_prev);
    __syncthreads();
    if (i > 0) {  // second projection (all previous rows normalised now)
      orth_dots(Qs, v, i, i, n, coef);
      __syncthreads();
      orth_update(Qs, v, coef, i, n, P, false, 0, 0.0, 1.0);
      __syncthreads();
    }
    pending = true;
    nrm0_prev = nrm0;
  }
  // the last row's norm
  double ss = 0.0;
  const double *vl = Qs + (int64_t)(b - 1) * n;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) ss += vl[e] * vl[e];
  const double nl = sqrt(block_sum(ss, red));
  if (!(nl > 1e-13 * nrm0_prev && nl > 0.0)) {
    __syncthreads();
    orth_row_redo(Qs, b - 1, n, seed, coef, red);
  } else {
    const double inv = 1.0 / nl;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) Qs[(int64_t)(b - 1) * n + e] *= inv;
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < (int64_t)b * n; e += blockDim.x) Qg[e] = Qs[e];
}

// Parallel cyclic Jacobi on the B x B symmetric T (shared memory), one CTA per
// matrix.  Each round rotates B/2 disjoint pairs (round-robin table built once
// in shared memory); the rotations are computed by B/2 threads, then
// T' = J^T T J is applied as independent 2x2 block updates and V' = V J in a
// single phase.  B is a template parameter so every index computation is a
// constant shift/mask.  Outputs eigenvalues sorted descending and the
// matching eigenvectors as rows of Vt.
// launch bound; RSB200_JACOBI_THREADS = 256 or 512 (default: one pass per
// rotation round at B = 24; C3 topeig 2.64 -> 2.47 ms, C2 0.367 -> 0.36 ms)
constexpr int JAC_THREADS = 512;

template <int B>
__global__ void __launch_bounds__(JAC_THREADS)
    k_jacobi(const double *__restrict__ Tall, double *__restrict__ evals,
             double *__restrict__ Vtall, int max_sweeps) {
  constexpr int LD = B + 1, HALF = B / 2;
  extern __shared__ double sm[];
  double *T = sm;                       // B x LD
  double *V = T + B * LD;               // B x LD
  double *rc = V + B * LD;              // HALF (c), HALF (s)
  double *rs = rc + HALF;
  int *pairs = (int *)(rs + HALF);      // (B-1) x HALF x 2
  int *flag = pairs + (B - 1) * B;
  const double *Tg = Tall + (int64_t)blockIdx.x * B * B;
  for (int e = threadIdx.x; e < B * B; e += blockDim.x) {
    const int r = e / B, c = e % B;
    T[r * LD + c] = 0.5 * (Tg[r * B + c] + Tg[c * B + r]);  // symmetrise
    V[r * LD + c] = (r == c) ? 1.0 : 0.0;
  }
  for (int e = threadIdx.x; e < (B - 1) * HALF; e += blockDim.x) {
    const int round = e / HALF, i = e % HALF;
    const int a0 = i, a1 = B - 1 - i;
    int p = a0 == 0 ? 0 : 1 + (a0 - 1 + round) % (B - 1);
    int q = a1 == 0 ? 0 : 1 + (a1 - 1 + round) % (B - 1);
    pairs[2 * e] = p < q ? p : q;
    pairs[2 * e + 1] = p < q ? q : p;
  }
  __syncthreads();
  double dmax = 0.0;
  for (int i = 0; i < B; ++i) dmax = fmax(dmax, fabs(T[i * LD + i]));
  // absolute floor at the rounding level of T: the Ritz values below it are
  // noise (their rotations only shuffle rounding errors, sweep after sweep)
  const double tol = 1e-16 * dmax;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int round = 0; round < B - 1; ++round) {
      const int *pr = pairs + round * B;
      if (threadIdx.x < HALF) {
        const int i = threadIdx.x;
        const int p = pr[2 * i], q = pr[2 * i + 1];
        const double app = T[p * LD + p], aqq = T[q * LD + q], apq = T[p * LD + q];
        double c = 1.0, s = 0.0;
        // rotate unless apq is rounding-level relative to the larger diagonal
        // entry or below the absolute floor (noise block of the Ritz matrix)
        if (fabs(apq) > tol && fabs(apq) > 1e-14 * fmax(fabs(app), fabs(aqq))) {
          const double d = aqq - app, e2 = apq + apq;
          const double t = (d >= 0.0 ? e2 : -e2) / (fabs(d) + sqrt(d * d + e2 * e2));
          c = rsqrt(1.0 + t * t);
          s = t * c;
          *flag = 1;
        }
        rc[i] = c;
        rs[i] = s;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < HALF * HALF + HALF * B; e += blockDim.x) {
        if (e < HALF * HALF) {
          const int i = e / HALF, j = e % HALF;
          const double ci = rc[i], si = rs[i], cj = rc[j], sj = rs[j];
          if (si == 0.0 && sj == 0.0) continue;
          const int p = pr[2 * i], q = pr[2 * i + 1], u = pr[2 * j], w = pr[2 * j + 1];
          const double tpu = T[p * LD + u], tpw = T[p * LD + w];
          const double tqu = T[q * LD + u], tqw = T[q * LD + w];
          const double ru_p = ci * tpu - si * tqu, rw_p = ci * tpw - si * tqw;
          const double ru_q = si * tpu + ci * tqu, rw_q = si * tpw + ci * tqw;
          T[p * LD + u] = cj * ru_p - sj * rw_p;
          T[p * LD + w] = sj * ru_p + cj * rw_p;
          T[q * LD + u] = cj * ru_q - sj * rw_q;
          T[q * LD + w] = sj * ru_q + cj * rw_q;
        } else {
          const int f = e - HALF * HALF;
          const int j = f / B, k = f % B;
          const double c = rc[j], s = rs[j];
          if (s == 0.0) continue;
          const int p = pr[2 * j], q = pr[2 * j + 1];
          const double vp = V[k * LD + p], vq = V[k * LD + q];
          V[k * LD + p] = c * vp - s * vq;
          V[k * LD + q] = s * vp + c * vq;
        }
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  double *ev = evals + (int64_t)blockIdx.x * B;
  double *Vt = Vtall + (int64_t)blockIdx.x * B * B;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const double ei = T[i * LD + i];
    int pos = 0;
    for (int j = 0; j < B; ++j) {
      const double ej = T[j * LD + j];
      pos += (ej > ei) || (ej == ei && j < i);
    }
    ev[pos] = ei;
    for (int k = 0; k < B; ++k) Vt[(int64_t)pos * B + k] = V[k * LD + i];
  }
}

template <int B>
static int launch_jacobi(const double *T, int nmat, double *evals, double *Vt, size_t reserve,
                         cudaStream_t s) {
  const size_t need = (size_t)(2 * B * (B + 1) + B) * 8 + (size_t)((B - 1) * B + 1) * 4;
  const size_t smem = std::max(need, reserve);
  cudaError_t e = smem_attr((const void *)k_jacobi<B>, (int)smem);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "jacobi smem: %s", cudaGetErrorString(e));
  static const int sweeps = getenv("RSB200_JACOBI_SWEEPS") ? atoi(getenv("RSB200_JACOBI_SWEEPS")) : 16;
  static const int threads = [] {
    const char *e = getenv("RSB200_JACOBI_THREADS");
    return e && atoi(e) == 256 ? 256 : JAC_THREADS;
  }();
  k_jacobi<B><<<(unsigned)nmat, threads, smem, s>>>(T, evals, Vt, sweeps);
  return check_launch("jacobi");
}

// cuSOLVER order (ascending values, eigenvectors as rows) -> the Jacobi
// kernel's (descending values, rows of Vt descending); one block per matrix
__global__ void k_flip_eig(const double *__restrict__ ev_asc, const double *__restrict__ V,
                           int b, double *__restrict__ evals, double *__restrict__ Vt) {
  const int64_t m = blockIdx.x;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int j = e / b, k = e - (e / b) * b;
    Vt[(m * b + j) * b + k] = V[(m * b + (b - 1 - j)) * b + k];
  }
  for (int j = threadIdx.x; j < b; j += blockDim.x) evals[m * b + j] = ev_asc[m * b + b - 1 - j];
}

// U[m][j][i] = sum_k Vt[m][j][k] Q[m][k][i]   (b x b times b x n, per matrix)
__global__ void k_ritz(const double *__restrict__ Vt, const double *__restrict__ Q, int b, int64_t n,
                       int nmat, double *__restrict__ U) {
  const int64_t total = (int64_t)nmat * b * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e % n, j = (e / n) % b, m = e / (n * b);
    const double *v = Vt + (m * b + j) * b;
    const double *q = Q + m * b * n + i;
    double acc = 0.0;
    for (int k = 0; k < b; ++k) acc = fma(v[k], q[(int64_t)k * n], acc);
    U[e] = acc;
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

// trace of each matrix (fixed-order warp reduction)
__global__ void k_trace(const double *__restrict__ G, int64_t n, double *__restrict__ tr) {
  const double *g = G + (int64_t)blockIdx.x * n * n;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 32) s += g[i * n + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) tr[blockIdx.x] = s;
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
using TileEigS = Tile<32, 32, 16, 16, 3>;  // skinny Ritz blocks (b <= 32): 4x the CTAs
// N just above a multiple of 64 (the Tucker operand GEMM at C5: N = r3 = 132 -> 3 x 64 = 192
// columns computed, 69 % useful): 48-wide tiles (3 x 48 = 144, 92 %)
using TileEigN48 = Tile<128, 48, 32, 24, 3>;

template <class T>
static int gemm_batched_t(const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb,
                          int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t M, int64_t N,
                          int64_t K, int nb, cudaStream_t s) {
  if (T::SMEM_BYTES > 48 * 1024) {
    cudaError_t e = smem_attr((const void *)k_gemm_nt_batched<T>, T::SMEM_BYTES);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
  }
  dim3 grid((unsigned)ceil_div(N, T::BN), (unsigned)ceil_div(M, T::BM), (unsigned)nb);
  k_gemm_nt_batched<T><<<grid, T::THREADS, T::SMEM_BYTES, s>>>(A, lda, sA, B, ldb, sB, C, ldc,
                                                                sC, M, N, K);
  return check_launch("eig gemm");
}

static int gemm_batched(const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb,
                        int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t M, int64_t N,
                        int64_t K, int nb, cudaStream_t s) {
  if (M <= 32 || N <= 32)
    return gemm_batched_t<TileEigS>(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, nb, s);
  if (M >= 256 && 100 * ceil_div(N, 48) * 48 <= 85 * ceil_div(N, 64) * 64)
    return gemm_batched_t<TileEigN48>(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, nb, s);
  return gemm_batched_t<TileEig>(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, nb, s);
}


int gemm_batched_nt(const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb,
                    int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t M, int64_t N,
                    int64_t K, int nb, cudaStream_t s) {
  return gemm_batched(A, lda, sA, B, ldb, sB, C, ldc, sC, M, N, K, nb, s);
}

}  // namespace rsb

using namespace rsb;

extern "C" {

int64_t rs_eigh_workspace_bytes(int64_t m, int64_t n);
int rs_eigh(double *G, int64_t m, int64_t n, double *evals, void *work, int64_t work_bytes,
            void *stream);
}  // extern "C"
namespace rsb {
int64_t orth_qr_workspace_bytes(int64_t m, int64_t b, int64_t n);
int orth_qr(double *Y, int64_t m, int64_t b, int64_t n, void *work, int64_t work_bytes,
            cudaStream_t s);
}  // namespace rsb
extern "C" {

// RSB200_ORTH_FUSED=0: the 10-barrier-per-row CGS2 kernel
static const bool g_orth_fused = [] {
  const char *e = getenv("RSB200_ORTH_FUSED");
  return !(e && e[0] == '0');
}();
// threads of the fused CGS2 CTA (RSB200_ORTH_THREADS = 256, 512 or 1024): the
// extra warps take one dot product each and split the projection sums.  1024
// measured no faster (C2 topeig 0.366 -> 0.39 ms, C3 equal): 256 stays.
static const int g_orth_threads = [] {
  const char *e = getenv("RSB200_ORTH_THREADS");
  const int t = e && *e ? atoi(e) : 256;
  return (t == 512 || t == 1024) ? t : 256;
}();

// the one-CTA CGS2 kernel keeps the block in shared memory up to ~200 KB; a
// larger block (C3/C4: 64 x 512/1024) re-reads it from L2 for every row and
// costs ~2.5 ms per pass at C3, where Householder QR (cuSOLVER) is faster
static bool orth_by_qr(int64_t n, int64_t b) {
  return b > 96 || (size_t)(n + b + 32 + b * n) * 8 > 200 * 1024;
}

int64_t rs_topeig_workspace_bytes(int64_t nmat, int64_t n, int64_t b) {
  // Q, Y (nmat*b*n each), T (nmat*b*b), Vt (nmat*b*b); b > 96: + ascending
  // Ritz values (nmat*b) + cuSOLVER workspace for the b x b Rayleigh quotients
  int64_t base = (2 * nmat * b * n + 2 * nmat * b * b) * 8 + 1024;
  if (orth_by_qr(n, b)) {
    const int64_t e = rs_eigh_workspace_bytes(nmat, b), q = orth_qr_workspace_bytes(nmat, b, n);
    if (e < 0 || q < 0) return -1;
    base += round_up(nmat * b * 8, 256) + std::max(e, q);
  }
  return base;
}

int rs_topeig(const double *G, int64_t nmat, int64_t n, int64_t b, int64_t iters, double *evals,
              double *U, double *trace, void *work, int64_t work_bytes, void *stream) {
  RS_REQUIRE(nmat >= 1 && n >= 2 && b >= 2 && b <= n && b % 2 == 0 && b <= 512 && iters >= 1,
             "rs_topeig: bad sizes (need 2 <= b <= min(n, 512), b even)");
  RS_REQUIRE(n % 2 == 0, "rs_topeig: n must be even");
  if (work_bytes < rs_topeig_workspace_bytes(nmat, n, b))
    return fail(RS_ERR_CAPACITY, "rs_topeig: workspace too small");
  cudaStream_t s = as_stream(stream);
  double *Q = (double *)work;
  double *Y = Q + nmat * b * n;
  double *T = Y + nmat * b * n;
  double *Vt = T + nmat * b * b;
  int st;
  ProfScope ps(s, "topeig");
  k_eig_start<<<grid_blocks(nmat * b * n), 256, 0, s>>>(Q, (int)nmat, (int)b, n, 12345);
  if ((st = check_launch("eig start"))) return st;
  const bool q_smem = (size_t)(n + b + 32 + b * n) * 8 <= 200 * 1024;
  // the latency-bound single-CTA kernels reserve a whole SM (shared-memory
  // request near the limit) so concurrent plane-GEMM blocks cannot co-reside
  const size_t reserve = 200 * 1024;
  size_t orth_smem = std::max<size_t>((size_t)(n + b + 32 + (q_smem ? b * n : 0)) * 8, reserve);
  const void *orth_fn = q_smem ? (g_orth_fused ? (const void *)k_orth_rows_fused
                                               : (const void *)k_orth_rows<true>)
                               : (const void *)k_orth_rows<false>;
  if (orth_smem > 48 * 1024) {
    cudaError_t e = smem_attr(orth_fn, (int)orth_smem);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "orth smem: %s", cudaGetErrorString(e));
  }
  // Y = Q G (rows), orth
  for (int64_t it = 0; it < iters; ++it) {
    if ((st = gemm_batched(Q, n, b * n, G, n, n * n, Y, n, b * n, b, n, n, (int)nmat, s))) return st;
    if (orth_by_qr(n, b)) {  // wide / large block: Householder QR (cuSOLVER), one thread/stream per matrix
      char *qw = (char *)work + round_up((2 * nmat * b * n + 2 * nmat * b * b) * 8 + 1024, 256) +
                 round_up(nmat * b * 8, 256);
      if ((st = orth_qr(Y, nmat, b, n, qw, work_bytes - (qw - (char *)work), s))) return st;
      std::swap(Q, Y);
      continue;
    }
    if (q_smem && g_orth_fused)
      k_orth_rows_fused<<<(unsigned)nmat, g_orth_threads, orth_smem, s>>>(Y, (int)b, n, b * n,
                                                                          777 + it);
    else if (q_smem)
      k_orth_rows<true><<<(unsigned)nmat, ORTH_THREADS, orth_smem, s>>>(Y, (int)b, n, b * n, 777 + it);
    else
      k_orth_rows<false><<<(unsigned)nmat, ORTH_THREADS, orth_smem, s>>>(Y, (int)b, n, b * n, 777 + it);
    if ((st = check_launch("orth"))) return st;
    std::swap(Q, Y);
  }
  // Rayleigh-Ritz: W = Q G (into Y), T = W Q^T
  if ((st = gemm_batched(Q, n, b * n, G, n, n * n, Y, n, b * n, b, n, n, (int)nmat, s))) return st;
  if ((st = gemm_batched(Y, n, b * n, Q, n, b * n, T, b, b * b, b, b, n, (int)nmat, s))) return st;
  if (b > 96) {  // Rayleigh quotients too large for the shared-memory Jacobi: cuSOLVER
    double *ev_asc = Vt + nmat * b * b;
    char *ew = (char *)work + round_up((2 * nmat * b * n + 2 * nmat * b * b) * 8 + 1024, 256) +
               round_up(nmat * b * 8, 256);
    const int64_t ebytes = work_bytes - (ew - (char *)work);
    if ((st = rs_eigh(T, nmat, b, ev_asc, ew, ebytes, stream))) return st;
    k_flip_eig<<<(unsigned)nmat, 256, 0, s>>>(ev_asc, T, (int)b, evals, Vt);
    if ((st = check_launch("flip eig"))) return st;
  } else switch (b) {
    case 16: st = launch_jacobi<16>(T, (int)nmat, evals, Vt, reserve, s); break;
    case 24: st = launch_jacobi<24>(T, (int)nmat, evals, Vt, reserve, s); break;
    case 32: st = launch_jacobi<32>(T, (int)nmat, evals, Vt, reserve, s); break;
    case 48: st = launch_jacobi<48>(T, (int)nmat, evals, Vt, reserve, s); break;
    case 64: st = launch_jacobi<64>(T, (int)nmat, evals, Vt, reserve, s); break;
    case 96: st = launch_jacobi<96>(T, (int)nmat, evals, Vt, reserve, s); break;
    default: return fail(RS_ERR_UNSUPPORTED, "rs_topeig: block size %lld not in {16,24,32,48,64,96}",
                         (long long)b);
  }
  if (st) return st;
  k_ritz<<<grid_blocks(nmat * b * n), 256, 0, s>>>(Vt, Q, (int)b, n, (int)nmat, U);
  if ((st = check_launch("ritz"))) return st;
  k_sign_rows<<<(unsigned)(nmat * b), 256, 0, s>>>(U, n);
  if ((st = check_launch("sign"))) return st;
  k_trace<<<(unsigned)nmat, 32, 0, s>>>(G, n, trace);
  return check_launch("trace");
}

}  // extern "C"

// ------------------------------------------------------------------------
// Full spectra of m Gram matrices, one cuSOLVER syevd per matrix on its own
// forked stream (the tridiagonal reduction of one n = 2048 matrix is
// latency-bound: the three modes overlap instead of running back to back),
// no host synchronisation (info stays on the device).  Reference:
// rankred.py:92 (np.linalg.eigh of the side Gram).
#include <cusolverDn.h>

#include <thread>

namespace {
constexpr int EIGH_SLOTS = 3;
struct EighCtx {
  cusolverDnHandle_t h[EIGH_SLOTS] = {};
  cudaStream_t s[EIGH_SLOTS] = {};
  cudaEvent_t fork = nullptr, join[EIGH_SLOTS] = {};
};
std::mutex g_eigh_mu;
EighCtx g_eigh[64];

int eigh_ctx(EighCtx **out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_eigh_mu);
  EighCtx &c = g_eigh[dev & 63];
  if (!c.fork) {
    for (int i = 0; i < EIGH_SLOTS; ++i) {
      if (cudaStreamCreateWithFlags(&c.s[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&c.join[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(RS_ERR_CUDA, "rs_eigh: stream/event");
      if (cusolverDnCreate(&c.h[i]) != CUSOLVER_STATUS_SUCCESS ||
          cusolverDnSetStream(c.h[i], c.s[i]) != CUSOLVER_STATUS_SUCCESS)
        return fail(RS_ERR_CUDA, "rs_eigh: cusolverDnCreate");
    }
    if (cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming) != cudaSuccess)
      return fail(RS_ERR_CUDA, "rs_eigh: event");
  }
  *out = &c;
  return RS_OK;
}
}  // namespace

extern "C" {

int64_t rs_eigh_workspace_bytes(int64_t m, int64_t n) {
  EighCtx *c = nullptr;
  if (m < 1 || n < 1 || eigh_ctx(&c)) return -1;
  int lwork = 0;
  if (cusolverDnDsyevd_bufferSize(c->h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                  (int)n, nullptr, (int)n, nullptr, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return -1;
  return m * (round_up((int64_t)lwork * 8, 256) + 256);
}

int rs_eigh(double *G, int64_t m, int64_t n, double *evals, void *work, int64_t work_bytes,
            void *stream) {
  RS_REQUIRE(G && evals && work && m >= 1 && n >= 1 && n < (1 << 30), "rs_eigh: bad arguments");
  EighCtx *c = nullptr;
  int st;
  if ((st = eigh_ctx(&c))) return st;
  int lwork = 0;
  if (cusolverDnDsyevd_bufferSize(c->h[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                  (int)n, G, (int)n, evals, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return fail(RS_ERR_CUDA, "rs_eigh: bufferSize");
  const int64_t per = round_up((int64_t)lwork * 8, 256) + 256;
  if (work_bytes < m * per)
    return fail(RS_ERR_CAPACITY, "rs_eigh: workspace %lld < %lld", (long long)work_bytes,
                (long long)(m * per));
  cudaStream_t s = as_stream(stream);
  if (cudaEventRecord(c->fork, s) != cudaSuccess) return fail(RS_ERR_CUDA, "rs_eigh: fork");
  int dev = 0;
  cudaGetDevice(&dev);
  // one host thread per slot: syevd synchronises internally (divide and
  // conquer bookkeeping), so issuing the modes from one thread serialises them
  for (int64_t i0 = 0; i0 < m; i0 += EIGH_SLOTS) {
    const int k = (int)std::min<int64_t>(EIGH_SLOTS, m - i0);
    int rc[EIGH_SLOTS] = {0, 0, 0};
    std::thread th[EIGH_SLOTS];
    for (int j = 0; j < k; ++j) {
      th[j] = std::thread([&, j] {
        const int64_t i = i0 + j;
        cudaSetDevice(dev);
        char *w = (char *)work + i * per;
        // symmetric input: row-major G is its own column-major transpose; the
        // eigenvectors come back column-major, i.e. as the ROWS of the
        // row-major (n, n) block, ascending eigenvalues
        if (cudaStreamWaitEvent(c->s[j], c->fork, 0) != cudaSuccess) { rc[j] = 1; return; }
        if (cusolverDnDsyevd(c->h[j], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n,
                             G + i * n * n, (int)n, evals + i * n, (double *)w, lwork,
                             (int *)(w + per - 256)) != CUSOLVER_STATUS_SUCCESS) {
          rc[j] = 2;
          return;
        }
        if (cudaEventRecord(c->join[j], c->s[j]) != cudaSuccess) rc[j] = 3;
      });
    }
    for (int j = 0; j < k; ++j) th[j].join();
    for (int j = 0; j < k; ++j) {
      if (rc[j]) return fail(RS_ERR_CUDA, "rs_eigh: syevd step %d failed on matrix %lld", rc[j],
                             (long long)(i0 + j));
      g_launches.fetch_add(1, std::memory_order_relaxed);
      if (cudaStreamWaitEvent(s, c->join[j], 0) != cudaSuccess)
        return fail(RS_ERR_CUDA, "rs_eigh: join");
    }
    if (i0 + EIGH_SLOTS < m && cudaEventRecord(c->fork, s) != cudaSuccess)
      return fail(RS_ERR_CUDA, "rs_eigh: fork");
  }
  return RS_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------
// Orthonormal basis of the b rows of each (b x n) block by Householder QR
// (cuSOLVER geqrf + orgqr on the column-major n x b view), one host thread
// and stream per matrix: the wide Ritz blocks (b = 192 at C5) where the
// one-CTA CGS2 kernel costs ~86 ms per pass.
namespace rsb {

int64_t orth_qr_workspace_bytes(int64_t m, int64_t b, int64_t n) {
  EighCtx *c = nullptr;
  if (m < 1 || b < 1 || n < b || eigh_ctx(&c)) return -1;
  int l1 = 0, l2 = 0;
  if (cusolverDnDgeqrf_bufferSize(c->h[0], (int)n, (int)b, nullptr, (int)n, &l1) !=
          CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDorgqr_bufferSize(c->h[0], (int)n, (int)b, (int)b, nullptr, (int)n, nullptr,
                                  &l2) != CUSOLVER_STATUS_SUCCESS)
    return -1;
  const int64_t lw = std::max(l1, l2);
  return m * (round_up((lw + b) * 8, 256) + 256);
}

int orth_qr(double *Y, int64_t m, int64_t b, int64_t n, void *work, int64_t work_bytes,
            cudaStream_t s) {
  EighCtx *c = nullptr;
  int st;
  if ((st = eigh_ctx(&c))) return st;
  int l1 = 0, l2 = 0;
  if (cusolverDnDgeqrf_bufferSize(c->h[0], (int)n, (int)b, Y, (int)n, &l1) !=
          CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDorgqr_bufferSize(c->h[0], (int)n, (int)b, (int)b, Y, (int)n, nullptr, &l2) !=
          CUSOLVER_STATUS_SUCCESS)
    return fail(RS_ERR_CUDA, "orth_qr: bufferSize");
  const int lw = std::max(l1, l2);
  const int64_t per = round_up(((int64_t)lw + b) * 8, 256) + 256;
  if (work_bytes < m * per) return fail(RS_ERR_CAPACITY, "orth_qr: workspace too small");
  if (cudaEventRecord(c->fork, s) != cudaSuccess) return fail(RS_ERR_CUDA, "orth_qr: fork");
  int dev = 0;
  cudaGetDevice(&dev);
  for (int64_t i0 = 0; i0 < m; i0 += EIGH_SLOTS) {
    const int k = (int)std::min<int64_t>(EIGH_SLOTS, m - i0);
    int rc[EIGH_SLOTS] = {0, 0, 0};
    std::thread th[EIGH_SLOTS];
    for (int j = 0; j < k; ++j) {
      th[j] = std::thread([&, j] {
        const int64_t i = i0 + j;
        cudaSetDevice(dev);
        double *A = Y + i * b * n;  // rows of the row-major b x n block = columns of n x b
        double *w = (double *)((char *)work + i * per);
        double *tau = w + lw;
        int *info = (int *)((char *)work + i * per + per - 256);
        if (cudaStreamWaitEvent(c->s[j], c->fork, 0) != cudaSuccess) { rc[j] = 1; return; }
        if (cusolverDnDgeqrf(c->h[j], (int)n, (int)b, A, (int)n, tau, w, lw, info) !=
            CUSOLVER_STATUS_SUCCESS) { rc[j] = 2; return; }
        if (cusolverDnDorgqr(c->h[j], (int)n, (int)b, (int)b, A, (int)n, tau, w, lw, info) !=
            CUSOLVER_STATUS_SUCCESS) { rc[j] = 3; return; }
        if (cudaEventRecord(c->join[j], c->s[j]) != cudaSuccess) rc[j] = 4;
      });
    }
    for (int j = 0; j < k; ++j) th[j].join();
    for (int j = 0; j < k; ++j) {
      if (rc[j]) return fail(RS_ERR_CUDA, "orth_qr: step %d failed on matrix %lld", rc[j],
                             (long long)(i0 + j));
      g_launches.fetch_add(2, std::memory_order_relaxed);
      if (cudaStreamWaitEvent(s, c->join[j], 0) != cudaSuccess)
        return fail(RS_ERR_CUDA, "orth_qr: join");
    }
    if (i0 + EIGH_SLOTS < m && cudaEventRecord(c->fork, s) != cudaSuccess)
      return fail(RS_ERR_CUDA, "orth_qr: fork");
  }
  return RS_OK;
}

}  // namespace rsb

// ------------------------------------------------------------------ chain
// The latency-bound long-range chain up to the host's rank decision in one
// host call, enqueued right behind rs_front: shift Grams (DMMA) -> top-b
// eigenpairs -> one packed vector [evals (3 b) | trace (3) | max snap
// displacement | duplicate-node key | occupied x3 count] copied into pinned
// host memory, then `done` recorded.  The host waits on `done` only.
namespace {
__global__ void k_pack_chain(const double *__restrict__ evals, int64_t ne,
                             const double *__restrict__ trace, const double *__restrict__ dmax,
                             const int64_t *__restrict__ dup_key, const int32_t *__restrict__ nb,
                             double *__restrict__ out) {
  for (int64_t i = threadIdx.x; i < ne + 6; i += blockDim.x) {
    double v;
    if (i < ne) v = evals[i];
    else if (i < ne + 3) v = trace[i - ne];
    else if (i == ne + 3) v = *dmax;
    else if (i == ne + 4) v = (double)*dup_key;
    else v = nb ? (double)*nb : 0.0;
    out[i] = v;
  }
}
}  // namespace

extern "C" {
int rs_gram_shifted(const double *table, int64_t ld_table, int64_t n, int64_t R, const double *c,
                    const double *wabs, double *G, void *work, int64_t work_bytes, void *stream);

int rs_chain_eig(const double *table, int64_t ld_table, int64_t n, int64_t R, const double *hist,
                 const double *wabs, double *G, void *gram_work, int64_t gram_work_bytes,
                 int64_t b, int64_t iters, double *evals, double *U, double *trace,
                 void *eig_work, int64_t eig_work_bytes, const double *dmax,
                 const int64_t *dup_key, const int32_t *nb, double *packed_dev,
                 double *packed_host, void *done, void *stream) {
  RS_REQUIRE(table && hist && wabs && G && evals && U && trace && dmax && dup_key && packed_dev &&
                 packed_host && done,
             "rs_chain_eig: bad arguments");
  cudaStream_t s = as_stream(stream);
  int st;
  if ((st = rs_gram_shifted(table, ld_table, n, R, hist, wabs, G, gram_work, gram_work_bytes,
                            stream)))
    return st;
  if ((st = rs_topeig(G, 3, n, b, iters, evals, U, trace, eig_work, eig_work_bytes, stream)))
    return st;
  k_pack_chain<<<1, 128, 0, s>>>(evals, 3 * b, trace, dmax, dup_key, nb, packed_dev);
  if ((st = check_launch("pack chain"))) return st;
  cudaError_t e = cudaMemcpyAsync(packed_host, packed_dev, (size_t)(3 * b + 6) * 8,
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaEventRecord((cudaEvent_t)done, s);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "rs_chain_eig: %s", cudaGetErrorString(e));
  return RS_OK;
}
}  // extern "C"
