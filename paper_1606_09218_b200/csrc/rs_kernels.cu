// sm_100a kernels + C ABI for the range-separated tensor assembly path.
// Declarations and the mapping to the reference functions: include/rs_b200.h.
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "rs_common.cuh"
#include "rs_dmma.cuh"
#include "rs_fused.cuh"

namespace rsb {
thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_pool;
std::mutex g_prof_mu;
bool g_prof_on = false;

// ===================================================================== snap
__global__ void k_snap(const double *__restrict__ pos, int64_t count, double h, int64_t n,
                       int64_t *__restrict__ idx, double *__restrict__ disp,
                       int64_t *__restrict__ key, double *__restrict__ snapped_out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= count) return;
  const double half = (double)(n / 2);
  double sq[3];
  int64_t ii[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    double x = pos[3 * p + l];
    double f = __dsub_rn(__dadd_rn(__ddiv_rn(x, h), half), 0.5);
    int64_t i = (int64_t)ceil(f);
    i = i < 1 ? 1 : (i > n - 1 ? n - 1 : i);
    idx[3 * p + l] = i;
    ii[l] = i;
    double snapped = __dmul_rn(__dsub_rn((double)i, half), h);
    if (snapped_out) snapped_out[3 * p + l] = snapped;
    double d = __dsub_rn(x, snapped);
    sq[l] = __dmul_rn(d, d);
  }
  disp[p] = __dsqrt_rn(__dadd_rn(__dadd_rn(sq[0], sq[1]), sq[2]));
  if (key) key[p] = (ii[2] * n + ii[1]) * n + ii[0];  // node key, x3-major
}

// After the key sort: copies in bucket order (c1, c2 int32, charges), window
// starts n - idx, the first duplicated node key (or -1) and the max snap
// displacement (as ordered bits of a non-negative double) -- deterministic.
__global__ void k_prep(const int64_t *__restrict__ ks, const int64_t *__restrict__ order,
                       const int64_t *__restrict__ idx, const double *__restrict__ z,
                       const double *__restrict__ disp, int64_t count, int64_t n,
                       int32_t *__restrict__ c1s, int32_t *__restrict__ c2s,
                       double *__restrict__ zqs, int64_t *__restrict__ starts,
                       unsigned long long *__restrict__ dup_pos,
                       unsigned long long *__restrict__ dmax_bits) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t p = order[i];
  c1s[i] = (int32_t)idx[3 * p];
  c2s[i] = (int32_t)idx[3 * p + 1];
  zqs[i] = z[p];
#pragma unroll
  for (int l = 0; l < 3; ++l) starts[3 * i + l] = n - idx[3 * i + l];
  if (i + 1 < count && ks[i] == ks[i + 1]) atomicMin(dup_pos, (unsigned long long)i);
  atomicMax(dmax_bits, (unsigned long long)__double_as_longlong(disp[i]));
}

// dup_pos -> duplicated node key (or -1), as int64 in place (one thread)
__global__ void k_prep_finish(const int64_t *__restrict__ ks, int64_t count,
                              unsigned long long *__restrict__ dup_pos) {
  const unsigned long long p = *dup_pos;
  *reinterpret_cast<long long *>(dup_pos) = p < (unsigned long long)count ? (long long)ks[p] : -1LL;
}

// ======================================================== window gather (K1)
__global__ void k_gather(const double *__restrict__ table, int64_t ld_table, int64_t n_rows,
                         const int64_t *__restrict__ starts, int64_t n_groups, int64_t n_terms,
                         int64_t term0, const double *__restrict__ gscale,
                         const double *__restrict__ tscale, double *__restrict__ out,
                         int64_t ld_out) {
  const int64_t cols = n_groups * n_terms;
  const int64_t total = n_rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, col = e - i * cols;
    int64_t g = col / n_terms, k = col - g * n_terms;
    double v = table[(starts[g] + i) * ld_table + term0 + k];
    if (gscale) v *= gscale[g];
    if (tscale) v *= tscale[k];
    out[i * ld_out + col] = v;
  }
}

// Shift-merged Gram operands of the three modes in one launch, occupied
// shifts only (empty shifts are zero columns of the reference's A):
// X[l][i][j*R + k] = sqrt(c[l][s]) |w_k| T[(s + i)*ld + k],  s = j-th occupied
// shift.  The shift list is built per block: block (i, l) scans
// the occupancy of mode l's histogram (fixed order, so every block of the
// mode gets the same list), then writes row i of X_l over the occupied shifts
// only; block (0, l) publishes kdev[l] = (occupied shifts) R, the K the
// SYRK re-slices in-kernel (C2: 50 of 256 shifts occupied).
__global__ void __launch_bounds__(256)
    k_gram_operands_rows(const double *__restrict__ table, int64_t ld_table, int64_t n,
                         int64_t R, const double *__restrict__ c,
                         const double *__restrict__ wabs, int32_t *__restrict__ kdev,
                         double *__restrict__ X, int64_t ldx) {
  extern __shared__ int32_t s_list[];  // n
  __shared__ int32_t wocc[8];
  __shared__ int32_t carry;
  const int64_t i = blockIdx.x;
  const int l = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double *cl = c + (int64_t)l * n;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t x = base + tid;
    const int32_t occ = (x < n && cl[x] != 0.0) ? 1 : 0;
    int32_t so = occ;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, so, o);
      if (lane >= o) so += t;
    }
    if (lane == 31) wocc[warp] = so;
    __syncthreads();
    int32_t po = carry;
    for (int w = 0; w < warp; ++w) po += wocc[w];
    if (occ) s_list[po + so - 1] = (int32_t)x;
    __syncthreads();
    if (tid == blockDim.x - 1) carry = po + so;
    __syncthreads();
  }
  const int64_t cols = (int64_t)carry * R;
  if (i == 0 && tid == 0) kdev[l] = (int32_t)cols;
  double *xr = X + ((int64_t)l * n + i) * ldx;
  for (int64_t col = tid; col < cols; col += blockDim.x) {
    const int64_t j = col / R, k = col - j * R;
    const int64_t sft = s_list[j];
    xr[col] = sqrt(cl[sft]) * wabs[k] * table[(sft + i) * ld_table + k];
  }
}

// effective K slices of a mode with K = kl columns: at least 64 columns each
__device__ __forceinline__ void syrk_slices(int64_t kl, int64_t sp_max, int64_t &sp, int64_t &ks) {
  sp = min(sp_max, max((int64_t)1, (kl + 63) / 64));
  ks = ((kl + sp - 1) / sp + 15) / 16 * 16;
}

// ============================================================ GEMM kernels
using TilePlane = Tile<128, 64, 32, 32, 3>;  // plane GEMM / generic NT GEMM
using TileSyrk = Tile<64, 64, 32, 32, 3>;    // Gram (square tiles)
// narrow x3 tiles for the short-range plane GEMM: the per-term bands add the
// tile width to every term's support, so narrow terms cost ~half with BN = 32
using TilePlaneN = Tile<128, 32, 32, 32, 3>;
// wide x3 tiles: fewer column tiles re-read each D row block (A traffic ~ tiles x (BN + 2 gamma))
using TilePlaneW = Tile<128, 128, 32, 32, 3>;
using TilePlane4 = Tile<128, 64, 32, 32, 4>;   // deeper cp.async ring
using TilePlaneM = Tile<128, 64, 64, 32, 3>;   // 64x32 warp tiles (fewer LDS per DMMA)
constexpr int PLANE_MIN_BN = 32;  // sizes the per-column-tile workspace tables

// C[m0.., n0..] = sum over the K ranges of this column tile of A B^T.
// ranges: per column tile, nr (lo, hi) pairs; NULL => single range [0, K).
template <class T, bool ACC>
__global__ void __launch_bounds__(T::THREADS)
    k_gemm_nt(const double *__restrict__ A, int64_t lda, const double *__restrict__ B, int64_t ldb,
              double *__restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K,
              const int64_t *__restrict__ ranges, int nr) {
  extern __shared__ __align__(16) double smem[];
  const int64_t n0 = (int64_t)blockIdx.x * T::BN;  // x: column tile (adjacent CTAs share A rows)
  const int64_t m0 = (int64_t)blockIdx.y * T::BM;
  Acc<T> acc;
  acc.zero();
  if (ranges) {
    for (int r = 0; r < nr; ++r) {
      int64_t lo = ranges[(blockIdx.x * nr + r) * 2], hi = ranges[(blockIdx.x * nr + r) * 2 + 1];
      mainloop<T>(smem, acc, A, lda, m0, M, B, ldb, n0, N, lo, hi);
    }
  } else {
    mainloop<T>(smem, acc, A, lda, m0, M, B, ldb, n0, N, 0, K);
  }
  store_tile<T, ACC>(acc, C, ldc, m0, M, n0, N);
}

__device__ __forceinline__ void tri_decode(int64_t t, int64_t &bi, int64_t &bj) {
  int64_t i = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  bi = i;
  bj = t - i * (i + 1) / 2;
}

// Lower-triangle Gram tiles, one K slice per blockIdx.y, partials to `part`.
__global__ void __launch_bounds__(TileSyrk::THREADS)
    k_syrk_part(const double *__restrict__ A, int64_t lda, int64_t n, int64_t K, int64_t kslice,
                double *__restrict__ part, int64_t a_stride, int64_t part_stride,
                const int32_t *__restrict__ kdev) {
  using T = TileSyrk;
  extern __shared__ __align__(16) double smem[];
  A += blockIdx.z * a_stride;
  part += blockIdx.z * part_stride;
  if (kdev) {  // K known on the device only: re-slice it over the first sp splits
    int64_t sp;
    K = kdev[blockIdx.z];
    syrk_slices(K, gridDim.y, sp, kslice);
    if (blockIdx.y >= sp) return;
  }
  int64_t bi, bj;
  tri_decode(blockIdx.x, bi, bj);
  const int64_t k_lo = (int64_t)blockIdx.y * kslice;
  const int64_t k_hi = k_lo + kslice < K ? k_lo + kslice : K;
  Acc<T> acc;
  acc.zero();
  mainloop<T>(smem, acc, A, lda, bi * T::BM, n, A, lda, bj * T::BN, n, k_lo, k_hi);
  double *dst = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (T::BM * T::BN);
  store_tile<T, false>(acc, dst, T::BN, 0, T::BM, 0, T::BN);
}

__global__ void k_syrk_reduce(const double *__restrict__ part, int64_t splits, int64_t ntiles,
                              int64_t n, double *__restrict__ G, int64_t part_stride,
                              const int32_t *__restrict__ kdev) {
  using T = TileSyrk;
  const int64_t per = T::BM * T::BN;
  part += blockIdx.z * part_stride;
  G += blockIdx.z * n * n;
  if (kdev) {
    int64_t ks;
    syrk_slices(kdev[blockIdx.z], splits, splits, ks);
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ntiles * per;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e / per, loc = e - t * per;
    int64_t bi, bj;
    tri_decode(t, bi, bj);
    int64_t r = bi * T::BM + loc / T::BN, c = bj * T::BN + loc % T::BN;
    if (r >= n || c >= n || c > r) continue;
    double s = 0.0;
    for (int64_t sp = 0; sp < splits; ++sp) s += part[(sp * ntiles + t) * per + loc];
    G[r * n + c] = s;
    G[c * n + r] = s;
  }
}

// ===================================================== shift projection (K4a)
// Block = (32 consecutive shifts, one term k); the table window T[s0 : s0+32+n, k]
// is staged in shared memory and every thread (a, s) streams Z[:, a].
constexpr int SP_SHIFTS = 32;
constexpr int SP_ICH = 64;  // Z rows staged per round

struct Proj3 {
  const double *Z[3];
  double *TT[3];
  int64_t r[3];
};

__global__ void __launch_bounds__(256)
    k_shift_project(Proj3 pj, int64_t n, const double *__restrict__ T, int64_t ld_table, int64_t R,
                    int64_t n_shift) {
  const double *__restrict__ Z = pj.Z[blockIdx.z];
  double *__restrict__ TT = pj.TT[blockIdx.z];
  const int64_t r = pj.r[blockIdx.z], ldz = r;
  extern __shared__ double win[];      // n + SP_SHIFTS, then SP_ICH * r
  double *zs = win + n + SP_SHIFTS;
  const int64_t s0 = (int64_t)blockIdx.x * SP_SHIFTS;
  const int64_t k = blockIdx.y;
  const int64_t len = n + SP_SHIFTS;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    int64_t row = s0 + e;
    win[e] = row < 2 * n ? T[row * ld_table + k] : 0.0;
  }
  // thread -> (a-slot, shift); up to 4 a values per thread
  const int sl = threadIdx.x % SP_SHIFTS, a0 = threadIdx.x / SP_SHIFTS;  // a0 < 8
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t a_base = 0; a_base < r; a_base += 32) {
    for (int u = 0; u < 4; ++u) acc[u] = 0.0;
    for (int64_t i0 = 0; i0 < n; i0 += SP_ICH) {
      const int64_t ni = n - i0 < SP_ICH ? n - i0 : SP_ICH;
      __syncthreads();
      for (int64_t e = threadIdx.x; e < ni * 32; e += blockDim.x) {
        int64_t ii = e / 32, aa = a_base + e % 32;
        zs[e] = aa < r ? Z[(i0 + ii) * ldz + aa] : 0.0;
      }
      __syncthreads();
      const double *w = win + sl + i0;
      for (int64_t ii = 0; ii < ni; ++ii) {
        const double wv = w[ii];
        const double *zr = zs + ii * 32 + a0;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = fma(zr[8 * u], wv, acc[u]);
      }
    }
    const int64_t s = s0 + sl;
    if (s < n_shift) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int64_t a = a_base + a0 + 8 * u;
        if (a < r) TT[(a * n_shift + s) * R + k] = acc[u];
      }
    }
  }
}

// The projections are read only at the shifts the particles occupy (mode l:
// n - c_l of some particle; C5: ~360 of 2048).  k_shift_flags marks them,
// k_shift_compact lists them in ascending order (one block per mode), and
// k_shift_project_list is k_shift_project over 32 consecutive LISTED shifts:
// its table window spans first..last listed shift + n rows (<= 2n).
__device__ __forceinline__ int block_exclusive_scan(int v, int *wsum, int *total);

__global__ void k_shift_flags(const int64_t *__restrict__ shift, int64_t count, int64_t n,
                              int *__restrict__ flags) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 3 * count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sft = shift[e];
    if (sft >= 0 && sft < n) flags[(e % 3) * n + sft] = 1;
  }
}

__global__ void __launch_bounds__(1024)
    k_shift_compact(const int *__restrict__ flags, int64_t n, int *__restrict__ list,
                    int *__restrict__ cnt) {
  __shared__ int wsum[32];
  const int l = blockIdx.x;
  int base = 0;
  for (int64_t s0 = 0; s0 < n; s0 += 1024) {
    const int64_t sft = s0 + threadIdx.x;
    const int f = sft < n ? flags[l * n + sft] : 0;
    int tot;
    const int pos = block_exclusive_scan(f, wsum, &tot);
    if (f) list[l * n + base + pos] = (int)sft;
    base += tot;
  }
  if (threadIdx.x == 0) cnt[l] = base;
}

__global__ void __launch_bounds__(256)
    k_shift_project_list(Proj3 pj, int64_t n, const double *__restrict__ T, int64_t ld_table,
                         int64_t R, int64_t n_shift, const int *__restrict__ list,
                         const int *__restrict__ cnt) {
  const int l = blockIdx.z;
  const int m = cnt[l];
  const int j0 = blockIdx.x * SP_SHIFTS;
  if (j0 >= m) return;
  const double *__restrict__ Z = pj.Z[l];
  double *__restrict__ TT = pj.TT[l];
  const int64_t r = pj.r[l], ldz = r;
  extern __shared__ double win[];      // up to 2n, then SP_ICH * 32
  const int *ls = list + (int64_t)l * n;
  const int nsh = min(SP_SHIFTS, m - j0);
  const int64_t s_first = ls[j0], s_last = ls[j0 + nsh - 1];
  const int64_t len = s_last - s_first + n;
  double *zs = win + 2 * n;
  const int64_t k = blockIdx.y;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    const int64_t row = s_first + e;
    win[e] = row < 2 * n ? T[row * ld_table + k] : 0.0;
  }
  const int sl = threadIdx.x % SP_SHIFTS, a0 = threadIdx.x / SP_SHIFTS;  // a0 < 8
  const int64_t sft = sl < nsh ? ls[j0 + sl] : s_first;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t a_base = 0; a_base < r; a_base += 32) {
    for (int u = 0; u < 4; ++u) acc[u] = 0.0;
    for (int64_t i0 = 0; i0 < n; i0 += SP_ICH) {
      const int64_t ni = n - i0 < SP_ICH ? n - i0 : SP_ICH;
      __syncthreads();
      for (int64_t e = threadIdx.x; e < ni * 32; e += blockDim.x) {
        int64_t ii = e / 32, aa = a_base + e % 32;
        zs[e] = aa < r ? Z[(i0 + ii) * ldz + aa] : 0.0;
      }
      __syncthreads();
      const double *w = win + (sft - s_first) + i0;
      for (int64_t ii = 0; ii < ni; ++ii) {
        const double wv = w[ii];
        const double *zr = zs + ii * 32 + a0;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = fma(zr[8 * u], wv, acc[u]);
      }
    }
    if (sl < nsh && sft < n_shift) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int64_t a = a_base + a0 + 8 * u;
        if (a < r) TT[(a * n_shift + sft) * R + k] = acc[u];
      }
    }
  }
}

// Per-mode shift histograms c[l][s] = sum_{p: n - idx[p][l] == s} z_p^2 and
// the x3 occupancy counts cnt[x] = #{p: idx[p][2] == x}.  Warp per (mode, s):
// lanes stride the particles (staged in shared memory, shared by the block's
// 8 warps), then a fixed shuffle tree -- deterministic.
constexpr int SH_CHUNK = 2048;

__global__ void __launch_bounds__(256)
    k_shift_hist(const int64_t *__restrict__ idx, const double *__restrict__ z, int64_t count,
                 int64_t n, double *__restrict__ c, int32_t *__restrict__ cnt3) {
  __shared__ int32_t key[SH_CHUNK];
  __shared__ double zz[SH_CHUNK];
  const int l = blockIdx.y;                      // mode
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * 8 + warp;
  double acc = 0.0;
  int32_t occ = 0;
  for (int64_t p0 = 0; p0 < count; p0 += SH_CHUNK) {
    const int m = (int)(count - p0 < SH_CHUNK ? count - p0 : SH_CHUNK);
    __syncthreads();
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
      key[e] = (int32_t)(n - idx[3 * (p0 + e) + l]);
      const double q = z[p0 + e];
      zz[e] = q * q;
    }
    __syncthreads();
    if (s < n) {
      for (int e = lane; e < m; e += 32) {
        const bool hit = key[e] == (int32_t)s;
        acc += hit ? zz[e] : 0.0;
        occ += (l == 2 && key[e] == (int32_t)(n - s)) ? 1 : 0;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    occ += __shfl_xor_sync(0xffffffffu, occ, o);
  }
  if (s < n && lane == 0) {
    c[(int64_t)l * n + s] = acc;
    if (l == 2) cnt3[s] = occ;
  }
}

// ============================================================ RHOSVD core (K4b)
// P_l[a][p*R + k] = TT_l[(a*n_shift + shift[3p+l])*R + k], mode 0 scaled by z_p w_k:
// the projected side matrices Z_l^T U_l (rankred.py:175) of the shift-structured
// long part, materialised once for the Khatri-Rao core GEMM.
__global__ void k_core_gather(const double *__restrict__ TT, int r, int64_t n_shift, int R,
                              const int64_t *__restrict__ shift, int l, const double *__restrict__ z,
                              const double *__restrict__ w, int64_t count, double *__restrict__ P) {
  const int64_t K = count * R;
  const int64_t total = (int64_t)r * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e / K, col = e - a * K;
    const int64_t p = col / R;
    const int k = (int)(col - p * R);
    double v = TT[(a * n_shift + shift[3 * p + l]) * R + k];
    if (l == 0) v *= z[p] * w[k];
    P[e] = v;
  }
}

// core[(a*r2+b), c] = sum_K P1[a,K] P2[b,K] P3[c,K] as a DMMA GEMM whose A tile is
// the Khatri-Rao product generated on the fly (never materialised); split-K
// partials reduced in fixed order by k_split_reduce.
using TileCore = Tile<128, 64, 32, 32, 2>;

__global__ void __launch_bounds__(TileCore::THREADS)
    k_core_kr(const double *__restrict__ P1, const double *__restrict__ P2,
              const double *__restrict__ P3, int r2, int64_t M, int64_t N, int64_t K,
              int64_t kslice, double *__restrict__ part) {
  using T = TileCore;
  __shared__ __align__(16) double sA[T::BM * T::LDS];
  __shared__ __align__(16) double sB[T::BN * T::LDS];
  const int64_t m0 = (int64_t)blockIdx.x * T::BM, n0 = (int64_t)blockIdx.y * T::BN;
  const int64_t k_lo = (int64_t)blockIdx.z * kslice;
  const int64_t k_hi = k_lo + kslice < K ? k_lo + kslice : K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / T::WARPS_N) * T::WM, wn0 = (warp % T::WARPS_N) * T::WN;
  const int gid = lane >> 2, tig = lane & 3;
  Acc<T> acc;
  acc.zero();
  // register double buffer: the next chunk's Khatri-Rao and P3 values are
  // fetched from L2 while the current chunk's DMMAs run
  constexpr int EA = T::BM * T::BK / T::THREADS, EB = T::BN * T::BK / T::THREADS;
  double ra[EA], rb[EB];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < EA; ++u) {
      const int e = threadIdx.x + u * T::THREADS;
      const int rr = e / T::BK, kk = e % T::BK;
      const int64_t row = m0 + rr, k = k0 + kk;
      double v = 0.0;
      if (row < M && k < k_hi) {
        const int64_t a = row / r2, b = row - a * r2;
        v = P1[a * K + k] * P2[b * K + k];
      }
      ra[u] = v;
    }
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int e = threadIdx.x + u * T::THREADS;
      const int rr = e / T::BK, kk = e % T::BK;
      const int64_t c = n0 + rr, k = k0 + kk;
      rb[u] = (c < N && k < k_hi) ? P3[c * K + k] : 0.0;
    }
  };
  if (k_lo < k_hi) fetch(k_lo);
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += T::BK) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < EA; ++u) {
      const int e = threadIdx.x + u * T::THREADS;
      sA[(e / T::BK) * T::LDS + e % T::BK] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int e = threadIdx.x + u * T::THREADS;
      sB[(e / T::BK) * T::LDS + e % T::BK] = rb[u];
    }
    __syncthreads();
    if (k0 + T::BK < k_hi) fetch(k0 + T::BK);
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
  store_tile<T, false>(acc, part + (int64_t)blockIdx.z * M * N, N, m0, M, n0, N);
}

__global__ void k_split_reduce(const double *__restrict__ part, int64_t splits, int64_t len,
                               double *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t sp = 0; sp < splits; ++sp) s += part[sp * len + e];
    out[e] = s;
  }
}

// ===================================================== grid assembly (K5)
// Yt[x1l, c, b] = sum_a V1[x1, a] core[a, b, c], zero-padded to (r3p, r2p): the
// B operand of the per-plane DMMA GEMM A[(x1l, x2), c] = sum_b V2[x2, b] Yt[x1l, c, b]
__global__ void k_tucker_yt(const double *__restrict__ core, int r1, int r2, int r3,
                            const double *__restrict__ V1, int64_t x1_lo, int r2p, int r3p,
                            int64_t planes, double *__restrict__ Yt) {
  const int64_t total = planes * r3p * r2p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e % r2p);
    const int64_t q = e / r2p;
    const int c = (int)(q % r3p);
    const int64_t x1l = q / r3p;
    double acc = 0.0;
    if (b < r2 && c < r3) {
      const double *v = V1 + (x1_lo + x1l) * r1;
      for (int a = 0; a < r1; ++a) acc = fma(v[a], core[((int64_t)a * r2 + b) * r3 + c], acc);
    }
    Yt[e] = acc;
  }
}

// coreT[(c r2p + b) r1p + a] = core[a, b, c] (zero-padded): the B operand of
// Yt[x1, (c, b)] = sum_a V1[x1, a] core[a, b, c] as one DMMA GEMM (large ranks)
__global__ void k_core_t(const double *__restrict__ core, int r1, int r2, int r3, int r1p,
                         int r2p, int r3p, double *__restrict__ coreT) {
  const int64_t total = (int64_t)r3p * r2p * r1p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e % r1p);
    const int64_t q = e / r1p;
    const int b = (int)(q % r2p), c = (int)(q / r2p);
    coreT[e] = (a < r1 && b < r2 && c < r3) ? core[((int64_t)a * r2 + b) * r3 + c] : 0.0;
  }
}

// V2p = V2 (n x r2) with columns zero-padded to r2p (16-byte aligned K rows)
__global__ void k_pad_cols(const double *__restrict__ V, int64_t n, int r, int rp,
                           double *__restrict__ Vp) {
  const int64_t total = n * rp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / rp;
    const int c = (int)(e - i * rp);
    Vp[e] = c < r ? V[i * r + c] : 0.0;
  }
}

constexpr int SR_MAXR = 24;  // largest short rank R_s of the row builder
#define SR_MAXR_DEV 24

__device__ __forceinline__ int block_exclusive_scan(int v, int *wsum, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int base = 0, tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (w < warp) base += wsum[w];
    tot += wsum[w];
  }
  *total = tot;
  __syncthreads();
  return base + x - v;
}

// Short-range rows on FP64 tensor cores.  For a bucket b and rank term k the
// (x1, x2) panel of D is a sum of rank-1 window products,
//   D_bk[x1, x2] = sum_{p in b} (zq_p wl_k ul[x1-c1p+g, k]) * ul[x2-c2p+g, k],
// i.e. a GEMM over the bucket's copies.  A CTA owns an 8-plane x 64-row tile
// and SD_BG consecutive buckets; each warp owns 8 rows and issues
// mma.m8n8k4.f64 with m = planes, n = rows, k = 4 copies, holding all R_s
// accumulators in registers.  The buckets' copies are one contiguous candidate
// range (x3-major node order); each pass stages 256 candidates, keeps those
// whose window meets the tile (block scan, order preserving, so each bucket's
// survivors stay contiguous) and runs the MMAs bucket by bucket; a bucket that
// straddles two passes keeps its accumulators.  Window factors are gathered
// from shared memory with clamped indices and a validity mask.
constexpr int SD_THREADS = 256;
constexpr int RB_ROWS = 128;  // row block of the plane GEMM's term table (TilePlane::BM)
constexpr int SD_TX1 = 8;    // planes per tile (MMA m)
constexpr int SD_TX2 = 64;   // rows per tile (8 warps x MMA n)
constexpr int SD_BG = 8;     // buckets per CTA
constexpr int SD_PADA = SD_TX1;  // plane offsets stay within [-TX1, W + TX1)
constexpr int SD_PADB = SD_TX2;  // row offsets stay within [-TX2, W + TX2)

// (two CTAs per SM at R_s <= 14 -- 128 registers -- measured no faster)
template <int GK>
__global__ void __launch_bounds__(SD_THREADS)
    k_short_dmma(const double *__restrict__ ul, const double *__restrict__ wl, int Rs, int G,
                 int gamma, const int32_t *__restrict__ c1, const int32_t *__restrict__ c2,
                 const double *__restrict__ zq, const int32_t *__restrict__ bstart,
                 const int32_t *__restrict__ nbp, int64_t n, int64_t x1_lo, int64_t planes,
                 double *__restrict__ A, int64_t lda, int64_t col0,
                 const int *__restrict__ kofd, const uint8_t *__restrict__ kr, int64_t ldk) {
  extern __shared__ double sm[];
  const int W = 2 * gamma + 1;
  constexpr int P = GK + 1;  // odd pitch (doubles): conflict-light row gathers
  const int WA = W + 2 * SD_PADA, WB = W + 2 * SD_PADB;
  double *uA = sm;                      // WA x P : wl_k ul[d, k], zero padded
  double *uB = uA + (int64_t)WA * P;    // WB x P : ul[d, k], zero padded
  double *szq = uB + (int64_t)WB * P;   // staged charges (SD_THREADS + 4)
  int *sc1 = (int *)(szq + SD_THREADS + 4);
  int *sc2 = sc1 + SD_THREADS + 4;
  int *sbk = sc2 + SD_THREADS + 4;     // staged copy -> local bucket
  int *wsum = sbk + SD_THREADS + 4;    // 32
  int *skofd = wsum + 32;              // gamma + 1: terms alive at (x1, x2) distance d
  __shared__ int s_bst[SD_BG + 1];     // bucket offsets in the candidate list
  __shared__ int s_slo[SD_BG + 1];     // bucket starts within the staged list
  __shared__ int s_plo[SD_BG];         // first candidate copy of each bucket
  const int nb = *nbp;
  const int b0 = blockIdx.z * SD_BG;
  if (b0 >= nb) return;
  const int nbk = min(SD_BG, nb - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t y0 = (int64_t)blockIdx.x * SD_TX2;
  const int64_t x1l0 = (int64_t)blockIdx.y * SD_TX1;
  const int64_t X0 = x1_lo + x1l0;
  for (int e = tid; e < (WA + WB) * P; e += SD_THREADS) uA[e] = 0.0;  // k >= Rs rows stay zero
  for (int d = tid; d <= gamma; d += SD_THREADS) skofd[d] = kofd ? kofd[d] : GK;
  __syncthreads();
  for (int e = tid; e < Rs * W; e += SD_THREADS) {  // coalesced read of ul (W x Rs)
    const int d = e / Rs, k = e - (e / Rs) * Rs;
    const double u = ul[e];
    uA[(d + SD_PADA) * P + k] = wl[k] * u;
    uB[(d + SD_PADB) * P + k] = u;
  }
  const int64_t yw = y0 + warp * 8;
  const int ar = lane >> 2, kq = lane & 3;  // fragment row (plane / row) and k slot
  const int64_t c1lo = X0 - gamma, c1hi = X0 + SD_TX1 - 1 + gamma;
  const int64_t c2lo = y0 - gamma, c2hi = y0 + SD_TX2 - 1 + gamma;
  if (tid < nbk) {  // per bucket: the copies whose x2 window meets the tile (c2 ascending)
    const int p_lo = bstart[b0 + tid], p_hi = bstart[b0 + tid + 1];
    int lo = p_lo, hi = p_hi;
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (c2[m] < c2lo) lo = m + 1; else hi = m;
    }
    int e = lo;
    hi = p_hi;
    while (e < hi) {
      const int m = (e + hi) >> 1;
      if (c2[m] <= c2hi) e = m + 1; else hi = m;
    }
    s_plo[tid] = lo;
    s_bst[tid + 1] = e - lo;
  }
  __syncthreads();
  if (tid == 0) {  // candidate offsets of the buckets in the concatenated c2 ranges
    s_bst[0] = 0;
    for (int j = 0; j < nbk; ++j) s_bst[j + 1] += s_bst[j];
  }
  __syncthreads();
  const int V = s_bst[nbk];
  double acc[GK][2];
#pragma unroll
  for (int k = 0; k < GK; ++k) acc[k][0] = acc[k][1] = 0.0;
  int jb = 0;  // first bucket not yet stored
  for (int cs = 0; cs < V; cs += SD_THREADS) {
    const int v = cs + tid;
    bool cov = false;
    int bk = 0, p = 0;
    if (v < V) {
      while (bk + 1 < nbk && s_bst[bk + 1] <= v) ++bk;
      p = s_plo[bk] + (v - s_bst[bk]);
      const int64_t a1 = c1[p];
      cov = a1 >= c1lo && a1 <= c1hi;
    }
    int tot;
    const int pos = block_exclusive_scan(cov ? 1 : 0, wsum, &tot);
    if (cov) {
      sc1[pos] = c1[p];
      sc2[pos] = c2[p];
      szq[pos] = zq[p];
      sbk[pos] = bk;
    }
    if (tid < 4) {  // guard entries: an MMA k-step may run past a bucket's end
      szq[tot + tid] = 0.0;
      sc1[tot + tid] = (int)X0;
      sc2[tid + tot] = (int)y0;
      sbk[tot + tid] = nbk;
    }
    __syncthreads();
    if (tid <= nbk) {  // first staged index of local bucket tid (sbk ascending)
      int lo = 0, hi = tot;
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (sbk[m] < tid) lo = m + 1; else hi = m;
      }
      s_slo[tid] = lo;
    }
    __syncthreads();
    const int cend = cs + SD_THREADS;
    for (int j = jb; j < nbk && s_bst[j] < cend; ++j) {
      const int q_lo = s_slo[j], q_hi = s_slo[j + 1];
#pragma unroll 2
      for (int q0 = q_lo; q0 < q_hi; q0 += 4) {
        // staged copies meet the tile, so both offsets land inside the padding;
        // slots past the bucket's end carry z = 0
        const int q = q0 + kq;
        const double z = q < q_hi ? szq[q] : 0.0;
        const int a1 = sc1[q], a2 = sc2[q];
        const double *pa = uA + ((int)(X0 + ar - a1) + gamma + SD_PADA) * P;
        const double *pb = uB + ((int)(yw + ar - a2) + gamma + SD_PADB) * P;
        // terms alive for this warp's 8 planes x 8 rows: kofd at the Chebyshev
        // distance of each of the 4 copies, max over them (warp-uniform); the
        // narrow terms of far copies are below RS_TERM_DROP there
        int kw = 0;
        if (q < q_hi) {
          const int dx = max(0, max((int)X0 - a1, a1 - (int)X0 - (SD_TX1 - 1)));
          const int dy = max(0, max((int)yw - a2, a2 - (int)yw - 7));
          const int d = max(dx, dy);
          kw = d <= gamma ? skofd[d] : 0;
        }
        kw = max(kw, __shfl_xor_sync(0xffffffffu, kw, 1));
        kw = max(kw, __shfl_xor_sync(0xffffffffu, kw, 2));
#pragma unroll
        for (int k = 0; k < GK; ++k)
          if (k < kw) dmma_884(acc[k], z * pa[k], pb[k]);
      }
      if (s_bst[j + 1] <= cend) {  // bucket complete: store its G-wide row segments
        const int64_t x1l = x1l0 + ar;
        if (x1l < planes) {
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int64_t x2 = yw + 2 * kq + jj;
            if (x2 < n) {
              const int64_t g = x1l * n + x2;
              // only the terms the plane GEMM reads for this row block
              const int kst = kr ? (int)kr[(g / RB_ROWS) * ldk + b0 + j] : GK;
              double *dst = A + g * lda + col0 + (int64_t)(b0 + j) * GK;
#pragma unroll
              for (int k = 0; k < GK; k += 2)
                if (k < kst)
                  *reinterpret_cast<double2 *>(dst + k) = make_double2(acc[k][jj], acc[k + 1][jj]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < GK; ++k) acc[k][0] = acc[k][1] = 0.0;
        jb = j + 1;
      }
    }
    __syncthreads();
  }
  // buckets without candidates after the last pass: zero segments
  const int64_t x1l = x1l0 + ar;
  for (int j = jb; j < nbk; ++j) {
    if (x1l < planes) {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int64_t x2 = yw + 2 * kq + jj;
        if (x2 < n) {
          const int64_t g = x1l * n + x2;
          const int kst = kr ? (int)kr[(g / RB_ROWS) * ldk + b0 + j] : GK;
          double *dst = A + g * lda + col0 + (int64_t)(b0 + j) * GK;
#pragma unroll
          for (int k = 0; k < GK; k += 2)
            if (k < kst) *reinterpret_cast<double2 *>(dst + k) = make_double2(0.0, 0.0);
        }
      }
    }
  }
}

// Per-term supports of the short part -> per-distance prefix widths.  Term k
// can contribute more than RS_TERM_DROP of the largest possible L0 entry only
// within gk[k] cells of its centre,
//   |wl_k ul[g+d,k]| max|ul_k|^2 > RS_TERM_DROP * sum_j |wl_j| max|ul_j|^3,
// and the narrow short-range Gaussians die out long before gamma (C4: 107 for
// the widest term, 1 for the narrowest).  kofd[d] = 1 + max{k : gk[k] >= d}:
// a bucket whose x3 index lies d cells outside a column tile needs only its
// first kofd[d] term columns (terms are ordered widest first).  What is
// dropped is below 1e-18 of max|L0| per (grid point, copy, term).
#define RS_TERM_DROP 1e-18
__global__ void __launch_bounds__(256)
    k_term_prefix(const double *__restrict__ ul, const double *__restrict__ wl, int Rs, int gamma,
                  int *__restrict__ kofd) {
  __shared__ double smx[SR_MAXR_DEV];
  __shared__ int sgk[SR_MAXR_DEV];
  __shared__ double stot;
  const int W = 2 * gamma + 1;
  const int k = threadIdx.x;
  double mx = 0.0;
  if (k < Rs) {
    for (int d = 0; d < W; ++d) mx = fmax(mx, fabs(ul[d * Rs + k]));
    smx[k] = mx;
  }
  __syncthreads();
  if (k == 0) {
    double t = 0.0;
    for (int j = 0; j < Rs; ++j) t += fabs(wl[j]) * smx[j] * smx[j] * smx[j];
    stot = t;
  }
  __syncthreads();
  if (k < Rs) {
    const double thr = RS_TERM_DROP * stot, f = fabs(wl[k]) * mx * mx;
    int g = 0;
    for (int d = gamma; d >= 0; --d)
      if (f * fmax(fabs(ul[(gamma + d) * Rs + k]), fabs(ul[(gamma - d) * Rs + k])) > thr) {
        g = d;
        break;
      }
    sgk[k] = g;
  }
  __syncthreads();
  for (int d = threadIdx.x; d <= gamma; d += blockDim.x) {
    int K = 0;
    for (int j = 0; j < Rs; ++j)
      if (sgk[j] >= d) K = j + 1;
    kofd[d] = K;
  }
}

// The plane GEMM: C[(x1,x2), x3] (=, +=) sum over K of A B^T where, per
// 64-wide x3 column tile, K = the Tucker columns [0, r3p) followed by, for
// every occupied x3 bucket b within gamma of the tile, the first
// kofd[distance] of its G term columns [r3p + b G, ...): per-term bands, so the
// narrow terms cost flops only near their buckets (C2-C4: ~0.5x the flops of
// the full band).  The segments (each rounded to an even width) are packed
// back to back into 16-column chunks of ONE cp.async pipeline: each thread
// always stages the same 2-column pair slot of a chunk, and a cursor walked
// identically by every thread maps the slot to its source column.
// nbp == NULL: Tucker columns only.
// Row-block term table: for GEMM row block rb (BM consecutive (x1, x2) rows of
// the plane range) and bucket b, kr[rb * ldk + b] = the number of leading
// terms that can be nonzero anywhere in that row block = kofd[d12] with d12
// the smallest Chebyshev (x1, x2) distance from the block to a copy of the
// bucket (0: no copy within gamma).  With the x3 distance of the GEMM's
// column tile this gives each (row block, column tile, bucket) its term
// count: the narrow terms only matter next to their copies in all three
// coordinates.  Copies of a bucket are c2-sorted: binary search of the x2
// window, scan of the candidates.
__global__ void k_rowblock_terms(const int32_t *__restrict__ c1, const int32_t *__restrict__ c2,
                                 const int32_t *__restrict__ bstart,
                                 const int32_t *__restrict__ nbp, const int *__restrict__ kofd,
                                 int gamma, int64_t n, int64_t x1_lo, int64_t rows, int BM,
                                 int64_t nrb, int64_t ldk, uint8_t *__restrict__ kr) {
  const int nb = *nbp;
  const int64_t total = nrb * ldk;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rb = e / ldk;
    const int b = (int)(e - rb * ldk);
    if (b >= nb) continue;
    const int64_t r0 = rb * BM, r1 = min(r0 + BM, rows) - 1;
    const int64_t xa = x1_lo + r0 / n, xb = x1_lo + r1 / n;
    const int64_t ya = xa == xb ? r0 % n : 0, yb = xa == xb ? r1 % n : n - 1;
    int l = bstart[b], h = bstart[b + 1];
    const int p_hi = h;
    while (l < h) {
      const int m = (l + h) >> 1;
      if (c2[m] < ya - gamma) l = m + 1; else h = m;
    }
    int64_t best = (int64_t)gamma + 1;
    for (int p = l; p < p_hi; ++p) {
      const int64_t y = c2[p];
      if (y > yb + gamma) break;
      const int64_t x = c1[p];
      const int64_t dx = x < xa ? xa - x : (x > xb ? x - xb : 0);
      const int64_t dy = y < ya ? ya - y : (y > yb ? y - yb : 0);
      const int64_t d = max(dx, dy);
      if (d < best) {
        best = d;
        if (d == 0) break;
      }
    }
    kr[e] = (uint8_t)(best <= gamma ? kofd[best] : 0);
  }
}

// Tucker-only plane GEMM with the A row block resident in shared memory:
//   C[g, x3] (+)= sum_{c < K} A[g, c] Bt[x3, c]   (K = r3p <= TR_KMAX)
// One 256-thread CTA per 128-row block walks ALL column tiles of 64: A (128 x
// K) is staged once, the Bt chunks of every (tile, 16-column K chunk) stream
// through one cp.async ring that never drains between tiles, and the old C
// values of a tile are requested into registers when its first chunk starts
// (their latency hides under the tile's MMAs), so neither the K-loop
// prologue nor the read-modify-write epilogue stalls the DMMA pipe per tile.
// With K ~ 132 (C5) these two bubbles cost the per-tile kernel ~40 % of peak.
namespace tr {
constexpr int BN = 64;
constexpr int WM = 32, WN = 32, WARPS_N = BN / WN, MT = WM / 8, NT = WN / 8;
constexpr int KMAX = 176;
__host__ __device__ constexpr int threads(int bm) { return (bm / WM) * WARPS_N * 32; }
// row pitch of the resident A block: K rounded up to a k-step, then to 4 mod 16
// doubles (conflict-free fragment reads)
__host__ __device__ constexpr int lda_s(int K) {
  int l = (K + 3) / 4 * 4;
  while (l % 16 != 4) l += 4;
  return l;
}
__host__ __device__ constexpr int smem_bytes(int bm, int K, int bk, int stages) {
  return (bm * lda_s(K) + stages * BN * (bk + 4)) * 8;
}
}  // namespace tr

// BM = 128: 8 warps, one CTA per SM; BM = 64: 4 warps, two CTAs per SM
template <int BM, bool ACC, int BK, int STAGES>
__global__ void __launch_bounds__(tr::threads(BM), BM == 64 ? 2 : 1)
    k_tucker_gemm_res(const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                      int64_t ldb, double *__restrict__ C, int64_t ldc, int64_t M, int64_t N,
                      int K) {
  using namespace tr;
  constexpr int THREADS = threads(BM), LDB = BK + 4;
  extern __shared__ __align__(16) double smem[];
  const int KC = (K + BK - 1) / BK, LDA = lda_s(K);
  double *sA = smem;
  double *sB = smem + BM * LDA;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int ntiles = (int)((N + BN - 1) / BN);
  const int total = ntiles * KC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;
  const int gid = lane >> 2, tig = lane & 3;
  // resident A block (zero past K and past M), first commit group with chunk 0
  for (int e = threadIdx.x; e < BM * (LDA / 2); e += THREADS) {
    const int r = e / (LDA / 2), kk = 2 * (e - r * (LDA / 2));
    const int64_t g = m0 + r;
    const bool ok = g < M && kk < K;
    const int bytes = ok ? (kk + 1 < K ? 16 : 8) : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                     smem_addr(sA + r * LDA + kk)),
                 "l"(ok ? A + g * lda + kk : A), "r"(bytes));
  }
  // Bt chunks are requested strictly in order (tile-major, chunk-minor), so the
  // loader keeps running state instead of decoding the chunk index: per thread
  // its SLOTS (row, column-pair) slots are fixed, the source pointers advance by
  // BK per chunk and by BN rows per tile, and only the last chunk of a tile
  // (K not a multiple of BK) and the last tile (N not a multiple of BN) take
  // the predicated path.  (The div/mod version spent ~45 % of the issue slots
  // of this 2-warps-per-scheduler kernel on addressing.)
  constexpr int SLOTS = BN * BK / 2 / THREADS;
  uint32_t sdst[SLOTS];
  const double *src[SLOTS];
#pragma unroll
  for (int u = 0; u < SLOTS; ++u) {
    const int e = u * THREADS + threadIdx.x, r = e / (BK / 2), pr = e % (BK / 2);
    sdst[u] = smem_addr(sB + r * LDB + 2 * pr);
    src[u] = B + (int64_t)r * ldb + 2 * pr;
  }
  int lt = 0, lkc = 0, lst = 0;
  const bool k_even = (K % BK) == 0;
  auto load_next = [&]() {
    const bool fast = (k_even || lkc < KC - 1) && (int64_t)(lt + 1) * BN <= N;
    const uint32_t soff = (uint32_t)(lst * BN * LDB * 8);
    if (fast) {
#pragma unroll
      for (int u = 0; u < SLOTS; ++u)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst[u] + soff),
                     "l"(src[u] + lkc * BK));
    } else {
#pragma unroll
      for (int u = 0; u < SLOTS; ++u) {
        const int e = u * THREADS + threadIdx.x;
        const int r = e / (BK / 2), kk = lkc * BK + 2 * (e % (BK / 2));
        const int64_t g = (int64_t)lt * BN + r;
        const bool ok = g < N && kk < K;
        const int bytes = ok ? (kk + 1 < K ? 16 : 8) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sdst[u] + soff),
                     "l"(ok ? src[u] + lkc * BK : B), "r"(bytes));
      }
    }
    if (++lkc == KC) {
      lkc = 0;
      ++lt;
#pragma unroll
      for (int u = 0; u < SLOTS; ++u) src[u] += (int64_t)BN * ldb;
    }
    if (++lst == STAGES) lst = 0;
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) load_next();
    cp_async_commit();
  }
  double acc[MT][NT][2], cold[MT][NT][2];
  // S k-steps of 4 columns of one staged chunk, fragments of step s+1 loaded
  // while the DMMAs of step s issue (the LDS latency off the tensor pipe)
  auto mma_steps = [&](const double *st, int kc, auto steps_c) {
    constexpr int S = decltype(steps_c)::value;
    double a[2][MT], b[2][NT];
#pragma unroll
    for (int i = 0; i < MT; ++i) a[0][i] = sA[(wm0 + i * 8 + gid) * LDA + kc * BK + tig];
#pragma unroll
    for (int j = 0; j < NT; ++j) b[0][j] = st[(wn0 + j * 8 + gid) * LDB + tig];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (s + 1 < S) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
          a[(s + 1) & 1][i] = sA[(wm0 + i * 8 + gid) * LDA + kc * BK + 4 * (s + 1) + tig];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[(s + 1) & 1][j] = st[(wn0 + j * 8 + gid) * LDB + 4 * (s + 1) + tig];
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_884(acc[i][j], a[s & 1][i], b[s & 1][j]);
    }
  };
  const int ksteps_last = (K - (KC - 1) * BK + 3) / 4;  // live 4-column steps of the last chunk
  int c = 0, cst = 0;
  for (int t = 0; t < ntiles; ++t) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        acc[i][j][0] = acc[i][j][1] = 0.0;
        cold[i][j][0] = cold[i][j][1] = 0.0;
        if (ACC) {
          const int64_t r = m0 + wm0 + i * 8 + gid, col = (int64_t)t * BN + wn0 + j * 8 + tig * 2;
          if (r < M && col + 1 < N) {
            const double2 o = __ldcs(reinterpret_cast<const double2 *>(C + r * ldc + col));
            cold[i][j][0] = o.x;
            cold[i][j][1] = o.y;
          } else if (r < M && col < N) {
            cold[i][j][0] = __ldcs(C + r * ldc + col);
          }
        }
      }
    for (int kc = 0; kc < KC; ++kc, ++c) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (c + STAGES - 1 < total) load_next();
      cp_async_commit();
      const double *st = sB + cst * BN * LDB;
      if (++cst == STAGES) cst = 0;
      const int ks = kc == KC - 1 ? ksteps_last : BK / 4;
      if (ks == BK / 4) {
        mma_steps(st, kc, std::integral_constant<int, BK / 4>{});
      } else {
        switch (ks) {   // live steps of a tile's last chunk
          case 1: mma_steps(st, kc, std::integral_constant<int, 1>{}); break;
          case 2: mma_steps(st, kc, std::integral_constant<int, 2>{}); break;
          case 3: mma_steps(st, kc, std::integral_constant<int, 3>{}); break;
          case 4: if constexpr (BK > 16) mma_steps(st, kc, std::integral_constant<int, 4>{}); break;
          case 5: if constexpr (BK > 16) mma_steps(st, kc, std::integral_constant<int, 5>{}); break;
          case 6: if constexpr (BK > 16) mma_steps(st, kc, std::integral_constant<int, 6>{}); break;
          default: if constexpr (BK > 16) mma_steps(st, kc, std::integral_constant<int, 7>{}); break;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int64_t r = m0 + wm0 + i * 8 + gid;
      if (r >= M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int64_t col = (int64_t)t * BN + wn0 + j * 8 + tig * 2;
        double *p = C + r * ldc + col;
        const double v0 = acc[i][j][0] + cold[i][j][0], v1 = acc[i][j][1] + cold[i][j][1];
        if (col + 1 < N) {
          __stcs(reinterpret_cast<double2 *>(p), make_double2(v0, v1));
        } else if (col < N) {
          __stcs(p, v0);
        }
      }
    }
  }
  cp_async_wait<0>();
}

constexpr int PLANE_SEGS = 1024;  // segments per column tile (1 + occupied x3 in the band)

template <class T, bool ACC>
__global__ void __launch_bounds__(T::THREADS)
    k_gemm_plane(const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                 int64_t ldb, double *__restrict__ C, int64_t ldc, int64_t M, int64_t N,
                 int64_t r3p, int64_t G, const int32_t *__restrict__ bc3,
                 const int32_t *__restrict__ nbp, int gamma, const int *__restrict__ kofd,
                 const uint8_t *__restrict__ kr, int64_t ldk) {
  constexpr int CH = T::BK / 2;                  // 2-column pair slots per chunk row
  static_assert(T::THREADS % CH == 0, "pair slot must be fixed per thread");
  constexpr int ROWS_PER_PASS = T::THREADS / CH;
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_col[PLANE_SEGS], s_len[PLANE_SEGS], s_pp[PLANE_SEGS];
  __shared__ int s_band[2], s_wsum[T::THREADS / 32];
  const int64_t n0 = (int64_t)blockIdx.x * T::BN;
  const int64_t m0 = (int64_t)blockIdx.y * T::BM;
  const int64_t top = min(n0 + T::BN, N) - 1;
  if (threadIdx.x == 0) {
    int a = 0, bb = 0;
    if (nbp) {
      const int nb = *nbp;
      const int64_t lo_x = n0 - gamma, hi_x = top + gamma;
      int l = 0, h = nb;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (bc3[m] < lo_x) l = m + 1; else h = m;
      }
      a = l;
      h = nb;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (bc3[m] <= hi_x) l = m + 1; else h = m;
      }
      bb = l;
    }
    s_band[0] = a;
    s_band[1] = bb;
  }
  __syncthreads();
  // segment list of this column tile in shared memory (order preserving) with
  // the exclusive prefix of their 2-column pair counts
  const int blo = s_band[0], bhi = s_band[1];
  int nseg = 0, npair = 0;
  if (r3p > 0) {
    if (threadIdx.x == 0) {
      s_col[0] = 0;
      s_len[0] = (int)r3p;
      s_pp[0] = 0;
    }
    nseg = 1;
    npair = (int)((r3p + 1) / 2);
  }
  for (int i0 = blo; i0 < bhi; i0 += T::THREADS) {
    const int bi = i0 + threadIdx.x;
    int K = 0;
    if (bi < bhi) {
      const int64_t s3 = bc3[bi];
      const int64_t d = max((int64_t)0, max(n0 - s3, s3 - top));
      K = d <= gamma ? kofd[d] : 0;
      if (kr) K = min(K, (int)kr[blockIdx.y * ldk + bi]);
    }
    int tot, ptot;
    const int pos = block_exclusive_scan(K > 0 ? 1 : 0, s_wsum, &tot);
    const int pp = block_exclusive_scan((K + 1) / 2, s_wsum, &ptot);
    if (K > 0 && nseg + pos < PLANE_SEGS) {
      s_col[nseg + pos] = (int)(r3p + (int64_t)bi * G);
      s_len[nseg + pos] = K;
      s_pp[nseg + pos] = npair + pp;
    }
    nseg += tot;
    npair += ptot;
  }
  nseg = min(nseg, PLANE_SEGS - 1);  // host guarantees 1 + BN + 2 gamma < PLANE_SEGS
  if (threadIdx.x == 0) s_pp[nseg] = npair;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / T::WARPS_N) * T::WM, wn0 = (warp % T::WARPS_N) * T::WN;
  const int gid = lane >> 2, tig = lane & 3;
  const int my = threadIdx.x % CH, row0 = threadIdx.x / CH;
  const int chunks = (npair + CH - 1) / CH;
  int si = 0;  // my slot's segment (advances monotonically)
  Acc<T> acc;
  acc.zero();
  auto load_chunk = [&](int c) {
    const int P = c * CH + my;
    int64_t col = 0;
    int bytes = 0;
    if (P < npair) {
      while (s_pp[si + 1] <= P) ++si;
      const int off = 2 * (P - s_pp[si]);
      col = s_col[si] + off;
      bytes = off + 1 < s_len[si] ? 16 : 8;
    }
    double *st = smem + (c % T::STAGES) * T::STAGE_DOUBLES;
#pragma unroll
    for (int r = row0; r < T::BM + T::BN; r += ROWS_PER_PASS) {
      const double *src;
      bool ok;
      if (r < T::BM) {
        const int64_t g = m0 + r;
        ok = bytes > 0 && g < M;
        src = ok ? A + g * lda + col : A;
      } else {
        const int64_t g = n0 + (r - T::BM);
        ok = bytes > 0 && g < N;
        src = ok ? B + g * ldb + col : B;
      }
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                       smem_addr(st + r * T::LDS + 2 * my)),
                   "l"(src), "r"(ok ? bytes : 0));
    }
  };
#pragma unroll
  for (int st = 0; st < T::STAGES - 1; ++st) {
    if (st < chunks) load_chunk(st);
    cp_async_commit();
  }
  for (int c = 0; c < chunks; ++c) {
    cp_async_wait<T::STAGES - 2>();
    __syncthreads();
    if (c + T::STAGES - 1 < chunks) load_chunk(c + T::STAGES - 1);
    cp_async_commit();
    stage_mma<T>(smem + (c % T::STAGES) * T::STAGE_DOUBLES, acc, wm0, wn0, gid, tig);
  }
  cp_async_wait<0>();
  store_tile<T, ACC>(acc, C, ldc, m0, M, n0, N);
}

// Tucker part of a plane slab for small r3 (HBM-bound: 2 r3 flops per 8-byte
// store, or per 16 bytes moved when accumulating):
//   out[g, x3] (+)= sum_c A[g, c] V3[x3, c],   g = (x1 - x1_lo) n + x2,
// with A = V2 Y_x1 from the batched DMMA stage.  Thread t of the CTA owns the
// column x3 = blockIdx.y blockDim + t and keeps V3[x3, :] in registers (zero
// past r3); the CTA stages its TA_ROWS rows of A in shared memory (one
// coalesced load) and walks them TA_U at a time: the TA_U old values are
// loaded first (accumulate), then each row is a run of broadcast LDS.128 +
// FMAs and one coalesced 8-byte store per thread.
template <int R, int U, bool ACC>
__global__ void __launch_bounds__(256, (R <= 16 && U <= 4) ? 3 : 2)
    k_tucker_apply(const double *__restrict__ A, int64_t lda, const double *__restrict__ V3,
                   int r3, int64_t n, int64_t rows, int rows_cta, double *__restrict__ out) {
  extern __shared__ __align__(16) double sA[];
  const int64_t x3 = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  const bool col = x3 < n;
  const int64_t g0 = (int64_t)blockIdx.x * rows_cta;
  const int64_t g1 = min(g0 + rows_cta, rows);
  // software pipeline: the old values of batch b + 1 are in flight while
  // batch b is computed and stored; the first batch is requested before the
  // A rows are staged
  double nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    nxt[u] = (ACC && col && g0 + u < g1) ? __ldcs(out + (g0 + u) * n + x3) : 0.0;
  for (int e = threadIdx.x; e < rows_cta * R; e += blockDim.x) {
    const int r = e / R, c = e - r * R;
    sA[e] = (g0 + r < g1 && c < r3) ? __ldg(A + (g0 + r) * lda + c) : 0.0;
  }
  double v[R];
#pragma unroll
  for (int c = 0; c < R; ++c) v[c] = (col && c < r3) ? __ldg(V3 + x3 * r3 + c) : 0.0;
  __syncthreads();
  if (!col) return;
  for (int64_t gb = g0; gb < g1; gb += U) {
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = nxt[u];
    if (ACC) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        nxt[u] = (gb + U + u < g1) ? __ldcs(out + (gb + U + u) * n + x3) : 0.0;
    }
    const double *a0 = sA + (gb - g0) * R;
#pragma unroll
    for (int c = 0; c < R; c += 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double2 ac = *reinterpret_cast<const double2 *>(a0 + u * R + c);
        acc[u] = fma(ac.y, v[c + 1], fma(ac.x, v[c], acc[u]));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (gb + u < g1) __stcs(out + (gb + u) * n + x3, acc[u]);
  }
}

// rows per CTA and rows per load batch (RSB200_TA_ROWS / RSB200_TA_U: A/B runs)
static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}
static const int g_ta_rows = env_int("RSB200_TA_ROWS", 64);
static const int g_ta_u = env_int("RSB200_TA_U", 4);

template <int R, int U>
static int launch_tucker_apply_ru(const double *A, int64_t lda, const double *V3, int r3,
                                  int64_t n, int64_t rows, double *out, bool acc, cudaStream_t s) {
  const int threads = (int)std::min<int64_t>(256, round_up(n, 32));
  const int rc = std::max(U, g_ta_rows / U * U);
  const dim3 grid((unsigned)ceil_div(rows, rc), (unsigned)ceil_div(n, threads));
  const size_t smem = (size_t)rc * R * 8;
  if (smem > 48 * 1024) return fail(RS_ERR_UNSUPPORTED, "tucker_apply: %d rows too many", rc);
  if (acc)
    k_tucker_apply<R, U, true><<<grid, threads, smem, s>>>(A, lda, V3, r3, n, rows, rc, out);
  else
    k_tucker_apply<R, U, false><<<grid, threads, smem, s>>>(A, lda, V3, r3, n, rows, rc, out);
  return check_launch("tucker_apply");
}

template <int R>
static int launch_tucker_apply_r(const double *A, int64_t lda, const double *V3, int r3,
                                 int64_t n, int64_t rows, double *out, bool acc, cudaStream_t s) {
  if (g_ta_u >= 16) return launch_tucker_apply_ru<R, 16>(A, lda, V3, r3, n, rows, out, acc, s);
  if (g_ta_u <= 4) return launch_tucker_apply_ru<R, 4>(A, lda, V3, r3, n, rows, out, acc, s);
  return launch_tucker_apply_ru<R, 8>(A, lda, V3, r3, n, rows, out, acc, s);
}

constexpr int TA_MAXR = 32;   // r3 = 40 (C4): the plane GEMM measured faster

static bool tucker_apply_ok(int64_t r3, int64_t n) {
  return r3 >= 1 && r3 <= TA_MAXR && n >= 2 && n % 2 == 0;
}

static int launch_tucker_apply(const double *A, int64_t lda, const double *V3, int r3, int64_t n,
                               int64_t rows, double *out, bool acc, cudaStream_t s) {
  switch ((r3 + 7) / 8) {
    case 1: return launch_tucker_apply_r<8>(A, lda, V3, r3, n, rows, out, acc, s);
    case 2: return launch_tucker_apply_r<16>(A, lda, V3, r3, n, rows, out, acc, s);
    case 3: return launch_tucker_apply_r<24>(A, lda, V3, r3, n, rows, out, acc, s);
    case 4: return launch_tucker_apply_r<32>(A, lda, V3, r3, n, rows, out, acc, s);
  }
  return fail(RS_ERR_UNSUPPORTED, "tucker_apply: r3=%d", r3);
}

// Bt[x3, :] = [V3[x3, :r3], 0 .. r3p, E[(b,k), x3]] with E = ul[x3 - bc3[b] + g, k] in
// the band (r3 = 0: no Tucker columns; Rs = 0: no short columns).
__global__ void k_build_bt(const double *__restrict__ V3, int r3, int r3p,
                           const double *__restrict__ ul, int Rs, int G, int gamma,
                           const int32_t *__restrict__ bc3, const int32_t *__restrict__ nbp,
                           int64_t n, double *__restrict__ Bt, int64_t ldb) {
  const int64_t nb = nbp ? *nbp : 0;
  const int64_t used = r3p + nb * G;  // columns past `used` are never read by the GEMM
  const int64_t total = n * used;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t x3 = e / used, col = e - x3 * used;
    double v = 0.0;
    if (col < r3) {
      v = V3[x3 * r3 + col];
    } else if (col >= r3p) {
      int64_t q = col - r3p, b = q / G;
      int k = (int)(q - b * G);
      if (k < Rs) {
        int64_t d = x3 - bc3[b];
        if (d >= -gamma && d <= gamma) v = ul[(d + gamma) * Rs + k];
      }
    }
    Bt[x3 * ldb + col] = v;
  }
}

// Per column tile t: range 0 = Tucker columns [0, r3p), range 1 = the buckets
// whose x3 index lies within gamma of the tile's x3 span (bc3 ascending).
__global__ void k_band_ranges(const int32_t *__restrict__ bc3, const int32_t *__restrict__ nbp,
                              int64_t n, int gamma, int BN, int64_t r3p, int G, int64_t ntiles,
                              int64_t *__restrict__ ranges) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int64_t nb = nbp ? *nbp : 0;
  int64_t top = t * BN + BN - 1 < n - 1 ? t * BN + BN - 1 : n - 1;
  int64_t lo_x = t * BN - gamma, hi_x = top + gamma;
  int64_t a = 0, b = nb;
  while (a < b) {
    int64_t m = (a + b) / 2;
    if (bc3[m] < lo_x) a = m + 1; else b = m;
  }
  int64_t blo = a;
  a = blo;
  b = nb;
  while (a < b) {
    int64_t m = (a + b) / 2;
    if (bc3[m] <= hi_x) a = m + 1; else b = m;
  }
  int64_t bhi = a;
  ranges[t * 4 + 0] = 0;
  ranges[t * 4 + 1] = r3p;
  ranges[t * 4 + 2] = r3p + blo * G;
  ranges[t * 4 + 3] = r3p + bhi * G;
}

// Buckets of the x3-sorted copies from the occupancy counts: bc3 = occupied x3
// values ascending, bstart = prefix sums of their counts, *nb = #buckets.
// One block, fixed-order scan (deterministic).
__global__ void __launch_bounds__(1024)
    k_short_layout(const int32_t *__restrict__ cnt3, int64_t n, int32_t *__restrict__ bstart,
                   int32_t *__restrict__ bc3, int32_t *__restrict__ nbp) {
  __shared__ int32_t wocc[32], wcnt[32];
  __shared__ int32_t carry_occ, carry_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry_occ = 0;
    carry_cnt = 0;
    bstart[0] = 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t x = base + tid;
    const int32_t c = x < n ? cnt3[x] : 0;
    const int32_t occ = c > 0 ? 1 : 0;
    int32_t so = occ, sc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t to = __shfl_up_sync(0xffffffffu, so, o), tc = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) {
        so += to;
        sc += tc;
      }
    }
    if (lane == 31) {
      wocc[warp] = so;
      wcnt[warp] = sc;
    }
    __syncthreads();
    int32_t po = carry_occ, pc = carry_cnt;
    for (int w = 0; w < warp; ++w) {
      po += wocc[w];
      pc += wcnt[w];
    }
    if (occ) {
      const int32_t pos = po + so - 1;  // exclusive index of this bucket
      bc3[pos] = (int32_t)x;
      bstart[pos + 1] = pc + sc;
    }
    __syncthreads();
    if (tid == blockDim.x - 1) {
      carry_occ = po + so;
      carry_cnt = pc + sc;
    }
    __syncthreads();
  }
  if (tid == 0) *nbp = carry_occ;
}

// ======================================================== point evaluation
// warp per point: Tucker value sum_abc core V1[i,a] V2[j,b] V3[l,c]
__global__ void k_eval_tucker(const double *__restrict__ core, int r1, int r2, int r3,
                              const double *__restrict__ V1, const double *__restrict__ V2,
                              const double *__restrict__ V3, const int64_t *__restrict__ idx,
                              int64_t m, double *__restrict__ out) {
  const int64_t pt = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (pt >= m) return;
  const double *v1 = V1 + idx[3 * pt] * r1;
  const double *v2 = V2 + idx[3 * pt + 1] * r2;
  const double *v3 = V3 + idx[3 * pt + 2] * r3;
  double acc = 0.0;
  for (int ab = lane; ab < r1 * r2; ab += 32) {
    int a = ab / r2, b = ab - a * r2;
    const double *cr = core + (int64_t)ab * r3;
    double t = 0.0;
    for (int c = 0; c < r3; ++c) t = fma(cr[c], v3[c], t);
    acc = fma(v1[a] * v2[b], t, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[pt] = acc;
}

// warp per point: short-range value and hit count (brute force over copies)
__global__ void k_eval_cct(const double *__restrict__ ul, const double *__restrict__ wl, int Rs,
                           int gamma, const int64_t *__restrict__ centers,
                           const double *__restrict__ zq, int64_t count,
                           const int64_t *__restrict__ idx, int64_t m, double *__restrict__ out,
                           int32_t *__restrict__ hits) {
  const int64_t pt = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (pt >= m) return;
  const int64_t i0 = idx[3 * pt], i1 = idx[3 * pt + 1], i2 = idx[3 * pt + 2];
  dd acc{0.0, 0.0};
  int h = 0;
  for (int64_t p = lane; p < count; p += 32) {
    int64_t o0 = i0 - centers[3 * p], o1 = i1 - centers[3 * p + 1], o2 = i2 - centers[3 * p + 2];
    if (o0 < -gamma || o0 > gamma || o1 < -gamma || o1 > gamma || o2 < -gamma || o2 > gamma)
      continue;
    ++h;
    const double *u0 = ul + (o0 + gamma) * Rs, *u1 = ul + (o1 + gamma) * Rs,
                 *u2 = ul + (o2 + gamma) * Rs;
    double s = 0.0;
    for (int k = 0; k < Rs; ++k) s = fma(wl[k], u0[k] * u1[k] * u2[k], s);
    acc = dd_add_d(acc, zq[p] * s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd other{__shfl_xor_sync(0xffffffffu, acc.hi, o), __shfl_xor_sync(0xffffffffu, acc.lo, o)};
    acc = dd_add(acc, other);
    h += __shfl_xor_sync(0xffffffffu, h, o);
  }
  if (lane == 0) {
    out[pt] = acc.hi + acc.lo;
    hits[pt] = h;
  }
}

// ============================================ windowed pair sums (K6: energy/forces)
constexpr int PS_THREADS = 256;

__device__ __forceinline__ double window_value(const double *__restrict__ T, int64_t ldt,
                                               int64_t n0, const double *__restrict__ w, int Rl,
                                               double h3, int64_t o0, int64_t o1, int64_t o2) {
  const double *r0 = T + (n0 + o0) * ldt, *r1 = T + (n0 + o1) * ldt, *r2 = T + (n0 + o2) * ldt;
  double s = 0.0;
  for (int k = 0; k < Rl; ++k) s = fma(__dmul_rn(__dmul_rn(r0[k], r1[k]), r2[k]), w[k], s);
  return s / h3;
}

__device__ dd block_reduce_dd(dd v, dd *scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd other{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = dd_add(v, other);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  dd r{0.0, 0.0};
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = dd_add(r, scratch[i]);
  return r;  // valid in thread 0
}

__global__ void __launch_bounds__(PS_THREADS)
    k_pair_sums(const double *__restrict__ T, int64_t ldt, int64_t n0, const double *__restrict__ w,
                int Rl, double h3, const int64_t *__restrict__ idx, const double *__restrict__ z,
                int64_t count, const int64_t *__restrict__ tgt, int mode,
                double *__restrict__ base, double *__restrict__ dshift) {
  __shared__ dd scratch[PS_THREADS / 32];
  const int64_t j = tgt[blockIdx.x];
  const int64_t j0 = idx[3 * j], j1 = idx[3 * j + 1], j2 = idx[3 * j + 2];
  if (mode == 0) {
    dd acc{0.0, 0.0};
    for (int64_t p = threadIdx.x; p < count; p += PS_THREADS) {
      double v = window_value(T, ldt, n0, w, Rl, h3, j0 - idx[3 * p], j1 - idx[3 * p + 1],
                              j2 - idx[3 * p + 2]);
      acc = dd_add_d(acc, __dmul_rn(z[p], v));
    }
    dd r = block_reduce_dd(acc, scratch);
    if (threadIdx.x == 0) base[blockIdx.x] = r.hi + r.lo;
  } else {
    dd acc[3] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int64_t p = threadIdx.x; p < count; p += PS_THREADS) {
      if (p == j) continue;
      int64_t o0 = j0 - idx[3 * p], o1 = j1 - idx[3 * p + 1], o2 = j2 - idx[3 * p + 2];
      double b0 = window_value(T, ldt, n0, w, Rl, h3, o0, o1, o2);
      double s0 = window_value(T, ldt, n0, w, Rl, h3, o0 - 1, o1, o2);
      double s1 = window_value(T, ldt, n0, w, Rl, h3, o0, o1 - 1, o2);
      double s2 = window_value(T, ldt, n0, w, Rl, h3, o0, o1, o2 - 1);
      if (mode == 2) {  // condition scale of the differences: sum |z| (|shifted| + |base|)
        const double za = fabs(z[p]);
        acc[0] = dd_add_d(acc[0], __dmul_rn(za, fabs(s0) + fabs(b0)));
        acc[1] = dd_add_d(acc[1], __dmul_rn(za, fabs(s1) + fabs(b0)));
        acc[2] = dd_add_d(acc[2], __dmul_rn(za, fabs(s2) + fabs(b0)));
        continue;
      }
      acc[0] = dd_add_d(acc[0], __dmul_rn(z[p], __dsub_rn(s0, b0)));
      acc[1] = dd_add_d(acc[1], __dmul_rn(z[p], __dsub_rn(s1, b0)));
      acc[2] = dd_add_d(acc[2], __dmul_rn(z[p], __dsub_rn(s2, b0)));
    }
    for (int a = 0; a < 3; ++a) {
      dd r = block_reduce_dd(acc[a], scratch);
      if (threadIdx.x == 0) dshift[3 * blockIdx.x + a] = r.hi + r.lo;
    }
  }
}

// ================================================= compensated vector sum
constexpr int SUM_THREADS = 256;
__global__ void __launch_bounds__(SUM_THREADS)
    k_sum_dd_part(const double *__restrict__ v, int64_t m, int64_t per, double *__restrict__ part) {
  __shared__ dd scratch[SUM_THREADS / 32];
  int64_t lo = blockIdx.x * per, hi = min(m, lo + per);
  dd acc{0.0, 0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += SUM_THREADS) acc = dd_add_d(acc, v[i]);
  dd r = block_reduce_dd(acc, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r.hi;
    part[2 * blockIdx.x + 1] = r.lo;
  }
}

__global__ void k_sum_dd_final(const double *__restrict__ part, int64_t np, double *__restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  dd acc{0.0, 0.0};
  for (int64_t i = 0; i < np; ++i) acc = dd_add(acc, dd{part[2 * i], part[2 * i + 1]});
  out[0] = acc.hi + acc.lo;
}

inline int grid_for(int64_t total, int threads) { return (int)grid_blocks(total, threads); }

template <class T>
int set_smem(const void *fn) {
  cudaError_t e =
      smem_attr(fn, T::SMEM_BYTES);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  return RS_OK;
}

}  // namespace rsb

namespace rsb {
int gemm_batched_nt(const double *A, int64_t lda, int64_t sA, const double *B, int64_t ldb,
                    int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t M, int64_t N,
                    int64_t K, int nb, cudaStream_t s);  // rs_eig.cu
}

using namespace rsb;

// ============================================================== C ABI
template <int GK>
static int launch_short_dmma_t(const double *ul, const double *wl, int Rs, int gamma,
                               const int32_t *c1, const int32_t *c2, const double *zq,
                               const int32_t *bstart, const int32_t *nb_dev, int64_t nb_max,
                               int64_t n, int64_t x1_lo, int64_t planes, double *A, int64_t lda,
                               int64_t col0, const int *kofd, const uint8_t *kr, int64_t ldk,
                               cudaStream_t s) {
  const int W = 2 * gamma + 1;
  const size_t smem = (size_t)(GK + 1) * (2 * W + 2 * SD_PADA + 2 * SD_PADB) * 8 +
                      (SD_THREADS + 4) * (8 + 4 + 4 + 4) + 32 * 4 + (size_t)(gamma + 1) * 4;
  cudaError_t e = smem_attr((const void *)k_short_dmma<GK>, (int)smem);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "short_dmma smem: %s", cudaGetErrorString(e));
  dim3 grid((unsigned)ceil_div(n, SD_TX2), (unsigned)ceil_div(planes, SD_TX1),
            (unsigned)ceil_div(nb_max, SD_BG));
  k_short_dmma<GK><<<grid, SD_THREADS, smem, s>>>(ul, wl, Rs, GK, gamma, c1, c2, zq, bstart, nb_dev,
                                                  n, x1_lo, planes, A, lda, col0, kofd, kr,
                                                  ldk);
  return check_launch("short_dmma");
}

// one instantiation per even row width G = R_s rounded up to even
static int launch_short_dmma(const double *ul, const double *wl, int Rs, int G, int gamma,
                             const int32_t *c1, const int32_t *c2, const double *zq,
                             const int32_t *bstart, const int32_t *nb_dev, int64_t nb_max,
                             int64_t n, int64_t x1_lo, int64_t planes, double *A, int64_t lda,
                             int64_t col0, const int *kofd, const uint8_t *kr, int64_t ldk,
                             cudaStream_t s) {
  switch (G) {
#define RS_SD(R)                                                                              \
  case R:                                                                                     \
    return launch_short_dmma_t<R>(ul, wl, Rs, gamma, c1, c2, zq, bstart, nb_dev, nb_max, n, \
                                  x1_lo, planes, A, lda, col0, kofd, kr, ldk, s);
    RS_SD(2) RS_SD(4) RS_SD(6) RS_SD(8) RS_SD(10) RS_SD(12) RS_SD(14) RS_SD(16) RS_SD(18)
    RS_SD(20) RS_SD(22) RS_SD(24)
#undef RS_SD
  }
  return fail(RS_ERR_UNSUPPORTED, "short_dmma: R_s=%d exceeds 24", Rs);
}

extern "C" {
int rs_oz_gemm_cols(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                    int64_t ldc, int64_t M, int64_t N, int64_t K, const int64_t *ranges, int nr,
                    int slices, int accumulate, void *work, int64_t work_bytes,
                    const int32_t *nb, int64_t r3p, int64_t G, void *stream, int phase);

int rs_abi_version(void) { return 1; }
const char *rs_last_error(void) { return g_err; }

int64_t rs_launch_count(void) { return g_launches.load(); }

int rs_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (on) {  // recycle the recorded events (no create/destroy in timed regions)
    for (auto &r : g_prof) {
      g_prof_pool.push_back(r.a);
      g_prof_pool.push_back(r.b);
    }
    g_prof.clear();
  }
  g_prof_on = on != 0;
  return RS_OK;
}

int rs_prof_query(const char *name, double *total_ms, int64_t *count) {
  RS_REQUIRE(name && total_ms && count, "rs_prof_query: null pointer");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double tot = 0.0;
  int64_t c = 0;
  for (auto &r : g_prof) {
    if (strcmp(r.name, name) != 0) continue;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "rs_prof_query: %s", cudaGetErrorString(e));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    tot += ms;
    ++c;
  }
  *total_ms = tot;
  *count = c;
  return RS_OK;
}

int rs_snap(const double *pos, int64_t count, double h, int64_t n, int64_t *idx, double *disp,
            int64_t *key, double *snapped, void *stream) {
  RS_REQUIRE(count >= 0 && n >= 2 && h > 0, "rs_snap: bad arguments");
  if (count == 0) return RS_OK;
  RS_REQUIRE(pos && idx && disp, "rs_snap: null pointer");
  k_snap<<<(unsigned)ceil_div(count, 256), 256, 0, as_stream(stream)>>>(pos, count, h, n, idx, disp,
                                                                       key, snapped);
  return check_launch("rs_snap");
}

int rs_prep(const int64_t *ks, const int64_t *order, const int64_t *idx, const double *z,
            const double *disp, int64_t count, int64_t n, int32_t *c1s, int32_t *c2s, double *zqs,
            int64_t *starts, uint64_t *dup_pos, uint64_t *dmax_bits, void *stream) {
  RS_REQUIRE(count >= 1 && n >= 2, "rs_prep: bad sizes");
  cudaStream_t s = as_stream(stream);
  cudaMemsetAsync(dup_pos, 0xff, 8, s);
  cudaMemsetAsync(dmax_bits, 0, 8, s);
  k_prep<<<(unsigned)ceil_div(count, 256), 256, 0, s>>>(
      ks, order, idx, z, disp, count, n, c1s, c2s, zqs, starts, (unsigned long long *)dup_pos,
      (unsigned long long *)dmax_bits);
  int st = check_launch("rs_prep");
  if (st) return st;
  k_prep_finish<<<1, 1, 0, s>>>(ks, count, (unsigned long long *)dup_pos);
  return check_launch("rs_prep finish");
}

int rs_gather_windows(const double *table, int64_t ld_table, int64_t n_rows, const int64_t *starts,
                      int64_t n_groups, int64_t n_terms, int64_t term0, const double *gscale,
                      const double *tscale, double *out, int64_t ld_out, void *stream) {
  RS_REQUIRE(n_rows >= 0 && n_groups >= 0 && n_terms >= 0 && term0 >= 0,
             "rs_gather_windows: negative size");
  RS_REQUIRE(ld_out >= n_groups * n_terms && ld_table >= term0 + n_terms,
             "rs_gather_windows: leading dimension too small");
  int64_t total = n_rows * n_groups * n_terms;
  if (total == 0) return RS_OK;
  k_gather<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      table, ld_table, n_rows, starts, n_groups, n_terms, term0, gscale, tscale, out, ld_out);
  return check_launch("rs_gather_windows");
}

static int64_t syrk_splits(int64_t n, int64_t K, int64_t *kslice) {
  const int64_t nt = ceil_div(n, TileSyrk::BM);
  const int64_t ntp = nt * (nt + 1) / 2;
  int64_t want = std::max<int64_t>(1, ceil_div(148 * 3, ntp));
  int64_t ks = round_up(std::max<int64_t>(ceil_div(K, want), 1), TileSyrk::BK);
  ks = std::max<int64_t>(ks, 64);
  *kslice = ks;
  return std::max<int64_t>(1, ceil_div(K, ks));
}

int64_t rs_syrk_workspace_bytes(int64_t n, int64_t K) {
  int64_t ks;
  int64_t sp = syrk_splits(n, K, &ks);
  int64_t nt = ceil_div(n, TileSyrk::BM);
  return sp * (nt * (nt + 1) / 2) * TileSyrk::BM * TileSyrk::BN * 8;
}

int rs_syrk(const double *A, int64_t lda, int64_t n, int64_t K, double *G, void *work,
            int64_t work_bytes, void *stream) {
  RS_REQUIRE(n >= 1 && K >= 0 && lda >= K, "rs_syrk: bad shape");
  RS_REQUIRE(lda % 2 == 0 && K % 2 == 0, "rs_syrk: lda and K must be even (pad with zeros)");
  RS_REQUIRE(((uintptr_t)A & 15) == 0, "rs_syrk: A must be 16-byte aligned");
  int64_t ks;
  int64_t sp = syrk_splits(n, K, &ks);
  int64_t nt = ceil_div(n, TileSyrk::BM), ntp = nt * (nt + 1) / 2;
  int64_t need = sp * ntp * TileSyrk::BM * TileSyrk::BN * 8;
  if (work_bytes < need) return fail(RS_ERR_CAPACITY, "rs_syrk: workspace %lld < %lld",
                                     (long long)work_bytes, (long long)need);
  int st = set_smem<TileSyrk>((const void *)k_syrk_part);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  double *part = (double *)work;
  {
    ProfScope ps(s, "syrk");
      k_syrk_part<<<dim3((unsigned)ntp, (unsigned)sp), TileSyrk::THREADS, TileSyrk::SMEM_BYTES, s>>>(
        A, lda, n, K, ks, part, 0, 0, nullptr);
  }
  if ((st = check_launch("rs_syrk part"))) return st;
  int64_t tot = ntp * TileSyrk::BM * TileSyrk::BN;
  k_syrk_reduce<<<grid_for(tot, 256), 256, 0, s>>>(part, sp, ntp, n, G, 0, nullptr);
  return check_launch("rs_syrk reduce");
}

int64_t rs_gram_shifted_workspace_bytes(int64_t n, int64_t R) {
  const int64_t ldx = round_up(n * R, 2);
  int64_t ks;
  const int64_t sp = syrk_splits(n, ldx, &ks);
  const int64_t nt = ceil_div(n, TileSyrk::BM);
  return round_up(3 * n * ldx * 8, 256) + 3 * sp * (nt * (nt + 1) / 2) * TileSyrk::BM * TileSyrk::BN * 8 +
         round_up(3 * n * 4, 256) + 256;
}

int rs_gram_shifted(const double *table, int64_t ld_table, int64_t n, int64_t R, const double *c,
                    const double *wabs, double *G, void *work, int64_t work_bytes, void *stream) {
  RS_REQUIRE(n >= 2 && R >= 1 && ld_table >= R, "rs_gram_shifted: bad shape");
  if (work_bytes < rs_gram_shifted_workspace_bytes(n, R))
    return fail(RS_ERR_CAPACITY, "rs_gram_shifted: workspace too small");
  const int64_t ldx = round_up(n * R, 2);
  int64_t ks;
  const int64_t sp = syrk_splits(n, ldx, &ks);
  const int64_t nt = ceil_div(n, TileSyrk::BM), ntp = nt * (nt + 1) / 2;
  const int64_t part_stride = sp * ntp * TileSyrk::BM * TileSyrk::BN;
  double *X = (double *)work;
  double *part = (double *)((char *)work + round_up(3 * n * ldx * 8, 256));
  int32_t *kdev = (int32_t *)((char *)part + 3 * part_stride * 8);
  cudaStream_t s = as_stream(stream);
  int st;
  // occupied shifts only: K per mode = (#occupied shifts) R instead of n R
  // (C2: 50 of 256 shifts, C5: 363 of 2048), known on the device
  k_gram_operands_rows<<<dim3((unsigned)n, 3), 256, (size_t)n * 4, s>>>(table, ld_table, n, R, c,
                                                                        wabs, kdev, X, ldx);
  if ((st = check_launch("gram operands"))) return st;
  if ((st = set_smem<TileSyrk>((const void *)k_syrk_part))) return st;
  {
    ProfScope ps(s, "syrk");
    k_syrk_part<<<dim3((unsigned)ntp, (unsigned)sp, 3), TileSyrk::THREADS, TileSyrk::SMEM_BYTES,
                  s>>>(X, ldx, n, ldx, ks, part, n * ldx, part_stride, kdev);
  }
  if ((st = check_launch("gram syrk"))) return st;
  const int64_t tot = ntp * TileSyrk::BM * TileSyrk::BN;
  k_syrk_reduce<<<dim3(grid_for(tot, 256), 1, 3), 256, 0, s>>>(part, sp, ntp, n, G, part_stride,
                                                                kdev);
  return check_launch("gram reduce");
}

int rs_gemm_nt(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
               int64_t M, int64_t N, int64_t K, void *stream) {
  RS_REQUIRE(M >= 0 && N >= 0 && K >= 0 && lda >= K && ldb >= K && ldc >= N, "rs_gemm_nt: bad shape");
  RS_REQUIRE(lda % 2 == 0 && ldb % 2 == 0 && K % 2 == 0, "rs_gemm_nt: lda, ldb, K must be even");
  RS_REQUIRE(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0, "rs_gemm_nt: operands must be 16-byte aligned");
  if (M == 0 || N == 0) return RS_OK;
  int st = set_smem<TilePlane>((const void *)k_gemm_nt<TilePlane, false>);
  if (st) return st;
  dim3 grid((unsigned)ceil_div(N, TilePlane::BN), (unsigned)ceil_div(M, TilePlane::BM));
  k_gemm_nt<TilePlane, false><<<grid, TilePlane::THREADS, TilePlane::SMEM_BYTES, as_stream(stream)>>>(
      A, lda, B, ldb, C, ldc, M, N, K, nullptr, 0);
  return check_launch("rs_gemm_nt");
}

int rs_shift_project(const double *Z, int64_t ldz, int64_t n, int64_t r, const double *table,
                     int64_t ld_table, int64_t R, int64_t n_shift, double *TT, void *stream) {
  RS_REQUIRE(n >= 1 && r >= 1 && R >= 1 && n_shift >= 1 && n_shift <= n && ldz >= r &&
                 ld_table >= R,
             "rs_shift_project: bad shape (table must have 2n rows, n_shift <= n)");
  size_t smem = (size_t)(n + SP_SHIFTS + SP_ICH * 32) * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = smem_attr((const void *)k_shift_project, (int)smem);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "shift_project smem: %s", cudaGetErrorString(e));
  }
  RS_REQUIRE(ldz == r, "rs_shift_project: Z must be contiguous (ldz == r)");
  Proj3 pj{{Z, Z, Z}, {TT, TT, TT}, {r, r, r}};
  {
    ProfScope ps(as_stream(stream), "shift_project");
    dim3 grid((unsigned)ceil_div(n_shift, SP_SHIFTS), (unsigned)R, 1);
    k_shift_project<<<grid, 256, smem, as_stream(stream)>>>(pj, n, table, ld_table, R, n_shift);
  }
  return check_launch("rs_shift_project");
}

int rs_shift_project3(const double *Z1, const double *Z2, const double *Z3, int64_t r1, int64_t r2,
                      int64_t r3, int64_t n, const double *table, int64_t ld_table, int64_t R,
                      int64_t n_shift, double *TT1, double *TT2, double *TT3, void *stream) {
  RS_REQUIRE(n >= 1 && r1 >= 1 && r2 >= 1 && r3 >= 1 && R >= 1 && n_shift >= 1 && n_shift <= n &&
                 ld_table >= R,
             "rs_shift_project3: bad shape");
  size_t smem = (size_t)(n + SP_SHIFTS + SP_ICH * 32) * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = smem_attr((const void *)k_shift_project, (int)smem);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "shift_project smem: %s", cudaGetErrorString(e));
  }
  Proj3 pj{{Z1, Z2, Z3}, {TT1, TT2, TT3}, {r1, r2, r3}};
  {
    ProfScope ps(as_stream(stream), "shift_project");
    dim3 grid((unsigned)ceil_div(n_shift, SP_SHIFTS), (unsigned)R, 3);
    k_shift_project<<<grid, 256, smem, as_stream(stream)>>>(pj, n, table, ld_table, R, n_shift);
  }
  return check_launch("rs_shift_project3");
}

}  // extern "C"

// (internal) rs_shift_project3 restricted to the shifts in `shift` (count x 3,
// n - c of the particles); list_work: (6 n + 8) ints.  Entries of TT at other
// shifts are left untouched (they are never read).
int rsb_shift_project3_listed(const double *Z1, const double *Z2, const double *Z3, int64_t r1,
                              int64_t r2, int64_t r3, int64_t n, const double *table,
                              int64_t ld_table, int64_t R, const int64_t *shift, int64_t count,
                              double *TT1, double *TT2, double *TT3, void *list_work,
                              cudaStream_t s) {
  int *flags = (int *)list_work, *list = flags + 3 * n, *cnt = list + 3 * n;
  if (cudaMemsetAsync(flags, 0, (size_t)(3 * n) * 4, s) != cudaSuccess)
    return fail(RS_ERR_CUDA, "shift list: memset");
  k_shift_flags<<<grid_blocks(3 * count), 256, 0, s>>>(shift, count, n, flags);
  k_shift_compact<<<3, 1024, 0, s>>>(flags, n, list, cnt);
  int st;
  if ((st = check_launch("shift list"))) return st;
  const size_t smem = (size_t)(2 * n + SP_ICH * 32) * 8;
  if (smem > 200 * 1024) return fail(RS_ERR_UNSUPPORTED, "shift_project: n too large");
  cudaError_t e = smem_attr((const void *)k_shift_project_list, (int)smem);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "shift_project smem: %s", cudaGetErrorString(e));
  Proj3 pj{{Z1, Z2, Z3}, {TT1, TT2, TT3}, {r1, r2, r3}};
  {
    ProfScope ps(s, "shift_project");
    dim3 grid((unsigned)ceil_div(n, SP_SHIFTS), (unsigned)R, 3);
    k_shift_project_list<<<grid, 256, smem, s>>>(pj, n, table, ld_table, R, n, list, cnt);
  }
  return check_launch("shift_project_list");
}

extern "C" {
int rs_shift_hist(const int64_t *idx, const double *z, int64_t count, int64_t n, double *c,
                  int32_t *cnt3, void *stream) {
  RS_REQUIRE(count >= 1 && n >= 2, "rs_shift_hist: bad sizes");
  k_shift_hist<<<dim3((unsigned)ceil_div(n, 8), 3), 256, 0, as_stream(stream)>>>(idx, z, count, n,
                                                                                 c, cnt3);
  return check_launch("rs_shift_hist");
}

static void core_plan(int64_t r1, int64_t r2, int64_t r3, int64_t K, int64_t *splits,
                      int64_t *kslice) {
  const int64_t tiles = ceil_div(r1 * r2, TileCore::BM) * ceil_div(r3, TileCore::BN);
  int64_t sp = std::max<int64_t>(1, ceil_div(148 * 2, tiles));
  sp = std::min<int64_t>(sp, std::max<int64_t>(1, K / 64));
  int64_t ks = round_up(ceil_div(K, sp), TileCore::BK);
  *kslice = ks;
  *splits = ceil_div(K, ks);
}

int64_t rs_core_workspace_bytes(int64_t r1, int64_t r2, int64_t r3, int64_t count, int64_t R) {
  int64_t sp, ks;
  const int64_t K = count * R;
  core_plan(r1, r2, r3, K, &sp, &ks);
  return round_up((r1 + r2 + r3) * K * 8, 256) + sp * r1 * r2 * r3 * 8;
}

int rs_core(const double *TT1, const double *TT2, const double *TT3, int64_t r1, int64_t r2,
            int64_t r3, int64_t n_shift, int64_t R, const int64_t *shift, const double *z,
            const double *w, int64_t count, double *core, void *work, int64_t work_bytes,
            void *stream) {
  RS_REQUIRE(r1 >= 1 && r2 >= 1 && r3 >= 1 && R >= 1 && count >= 1, "rs_core: bad shape");
  const int64_t K = count * R;
  if (work_bytes < rs_core_workspace_bytes(r1, r2, r3, count, R))
    return fail(RS_ERR_CAPACITY, "rs_core: workspace too small");
  int64_t sp, ks;
  core_plan(r1, r2, r3, K, &sp, &ks);
  cudaStream_t s = as_stream(stream);
  double *P1 = (double *)work;
  double *P2 = P1 + r1 * K;
  double *P3 = P2 + r2 * K;
  double *part = (double *)((char *)work + round_up((r1 + r2 + r3) * K * 8, 256));
  const double *TTs[3] = {TT1, TT2, TT3};
  double *Ps[3] = {P1, P2, P3};
  const int64_t rs_[3] = {r1, r2, r3};
  int st;
  ProfScope ps(s, "core");
  for (int l = 0; l < 3; ++l) {
    k_core_gather<<<grid_for(rs_[l] * K, 256), 256, 0, s>>>(TTs[l], (int)rs_[l], n_shift, (int)R,
                                                            shift, l, z, w, count, Ps[l]);
    if ((st = check_launch("rs_core gather"))) return st;
  }
  dim3 grid((unsigned)ceil_div(r1 * r2, TileCore::BM), (unsigned)ceil_div(r3, TileCore::BN),
            (unsigned)sp);
  k_core_kr<<<grid, TileCore::THREADS, 0, s>>>(P1, P2, P3, (int)r2, r1 * r2, r3, K, ks, part);
  if ((st = check_launch("rs_core kr"))) return st;
  const int64_t len = r1 * r2 * r3;
  k_split_reduce<<<grid_for(len, 256), 256, 0, s>>>(part, sp, len, core);
  return check_launch("rs_core reduce");
}

// workspace: A (planes*n x lda) | Bt (n x lda) | Y (planes x r2 r3) | ranges
// x3 tile width of the short-range plane GEMM (RSB200_PLANE_BN = 32 or 64)
static const int g_plane_bn = [] {
  const char *e = getenv("RSB200_PLANE_BN");
  return (e && (atoi(e) == 32 || atoi(e) == 128)) ? atoi(e) : 64;
}();

// (internal, not part of the ABI header) the per-distance live-term table at
// offset 0 of an rs_assemble_planes workspace (depends on the plan only:
// rs_front fills it before its wait on the front)
int rsb_asm_term_prefix(const double *ul, const double *wl, int Rs, int gamma, void *work,
                        cudaStream_t s) {
  k_term_prefix<<<1, 256, 0, s>>>(ul, wl, Rs, gamma, (int *)work);
  return check_launch("term_prefix");
}

// short-range plane GEMM tile variant (RSB200_PLANE_TILE: 0 default, 1 four
// stages, 2 64x32 warp tiles) -- A/B measurements
static const int g_plane_tile = [] {
  const char *e = getenv("RSB200_PLANE_TILE");
  return e && *e ? atoi(e) : 2;   // 64x32 warp tiles: C2 GEMM -4 %, C3 -6 %, C4 -5 %
}();
// RSB200_TUCKER_RES=0: the Tucker-only plane GEMM as one CTA per (row block,
// column tile) instead of the A-resident kernel
// (RSB200_TUCKER_RES=128: 128-row blocks, one CTA per SM; default 64-row
// blocks, two CTAs per SM: C4 Tucker 7.18 -> 4.67 ms, C5 109.8 -> 99.7 ms)
static const int g_tucker_res = [] {
  const char *e = getenv("RSB200_TUCKER_RES");
  if (e && e[0] == '0') return 0;
  return e && atoi(e) == 128 ? 128 : 64;
}();
// RSB200_PLANE_RBG: row blocks per plane-GEMM launch (0: one launch)
static const int64_t g_plane_rbg = [] {
  const char *e = getenv("RSB200_PLANE_RBG");
  return (int64_t)(e && *e ? atoll(e) : 0);
}();
static const int g_tucker_tile = [] {
  const char *e = getenv("RSB200_TUCKER_TILE");
  return e && *e ? atoi(e) : 0;
}();

// RSB200_TUCKER_APPLY=0: the Tucker part through the plane GEMM as before
static const bool g_tucker_apply = [] {
  const char *e = getenv("RSB200_TUCKER_APPLY");
  return !(e && e[0] == '0');
}();

// RSB200_ROW_CUT=0: the row builder computes every term of every copy
static const bool g_row_cut = [] {
  const char *e = getenv("RSB200_ROW_CUT");
  return !(e && e[0] == '0');
}();

// The Tucker part of the grid at large ranks (96 < r3 <= 160: C5) runs as an
// Ozaki-split GEMM on the int8 tensor cores (tcgen05, rs_tc8.cu: k_oz_res) instead of
// the FP64 DMMA kernel: C5 slab of 64 planes 2.77 -> 1.88 ms.  RSB200_TUCKER_OZ=0
// keeps the DMMA kernel, 6 | 7 sets the slice count.  Explicit slices in `flags` win.
static int tucker_oz_policy(int flags, int64_t r3, int64_t n) {
  static const int env = [] {
    const char *e = getenv("RSB200_TUCKER_OZ");
    const int v = e && *e ? atoi(e) : 7;
    return (v == 6 || v == 7) ? v : 0;
  }();
  if (((flags >> 8) & 0xF) || !(flags & RS_ASM_LONG) || (flags & RS_ASM_SHORT) || !env) return flags;
  const int64_t r3p = round_up(std::max<int64_t>(r3, 1), 2);
  if (r3p > 96 && r3p <= 160 && n >= 256) flags |= env << 8;
  return flags;
}

static void asm_layout(int64_t n, int64_t planes, int64_t rmax, int64_t r3, int64_t nb_max,
                       int64_t Rs, int flags, int64_t *lda, int64_t *r3p, int64_t *G, int64_t *offA,
                       int64_t *offB, int64_t *offY, int64_t *offR, int64_t *total) {
  const bool with_long = flags & RS_ASM_LONG, with_short = (flags & RS_ASM_SHORT) && Rs > 0;
  *r3p = with_long ? round_up(std::max<int64_t>(r3, 1), 2) : 0;
  *G = round_up(std::max<int64_t>(Rs, 1), 2);
  *lda = std::max<int64_t>(*r3p + (with_short ? nb_max * *G : 0), 2);
  int64_t a = round_up(planes * n * *lda * 8, 256);
  int64_t b = round_up(n * *lda * 8, 256);
  const int64_t rp = round_up(std::max<int64_t>(rmax, 1), 2);
  // Yt (planes x r3p x r2p) | V2p (n x r2p) | V1p (n x r1p) | coreT (r3p r2p x r1p)
  int64_t y = with_long ? round_up((planes * rp * rp + 2 * n * rp + rp * rp * rp) * 8, 256) : 0;
  int64_t ntiles = ceil_div(n, PLANE_MIN_BN);
  // kofd first (fixed offset 0 for every plane count: rs_front fills it ahead
  // of the chunks) | A | Bt | Y | ranges | row-block term table (uint8)
  const int64_t k0 = round_up((n + 1) * 4, 256);
  int64_t rr = round_up(ntiles * 4 * 8, 256) +
               (with_short ? round_up(ceil_div(planes * n, TilePlane::BM) * round_up(nb_max, 16), 256)
                           : 0);
  *offA = k0;
  *offB = k0 + a;
  *offY = k0 + a + b;
  *offR = k0 + a + b + y;
  *total = k0 + a + b + y + rr;
  const int slices = (flags >> 8) & 0xF;
  if (slices) *total += round_up(rs_oz_workspace_bytes(planes * n, n, *lda, slices), 256);
}

int64_t rs_assemble_workspace_bytes(int64_t n, int64_t planes, int64_t rmax, int64_t nb_max,
                                    int64_t Rs, int flags) {
  int64_t lda, r3p, G, oA, oB, oY, oR, tot;
  asm_layout(n, planes, rmax, rmax, nb_max, Rs, tucker_oz_policy(flags, rmax, n), &lda, &r3p, &G,
             &oA, &oB, &oY, &oR, &tot);
  return tot;
}

int rs_short_layout(const int32_t *cnt3, int64_t n, int32_t *bstart, int32_t *bc3, int32_t *nb,
                    void *stream) {
  RS_REQUIRE(n >= 1 && cnt3 && bstart && bc3 && nb, "rs_short_layout: bad arguments");
  k_short_layout<<<1, 1024, 0, as_stream(stream)>>>(cnt3, n, bstart, bc3, nb);
  return check_launch("rs_short_layout");
}

int rs_assemble_planes(const double *core, int64_t r1, int64_t r2, int64_t r3, const double *V1,
                       const double *V2, const double *V3, int64_t n, const double *ul,
                       const double *wl, int64_t Rs, int64_t gamma, const int32_t *c1,
                       const int32_t *c2, const double *zq, const int32_t *bstart,
                       const int32_t *bc3, const int32_t *nb_dev, int64_t nb_max, int64_t x1_lo,
                       int64_t x1_hi, int flags, double *out, void *work, int64_t work_bytes,
                       void *stream) {
  const bool with_long = flags & RS_ASM_LONG;
  const bool with_short = (flags & RS_ASM_SHORT) && Rs > 0 && nb_max > 0;
  const bool accumulate = flags & RS_ASM_ACCUMULATE;
  RS_REQUIRE(n >= 2 && n % 2 == 0, "rs_assemble_planes: n must be even");
  RS_REQUIRE(!with_long || (r1 >= 1 && r2 >= 1 && r3 >= 1 && core && V1 && V2 && V3),
             "rs_assemble_planes: bad long part");
  RS_REQUIRE(0 <= x1_lo && x1_lo < x1_hi && x1_hi <= n, "rs_assemble_planes: bad plane range");
  RS_REQUIRE(Rs >= 0 && Rs <= SR_MAXR, "rs_assemble_planes: Rs=%lld exceeds %d", (long long)Rs,
             SR_MAXR);
  RS_REQUIRE(gamma >= 0 && gamma < n, "rs_assemble_planes: bad gamma");
  RS_REQUIRE(1 + TilePlaneW::BN + 2 * gamma < PLANE_SEGS,
             "rs_assemble_planes: gamma=%lld too wide for the plane GEMM's segment list",
             (long long)gamma);
  RS_REQUIRE(!with_short || (c1 && c2 && zq && bstart && bc3 && nb_dev && ul && wl),
             "rs_assemble_planes: bad short part");
  RS_REQUIRE(with_long || with_short || accumulate, "rs_assemble_planes: nothing to do");
  const int64_t planes = x1_hi - x1_lo;
  const int64_t rmax = std::max<int64_t>(std::max<int64_t>(r1, r2), r3);
  int64_t lda, r3p, G, oA, oB, oY, oR, tot;
  {
    const int pf = tucker_oz_policy(flags, r3, n);
    asm_layout(n, planes, rmax, r3, nb_max, Rs, pf, &lda, &r3p, &G, &oA, &oB, &oY, &oR, &tot);
    if (pf != flags && work_bytes < tot)   // caller sized the workspace without the slices
      asm_layout(n, planes, rmax, r3, nb_max, Rs, flags, &lda, &r3p, &G, &oA, &oB, &oY, &oR, &tot);
    else
      flags = pf;
  }
  if (work_bytes < tot)
    return fail(RS_ERR_CAPACITY, "rs_assemble_planes: workspace %lld < %lld",
                (long long)work_bytes, (long long)tot);
  if (!with_long && !with_short) {  // accumulate nothing: out unchanged
    return RS_OK;
  }
  char *wb = (char *)work;
  double *A = (double *)(wb + oA);
  double *Bt = (double *)(wb + oB);
  double *Y = (double *)(wb + oY);
  int64_t *ranges = (int64_t *)(wb + oR);
  cudaStream_t s = as_stream(stream);
  int st;
  const bool f_only = with_long && !with_short && (flags & RS_ASM_F_ONLY);
  const bool f_ready = with_long && !with_short && (flags & RS_ASM_F_READY);
  if (with_long && !f_ready) {
    ProfScope ps(s, "tucker_f");
    const int64_t rp = round_up(rmax, 2), r2p = round_up(r2, 2);
    double *Yt = Y;
    double *V2p = Yt + planes * rp * rp;
    if (r1 * r2 * r3 >= 32768) {  // large ranks (C4, C5): Yt as one DMMA GEMM over r1
      const int64_t r1p = round_up(r1, 2);
      double *V1p = V2p + n * rp, *coreT = V1p + n * rp;
      k_pad_cols<<<grid_for(n * r1p, 256), 256, 0, s>>>(V1, n, (int)r1, (int)r1p, V1p);
      k_core_t<<<grid_for(r3p * r2p * r1p, 256), 256, 0, s>>>(core, (int)r1, (int)r2, (int)r3,
                                                              (int)r1p, (int)r2p, (int)r3p, coreT);
      if ((st = check_launch("tucker core_t"))) return st;
      if ((st = rs_gemm_nt(V1p + x1_lo * r1p, r1p, coreT, r1p, Yt, r3p * r2p, planes, r3p * r2p,
                           r1p, stream)))
        return st;
    } else {
      k_tucker_yt<<<grid_for(planes * r3p * r2p, 256), 256, 0, s>>>(
          core, (int)r1, (int)r2, (int)r3, V1, x1_lo, (int)r2p, (int)r3p, planes, Yt);
      if ((st = check_launch("tucker_yt"))) return st;
    }
    k_pad_cols<<<grid_for(n * r2p, 256), 256, 0, s>>>(V2, n, (int)r2, (int)r2p, V2p);
    if ((st = check_launch("pad_cols"))) return st;
    // per plane: A[x1l][x2, c] = V2p[x2, :] . Yt[x1l][c, :]  (DMMA, batched over planes)
    if ((st = gemm_batched_nt(V2p, r2p, 0, Yt, r2p, r3p * r2p, A, lda, n * lda, n, r3p, r2p,
                              (int)planes, s)))
      return st;
  }
  const int64_t ntiles0 = ceil_div(n, PLANE_MIN_BN);
  int *kofd = (int *)wb;
  const int64_t nrb = ceil_div(planes * n, TilePlane::BM), ldk = round_up(nb_max, 16);
  uint8_t *kr = (uint8_t *)((char *)ranges + round_up(ntiles0 * 4 * 8, 256));
  const int slices = (flags >> 8) & 0xF;
  if (with_short) {
    // per-distance live-term counts and the row-block term table: the row
    // builder's and the GEMM's term cuts (the builder stores only the terms
    // the GEMM reads; the Ozaki path reads whole bands, so it gets them all)
    if (!(flags & RS_ASM_KOFD_READY)) {
      k_term_prefix<<<1, 256, 0, s>>>(ul, wl, (int)Rs, (int)gamma, kofd);
      if ((st = check_launch("term_prefix"))) return st;
    }
    k_rowblock_terms<<<grid_for(nrb * ldk, 256), 256, 0, s>>>(
        c1, c2, bstart, nb_dev, kofd, (int)gamma, n, x1_lo, planes * n, TilePlane::BM, nrb, ldk,
        kr);
    if ((st = check_launch("rowblock_terms"))) return st;
    ProfScope ps(s, "short_rows");
    if ((st = launch_short_dmma(ul, wl, (int)Rs, (int)G, (int)gamma, c1, c2, zq, bstart, nb_dev,
                                nb_max, n, x1_lo, planes, A, lda, r3p,
                                g_row_cut ? kofd : nullptr,
                                (g_row_cut && !slices) ? kr : nullptr, ldk, s)))
      return st;
  }
  if (with_short && (st = check_launch("short_rows"))) return st;
  const int slices0 = (flags >> 8) & 0xF;
  if (f_only) {
    if (slices0) {   // Ozaki Tucker GEMM: the operands' exponents and slices belong to this phase
      k_build_bt<<<grid_for(n * lda, 256), 256, 0, s>>>(V3, (int)r3, (int)r3p, ul, 0, (int)G,
                                                         (int)gamma, bc3, nullptr, n, Bt, lda);
      if ((st = check_launch("build_bt"))) return st;
      ProfScope ps(s, "tucker_f");
      const int64_t oz_off = tot - round_up(rs_oz_workspace_bytes(planes * n, n, lda, slices0), 256);
      return rs_oz_gemm_cols(A, lda, Bt, lda, out, n, planes * n, n, lda, nullptr, 2, slices0, 0,
                             wb + oz_off, tot - oz_off, nullptr, r3p, G, stream, 1);
    }
    return RS_OK;
  }
  if (with_long && !with_short && !slices0 && g_tucker_apply && tucker_apply_ok(r3, n)) {
    // small r3: the HBM-bound row kernel instead of the plane GEMM
    ProfScope ps(s, "gemm_tucker");
    return launch_tucker_apply(A, lda, V3, (int)r3, n, planes * n, out, accumulate, s);
  }
  k_build_bt<<<grid_for(n * lda, 256), 256, 0, s>>>(with_long ? V3 : nullptr,
                                                     with_long ? (int)r3 : 0, (int)r3p, ul,
                                                     with_short ? (int)Rs : 0, (int)G, (int)gamma,
                                                     bc3, with_short ? nb_dev : nullptr, n, Bt, lda);
  if ((st = check_launch("build_bt"))) return st;
  const int64_t ntiles = ceil_div(n, TilePlane::BN);
  if (slices) {  // Ozaki-split FP64 on the int8 tensor cores (same tiles, same K ranges)
    if (with_short) {
      k_band_ranges<<<(unsigned)ceil_div(ntiles, 128), 128, 0, s>>>(
          bc3, nb_dev, n, (int)gamma, TilePlane::BN, r3p, (int)G, ntiles, ranges);
      if ((st = check_launch("band_ranges"))) return st;
    }
    ProfScope ps(s, with_long && with_short ? "gemm_plane" : (with_short ? "gemm_short" : "gemm_tucker"));
    const int64_t oz_off = tot - round_up(rs_oz_workspace_bytes(planes * n, n, lda, slices), 256);
    // Tucker columns only: one dense K range (ranges = NULL -> the A-resident kernel)
    return rs_oz_gemm_cols(A, lda, Bt, lda, out, n, planes * n, n, lda,
                           with_short ? ranges : nullptr, 2, slices,
                           accumulate ? 1 : 0, wb + oz_off, tot - oz_off,
                           with_short ? nb_dev : nullptr, r3p, G, stream, f_ready ? 2 : 3);
  }

  {
    ProfScope ps(s, with_long && with_short ? "gemm_plane" : (with_short ? "gemm_short" : "gemm_tucker"));
    const int32_t *nbs = with_short ? nb_dev : nullptr;
    const uint8_t *krp = with_short ? kr : nullptr;
    auto launch = [&](auto tile) -> int {
      using T = decltype(tile);
      auto fn = accumulate ? k_gemm_plane<T, true> : k_gemm_plane<T, false>;
      int e;
      if ((e = set_smem<T>((const void *)fn))) return e;
      const int64_t M = planes * n, nrb_all = ceil_div(M, T::BM);
      // row-block groups: every launch is at most one wave, so the column tiles
      // of a row block start together and share its D rows in L2
      const int64_t rbg = g_plane_rbg > 0 ? g_plane_rbg : nrb_all;
      for (int64_t rb0 = 0; rb0 < nrb_all; rb0 += rbg) {
        const int64_t m0 = rb0 * T::BM, mg = min(M - m0, rbg * T::BM);
        dim3 grid((unsigned)ceil_div(n, T::BN), (unsigned)ceil_div(mg, T::BM));
        fn<<<grid, T::THREADS, T::SMEM_BYTES, s>>>(A + m0 * lda, lda, Bt, lda, out + m0 * n, n,
                                                   mg, n, r3p, G, bc3, nbs, (int)gamma, kofd,
                                                   krp ? krp + rb0 * ldk : nullptr, ldk);
      }
      return 0;
    };
    if (with_long && !with_short && g_tucker_res && r3p <= tr::KMAX && n % 2 == 0) {
      // A-resident Tucker GEMM: one CTA per 64-row block (default; RSB200_TUCKER_RES=128: 128 rows)
      // over all column tiles
      // Bt chunk width x ring depth: 16 columns x 3 stages, or 32 x 2 for short K
      // (same-job A/B: C5, K = 132: 2.82 vs 2.98 ms per 64 planes; C4, K = 40:
      // 0.381 vs 0.355 ms); RSB200_TUCKER_BK=16|32 forces one
      static const int bk_env = [] {
        const char *e = getenv("RSB200_TUCKER_BK");
        return e ? atoi(e) : 0;
      }();
      const int bk = bk_env == 16 || bk_env == 32 ? bk_env : (r3p <= 64 ? 32 : 16);
      auto go = [&](auto bm_c) -> int {
        constexpr int BM = decltype(bm_c)::value;
        auto run = [&](auto bk_c, auto st_c) -> int {
          constexpr int BK = decltype(bk_c)::value, STG = decltype(st_c)::value;
          const int smem = tr::smem_bytes(BM, (int)r3p, BK, STG);
          auto fn = accumulate ? k_tucker_gemm_res<BM, true, BK, STG>
                               : k_tucker_gemm_res<BM, false, BK, STG>;
          cudaError_t e = smem_attr((const void *)fn, smem);
          if (e != cudaSuccess)
            return fail(RS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
          fn<<<(unsigned)ceil_div(planes * n, (int64_t)BM), tr::threads(BM), smem, s>>>(
              A, lda, Bt, lda, out, n, planes * n, n, (int)r3p);
          return 0;
        };
        return bk == 16 ? run(std::integral_constant<int, 16>{}, std::integral_constant<int, 3>{})
                        : run(std::integral_constant<int, 32>{}, std::integral_constant<int, 2>{});
      };
      if ((st = g_tucker_res == 128 ? go(std::integral_constant<int, 128>{})
                                    : go(std::integral_constant<int, 64>{})))
        return st;
    } else if ((with_short && !with_long && g_plane_tile == 1) ||
        (with_long && !with_short && g_tucker_tile == 1)) {
      if ((st = launch(TilePlane4{}))) return st;
    } else if (with_long && !with_short && g_tucker_tile == 3) {
      if ((st = launch(TilePlaneW{}))) return st;
    } else if ((with_short && !with_long && g_plane_tile == 2) ||
               (with_long && !with_short && g_tucker_tile == 2)) {
      if ((st = launch(TilePlaneM{}))) return st;
    } else if (with_short && !with_long && g_plane_bn == 128) {
      if ((st = launch(TilePlaneW{}))) return st;
    } else if (with_short && !with_long && g_plane_bn == 32) {
      if ((st = launch(TilePlaneN{}))) return st;
    } else {
      if ((st = launch(TilePlane{}))) return st;
    }
  }
  return check_launch("plane_gemm");
}

int rs_assemble_fused_l0(int64_t r1, int64_t r2, int64_t r3, const double *V3, int64_t n,
                         const double *L0, int64_t gamma, const int32_t *c1, const int32_t *c2,
                         const double *zq, const int32_t *bstart, const int32_t *bc3,
                         const int32_t *nb_dev, int64_t a_lo, int64_t a_hi, int64_t x1_lo,
                         int64_t x1_hi, double *out, void *work, int64_t work_bytes,
                         void *stream) {
  RS_REQUIRE(r1 >= 1 && r2 >= 1 && r3 >= 1 && V3 && L0 && c1 && c2 && zq && bstart && bc3 &&
                 nb_dev && out && work,
             "rs_assemble_fused_l0: bad arguments");
  RS_REQUIRE(0 <= a_lo && a_lo <= x1_lo && x1_lo < x1_hi && x1_hi <= a_hi && a_hi <= n,
             "rs_assemble_fused_l0: plane range [%lld, %lld) outside the formed operands "
             "[%lld, %lld)", (long long)x1_lo, (long long)x1_hi, (long long)a_lo, (long long)a_hi);
  // the workspace layout of the RS_ASM_F_ONLY call that formed A for [a_lo, a_hi)
  const int64_t rmax = std::max<int64_t>(std::max<int64_t>(r1, r2), r3);
  int64_t lda, r3p, G, oA, oB, oY, oR, tot;
  asm_layout(n, a_hi - a_lo, rmax, r3, 0, 0, RS_ASM_LONG | RS_ASM_ACCUMULATE, &lda, &r3p, &G, &oA,
             &oB, &oY, &oR, &tot);
  if (work_bytes < tot)
    return fail(RS_ERR_CAPACITY, "rs_assemble_fused_l0: workspace %lld < %lld",
                (long long)work_bytes, (long long)tot);
  RS_REQUIRE(fused_l0_supported(n, r3p, gamma), "rs_assemble_fused_l0: unsupported shape");
  char *wb = (char *)work;
  const double *A = (const double *)(wb + oA) + (x1_lo - a_lo) * n * lda;
  double *Bt = (double *)(wb + oB);
  cudaStream_t s = as_stream(stream);
  k_build_bt<<<grid_for(n * lda, 256), 256, 0, s>>>(V3, (int)r3, (int)r3p, nullptr, 0, 2, 0,
                                                     nullptr, nullptr, n, Bt, lda);
  int st;
  if ((st = check_launch("build_bt"))) return st;
  return launch_fused_l0(A, lda, Bt, lda, r3p, L0, gamma, n, c1, c2, zq, bstart, bc3, nb_dev,
                         x1_lo, x1_hi, out, s);
}

int rs_fused_l0_supported(int64_t n, int64_t r3, int64_t gamma) {
  return fused_l0_supported(n, round_up(std::max<int64_t>(r3, 1), 2), gamma) ? 1 : 0;
}

int rs_eval_tucker(const double *core, int64_t r1, int64_t r2, int64_t r3, const double *V1,
                   const double *V2, const double *V3, const int64_t *idx, int64_t m, double *out,
                   void *stream) {
  RS_REQUIRE(r1 >= 1 && r2 >= 1 && r3 >= 1 && m >= 0, "rs_eval_tucker: bad shape");
  if (m == 0) return RS_OK;
  k_eval_tucker<<<(unsigned)ceil_div(m * 32, 256), 256, 0, as_stream(stream)>>>(
      core, (int)r1, (int)r2, (int)r3, V1, V2, V3, idx, m, out);
  return check_launch("rs_eval_tucker");
}

int rs_eval_cct(const double *ul, const double *wl, int64_t Rs, int64_t gamma,
                const int64_t *centers, const double *zq, int64_t count, const int64_t *idx,
                int64_t m, double *out, int32_t *hits, void *stream) {
  RS_REQUIRE(Rs >= 1 && gamma >= 0 && count >= 0 && m >= 0, "rs_eval_cct: bad shape");
  if (m == 0) return RS_OK;
  k_eval_cct<<<(unsigned)ceil_div(m * 32, 256), 256, 0, as_stream(stream)>>>(
      ul, wl, (int)Rs, (int)gamma, centers, zq, count, idx, m, out, hits);
  return check_launch("rs_eval_cct");
}

int rs_pair_sums(const double *table, int64_t ld_table, int64_t n0, const double *w, int64_t Rl,
                 double h3, const int64_t *idx, const double *z, int64_t count, const int64_t *tgt,
                 int64_t m, int mode, double *base, double *dshift, void *stream) {
  RS_REQUIRE(Rl >= 1 && count >= 1 && m >= 0 && mode >= 0 && mode <= 2 && h3 > 0,
             "rs_pair_sums: bad arguments");
  if (m == 0) return RS_OK;
  k_pair_sums<<<(unsigned)m, PS_THREADS, 0, as_stream(stream)>>>(
      table, ld_table, n0, w, (int)Rl, h3, idx, z, count, tgt, mode, base, dshift);
  return check_launch("rs_pair_sums");
}

int64_t rs_sum_workspace_bytes(int64_t m) {
  int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(1024, ceil_div(m, 4096)));
  return blocks * 16;
}

int rs_sum_dd(const double *v, int64_t m, double *out, void *work, int64_t work_bytes,
              void *stream) {
  RS_REQUIRE(m >= 0, "rs_sum_dd: bad size");
  int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(1024, ceil_div(m, 4096)));
  if (work_bytes < blocks * 16) return fail(RS_ERR_CAPACITY, "rs_sum_dd: workspace too small");
  int64_t per = std::max<int64_t>(1, ceil_div(m, blocks));
  cudaStream_t s = as_stream(stream);
  k_sum_dd_part<<<(unsigned)blocks, SUM_THREADS, 0, s>>>(v, m, per, (double *)work);
  int st = check_launch("rs_sum_dd part");
  if (st) return st;
  k_sum_dd_final<<<1, 32, 0, s>>>((double *)work, blocks, out);
  return check_launch("rs_sum_dd final");
}

}  // extern "C"
