// Fused single-pass grid store for the low-overlap (dense-L0) regime:
//
//   out[x1, x2, x3] = Tucker[x1, x2, x3] + sum_p z_p L0[x - c_p + gamma]
//
// (formats.py:448-453 dense_rs = TuckerTensor.dense (formats.py:173-176) +
// dense_cct (formats.py:423-445)).  The two-kernel route stores the short
// part (8 B/pt) and then read-modify-writes it with the Tucker GEMM (16 B/pt);
// the Tucker GEMM is FP64-tensor (DMMA) bound and the gather is L2-load bound,
// so run back to back neither resource is busy while the other works.  Here
// one CTA owns a 64-row block of x2 rows for PL consecutive x1 planes and
// walks every 64-wide x3 tile of each plane (steps u = plane * tiles + tile):
//
//   * warps 0-7 (MMA), two independent groups of four: the A-resident Tucker
//     GEMM of k_tucker_gemm_res -- the plane's A rows (64 x K, K = r3 padded)
//     staged in shared memory, the V3 chunks of every (step, 16-column K
//     chunk) through the group's own cp.async ring, DMMA m8n8k4, 32 x 32 per
//     warp; group g takes the steps u = g mod 2, so one group's chunk barrier
//     never drains the other's tensor pipe.  The epilogue adds the short tile
//     from shared memory and stores the final grid values once (streaming
//     16-byte stores);
//   * warps 8-15 (gather): the short-range tile of the same 64 x 64 points
//     from the L2-resident pair table of L0 (rs_l0.cuh: one 16-byte load per
//     row and copy covers a lane's two x3 neighbours; loads predicated so two
//     copies' loads are in flight together), 8 rows per warp, into a
//     double-buffered shared tile.
//
// Named barriers hand the short tiles over (full[b]: gather -> MMA group b,
// empty[b]: group b -> gather), so the gather of step u+1 overlaps the MMAs of
// step u.  The copies whose windows meet the CTA's rows are found once per
// CTA (x3 bucket layout of rs_front: binary search of the x2 window in each
// c2-sorted bucket, x1 filter by an order-preserving scan) and kept in shared
// memory in bucket (= x3) order; a tile's copies are a contiguous range of
// that list.  A CTA with more copies than the list holds falls back to
// per-tile lists in pages (correct for any density, slower).
//
// The accumulation orders equal those of k_short_l0 (copies in bucket order,
// c2 ascending inside a bucket, fma(z, L0, acc) from 0) and of
// k_tucker_gemm_res (same K order, then acc + short), so the fused grid is
// bitwise equal to the two-kernel route.
#include "rs_dmma.cuh"
#include "rs_fused.cuh"
#include "rs_l0.cuh"

#include <stdlib.h>

namespace rsb {
namespace fz {
constexpr int BM = 64, BN = 64, BK = 16, LDB = BK + 4, STAGES = 3;
constexpr int NMMA = 8, NGATH = 8, THREADS = (NMMA + NGATH) * 32, GTHREADS = NGATH * 32;
constexpr int NGRP = 2, GRP_THREADS = NMMA * 32 / NGRP;  // MMA groups of 4 warps
constexpr int FULL_COUNT = GTHREADS + GRP_THREADS;        // gather warps + one MMA group
constexpr int WM = 32, WN = 32, WARPS_N = BN / WN, MT = WM / 8, NT = WN / 8;
constexpr int PL = 4;                // x1 planes per CTA (one copy list for all of them)
constexpr int LDS_S = BN + 2;        // short tile row stride (doubles)
constexpr int GROWS = BM / NGATH;    // rows per gather warp
constexpr int CAP = 1024;            // staged copies (16 B each)
constexpr int GU = 3;                // copies per gather step
constexpr int KMAX = 176;
// named barriers (0 is __syncthreads)
constexpr int BAR_MMA = 1, BAR_MMA_ALL = 3, BAR_G = 4, BAR_FULL = 5, BAR_EMPTY = 7;

__host__ __device__ constexpr int lda_s(int kc) { return kc * BK + 4; }
__host__ __device__ constexpr int smem_bytes(int kc) {
  return (BM * lda_s(kc) + NGRP * STAGES * BN * LDB + 2 * BM * LDS_S) * 8 + CAP * 16 +
         3 * GTHREADS * 4 + 64;
}

struct Cand {
  int c12;   // c1 | c2 << 16
  int c3;
  double z;
};
}  // namespace fz

namespace {

__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// exclusive scan over the gather threads (named barrier BAR_G)
__device__ __forceinline__ int g_scan(int v, int gtid, int *wsum, int *total) {
  const int lane = gtid & 31, w = gtid >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) wsum[w] = x;
  nbar_sync(fz::BAR_G, fz::GTHREADS);
  int base = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < fz::NGATH; ++k) {
    if (k < w) base += wsum[k];
    tot += wsum[k];
  }
  *total = tot;
  nbar_sync(fz::BAR_G, fz::GTHREADS);
  return base + x - v;
}

// The copies of buckets [b_lo, b_hi) whose window meets planes [x1a, x1b] and rows
// [c2lo + gamma, c2hi - gamma]: filtered copies number `skip` .. skip + CAP - 1
// of that stream are stored (bucket order).  Returns the stream length.
__device__ int g_build(int b_lo, int b_hi, int skip, int gtid, int64_t x1a, int64_t x1b, int gamma,
                       int64_t c2lo, int64_t c2hi, const int32_t *__restrict__ c1,
                       const int32_t *__restrict__ c2, const double *__restrict__ zq,
                       const int32_t *__restrict__ bstart, const int32_t *__restrict__ bc3,
                       fz::Cand *list, int *s_lo, int *s_off, int *s_b3, int *wsum) {
  int count = 0;
  for (int g = b_lo; g < b_hi; g += fz::GTHREADS) {
    const int b = g + gtid;
    int lo = 0, cnt = 0, b3 = 0;
    if (b < b_hi) {
      const int p_lo = bstart[b], p_hi = bstart[b + 1];
      int l = p_lo, h = p_hi;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (c2[m] < c2lo) l = m + 1; else h = m;
      }
      int e = l;
      h = p_hi;
      while (e < h) {
        const int m = (e + h) >> 1;
        if (c2[m] <= c2hi) e = m + 1; else h = m;
      }
      lo = l;
      cnt = e - l;
      b3 = bc3[b];
    }
    int tot;
    const int off = g_scan(cnt, gtid, wsum, &tot);
    s_lo[gtid] = lo;
    s_off[gtid] = off;
    s_b3[gtid] = b3;
    const int nbk = min(fz::GTHREADS, b_hi - g);
    nbar_sync(fz::BAR_G, fz::GTHREADS);
    for (int cs = 0; cs < tot; cs += fz::GTHREADS) {
      const int v = cs + gtid;
      bool cov = false;
      int p = 0, k = 0, a1 = 0;
      if (v < tot) {
        int l = 0, h = nbk;
        while (h - l > 1) {
          const int m = (l + h) >> 1;
          if (s_off[m] <= v) l = m; else h = m;
        }
        k = l;
        p = s_lo[k] + (v - s_off[k]);
        a1 = c1[p];
        cov = a1 >= x1a - gamma && a1 <= x1b + gamma;
      }
      int t2;
      const int pos = g_scan(cov ? 1 : 0, gtid, wsum, &t2);
      const int gi = count + pos - skip;
      if (cov && gi >= 0 && gi < fz::CAP) {
        fz::Cand c;
        c.c12 = a1 | (c2[p] << 16);
        c.c3 = s_b3[k];
        c.z = zq[p];
        list[gi] = c;
      }
      count += t2;
    }
    nbar_sync(fz::BAR_G, fz::GTHREADS);
  }
  return count;
}

__global__ void __launch_bounds__(fz::THREADS, 1)
    k_fused_l0(const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
               int64_t ldb, int K, const double *__restrict__ P, int gamma, int64_t n,
               const int32_t *__restrict__ c1, const int32_t *__restrict__ c2,
               const double *__restrict__ zq, const int32_t *__restrict__ bstart,
               const int32_t *__restrict__ bc3, const int32_t *__restrict__ nbp, int64_t x1_lo,
               int64_t x1_hi, double *__restrict__ C, int mode) {
  using namespace fz;
  extern __shared__ __align__(16) double smem[];
  const int KC = (K + BK - 1) / BK, LDA = lda_s(KC);
  double *sA = smem;
  double *sB = sA + BM * LDA;                       // one ring per MMA group
  double *sS = sB + NGRP * STAGES * BN * LDB;
  Cand *list = reinterpret_cast<Cand *>(sS + 2 * BM * LDS_S);
  int *s_lo = reinterpret_cast<int *>(list + CAP);
  int *s_off = s_lo + GTHREADS, *s_b3 = s_off + GTHREADS;
  int *wsum = s_b3 + GTHREADS;
  const int64_t nx2b = n / BM;
  const int64_t X1 = x1_lo + (int64_t)(blockIdx.x / nx2b) * PL;
  const int64_t X2 = (int64_t)(blockIdx.x % nx2b) * BM;
  const int npl = (int)min((int64_t)PL, x1_hi - X1);
  const int ntiles = (int)((n + BN - 1) / BN);
  const int utot = npl * ntiles;  // (plane, x3 tile) steps of this CTA, u = pl ntiles + t
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp < NMMA) {
    // ------------------------------------------------------------ MMA warps
    // two independent groups of 4 warps (64 x 64 tiles, 32 x 32 per warp):
    // group g takes the steps u = g, g + 2, ... with its own cp.async ring
    // and barrier, so one group's chunk barrier never drains the other's DMMAs
    const int grp = warp / (NMMA / NGRP), gtid = threadIdx.x - grp * GRP_THREADS;
    const int gwarp = warp - grp * (NMMA / NGRP);
    const int nmine = (utot - grp + 1) / 2;
    const int total = nmine * KC;
    const int wm0 = (gwarp / WARPS_N) * WM, wn0 = (gwarp % WARPS_N) * WN;
    const int gid = lane >> 2, tig = lane & 3;
    double *ring = sB + grp * STAGES * BN * LDB;
    auto load_a = [&](int pl) {  // resident A rows of plane X1 + pl (zero past K), all MMA warps
      const double *Ap = A + ((X1 + pl - x1_lo) * n + X2) * lda;
      for (int e = threadIdx.x; e < BM * (KC * BK / 2); e += NMMA * 32) {
        const int r = e / (KC * BK / 2), kk = 2 * (e - r * (KC * BK / 2));
        const bool ok = kk < K;
        const int bytes = ok ? (kk + 1 < K ? 16 : 8) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                         smem_addr(sA + r * LDA + kk)),
                     "l"(ok ? Ap + r * lda + kk : Ap), "r"(bytes));
      }
    };
    auto load_b = [&](int c) {
      const int k = c / KC, kc = c - k * KC, t = (grp + 2 * k) % ntiles;
      double *st = ring + (c % STAGES) * BN * LDB;
#pragma unroll
      for (int e0 = 0; e0 < BN * BK / 2; e0 += GRP_THREADS) {
        const int e = e0 + gtid;
        const int r = e / (BK / 2), kk = kc * BK + 2 * (e % (BK / 2));
        const int64_t g = (int64_t)t * BN + r;
        const bool ok = g < n && kk < K;
        const int bytes = ok ? (kk + 1 < K ? 16 : 8) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                         smem_addr(st + r * LDB + 2 * (e % (BK / 2)))),
                     "l"(ok ? B + g * ldb + kk : B), "r"(bytes));
      }
    };
    load_a(0);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < total) load_b(s);
      cp_async_commit();
    }
    cp_async_wait<0>();
    nbar_sync(BAR_MMA_ALL, NMMA * 32);  // sA complete for both groups
    double acc[MT][NT][2];
    int cur_pl = 0;
    for (int c = 0; c < total; ++c) {
      const int k = c / KC, kc = c - k * KC;
      const int u = grp + 2 * k, pl = u / ntiles, t = u - pl * ntiles;
      if (kc == 0) {
        if (pl != cur_pl) {  // next plane: both groups are done with sA
          nbar_sync(BAR_MMA_ALL, NMMA * 32);
          load_a(pl);
          cp_async_commit();
          cp_async_wait<0>();
          nbar_sync(BAR_MMA_ALL, NMMA * 32);
          cur_pl = pl;
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      }
      cp_async_wait<STAGES - 2>();
      nbar_sync(BAR_MMA + grp, GRP_THREADS);
      if (c + STAGES - 1 < total) load_b(c + STAGES - 1);
      cp_async_commit();
      const double *st = ring + (c % STAGES) * BN * LDB;
      const int kv = (mode & 2) ? 0 : min(BK, K - kc * BK);  // mode 2: no MMAs (diagnostic)
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        if (kk >= kv) break;
        double a[MT], b[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = sA[(wm0 + i * 8 + gid) * LDA + kc * BK + kk + tig];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = st[(wn0 + j * 8 + gid) * LDB + kk + tig];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma_884(acc[i][j], a[i], b[j]);
      }
      if (kc == KC - 1) {
        const int bf = u & 1;  // == grp
        nbar_sync(BAR_FULL + bf, FULL_COUNT);
        const double *S = sS + bf * BM * LDS_S;
        double *Cp = C + ((X1 + pl - x1_lo) * n + X2) * n + (int64_t)t * BN;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int rl = wm0 + i * 8 + gid;
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int cl = wn0 + j * 8 + tig * 2;
            const double2 sv = *reinterpret_cast<const double2 *>(S + rl * LDS_S + cl);
            const double v0 = acc[i][j][0] + sv.x, v1 = acc[i][j][1] + sv.y;
            if ((int64_t)t * BN + cl < n)   // n even: the pair is inside
              __stcs(reinterpret_cast<double2 *>(Cp + (int64_t)rl * n + cl), make_double2(v0, v1));
          }
        }
        if (u + 2 < utot) nbar_arrive(BAR_EMPTY + bf, FULL_COUNT);
      }
    }
    cp_async_wait<0>();
    return;
  }

  // -------------------------------------------------------------- gather warps
  const int gtid = threadIdx.x - NMMA * 32, gw = warp - NMMA;
  const int W = 2 * gamma + 1;
  const int64_t c2lo = X2 - gamma, c2hi = min(X2 + BM, n) - 1 + gamma;
  const int nb = *nbp;
  const int total0 = g_build(0, nb, 0, gtid, X1, X1 + npl - 1, gamma, c2lo, c2hi, c1, c2, zq,
                             bstart, bc3, list, s_lo, s_off, s_b3, wsum);
  const bool paged = total0 > CAP;
  const uint64_t pol = l0_evict_last();
  const int r0 = gw * GROWS;
  const int64_t xr0 = X2 + r0;
  for (int u = 0; u < utot; ++u) {
    const int pl = u / ntiles, t = u - pl * ntiles;
    const int64_t x1 = X1 + pl;
    const int bf = u & 1;
    const int64_t X3 = (int64_t)t * BN;
    const int64_t lo_x = X3 - gamma, hi_x = min(X3 + BN, n) - 1 + gamma;
    double2 acc[GROWS];
#pragma unroll
    for (int r = 0; r < GROWS; ++r) acc[r] = make_double2(0.0, 0.0);
    // lane l: x3 pair (2l, 2l + 1) of the tile, one 16-byte L0 load per row
    auto one = [&](const Cand &cd, double2 (&v)[GROWS]) {
      const int da = abs((int)(x1 - (cd.c12 & 0xFFFF)));
      const int cA = (int)(X3 + 2 * lane - cd.c3) + gamma;
      const int par = cA & 1;
      const int b0 = (int)(xr0 - (cd.c12 >> 16)) + gamma;
      const bool ok = da <= gamma && (unsigned)(cA + 1) <= (unsigned)W;
      const double *p = P + l0_off(par, min(da, gamma), b0, cA, gamma);
#pragma unroll
      for (int r = 0; r < GROWS; ++r)
        v[r] = l0_ld2(p + r * L0_PITCH, ok && (unsigned)(b0 + r) < (unsigned)W, pol);
    };
    auto gather = [&](int e0, int e1) {
      int e = e0;
      for (; e + GU <= e1; e += GU) {  // GU copies' loads in flight together
        Cand cs[GU];
        double2 v[GU][GROWS];
#pragma unroll
        for (int q = 0; q < GU; ++q) {
          cs[q] = list[e + q];
          one(cs[q], v[q]);
        }
#pragma unroll
        for (int q = 0; q < GU; ++q)
#pragma unroll
          for (int r = 0; r < GROWS; ++r) {
            acc[r].x = fma(cs[q].z, v[q][r].x, acc[r].x);
            acc[r].y = fma(cs[q].z, v[q][r].y, acc[r].y);
          }
      }
      for (; e < e1; ++e) {
        const Cand ca = list[e];
        double2 va[GROWS];
        one(ca, va);
#pragma unroll
        for (int r = 0; r < GROWS; ++r) {
          acc[r].x = fma(ca.z, va[r].x, acc[r].x);
          acc[r].y = fma(ca.z, va[r].y, acc[r].y);
        }
      }
    };
    if (mode & 1) {  // diagnostic: no gather
    } else if (!paged) {
      // the list is in bucket (x3) order: the tile's copies are [e_lo, e_hi)
      int l = 0, h = total0;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (list[m].c3 < lo_x) l = m + 1; else h = m;
      }
      const int e_lo = l;
      h = total0;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (list[m].c3 <= hi_x) l = m + 1; else h = m;
      }
      gather(e_lo, l);
    } else {
      // per-tile lists of the tile's x3 band, in pages of CAP copies
      int l = 0, h = nb;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (bc3[m] < lo_x) l = m + 1; else h = m;
      }
      const int b_lo = l;
      h = nb;
      while (l < h) {
        const int m = (l + h) >> 1;
        if (bc3[m] <= hi_x) l = m + 1; else h = m;
      }
      const int b_hi = l;
      for (int skip = 0;; skip += CAP) {
        nbar_sync(BAR_G, GTHREADS);  // every gather warp is done with the list
        const int tot = g_build(b_lo, b_hi, skip, gtid, x1, x1, gamma, c2lo, c2hi, c1, c2, zq,
                                bstart, bc3, list, s_lo, s_off, s_b3, wsum);
        gather(0, min(CAP, tot - skip));
        if (tot <= skip + CAP) break;
      }
    }
    if (u >= 2) nbar_sync(BAR_EMPTY + bf, FULL_COUNT);
    double *S = sS + bf * BM * LDS_S;
#pragma unroll
    for (int r = 0; r < GROWS; ++r)
      *reinterpret_cast<double2 *>(S + (r0 + r) * LDS_S + 2 * lane) = acc[r];
    nbar_arrive(BAR_FULL + bf, FULL_COUNT);
  }
}

}  // namespace

int fused_l0_smem_bytes(int64_t K) { return fz::smem_bytes((int)ceil_div(K, fz::BK)); }

bool fused_l0_supported(int64_t n, int64_t K, int64_t gamma) {
  return K >= 1 && K <= fz::KMAX && n % (2 * fz::BN) == 0 && n <= 32768 && l0_gamma_ok(gamma) &&
         fused_l0_smem_bytes(K) <= 227 * 1024;
}

int launch_fused_l0(const double *A, int64_t lda, const double *Bt, int64_t ldb, int64_t K,
                    const double *L0, int64_t gamma, int64_t n, const int32_t *c1,
                    const int32_t *c2, const double *zq, const int32_t *bstart,
                    const int32_t *bc3, const int32_t *nb_dev, int64_t x1_lo, int64_t x1_hi,
                    double *out, cudaStream_t s) {
  RS_REQUIRE(fused_l0_supported(n, K, gamma), "fused_l0: unsupported shape (n=%lld K=%lld)",
             (long long)n, (long long)K);
  const int smem = fused_l0_smem_bytes(K);
  cudaError_t e = smem_attr((const void *)k_fused_l0, smem);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  const int mode = getenv("RSB200_FUSED_MODE") ? atoi(getenv("RSB200_FUSED_MODE")) : 0;
  ProfScope ps(s, "fused_l0");
  const int64_t ctas = ceil_div(x1_hi - x1_lo, fz::PL) * (n / fz::BM);
  k_fused_l0<<<(unsigned)ctas, fz::THREADS, smem, s>>>(A, lda, Bt, ldb, (int)K, L0, (int)gamma, n,
                                                       c1, c2, zq, bstart, bc3, nb_dev, x1_lo,
                                                       x1_hi, out, mode);
  return check_launch("fused_l0");
}

}  // namespace rsb
