// Short-range agglomeration fused onto the FP64 tensor cores
// (formats.py:423-445, dense_cct):
//
//   P_short[x] = sum_p z_p sum_k wl_k ul_k[x1-c1p+g] ul_k[x2-c2p+g] ul_k[x3-c3p+g]
//
// Output-stationary: a CTA owns an 8 (x1) x 16 (x2) x 64 (x3) tile and, for it,
// the GEMM  C[(x1,x2), x3] = sum_col A[(x1,x2), col] B[x3, col]  whose columns
// are (x3 bucket s, term k) pairs:
//
//   A[(x1,x2),(s,k)] = sum_{p in bucket s near the tile} z_p v_k[x1-c1p] v_k[x2-c2p]
//   B[x3,(s,k)]      = v_k[x3-s],            v_k = cbrt(wl_k) ul_k (zero off the window)
//
// Neither operand ever exists in memory.  The per-particle 1-D factors v_k are
// staged once per CTA in shared memory (k-major, zero margins, pitch = 4 mod 16
// doubles so the fragment gathers below are bank-conflict free); every lane
// forms its own mma.m8n8k4 A fragment -- the outer product of the staged
// factors summed over the bucket's candidate copies, 1 DMUL + 2 DFMA per copy
// against the 16 DMMAs (4096 FMAs) the fragment feeds -- and gathers its B
// fragment straight from the same table.  Warp w owns plane x1 = X0 + w, so
// the x1 factor is one value per (copy, term) and lane; there is no operand
// staging, no barrier and no cp.async pipeline inside the K loop.
//
// Sparsity (the same 1e-18 drop rule as the plane GEMM's bands, k_term_prefix):
// a copy contributes term k to a tile only when the tile lies within g_k cells
// of it in all three coordinates; terms are ordered widest first, so copy p
// brings its first kofd[Chebyshev distance(tile, p)] terms and a bucket's
// column count is the maximum over its copies.  Buckets without a copy near
// the tile cost nothing.
//
// Candidates come from rs_front's x3-bucket layout (bucket range by binary
// search over bc3, x2 window by binary search in the c2-sorted bucket, x1
// filter + order-preserving block scan), are staged SM_CAP at a time and
// consumed in bucket order: deterministic.  CTAs take tiles from an atomic
// counter, x3 fastest, and retire after a bounded number of them (the factor
// table is staged once per CTA).
// Roofline: FP64 tensor pipe (DMMA); algorithmic work 2 flops per (grid
// point, covering copy) pair.
#include "rs_common.cuh"
#include "rs_dmma.cuh"

#include <algorithm>
#include <stdlib.h>
#include <string.h>

extern "C" int rsb_asm_term_prefix(const double *ul, const double *wl, int Rs, int gamma,
                                   void *work, cudaStream_t s);  // rs_kernels.cu

namespace rsb {
namespace {

constexpr int SM_T1 = 8;       // x1 planes per tile = warps per CTA
constexpr int SM_T2 = 16;      // x2 rows per tile (2 MMA row groups)
constexpr int SM_T3 = 64;      // x3 columns per tile (8 MMA column groups)
constexpr int SM_THREADS = 256;
constexpr int SM_PAD = 64;     // zero margin of the factor table, >= every tile edge
constexpr int SM_CAP = 512;    // staged candidate copies per MMA phase
constexpr int SM_MAXR = 24;    // largest short rank
constexpr int SM_MAXT3 = 256;  // x3 tiles per grid row (n <= 16384)
constexpr int SM_ACH = 16;     // columns per staged A chunk (builder variant)
constexpr int SM_GRP = 4;      // x3 tiles per candidate search (low-overlap systems)
constexpr int SM_ALD = 132;    // doubles per A column: 8 planes x 16 rows + 4 (= 4 mod 16)

__host__ __device__ inline int sm_pitch(int gamma) {
  int ld = 2 * gamma + 1 + 2 * SM_PAD;
  while (ld % 16 != 4) ++ld;
  return ld;
}

struct SmLayout {
  int table, rec, cb, kn, seg, grp, kofd, abuf, d12, total;  // byte offsets
};

// one staged candidate copy: charge and the two table offsets of its window
struct __align__(16) SmRec {
  double z;
  int o1, o2;   // X0 - c1 + gamma + PAD,  Y0 - c2 + gamma + PAD
};

// one segment (= bucket run) of an MMA phase
struct __align__(16) SmSeg {
  int q_lo;     // first staged copy
  int col;      // columns before this segment
  int K;        // its column count (live terms)
  int bo;       // B offset Z0 - s + gamma + PAD
};

__host__ __device__ inline SmLayout sm_layout(int gamma, int Rs, bool build = false,
                                              bool grouped = false) {
  SmLayout L;
  int o = 0;
  L.table = o; o += Rs * sm_pitch(gamma) * 8;
  L.rec = o;   o += SM_CAP * 16;
  L.seg = o;   o += (SM_CAP + 1) * 16;           // + sentinel
  L.cb = o;    o += (SM_CAP + 4) * 4;            // bucket id (B offset) per staged copy
  L.kn = o;    o += (SM_CAP + 4) * 4;            // live terms per staged copy
  L.grp = o;   o += 3 * SM_THREADS * 4 + 64;     // per-bucket lo / offset / x3 of a group
  L.kofd = o;  o += (gamma + 2) * 4;
  o = (o + 15) & ~15;
  L.abuf = o;  o += build ? 2 * SM_ACH * SM_ALD * 8 : 0;   // two A chunks (builder variant)
  L.d12 = o;   o += grouped ? (SM_CAP + 4) * 4 : 0;        // (x1, x2) distance per staged copy
  L.total = (o + 15) & ~15;
  return L;
}

__device__ __forceinline__ int sm_block_scan(int v, int *wsum, int *total) {
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
#pragma unroll
  for (int w = 0; w < SM_THREADS / 32; ++w) {
    if (w < warp) base += wsum[w];
    tot += wsum[w];
  }
  *total = tot;
  __syncthreads();
  return base + x - v;
}

// Coarse x2 index of the bucket-ordered copies: y16[b * ldy + j] = first copy p
// of bucket b (c2 ascending inside a bucket) with c2[p] >= 16 j; the last
// entry is the bucket's end.  Two lookups replace the two binary searches a
// tile would run per bucket.
__global__ void k_x2_index(const int32_t *__restrict__ c2, const int32_t *__restrict__ bstart,
                           const int32_t *__restrict__ nbp, int ldy, int32_t *__restrict__ y16) {
  const int nb = *nbp;
  const int64_t total = (int64_t)nb * ldy;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / ldy), j = (int)(e - (int64_t)b * ldy);
    int l = bstart[b], h = bstart[b + 1];
    const int key = 16 * j;
    while (l < h) {
      const int m = (l + h) >> 1;
      if (c2[m] < key) l = m + 1; else h = m;
    }
    y16[e] = j == ldy - 1 ? bstart[b + 1] : l;
  }
}

// explicit shared-space loads (32-bit addresses): the generic-pointer form made
// the compiler rebuild the shared window base inside the K loop
__device__ __forceinline__ double sm_lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
template <int OFF>
__device__ __forceinline__ double sm_lds_at(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
  return v;
}
__device__ __forceinline__ void sm_lds_rec(uint32_t a, double &z, int &o1, int &o2) {
  int lo, hi;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(lo), "=r"(hi), "=r"(o1), "=r"(o2)
               : "r"(a));
  z = __hiloint2double(hi, lo);
}

// 8-bit mask of the 8-wide x3 blocks j of a tile in which column (bucket s,
// term k) can be nonzero: |Z0 + 8 j + t - s| <= g_k for some t in [0, 8).
// e = Z0 - s.  Beyond g_k the term is below the drop threshold (k_term_prefix).
__device__ __forceinline__ unsigned sm_live_blocks(int e, int g) {
  const int jlo = max((-e - g) >> 3, 0), jhi = min((g - e) >> 3, 7);
  return jhi < jlo ? 0u : ((2u << jhi) - 1u) & ~((1u << jlo) - 1u);
}

template <bool ACC, bool BUILD, bool SKIP, int GRP, int NJ>
__global__ void __launch_bounds__(SM_THREADS, NJ == 4 ? 3 : 2)
    k_short_mma(const double *__restrict__ ul, const double *__restrict__ wl, int Rs, int gamma,
                int64_t n, const int32_t *__restrict__ c1, const int32_t *__restrict__ c2,
                const double *__restrict__ zq, const int32_t *__restrict__ bstart,
                const int32_t *__restrict__ bc3, const int32_t *__restrict__ nbp,
                const int *__restrict__ kofd_g, const int32_t *__restrict__ y16, int ldy,
                int64_t x1_lo, int64_t x1_hi, int *__restrict__ counter, int tiles_per_cta,
                int one, double *__restrict__ out) {
  constexpr int T3 = 8 * NJ;   // x3 columns per tile: NJ MMA column blocks
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const SmLayout L = sm_layout(gamma, Rs, BUILD, GRP > 1);
  double *ut = (double *)(sm_raw + L.table);
  SmRec *s_rec = (SmRec *)(sm_raw + L.rec);
  SmSeg *s_seg = (SmSeg *)(sm_raw + L.seg);
  int *s_cb = (int *)(sm_raw + L.cb);
  int *s_kn = (int *)(sm_raw + L.kn);
  int *s_lo = (int *)(sm_raw + L.grp);
  int *s_off = s_lo + SM_THREADS;
  int *s_b3 = s_off + SM_THREADS;
  int *skofd = (int *)(sm_raw + L.kofd);
  int *s_d12 = (int *)(sm_raw + L.d12);
  __shared__ int wsum[SM_THREADS / 32];
  __shared__ int s_tile[2];
  __shared__ int s_bands[2 * SM_MAXT3];   // bucket band [lo, hi) of every x3 tile
  __shared__ int s_gk[SM_MAXR];           // reach g_k of term k (cells), from kofd

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int W = 2 * gamma + 1, LD = sm_pitch(gamma);
  const int nb = *nbp;
  // x1 tiles sit on absolute multiples of SM_T1, so a slab's values do not
  // depend on where the slab starts (same candidates, same term cuts, same sums)
  const int64_t x1_base = x1_lo - x1_lo % SM_T1;
  const int n3t = (int)((n + T3 - 1) / T3), n2t = (int)((n + SM_T2 - 1) / SM_T2);
  // work items: groups of GRP consecutive x3 tiles (one candidate search per group)
  const int n3g = (n3t + GRP - 1) / GRP;
  const int64_t ntiles = (int64_t)n3g * n2t * ((x1_hi - x1_base + SM_T1 - 1) / SM_T1);

  // the factor table, once per CTA: v_k[d] = cbrt(wl_k) ul[d, k] inside the
  // window, zero in the margins
  for (int e = tid; e < Rs * LD; e += SM_THREADS) ut[e] = 0.0;
  for (int d = tid; d <= gamma; d += SM_THREADS) skofd[d] = kofd_g[d];
  __syncthreads();
  for (int e = tid; e < Rs * W; e += SM_THREADS) {   // coalesced read of ul (W x Rs)
    const int d = e / Rs, k = e - d * Rs;
    ut[k * LD + SM_PAD + d] = cbrt(wl[k]) * ul[e];
  }
  if (tid < Rs) {   // g_k = the largest distance at which term k is still kept
    int g = -1;
    for (int d = 0; d <= gamma; ++d)
      if (skofd[d] > tid) g = d;
    s_gk[tid] = g;
  }
  // occupied x3 buckets within gamma of each x3 tile: found once per CTA, all
  // tiles in parallel (per tile this was ~18 dependent global loads by one
  // thread with the CTA waiting at a barrier)
  for (int t3 = tid; t3 < n3t; t3 += SM_THREADS) {
    const int lo_x = t3 * T3 - gamma, hi_x = t3 * T3 + T3 - 1 + gamma;
    int l = 0, h = nb;
    while (l < h) {
      const int m = (l + h) >> 1;
      if (bc3[m] < lo_x) l = m + 1; else h = m;
    }
    s_bands[2 * t3] = l;
    h = nb;
    while (l < h) {
      const int m = (l + h) >> 1;
      if (bc3[m] <= hi_x) l = m + 1; else h = m;
    }
    s_bands[2 * t3 + 1] = l;
  }

  // a CTA retires after tiles_per_cta tiles: the turnover lets the kernels of a
  // higher-priority stream (the latency-bound Gram / eigen / core chain) onto
  // the SMs between two CTAs instead of behind the whole grid
  if (tid == 0) s_tile[0] = atomicAdd(counter, 1);
  for (int done = 0; done < tiles_per_cta; ++done) {
    __syncthreads();   // previous tile done with the staging arrays; table complete
    const int64_t tile = s_tile[done & 1];
    if (tile >= ntiles) break;
    // the next tile's index is requested now: the atomic's latency hides under this tile
    if (tid == 0 && done + 1 < tiles_per_cta) s_tile[(done + 1) & 1] = atomicAdd(counter, 1);
    const int t3g = (int)(tile % n3g), t2 = (int)((tile / n3g) % n2t);
    const int64_t t1 = tile / ((int64_t)n3g * n2t);
    const int X0 = (int)(x1_base + t1 * SM_T1), Y0 = t2 * SM_T2;
    const int t3_lo = t3g * GRP, t3_hi = min(t3_lo + GRP, n3t);
    int Z0 = t3_lo * T3;   // the x3 tile in work (set per tile below)

    double acc[2][NJ][2];
    auto zero_acc = [&]() {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    };

    // one MMA phase over the staged copies [base, base + len) (s_cb = their x3 index, s_kn =
    // their live terms for the tile at Z0): segments = runs of equal bucket, column count =
    // max live terms of the run's copies
    auto flush = [&](int base, int len) {
      __syncthreads();
      const int end = base + len;
      int nseg = 0, ncol = 0;
      for (int i0 = 0; i0 < len; i0 += SM_THREADS) {
        const int i = base + i0 + tid;
        const bool start = i < end && (i == base || s_cb[i] != s_cb[i - 1]);
        int K = 0;
        if (start) {   // the run is short (copies of one bucket near the tile)
          const int id = s_cb[i];
          for (int q = i; q < end && s_cb[q] == id; ++q) K = max(K, s_kn[q]);
        }
        int tot;   // one scan for both the segment index (low half) and the column prefix
        const int pre = sm_block_scan(start ? (K << 12) | 1 : 0, wsum, &tot);
        if (start) {
          SmSeg sg;
          sg.q_lo = i;
          sg.col = ncol + (pre >> 12);
          sg.K = K;
          sg.bo = Z0 - s_cb[i] + gamma + SM_PAD;   // B offset of the bucket for this tile
          s_seg[nseg + (pre & 0xFFF)] = sg;
        }
        nseg += tot & 0xFFF;
        ncol += tot >> 12;
      }
      if (tid == 0) {
        SmSeg sg;
        sg.q_lo = end;
        sg.col = ncol;
        sg.K = 0;
        sg.bo = 0;
        s_seg[nseg] = sg;
      }
      __syncthreads();
      if (one < 0) ncol = 0;
      if constexpr (!BUILD) {
        const int steps = (ncol + 3) >> 2;
        int si = -1, seg_end = 0, col0 = 0, e3 = 0;
        uint32_t qa_lo = 0, qa_hi = 0, bob = 0;
        const uint32_t ut_s = smem_addr(ut), rec_s = smem_addr(s_rec), seg_s = smem_addr(s_seg);
        const uint32_t ut1_s = ut_s + 8 * warp, ut2_s = ut_s + 8 * gid;
        const int LDb = LD * 8;
        for (int st = 0; st < steps; ++st) {
          const int c = 4 * st + tig;
          double a0 = 0.0, a1 = 0.0, b[NJ];
          unsigned own = 0;   // x3 blocks of the tile this lane's column reaches
          uint32_t ub = ut2_s;
          if (c < ncol) {
            if (c >= seg_end) {   // this lane's column enters a new segment
              int q_lo, K, bo, nq;
              do {
                ++si;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(q_lo), "=r"(col0), "=r"(K), "=r"(bo)
                             : "r"(seg_s + 16 * si));
                seg_end = col0 + K;
              } while (c >= seg_end);
              asm volatile("ld.shared.b32 %0, [%1+16];" : "=r"(nq) : "r"(seg_s + 16 * si));
              qa_lo = rec_s + 16 * q_lo;
              qa_hi = rec_s + 16 * nq;
              bob = 8 * bo;
              e3 = bo - gamma - SM_PAD;
            }
            own = SKIP ? sm_live_blocks(e3, s_gk[c - col0]) : (1u << NJ) - 1u;
            const uint32_t koff = (uint32_t)((c - col0) * LDb);
            const uint32_t u1 = ut1_s + koff, u2 = ut2_s + koff;
  #pragma unroll 2
            for (uint32_t qa = qa_lo; qa < qa_hi; qa += 16) {
              double z;
              int o1, o2;
              sm_lds_rec(qa, z, o1, o2);
              const double t = z * sm_lds(u1 + o1);
              const uint32_t w2 = u2 + o2;
              a0 = fma(t, sm_lds(w2), a0);
              a1 = fma(t, sm_lds_at<64>(w2), a1);
            }
            ub = u2 + bob;
          }
          // the step's 4 columns (mostly consecutive terms of one bucket) reach only
          // some of the tile's 8 x3 blocks: the others' MMAs and B loads are skipped
          const unsigned live = SKIP ? __reduce_or_sync(0xffffffffu, own) : (1u << NJ) - 1u;
#pragma unroll
          for (int j = 0; j < NJ; ++j) b[j] = (own & (1u << j)) ? sm_lds(ub + 64 * j) : 0.0;
  #pragma unroll
          for (int j = 0; j < NJ; ++j) {
            if (SKIP) {
              // a predicated-off DMMA costs the pipe as much as a live one
              // (tools/probe_dmma_pred.cu), and ptxas if-converts any plain `if` around
              // the pair: the trip count `one` (= 1, a kernel argument) keeps the branch
              if (live & (1u << j)) {
  #pragma unroll 1
                for (int r = 0; r < one; ++r) {
                  dmma_884(acc[0][j], a0, b[j]);
                  dmma_884(acc[1][j], a1, b[j]);
                }
              }
            } else {
              dmma_884(acc[0][j], a0, b[j]);
              dmma_884(acc[1][j], a1, b[j]);
            }
          }
        }
      } else {
        // Builder variant (many copies per bucket: C2-C4).  The 128 A values of a
        // column, A[(x1,x2)] = sum_p (z_p v_k[x1-c1p]) v_k[x2-c2p], are a rank-(copies)
        // product P (8 x copies) Q (copies x 16): ONE warp forms them with
        // mma.m8n8k4 itself (2 DMMAs per 4 copies) from 3 table loads per lane and
        // 4 copies, instead of every lane of every warp re-reading the copies'
        // records and x2 factors (8x redundant across the planes, and the shared-
        // memory bandwidth bound of the per-lane form).  Columns go through a
        // double-buffered shared A chunk of 16; warp w builds columns 2w, 2w + 1 of
        // the next chunk, then runs the 4 k-steps of the current one: one barrier
        // per chunk.
        const uint32_t ut_s = smem_addr(ut), rec_s = smem_addr(s_rec), seg_s = smem_addr(s_seg);
        const uint32_t ab_s = smem_addr(sm_raw + L.abuf);
        const int LDb = LD * 8;
        const int nchunks = (ncol + SM_ACH - 1) / SM_ACH;
        int bsi = -1, bseg_end = 0, bcol0 = 0;      // builder cursor (warp-uniform)
        uint32_t bqa_lo = 0, bqa_hi = 0;
        auto build = [&](int ch) {
          const uint32_t buf = ab_s + (uint32_t)((ch & 1) * SM_ACH * SM_ALD * 8);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int cl = 2 * warp + u, c = ch * SM_ACH + cl;
            double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
            if (c < ncol) {
              if (c >= bseg_end) {
                int q_lo, K, bo, nq;
                do {
                  ++bsi;
                  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(q_lo), "=r"(bcol0), "=r"(K), "=r"(bo)
                               : "r"(seg_s + 16 * bsi));
                  bseg_end = bcol0 + K;
                } while (c >= bseg_end);
                asm volatile("ld.shared.b32 %0, [%1+16];" : "=r"(nq) : "r"(seg_s + 16 * bsi));
                bqa_lo = rec_s + 16 * q_lo;
                bqa_hi = rec_s + 16 * nq;
              }
              const uint32_t ug = ut_s + (uint32_t)((c - bcol0) * LDb) + 8 * gid;
              for (uint32_t qa = bqa_lo; qa < bqa_hi; qa += 64) {   // 4 copies per step
                const uint32_t mine = qa + 16 * tig;
                double z = 0.0;
                int o1 = 0, o2 = 0;                 // offset 0: the table's zero margin
                if (mine < bqa_hi) sm_lds_rec(mine, z, o1, o2);
                const double av = z * sm_lds(ug + o1);
                const uint32_t w2 = ug + o2;
                dmma_884(d0, av, sm_lds(w2));
                dmma_884(d1, av, sm_lds_at<64>(w2));
              }
            }
            // A[col][x1 = gid][x2 = 2 tig .. +1] and [x2 = 8 + 2 tig .. +1]
            const uint32_t dst = buf + (uint32_t)((cl * SM_ALD + gid * 16 + 2 * tig) * 8);
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(dst), "d"(d0[0]), "d"(d0[1]));
            asm volatile("st.shared.v2.f64 [%0+64], {%1, %2};" ::"r"(dst), "d"(d1[0]), "d"(d1[1]));
          }
        };
        int si = -1, seg_end = 0, col0 = 0, e3 = 0;  // per-lane cursor of the main loop
        uint32_t bob = 0;
        const uint32_t ut2_s = ut_s + 8 * gid;
        if (nchunks > 0) build(0);
        __syncthreads();
        for (int ch = 0; ch < nchunks; ++ch) {
          if (ch + 1 < nchunks) build(ch + 1);
          const uint32_t buf = ab_s + (uint32_t)((ch & 1) * SM_ACH * SM_ALD * 8) +
                               (uint32_t)((warp * 16 + gid) * 8);
#pragma unroll
          for (int ks = 0; ks < SM_ACH / 4; ++ks) {
            const int c = ch * SM_ACH + 4 * ks + tig;
            if (4 * ks + ch * SM_ACH >= ncol) break;   // uniform: no live column in this step
            const uint32_t ap = buf + (uint32_t)((4 * ks + tig) * SM_ALD * 8);
            const double a0 = sm_lds(ap), a1 = sm_lds_at<64>(ap);
            double b[NJ];
            unsigned own = 0;
            uint32_t ub = ut2_s;
            if (c < ncol) {
              if (c >= seg_end) {
                int q_lo, K, bo;
                do {
                  ++si;
                  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(q_lo), "=r"(col0), "=r"(K), "=r"(bo)
                               : "r"(seg_s + 16 * si));
                  seg_end = col0 + K;
                } while (c >= seg_end);
                bob = 8 * bo;
                e3 = bo - gamma - SM_PAD;
              }
              own = SKIP ? sm_live_blocks(e3, s_gk[c - col0]) : (1u << NJ) - 1u;
              ub = ut2_s + (uint32_t)((c - col0) * LDb) + bob;
            }
            const unsigned live = SKIP ? __reduce_or_sync(0xffffffffu, own) : (1u << NJ) - 1u;
#pragma unroll
            for (int j = 0; j < NJ; ++j) b[j] = (own & (1u << j)) ? sm_lds(ub + 64 * j) : 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              if (SKIP) {
                if (live & (1u << j)) {
#pragma unroll 1
                  for (int r = 0; r < one; ++r) {
                    dmma_884(acc[0][j], a0, b[j]);
                    dmma_884(acc[1][j], a1, b[j]);
                  }
                }
              } else {
                dmma_884(acc[0][j], a0, b[j]);
                dmma_884(acc[1][j], a1, b[j]);
              }
            }
          }
          __syncthreads();
        }
      }
    };

    const int c1lo = X0 - gamma, c1hi = X0 + SM_T1 - 1 + gamma;
    const int c2lo = Y0 - gamma, c2hi = Y0 + SM_T2 - 1 + gamma;

    // epilogue: every grid point of the tile at Z0 is written once
    auto epilogue = [&]() {
      const int64_t x1 = X0 + warp;
      if (x1 >= x1_lo && x1 < x1_hi) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int64_t x2 = Y0 + 8 * i + gid;
          if (x2 >= n) continue;
          double *row = out + ((x1 - x1_lo) * n + x2) * n + Z0 + 2 * tig;
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const int64_t x3 = Z0 + 8 * j + 2 * tig;
            double v0 = acc[i][j][0], v1 = acc[i][j][1];
            if (x3 + 1 < n) {
              double2 *p = reinterpret_cast<double2 *>(row + 8 * j);
              if (ACC) {
                const double2 o = __ldcs(p);
                v0 += o.x;
                v1 += o.y;
              }
              __stcs(p, make_double2(v0, v1));
            } else if (x3 < n) {
              if (ACC) v0 += __ldcs(row + 8 * j);
              __stcs(row + 8 * j, v0);
            }
          }
        }
      }
    };

    // Candidate copies of the x3 tiles [ta, tb) (same x1, x2 window; the union of
    // their bucket bands), bucket group by bucket group, staged in bucket order.
    // grouped = false: one tile; the live terms are known at staging and a full
    // staging area is flushed on the way (returns the copies still staged).
    // grouped = true: nothing is flushed; returns -1 when the area overflows.
    auto search = [&](int ta, int tb, bool grouped) -> int {
      const int blo = s_bands[2 * ta], bhi = s_bands[2 * (tb - 1) + 1];
      int len = 0;
      bool over = false;
      for (int g = blo; g < bhi; g += SM_THREADS) {
        const int bi = g + tid;
        int lo = 0, cnt = 0, b3 = 0;
        if (bi < bhi) {  // the bucket's copies in the 16-cell x2 blocks the window meets
          b3 = bc3[bi];
          const int32_t *yr = y16 + (int64_t)bi * ldy;
          lo = yr[max(c2lo, 0) >> 4];
          cnt = yr[min((c2hi >> 4) + 1, ldy - 1)] - lo;
        }
        int tot;
        const int off = sm_block_scan(cnt, wsum, &tot);
        s_lo[tid] = lo;
        s_off[tid] = off;
        s_b3[tid] = b3;
        const int nbk = min(SM_THREADS, bhi - g);
        __syncthreads();
        for (int cs = 0; cs < tot; cs += SM_THREADS) {
          if (len > SM_CAP - SM_THREADS) {   // uniform
            if (grouped) {
              over = true;
              break;
            }
            flush(0, len);
            __syncthreads();
            len = 0;
          }
          const int v = cs + tid;
          bool cov = false;
          int kn = 0, a3 = 0, d12 = 0;
          SmRec rec;
          if (v < tot) {   // last bucket with offset <= v (empty buckets share offsets)
            int l = 0, h = nbk;
            while (h - l > 1) {
              const int m = (l + h) >> 1;
              if (s_off[m] <= v) l = m; else h = m;
            }
            const int p = s_lo[l] + (v - s_off[l]);
            const int a1 = c1[p], a2 = c2[p];
            const double zp = zq[p];   // with the coordinates: one memory round trip, not two
            if (a1 >= c1lo && a1 <= c1hi && a2 >= c2lo && a2 <= c2hi) {
              a3 = s_b3[l];
              const int d1 = max(0, max(X0 - a1, a1 - (X0 + SM_T1 - 1)));
              const int d2 = max(0, max(Y0 - a2, a2 - (Y0 + SM_T2 - 1)));
              d12 = max(d1, d2);
              if (grouped) {
                kn = skofd[d12];   // an upper bound: the tile's x3 distance cuts it further
              } else {
                const int d3 = max(0, max(Z0 - a3, a3 - (Z0 + T3 - 1)));
                kn = skofd[max(d12, d3)];
              }
              if (kn > 0) {
                cov = true;
                rec.z = zp;
                rec.o1 = 8 * (X0 - a1 + gamma + SM_PAD);   // byte offsets into a table row
                rec.o2 = 8 * (Y0 - a2 + gamma + SM_PAD);
              }
            }
          }
          int t2;
          const int pos = sm_block_scan(cov ? 1 : 0, wsum, &t2);
          if (cov) {
            s_rec[len + pos] = rec;
            s_kn[len + pos] = kn;
            s_cb[len + pos] = a3;   // the bucket's x3 index (ascending along the staging area)
            if (GRP > 1) s_d12[len + pos] = d12;
          }
          len += t2;
        }
        __syncthreads();
        if (over) return -1;
      }
      return len;
    };

    auto tile_alone = [&](int t3) {
      Z0 = t3 * T3;
      zero_acc();
      const int len = search(t3, t3 + 1, false);
      if (len > 0) flush(0, len);
      epilogue();
    };

    if constexpr (GRP == 1) {
      tile_alone(t3_lo);
    } else {
      // one search for the group's tiles (low overlap: a few dozen copies): every tile
      // then takes the staged copies whose bucket lies within gamma of it -- a
      // contiguous range, the area is in bucket order -- with the live terms of its
      // own x3 distance.  An overflowing group falls back to tile-by-tile searches.
      const int glen = search(t3_lo, t3_hi, true);
      if (glen < 0) {
        for (int t3 = t3_lo; t3 < t3_hi; ++t3) {
          __syncthreads();
          tile_alone(t3);
        }
      } else {
        for (int t3 = t3_lo; t3 < t3_hi; ++t3) {
          __syncthreads();   // previous tile's MMA phase done with s_kn / s_seg
          Z0 = t3 * T3;
          zero_acc();
          const int zlo = Z0 - gamma, zhi = Z0 + T3 - 1 + gamma;
          int qa = 0, qb = glen;   // first staged copy with x3 >= zlo, first with x3 > zhi
          {
            int l = 0, h = glen;
            while (l < h) {
              const int m = (l + h) >> 1;
              if (s_cb[m] < zlo) l = m + 1; else h = m;
            }
            qa = l;
            h = glen;
            while (l < h) {
              const int m = (l + h) >> 1;
              if (s_cb[m] <= zhi) l = m + 1; else h = m;
            }
            qb = l;
          }
          for (int q = qa + tid; q < qb; q += SM_THREADS) {
            const int a3 = s_cb[q];
            const int d3 = max(0, max(Z0 - a3, a3 - (Z0 + T3 - 1)));
            s_kn[q] = skofd[max(s_d12[q], d3)];
          }
          if (qb > qa) flush(qa, qb - qa);   // (starts with a barrier: s_kn complete)
          epilogue();
        }
      }
    }
  }
}

}  // namespace
}  // namespace rsb

using namespace rsb;

extern "C" {

int rs_short_mma_supported(int64_t n, int64_t gamma, int64_t Rs) {
  if (n < 2 || n % 2 || gamma < 0 || Rs < 1 || Rs > SM_MAXR) return 0;
  if (ceil_div(n, SM_T3) > SM_MAXT3) return 0;
  const SmLayout L = sm_layout((int)gamma, (int)Rs);
  return L.total + 4096 <= 227 * 1024 ? 1 : 0;
}

static int64_t sm_ldy(int64_t n) { return ceil_div(n, 16) + 1; }

// kofd (gamma + 2 ints) | tile counter | x2 index (n buckets x ldy)
int64_t rs_short_mma_workspace_bytes(int64_t n, int64_t gamma) {
  return round_up((gamma + 2) * 4, 256) + 256 + round_up(n * sm_ldy(n) * 4, 256);
}

/* (a13) dense_cct on planes [x1_lo, x1_hi) by the fused tensor-core kernel.
 * flags: RS_ASM_ACCUMULATE adds to `out`; RS_ASM_KOFD_READY: the term table at
 * offset 0 of `work` is already filled (rsb_asm_term_prefix). */
int rs_assemble_short_mma(const double *ul, const double *wl, int64_t Rs, int64_t gamma, int64_t n,
                          int64_t count, const int32_t *c1, const int32_t *c2, const double *zq,
                          const int32_t *bstart, const int32_t *bc3, const int32_t *nb_dev,
                          int64_t x1_lo, int64_t x1_hi, int flags, double *out, void *work,
                          int64_t work_bytes, void *stream) {
  RS_REQUIRE(ul && wl && c1 && c2 && zq && bstart && bc3 && nb_dev && out && work,
             "rs_assemble_short_mma: bad arguments");
  RS_REQUIRE(0 <= x1_lo && x1_lo < x1_hi && x1_hi <= n, "rs_assemble_short_mma: bad plane range");
  RS_REQUIRE(rs_short_mma_supported(n, gamma, Rs),
             "rs_assemble_short_mma: unsupported shape (n=%lld gamma=%lld Rs=%lld)", (long long)n,
             (long long)gamma, (long long)Rs);
  if (work_bytes < rs_short_mma_workspace_bytes(n, gamma))
    return fail(RS_ERR_CAPACITY, "rs_assemble_short_mma: workspace too small");
  cudaStream_t s = as_stream(stream);
  int st;
  int *kofd = (int *)work;
  int *counter = (int *)((char *)work + round_up((gamma + 2) * 4, 256));
  if (!(flags & RS_ASM_KOFD_READY) &&
      (st = rsb_asm_term_prefix(ul, wl, (int)Rs, (int)gamma, kofd, s)))
    return st;
  if (cudaMemsetAsync(counter, 0, 4, s) != cudaSuccess)
    return fail(RS_ERR_CUDA, "rs_assemble_short_mma: memset");
  int32_t *y16 = (int32_t *)((char *)counter + 256);
  const int ldy = (int)sm_ldy(n);
  k_x2_index<<<grid_blocks(n * ldy), 256, 0, s>>>(c2, bstart, nb_dev, ldy, y16);
  if ((st = check_launch("short_mma x2 index"))) return st;
  // many copies per bucket and tile (C2-C4): the DMMA builder variant; few (C5): the
  // per-lane form.  RSB200_MMA_BUILD=0|1 forces one.
  const char *benv = getenv("RSB200_MMA_BUILD");   // (read per call: the tests switch it)
  const int build_env = benv && *benv ? atoi(benv) : -1;
  const double w0 = (double)std::min<int64_t>(2 * gamma + 1, n);
  const double ov0 = (double)std::max<int64_t>(count, 1) * (w0 / n) * (w0 / n) * (w0 / n);
  bool build = build_env >= 0 ? build_env != 0 : ov0 >= 64.0;
  if (build && sm_layout((int)gamma, (int)Rs, true).total + 4096 > 227 * 1024) build = false;
  const bool acc = flags & RS_ASM_ACCUMULATE;
  // RSB200_MMA_SKIP=1: the MMAs (and B loads) of the 8-wide x3 blocks a step's columns
  // cannot reach are skipped -- 25 % (C5) / 15 % (C4) fewer DMMAs.  Measured no faster
  // (C5 75.5 -> 75.1 ms) or slower (C4 113 -> 124 ms): with every DMMA removed the
  // kernel still takes 56 ms (C5) / 93 ms (C4) (RSB200_MMA_DBG=1) -- operand forming and
  // the candidate search dominate, not the tensor pipe -- so the default issues them all.
  const char *senv = getenv("RSB200_MMA_SKIP");
  const bool skip = senv && senv[0] == '1';
  // RSB200_MMA_GROUP=1, low overlap (C5: ~25 candidate copies per tile): one candidate
  // search per group of SM_GRP consecutive x3 tiles.  Measured no faster (C5 75.8 vs
  // 76.2 ms: of the 21 ms the kernel takes without its K loop, 11 are the grid store
  // itself and the per-tile segmentation stays), so the default searches per tile.
  const char *genv = getenv("RSB200_MMA_GROUP");
  const bool grouped = !build && !skip && ov0 <= 64.0 && genv && genv[0] == '1';
  const SmLayout L = sm_layout((int)gamma, (int)Rs, build, grouped);
  // RSB200_MMA_T3=32: 32-wide x3 tiles (half the accumulators: three CTAs per SM)
  const char *tenv = getenv("RSB200_MMA_T3");
  const bool narrow = tenv && atoi(tenv) == 32 && !grouped && !skip && ceil_div(n, 32) <= SM_MAXT3;
  const int t3w = narrow ? 32 : SM_T3;
  auto fn = narrow ? (build ? (acc ? k_short_mma<true, true, false, 1, 4> : k_short_mma<false, true, false, 1, 4>)
                            : (acc ? k_short_mma<true, false, false, 1, 4>
                                   : k_short_mma<false, false, false, 1, 4>))
            : grouped ? (acc ? k_short_mma<true, false, false, SM_GRP, 8>
                             : k_short_mma<false, false, false, SM_GRP, 8>)
            : skip ? (build ? (acc ? k_short_mma<true, true, true, 1, 8> : k_short_mma<false, true, true, 1, 8>)
                            : (acc ? k_short_mma<true, false, true, 1, 8> : k_short_mma<false, false, true, 1, 8>))
                   : (build ? (acc ? k_short_mma<true, true, false, 1, 8> : k_short_mma<false, true, false, 1, 8>)
                            : (acc ? k_short_mma<true, false, false, 1, 8>
                                   : k_short_mma<false, false, false, 1, 8>));
  // RSB200_MMA_PAD_KB: extra dynamic shared memory per CTA (occupancy experiments:
  // one CTA per SM leaves room for another kernel's CTAs)
  const char *penv = getenv("RSB200_MMA_PAD_KB");
  const int smem_bytes = std::min(L.total + (penv ? atoi(penv) * 1024 : 0), 227 * 1024);
  cudaError_t e = smem_attr((const void *)fn, smem_bytes);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "short_mma smem: %s", cudaGetErrorString(e));
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int per_sm = (narrow && smem_bytes + 1024 <= 75 * 1024) ? 3 : smem_bytes + 1024 <= 113 * 1024 ? 2 : 1;
  // work items: x3 tile groups (of one tile unless grouped)
  const int64_t ntiles = ceil_div(ceil_div(n, t3w), grouped ? SM_GRP : 1) * ceil_div(n, SM_T2) *
                         ceil_div(x1_hi - (x1_lo - x1_lo % SM_T1), SM_T1);
  static const int waves = [] {   // RSB200_MMA_WAVES: CTA generations per SM slot
    const char *e = getenv("RSB200_MMA_WAVES");
    return e && atoi(e) > 0 ? atoi(e) : 256;
  }();
  const int64_t slots = (int64_t)sms * per_sm;
  // tiles per CTA: at least ~100 us of work per staged factor table (a tile
  // costs ~0.3 us per window covering a grid point: C5 ~5 us, C2-C4 ~100 us)
  // when the launch has that many tiles per SM slot, and no more than
  // 1/waves of a slot's share, so CTAs keep turning over
  const double w = (double)std::min<int64_t>(2 * gamma + 1, n);
  const double ov = std::max(1.0, (double)std::max<int64_t>(count, 1) * (w / n) * (w / n) * (w / n));
  const int64_t t_min = std::max<int64_t>(1, std::min<int64_t>(16, (int64_t)(100.0 / (0.3 * ov))) /
                                             (grouped ? SM_GRP : 1));
  const int tiles_per_cta = (int)std::max<int64_t>(
      ceil_div(ntiles, slots * waves), std::min<int64_t>(t_min, ceil_div(ntiles, slots)));
  const unsigned grid = (unsigned)ceil_div(ntiles, tiles_per_cta);
  // RSB200_MMA_DBG (diagnostics, results wrong): 1 = no DMMA issued, 2 = no K loop at all
  const char *denv = getenv("RSB200_MMA_DBG");
  const int one = denv && *denv ? 1 - atoi(denv) : 1;
  ProfScope ps(s, "short_mma");
  fn<<<grid, SM_THREADS, smem_bytes, s>>>(ul, wl, (int)Rs, (int)gamma, n, c1, c2, zq, bstart, bc3,
                                       nb_dev, kofd, y16, ldy, x1_lo, x1_hi, counter, tiles_per_cta, one, out);
  return check_launch("short_mma");
}

}  // extern "C"
