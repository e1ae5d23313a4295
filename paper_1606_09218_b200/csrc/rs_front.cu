// Front of the RS build in one host call: snap -> node sort -> bucket-ordered
// copies -> shift histograms -> short-range bucket table, all enqueued on one
// stream from C++ (the Python driver's per-call overhead was the critical
// path of a C2 step).  Buffers live in one caller-owned region whose layout
// rs_front_offsets describes.  Reference: particles.py:302-329 (snap),
// assembly.py:139-184 / formats.py:179-244 (CCT buckets), rankred.py:82-126
// (the shift regrouping behind the histograms).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "rs_common.cuh"
#include "rs_dmma.cuh"

using namespace rsb;

extern "C" {
int rs_snap(const double *pos, int64_t count, double h, int64_t n, int64_t *idx, double *disp,
            int64_t *key, double *snapped, void *stream);
int rs_prep(const int64_t *ks, const int64_t *order, const int64_t *idx, const double *z,
            const double *disp, int64_t count, int64_t n, int32_t *c1s, int32_t *c2s, double *zqs,
            int64_t *starts, uint64_t *dup_pos, uint64_t *dmax_bits, void *stream);
int rs_shift_hist(const int64_t *idx, const double *z, int64_t count, int64_t n, double *c,
                  int32_t *cnt3, void *stream);
int rs_short_layout(const int32_t *cnt3, int64_t n, int32_t *bstart, int32_t *bc3, int32_t *nb,
                    void *stream);
int64_t rs_assemble_workspace_bytes(int64_t n, int64_t planes, int64_t rmax, int64_t nb_max,
                                    int64_t Rs, int flags);
int rs_assemble_planes(const double *core, int64_t r1, int64_t r2, int64_t r3, const double *V1,
                       const double *V2, const double *V3, int64_t n, const double *ul,
                       const double *wl, int64_t Rs, int64_t gamma, const int32_t *c1,
                       const int32_t *c2, const double *zq, const int32_t *bstart,
                       const int32_t *bc3, const int32_t *nb_dev, int64_t nb_max, int64_t x1_lo,
                       int64_t x1_hi, int flags, double *out, void *work, int64_t work_bytes,
                       void *stream);
}

int rsb_shift_project3_listed(const double *Z1, const double *Z2, const double *Z3, int64_t r1,
                              int64_t r2, int64_t r3, int64_t n, const double *table,
                              int64_t ld_table, int64_t R, const int64_t *shift, int64_t count,
                              double *TT1, double *TT2, double *TT3, void *list_work,
                              cudaStream_t s);  // rs_kernels.cu
extern "C" int rsb_asm_term_prefix(const double *ul, const double *wl, int Rs, int gamma,
                                   void *work, cudaStream_t s);

namespace {

enum Slot {
  F_IDX, F_DISP, F_KEY, F_SNAPPED, F_KS, F_ORDER, F_C1, F_C2, F_ZQ, F_STARTS, F_SCAL, F_HIST,
  F_CNT3, F_BSTART, F_BC3, F_NB, F_IOTA, F_CUB, F_END
};

__global__ void k_iota(int64_t *v, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

int key_bits(int64_t n) {  // node keys are < n^3
  int b = 1;
  while (b < 63 && ((int64_t)1 << b) < n * n * n) ++b;
  return b;
}

size_t cub_bytes(int64_t count, int64_t n) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const int64_t *)nullptr, (int64_t *)nullptr,
                                  (const int64_t *)nullptr, (int64_t *)nullptr, (int)count, 0,
                                  key_bits(n));
  return t;
}

void layout(int64_t count, int64_t n, int64_t *off) {
  const int64_t c = std::max<int64_t>(count, 1);
  const int64_t sz[F_END] = {c * 24, c * 8, c * 8, c * 24, c * 8, c * 8, c * 4, c * 4, c * 8,
                             c * 24, 16,    3 * n * 8, n * 4, (n + 1) * 4, n * 4, 4, c * 8,
                             (int64_t)cub_bytes(c, n)};
  int64_t o = 0;
  for (int i = 0; i < F_END; ++i) {
    off[i] = o;
    o += round_up(std::max<int64_t>(sz[i], 1), 256);
  }
  off[F_END] = o;
}

}  // namespace

extern "C" {

/* Byte offsets of the front buffers (F_END + 1 entries, last = total):
 * idx (count,3) i64 | disp f64 | key i64 | snapped (count,3) f64 | sorted keys |
 * order | c1 i32 | c2 i32 | zq f64 | starts (count,3) i64 | scal (dup key i64,
 * dmax f64) | hist (3,n) f64 | cnt3 (n) i32 | bstart (n+1) i32 | bc3 (n) i32 |
 * nb i32 | iota | sort scratch. */
int rs_front_offsets(int64_t count, int64_t n, int64_t *offsets) {
  RS_REQUIRE(count >= 1 && n >= 2 && offsets, "rs_front_offsets: bad arguments");
  layout(count, n, offsets);
  return RS_OK;
}

/* snap + sort + prep + histograms + bucket table for `count` particles; with
 * `side` != NULL also the short-range planes [x1_lo, x1_hi) into `out` on
 * the side stream (after the bucket table, chunked by `work_bytes`). */
int rs_front(const double *pos, const double *z, int64_t count, double h, int64_t n, void *buf,
             int64_t buf_bytes, void *stream, const double *ul, const double *wl, int64_t Rs,
             int64_t gamma, int64_t x1_lo, int64_t x1_hi, double *out, void *work,
             int64_t work_bytes, void *side, int oz_slices, int64_t group, void **events) {
  RS_REQUIRE(count >= 1 && n >= 2 && h > 0 && pos && z && buf, "rs_front: bad arguments");
  int64_t off[F_END + 1];
  layout(count, n, off);
  if (buf_bytes < off[F_END])
    return fail(RS_ERR_CAPACITY, "rs_front: buffer %lld < %lld", (long long)buf_bytes,
                (long long)off[F_END]);
  char *b = (char *)buf;
  auto P = [&](int s) { return (void *)(b + off[s]); };
  cudaStream_t s = as_stream(stream);
  int st;
  if ((st = rs_snap(pos, count, h, n, (int64_t *)P(F_IDX), (double *)P(F_DISP),
                    (int64_t *)P(F_KEY), (double *)P(F_SNAPPED), stream)))
    return st;
  k_iota<<<(unsigned)std::min<int64_t>(ceil_div(count, 256), 1024), 256, 0, s>>>(
      (int64_t *)P(F_IOTA), count);
  if ((st = check_launch("rs_front iota"))) return st;
  size_t tb = (size_t)(off[F_CUB + 1] - off[F_CUB]);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(
      P(F_CUB), tb, (const int64_t *)P(F_KEY), (int64_t *)P(F_KS), (const int64_t *)P(F_IOTA),
      (int64_t *)P(F_ORDER), (int)count, 0, key_bits(n), s);
  if (e != cudaSuccess) return fail(RS_ERR_CUDA, "rs_front sort: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if ((st = rs_prep((const int64_t *)P(F_KS), (const int64_t *)P(F_ORDER),
                    (const int64_t *)P(F_IDX), z, (const double *)P(F_DISP), count, n,
                    (int32_t *)P(F_C1), (int32_t *)P(F_C2), (double *)P(F_ZQ),
                    (int64_t *)P(F_STARTS), (uint64_t *)P(F_SCAL),
                    (uint64_t *)((char *)P(F_SCAL) + 8), stream)))
    return st;
  if ((st = rs_shift_hist((const int64_t *)P(F_IDX), z, count, n, (double *)P(F_HIST),
                          (int32_t *)P(F_CNT3), stream)))
    return st;
  if ((st = rs_short_layout((const int32_t *)P(F_CNT3), n, (int32_t *)P(F_BSTART),
                            (int32_t *)P(F_BC3), (int32_t *)P(F_NB), stream)))
    return st;
  if (!side) return RS_OK;
  RS_REQUIRE(out && ul && wl && Rs >= 1 && 0 <= x1_lo && x1_lo < x1_hi && x1_hi <= n,
             "rs_front: bad prefetch arguments");
  static thread_local cudaEvent_t ev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!ev[dev & 63] && cudaEventCreateWithFlags(&ev[dev & 63], cudaEventDisableTiming) != cudaSuccess)
    return fail(RS_ERR_CUDA, "rs_front: event");
  const int method = rs_short_method(n, count, gamma, Rs);
  const bool l0_path = method == RS_SHORT_L0;
  if (!l0_path) {  // plan-only term table: ahead of the wait, overlapping the front
    if (work_bytes < (int64_t)((n + 1) * 4))
      return fail(RS_ERR_CAPACITY, "rs_front: workspace too small");
    if ((st = rsb_asm_term_prefix(ul, wl, (int)Rs, (int)gamma, work, as_stream(side)))) return st;
  }
  if (cudaEventRecord(ev[dev & 63], s) != cudaSuccess ||
      cudaStreamWaitEvent(as_stream(side), ev[dev & 63], 0) != cudaSuccess)
    return fail(RS_ERR_CUDA, "rs_front: stream dependency");
  // planes are produced in groups of `group` (<= 0: one group); events[g]
  // (caller-created, may be NULL) is recorded on `side` when group g is done,
  // so a consumer can start on the first planes (e.g. their D2H) early
  const int64_t span = x1_hi - x1_lo;
  const int64_t grp = group > 0 ? std::min<int64_t>(group, span) : span;
  auto mark = [&](int64_t p1) -> int {
    if (!events) return RS_OK;
    if ((p1 - x1_lo) % grp != 0 && p1 != x1_hi) return RS_OK;
    cudaEvent_t e = (cudaEvent_t)events[(p1 - x1_lo - 1) / grp];
    if (e && cudaEventRecord(e, as_stream(side)) != cudaSuccess)
      return fail(RS_ERR_CUDA, "rs_front: group event");
    return RS_OK;
  };
  if (l0_path) {  // dense-L0 gather, L0 in `work`
    if (work_bytes < rs_short_l0_bytes(gamma))
      return fail(RS_ERR_CAPACITY, "rs_front: workspace %lld < L0 %lld", (long long)work_bytes,
                  (long long)rs_short_l0_bytes(gamma));
    double *L0 = (double *)work;
    if ((st = rs_short_l0_table(ul, wl, Rs, gamma, L0, side))) return st;
    for (int64_t p0 = x1_lo; p0 < x1_hi; p0 += grp) {
      const int64_t p1 = std::min<int64_t>(x1_hi, p0 + grp);
      if ((st = rs_assemble_short_l0(L0, gamma, n, (const int32_t *)P(F_C1),
                                     (const int32_t *)P(F_C2), (const double *)P(F_ZQ),
                                     (const int32_t *)P(F_BSTART), (const int32_t *)P(F_BC3),
                                     (const int32_t *)P(F_NB), p0, p1, 0,
                                     out + (p0 - x1_lo) * n * n, side)) ||
          (st = mark(p1)))
        return st;
    }
    return RS_OK;
  }
  if (method == RS_SHORT_MMA) {  // fused tensor-core kernel, term table at work[0]
    for (int64_t p0 = x1_lo; p0 < x1_hi; p0 += grp) {
      const int64_t p1 = std::min<int64_t>(x1_hi, p0 + grp);
      if ((st = rs_assemble_short_mma(ul, wl, Rs, gamma, n, count, (const int32_t *)P(F_C1),
                                      (const int32_t *)P(F_C2), (const double *)P(F_ZQ),
                                      (const int32_t *)P(F_BSTART), (const int32_t *)P(F_BC3),
                                      (const int32_t *)P(F_NB), p0, p1, RS_ASM_KOFD_READY,
                                      out + (p0 - x1_lo) * n * n, work, work_bytes, side)) ||
          (st = mark(p1)))
        return st;
    }
    return RS_OK;
  }
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(n, count));
  const int flags = RS_ASM_SHORT | RS_ASM_OZ(oz_slices) | RS_ASM_KOFD_READY;
  const int64_t one = rs_assemble_workspace_bytes(n, 1, 1, nb_max, Rs, flags);
  const int64_t per = rs_assemble_workspace_bytes(n, 2, 1, nb_max, Rs, flags) - one;
  const int64_t chunk = std::max<int64_t>(
      1, std::min<int64_t>(grp, (work_bytes - (one - per)) / std::max<int64_t>(per, 1)));
  for (int64_t g0 = x1_lo; g0 < x1_hi; g0 += grp) {
    const int64_t g1 = std::min<int64_t>(x1_hi, g0 + grp);
    for (int64_t p0 = g0; p0 < g1; p0 += chunk) {
      const int64_t p1 = std::min<int64_t>(g1, p0 + chunk);
      if ((st = rs_assemble_planes(nullptr, 1, 1, 1, nullptr, nullptr, nullptr, n, ul, wl, Rs,
                                   gamma, (const int32_t *)P(F_C1), (const int32_t *)P(F_C2),
                                   (const double *)P(F_ZQ), (const int32_t *)P(F_BSTART),
                                   (const int32_t *)P(F_BC3), (const int32_t *)P(F_NB), nb_max,
                                   p0, p1, flags, out + (p0 - x1_lo) * n * n, work, work_bytes,
                                   side)))
        return st;
    }
    if ((st = mark(g1))) return st;
  }
  return RS_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ back
// After the host picked the ranks: Ritz rows -> Tucker factors (transpose),
// per-shift projections and the RHOSVD core, in one host call (reference:
// rankred.py:151-177 with the shift regrouping of rankred.py:82-126).
namespace {
__global__ void k_ritz_to_factors(const double *__restrict__ U, int64_t b, int64_t n, int r1,
                                  int r2, int r3, double *__restrict__ Z1, double *__restrict__ Z2,
                                  double *__restrict__ Z3) {
  const int64_t tot = n * (int64_t)(r1 + r2 + r3);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / (r1 + r2 + r3);
    int a = (int)(e - i * (r1 + r2 + r3));
    int l = 0;
    double *Z = Z1;
    int r = r1;
    if (a >= r1) {
      a -= r1;
      l = 1;
      Z = Z2;
      r = r2;
      if (a >= r2) {
        a -= r2;
        l = 2;
        Z = Z3;
        r = r3;
      }
    }
    Z[i * r + a] = U[((int64_t)l * b + a) * n + i];
  }
}
// Core by mode-3 buckets: core[(a,b), c] = sum_{(q,k)} H[(a,b),(q,k)] T3[c,(q,k)]
// with H[(a,b),(q,k)] = sum_{i in bucket q} zq_i w_k TT1[a, n-c1_i, k] TT2[b, n-c2_i, k]
// and T3[c,(q,k)] = TT3[c, n - x3_q, k]: the K of the core GEMM drops from
// N R_l (particles x terms) to (occupied x3 values) x R_l.
constexpr int CH_CHUNK = 64;   // bucket copies staged per pass (32: C5 core_h 6.9 ms)
constexpr int CH_RMAX = 24;

// TTt[s][k][a] = TT[a][s][k]: per-(shift, term) vectors contiguous in a
__global__ void k_tt_transpose(const double *__restrict__ TT, int r, int64_t n, int R,
                               double *__restrict__ TTt) {
  const int64_t tot = (int64_t)r * n * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e % r, sk = e / r;  // output order (s, k, a)
    const int64_t sh = sk / R, k = sk - sh * R;
    TTt[e] = TT[(a * n + sh) * R + k];
  }
}

// Block = (bucket q, CH_TA consecutive a, CH_KG consecutive terms k); thread =
// one b (blockDim >= r2).  Per staged chunk of the bucket's copies and per
// term k: the copies' TT2 vectors (all b) and TT1 entries (the block's a) land
// in shared memory with coalesced loads; every thread accumulates CH_TA x
// CH_KG outputs in registers and finally writes, per row, one aligned CH_KG-
// wide segment.  The TT2 panel of a (copy, term) is re-read once per a-tile:
// 16 a per block instead of 2 cut the L2 traffic of this stage 8x (C5 core
// 27 -> see DESIGN).
constexpr int CH_TA = 16;
constexpr int CH_KG = 4;
__global__ void __launch_bounds__(256)
    k_core_h(const double *__restrict__ TT1t, const double *__restrict__ TT2t, int r1,
             int r2, int64_t n, int R, const double *__restrict__ w,
             const int32_t *__restrict__ c1, const int32_t *__restrict__ c2,
             const double *__restrict__ zq, const int32_t *__restrict__ bstart,
             double *__restrict__ H, int64_t ldH) {
  extern __shared__ double sh[];
  double *sY = sh;                          // CH_CHUNK x r2
  double *sX = sh + CH_CHUNK * r2;          // CH_CHUNK x CH_TA
  const int q = blockIdx.y;
  const int a0 = blockIdx.x * CH_TA;
  const int k0 = blockIdx.z * CH_KG;
  const int bcol = threadIdx.x;
  double acc[CH_TA][CH_KG];
#pragma unroll
  for (int u = 0; u < CH_TA; ++u)
#pragma unroll
    for (int k = 0; k < CH_KG; ++k) acc[u][k] = 0.0;
  const int p_lo = bstart[q], p_hi = bstart[q + 1];
  for (int i0 = p_lo; i0 < p_hi; i0 += CH_CHUNK) {
    const int cnt = min(CH_CHUNK, p_hi - i0);
#pragma unroll
    for (int kk = 0; kk < CH_KG; ++kk) {
      const int k = k0 + kk;
      if (k < R) {   // uniform
        for (int e = threadIdx.x; e < cnt * r2; e += blockDim.x) {
          const int j = e / r2, t = e - j * r2;
          sY[e] = TT2t[((int64_t)(n - c2[i0 + j]) * R + k) * r2 + t];
        }
        for (int e = threadIdx.x; e < cnt * CH_TA; e += blockDim.x) {
          const int j = e / CH_TA, u = e - j * CH_TA;
          const int i = i0 + j;
          sX[e] = a0 + u < r1 ? zq[i] * w[k] * TT1t[((int64_t)(n - c1[i]) * R + k) * r1 + a0 + u]
                              : 0.0;
        }
        __syncthreads();
        if (bcol < r2) {
          for (int j = 0; j < cnt; ++j) {
            const double y = sY[j * r2 + bcol];
            const double2 *xs = reinterpret_cast<const double2 *>(sX + j * CH_TA);
#pragma unroll
            for (int u = 0; u < CH_TA; u += 2) {
              const double2 x = xs[u >> 1];
              acc[u][kk] = fma(x.x, y, acc[u][kk]);
              acc[u + 1][kk] = fma(x.y, y, acc[u + 1][kk]);
            }
          }
        }
        __syncthreads();
      }
    }
  }
  if (bcol < r2) {
#pragma unroll
    for (int u = 0; u < CH_TA; ++u) {
      const int a = a0 + u;
      if (a >= r1) continue;
      double *dst = H + ((int64_t)a * r2 + bcol) * ldH + (int64_t)q * R + k0;
#pragma unroll
      for (int kk = 0; kk < CH_KG; ++kk)
        if (k0 + kk < R) dst[kk] = acc[u][kk];
      if (q == (int)gridDim.y - 1 && blockIdx.z == gridDim.z - 1)  // even-K padding column(s)
        for (int64_t c = (int64_t)(q + 1) * R; c < ldH; ++c) H[((int64_t)a * r2 + bcol) * ldH + c] = 0.0;
    }
  }
}

// The same H stage on the FP64 tensor cores: for a (bucket q, term k) the (a, b) panel
// is X^T Y with X = (z w_k TT1[a]) (copies x a) and Y = TT2 (copies x b), K = the
// bucket's copies (C5: ~86) -- mma.m8n8k4 with a = m, copy = k, b = n.  Block = (bucket,
// 16 a, 4 terms) as above; warp w owns the 8-wide b blocks w, w + 8, w + 16 for both
// 8-row a blocks and all 4 terms (48 accumulators per thread); operands are staged per
// term with the pitch = 4 mod 16 doubles that keeps the fragment gathers conflict free.
// C5 core_h 6.7 -> see DESIGN (the CUDA-core form ran at 9 % of the FP64 peak).
constexpr int CHM_NB = 3;      // b blocks per warp: r2 <= 8 * 8 * 3 = 192
__host__ __device__ inline int chm_pitch(int r) {
  int p = (r + 7) / 8 * 8;
  while (p % 16 != 4) ++p;
  return p;
}
__global__ void __launch_bounds__(256)
    k_core_h_mma(const double *__restrict__ TT1t, const double *__restrict__ TT2t, int r1, int r2,
                 int64_t n, int R, const double *__restrict__ w, const int32_t *__restrict__ c1,
                 const int32_t *__restrict__ c2, const double *__restrict__ zq,
                 const int32_t *__restrict__ bstart, double *__restrict__ H, int64_t ldH) {
  extern __shared__ double sh[];
  const int PY = chm_pitch(r2), PX = 20;
  double *sY = sh;                      // CH_CHUNK x PY
  double *sX = sh + CH_CHUNK * PY;      // CH_CHUNK x PX (16 a + pad)
  const int q = blockIdx.y, a0 = blockIdx.x * CH_TA, k0 = blockIdx.z * CH_KG;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gid = lane >> 2, tig = lane & 3;
  const int nbk = (r2 + 7) / 8;
  double acc[CH_KG][CHM_NB][2][2];
#pragma unroll
  for (int k = 0; k < CH_KG; ++k)
#pragma unroll
    for (int b = 0; b < CHM_NB; ++b)
#pragma unroll
      for (int m = 0; m < 2; ++m) acc[k][b][m][0] = acc[k][b][m][1] = 0.0;
  const int p_lo = bstart[q], p_hi = bstart[q + 1];
  for (int i0 = p_lo; i0 < p_hi; i0 += CH_CHUNK) {
    const int cnt = min(CH_CHUNK, p_hi - i0), cnt4 = (cnt + 3) & ~3;
#pragma unroll
    for (int kk = 0; kk < CH_KG; ++kk) {
      const int k = k0 + kk;
      if (k < R) {   // uniform
        for (int e = tid; e < cnt4 * r2; e += 256) {
          const int j = e / r2, t = e - j * r2;
          sY[j * PY + t] = j < cnt ? TT2t[((int64_t)(n - c2[i0 + j]) * R + k) * r2 + t] : 0.0;
        }
        for (int e = tid; e < cnt4 * CH_TA; e += 256) {
          const int j = e / CH_TA, u = e - j * CH_TA;
          const int i = i0 + j;
          sX[j * PX + u] = (j < cnt && a0 + u < r1)
                               ? zq[i] * w[k] * TT1t[((int64_t)(n - c1[i]) * R + k) * r1 + a0 + u]
                               : 0.0;
        }
        __syncthreads();
        for (int j0 = 0; j0 < cnt4; j0 += 4) {
          const double xa0 = sX[(j0 + tig) * PX + gid], xa1 = sX[(j0 + tig) * PX + 8 + gid];
#pragma unroll
          for (int b = 0; b < CHM_NB; ++b) {
            const int nb = warp + 8 * b;
            if (nb < nbk) {   // warp-uniform
              const double yb = sY[(j0 + tig) * PY + 8 * nb + gid];
              dmma_884(acc[kk][b][0], xa0, yb);
              dmma_884(acc[kk][b][1], xa1, yb);
            }
          }
        }
        __syncthreads();
      }
    }
  }
  // c[0], c[1]: row a = 8 m + gid, columns b = 8 nb + 2 tig + {0, 1}; per (a, b) one
  // aligned CH_KG-wide segment of H
#pragma unroll
  for (int b = 0; b < CHM_NB; ++b) {
    const int nb = warp + 8 * b;
    if (nb >= nbk) continue;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int a = a0 + 8 * m + gid;
      if (a >= r1) continue;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int bc = 8 * nb + 2 * tig + c;
        if (bc >= r2) continue;
        double *dst = H + ((int64_t)a * r2 + bc) * ldH + (int64_t)q * R + k0;
#pragma unroll
        for (int kk = 0; kk < CH_KG; ++kk)
          if (k0 + kk < R) dst[kk] = acc[kk][b][m][c];
        if (q == (int)gridDim.y - 1 && blockIdx.z == gridDim.z - 1)  // even-K padding column(s)
          for (int64_t cc = (int64_t)(q + 1) * R; cc < ldH; ++cc) H[((int64_t)a * r2 + bc) * ldH + cc] = 0.0;
      }
    }
  }
}

// T3[c, q*R + k] = TT3[c, n - bc3[q], k] for occupied buckets, 0 past *nb
__global__ void k_core_t3(const double *__restrict__ TT3, int r3, int64_t n, int R,
                          const int32_t *__restrict__ bc3, const int32_t *__restrict__ nbp,
                          int64_t nq, double *__restrict__ T3, int64_t ldT, int q_off) {
  const int64_t tot = (int64_t)r3 * ldT;
  const int nb = *nbp - q_off;   // bc3 already points at bucket q_off
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / ldT, col = e - c * ldT;
    const int64_t q = col / R;
    const int k = (int)(col - q * R);
    T3[e] = (q < nb && q < nq) ? TT3[((int64_t)c * n + (n - bc3[q])) * R + k] : 0.0;
  }
}
}  // namespace

extern "C" {
int rs_gemm_nt(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
               int64_t M, int64_t N, int64_t K, void *stream);
int rs_shift_project3(const double *Z1, const double *Z2, const double *Z3, int64_t r1, int64_t r2,
                      int64_t r3, int64_t n, const double *table, int64_t ld_table, int64_t R,
                      int64_t n_shift, double *TT1, double *TT2, double *TT3, void *stream);
int64_t rs_core_workspace_bytes(int64_t r1, int64_t r2, int64_t r3, int64_t count, int64_t R);
int rs_core(const double *TT1, const double *TT2, const double *TT3, int64_t r1, int64_t r2,
            int64_t r3, int64_t n_shift, int64_t R, const int64_t *shift, const double *z,
            const double *w, int64_t count, double *core, void *work, int64_t work_bytes,
            void *stream);

static int64_t ldh_of(int64_t nq, int64_t R) { return round_up(std::max<int64_t>(nq * R, 2), 2); }

int64_t rs_back_workspace_bytes(int64_t n, int64_t r1, int64_t r2, int64_t r3, int64_t count,
                                int64_t R, int64_t nq_host) {
  // projections | max(particle-K core scratch, bucket-K H + T3)
  const int64_t nq = nq_host > 0 ? nq_host : std::min<int64_t>(n, count), ld = ldh_of(nq, R);
  const int64_t hb = round_up(r1 * r2 * ld * 8, 256) + round_up(r3 * ld * 8, 256) +
                     (r1 + r2) * n * R * 8;
  return round_up((r1 + r2 + r3) * n * R * 8, 256) + round_up((6 * n + 8) * 4, 256) +
         std::max<int64_t>(rs_core_workspace_bytes(r1, r2, r3, count, R), hb);
}

/* U: (3, b, n) Ritz rows (descending); Z_l (n, r_l) = U[l, :r_l]^T; core
 * (r1, r2, r3) of the shift-structured long part. */
}  // extern "C"

// rs_back / rs_back_shard.  A shard (rank of `world`) sums only its share of
// the core's K dimension: the x3 buckets [q_lo, q_hi) on the bucket-K path,
// the particles [p_lo, p_hi) on the particle-K path (which of the two runs
// depends only on sizes every rank agrees on).  q_lo < 0: everything.
static int back_impl(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
            const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
            const double *z, const double *w, int64_t count, double *Z1, double *Z2, double *Z3,
            double *core, void *work, int64_t work_bytes, void *stream,
            const int32_t *c1, const int32_t *c2, const double *zq, const int32_t *bstart,
            const int32_t *bc3, const int32_t *nb, int64_t nq_host, int64_t q_lo, int64_t q_hi,
            int64_t p_lo, int64_t p_hi) {
  RS_REQUIRE(r1 >= 1 && r2 >= 1 && r3 >= 1 && r1 <= b && r2 <= b && r3 <= b && n >= 2,
             "rs_back: bad ranks");
  const bool shard = q_lo >= 0;
  RS_REQUIRE(!shard || (q_lo <= q_hi && q_hi <= std::max<int64_t>(nq_host, 0) && 0 <= p_lo &&
                        p_lo <= p_hi && p_hi <= count),
             "rs_back_shard: bad shard bounds");
  if (work_bytes < rs_back_workspace_bytes(n, r1, r2, r3, count, R, nq_host))
    return fail(RS_ERR_CAPACITY, "rs_back: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t tot = n * (r1 + r2 + r3);
  k_ritz_to_factors<<<(unsigned)std::min<int64_t>(ceil_div(tot, 256), 1024), 256, 0, s>>>(
      U, b, n, (int)r1, (int)r2, (int)r3, Z1, Z2, Z3);
  int st;
  if ((st = check_launch("rs_back factors"))) return st;
  double *TT1 = (double *)work, *TT2 = TT1 + r1 * n * R, *TT3 = TT2 + r2 * n * R;
  // projections at the occupied shifts only (the core reads no others)
  char *lw = (char *)work + round_up((r1 + r2 + r3) * n * R * 8, 256);
  if (n <= 8192) {
    if ((st = rsb_shift_project3_listed(Z1, Z2, Z3, r1, r2, r3, n, table, ld_table, R, starts,
                                        count, TT1, TT2, TT3, lw, s)))
      return st;
  } else if ((st = rs_shift_project3(Z1, Z2, Z3, r1, r2, r3, n, table, ld_table, R, n, TT1, TT2,
                                     TT3, stream))) {
    return st;
  }
  char *cw = lw + round_up((6 * n + 8) * 4, 256);
  // the particle-K Khatri-Rao GEMM is latency-bound and cheap below ~1e10
  // flops (C1-C3); the bucket-K form wins once N R_l r1 r2 r3 dominates (C4, C5)
  const double kr_flops = 2.0 * (double)r1 * r2 * r3 * (double)count * R;
  if (!bstart || nq_host <= 0 || R > CH_RMAX || kr_flops < 1e10 || r2 > 256) {
    if (!shard)
      return rs_core(TT1, TT2, TT3, r1, r2, r3, n, R, starts, z, w, count, core, cw,
                     rs_core_workspace_bytes(r1, r2, r3, count, R), stream);
    if (p_hi == p_lo) {  // empty particle shard: a zero partial
      if (cudaMemsetAsync(core, 0, (size_t)(r1 * r2 * r3) * 8, s) != cudaSuccess)
        return fail(RS_ERR_CUDA, "rs_back_shard: memset");
      return RS_OK;
    }
    return rs_core(TT1, TT2, TT3, r1, r2, r3, n, R, starts + 3 * p_lo, z + p_lo, w, p_hi - p_lo,
                   core, cw, rs_core_workspace_bytes(r1, r2, r3, p_hi - p_lo, R), stream);
  }
  if (shard) {  // this rank's buckets: the tables are indexed from q_lo
    if (q_hi == q_lo) {
      if (cudaMemsetAsync(core, 0, (size_t)(r1 * r2 * r3) * 8, s) != cudaSuccess)
        return fail(RS_ERR_CUDA, "rs_back_shard: memset");
      return RS_OK;
    }
    bstart += q_lo;
    bc3 += q_lo;
    nq_host = q_hi - q_lo;
  }
  const int q_off = shard ? (int)q_lo : 0;
  // bucket-K core: H (r1 r2 x nq R) on CUDA cores, then one DMMA GEMM
  // nq_host: the occupied x3 count the host read back (0: the upper bound)
  const int64_t nq = nq_host > 0 ? nq_host : std::min<int64_t>(n, count), ldH = ldh_of(nq, R);
  double *H = (double *)cw;
  double *T3 = (double *)(cw + round_up(r1 * r2 * ldH * 8, 256));
  double *TT1t = (double *)((char *)T3 + round_up(r3 * ldH * 8, 256));
  double *TT2t = TT1t + r1 * n * R;
  ProfScope ps(s, "core");
  k_tt_transpose<<<(unsigned)std::min<int64_t>(ceil_div(r1 * n * R, 256), 4096), 256, 0, s>>>(
      TT1, (int)r1, n, (int)R, TT1t);
  k_tt_transpose<<<(unsigned)std::min<int64_t>(ceil_div(r2 * n * R, 256), 4096), 256, 0, s>>>(
      TT2, (int)r2, n, (int)R, TT2t);
  if ((st = check_launch("core transpose"))) return st;
  RS_REQUIRE(r2 <= 256, "rs_back: r2 = %lld exceeds the H kernel's block", (long long)r2);
  // RSB200_CORE_H=cuda: the CUDA-core H stage (also beyond the tensor form's r2 <= 192)
  static const bool h_mma = [] {
    const char *e = getenv("RSB200_CORE_H");
    return !(e && e[0] == 'c');
  }();
  const dim3 hgrid((unsigned)ceil_div(r1, CH_TA), (unsigned)nq, (unsigned)ceil_div(R, CH_KG));
  if (h_mma && r2 <= 8 * 8 * CHM_NB) {
    const size_t smem = (size_t)CH_CHUNK * (chm_pitch((int)r2) + 20) * 8;
    cudaError_t e = smem_attr((const void *)k_core_h_mma, (int)smem);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "core_h smem: %s", cudaGetErrorString(e));
    k_core_h_mma<<<hgrid, 256, smem, s>>>(TT1t, TT2t, (int)r1, (int)r2, n, (int)R, w, c1, c2, zq,
                                          bstart, H, ldH);
  } else {
    const int threads = (int)round_up(r2, 32);
    const size_t smem = (size_t)CH_CHUNK * (r2 + CH_TA) * 8;
    cudaError_t e = smem_attr((const void *)k_core_h, (int)smem);
    if (e != cudaSuccess) return fail(RS_ERR_CUDA, "core_h smem: %s", cudaGetErrorString(e));
    k_core_h<<<hgrid, threads, smem, s>>>(TT1t, TT2t, (int)r1, (int)r2, n, (int)R, w, c1, c2, zq,
                                          bstart, H, ldH);
  }
  if ((st = check_launch("core_h"))) return st;
  k_core_t3<<<(unsigned)std::min<int64_t>(ceil_div(r3 * ldH, 256), 4096), 256, 0, s>>>(
      TT3, (int)r3, n, (int)R, bc3, nb, nq, T3, ldH, q_off);
  if ((st = check_launch("core_t3"))) return st;
  return rs_gemm_nt(H, ldH, T3, ldH, core, r3, r1 * r2, r3, ldH, stream);
}

extern "C" {
int rs_back(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
            const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
            const double *z, const double *w, int64_t count, double *Z1, double *Z2, double *Z3,
            double *core, void *work, int64_t work_bytes, void *stream,
            const int32_t *c1, const int32_t *c2, const double *zq, const int32_t *bstart,
            const int32_t *bc3, const int32_t *nb, int64_t nq_host) {
  return back_impl(U, b, n, r1, r2, r3, table, ld_table, R, starts, z, w, count, Z1, Z2, Z3, core,
                   work, work_bytes, stream, c1, c2, zq, bstart, bc3, nb, nq_host, -1, -1, 0, 0);
}

int rs_back_shard(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
                  const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
                  const double *z, const double *w, int64_t count, double *Z1, double *Z2,
                  double *Z3, double *core, void *work, int64_t work_bytes, void *stream,
                  const int32_t *c1, const int32_t *c2, const double *zq, const int32_t *bstart,
                  const int32_t *bc3, const int32_t *nb, int64_t nq_host, int64_t q_lo,
                  int64_t q_hi, int64_t p_lo, int64_t p_hi) {
  RS_REQUIRE(q_lo >= 0, "rs_back_shard: bad shard bounds");
  return back_impl(U, b, n, r1, r2, r3, table, ld_table, R, starts, z, w, count, Z1, Z2, Z3, core,
                   work, work_bytes, stream, c1, c2, zq, bstart, bc3, nb, nq_host, q_lo, q_hi,
                   p_lo, p_hi);
}

/* rs_back, then (after `wait_event` when given) the Tucker part of planes
 * [x1_lo, x1_hi) accumulated into `out` (the prefetched short-range slab) in
 * chunks of `chunk` planes: the post-synchronisation device work of build_rs
 * in one host call.  Reference: rankred.py:151-177 + formats.py:173-176. */
int rs_back_tucker(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
                   const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
                   const double *z, const double *w, int64_t count, double *Z1, double *Z2,
                   double *Z3, double *core, void *work, int64_t work_bytes, void *stream,
                   const int32_t *c1, const int32_t *c2, const double *zq,
                   const int32_t *bstart, const int32_t *bc3, const int32_t *nb, int64_t nq_host,
                   double *out, int64_t x1_lo, int64_t x1_hi, int64_t chunk, void *asm_work,
                   int64_t asm_work_bytes, void *wait_event) {
  RS_REQUIRE(out && asm_work && 0 <= x1_lo && x1_lo < x1_hi && x1_hi <= n && chunk >= 1,
             "rs_back_tucker: bad slab arguments");
  int st = rs_back(U, b, n, r1, r2, r3, table, ld_table, R, starts, z, w, count, Z1, Z2, Z3, core,
                   work, work_bytes, stream, c1, c2, zq, bstart, bc3, nb, nq_host);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  int flags = RS_ASM_LONG | RS_ASM_ACCUMULATE;
  if (chunk >= x1_hi - x1_lo) {
    // one chunk: the Tucker operands do not depend on the short-range planes,
    // so they are formed before the wait (C5: 24 ms that overlap the prefetch)
    if ((st = rs_assemble_planes(core, r1, r2, r3, Z1, Z2, Z3, n, nullptr, nullptr, 0, 0, nullptr,
                                 nullptr, nullptr, nullptr, nullptr, nullptr, 0, x1_lo, x1_hi,
                                 flags | RS_ASM_F_ONLY, out, asm_work, asm_work_bytes, stream)))
      return st;
    flags |= RS_ASM_F_READY;
  }
  if (wait_event && cudaStreamWaitEvent(s, (cudaEvent_t)wait_event, 0) != cudaSuccess)
    return fail(RS_ERR_CUDA, "rs_back_tucker: wait");
  for (int64_t p0 = x1_lo; p0 < x1_hi; p0 += chunk) {
    const int64_t p1 = std::min<int64_t>(x1_hi, p0 + chunk);
    if ((st = rs_assemble_planes(core, r1, r2, r3, Z1, Z2, Z3, n, nullptr, nullptr, 0, 0, nullptr,
                                 nullptr, nullptr, nullptr, nullptr, nullptr, 0, p0, p1, flags,
                                 out + (p0 - x1_lo) * n * n, asm_work, asm_work_bytes, stream)))
      return st;
  }
  return RS_OK;
}
}  // extern "C"

// ------------------------------------------------------------ rank rule
// Host-side eps-rank of the top-b Ritz values (rankred.truncated_spectrum /
// rank_rule_fast in C: it sits between the eigen block's synchronisation and
// the back launch).  Reference: rankred.py:129-148 (_eps_rank).
namespace {
// numpy's float64 add.reduce of a contiguous vector: pairwise sum (8
// accumulators up to 128 elements, halves above)
double np_pairwise(const double *a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}
double np_sum(const double *a, int64_t n) {
  return n <= 0 ? 0.0 : np_pairwise(a, n);
}
}  // namespace

extern "C" {
int rs_rank_rule(const double *thetas, const double *traces, int64_t m, int64_t b, int64_t n,
                 double eps, const int64_t *forced, int64_t limit, int64_t iters,
                 int64_t *rank_out, double *tail_out, double *total_out) {
  RS_REQUIRE(thetas && traces && m >= 1 && b >= 1 && b <= 4096 && rank_out && tail_out &&
                 total_out,
             "rs_rank_rule: bad arguments");
  std::vector<double> th((size_t)b), tails((size_t)b);
  for (int64_t l = 0; l < m; ++l) {
    for (int64_t k = 0; k < b; ++k) th[k] = thetas[l * b + k] > 0.0 ? thetas[l * b + k] : 0.0;
    const double tot_th = np_sum(th.data(), b);
    const double rem = b < n ? std::max(traces[l] - tot_th, 0.0) : 0.0;
    const double total = tot_th + rem;
    double acc = 0.0;
    for (int64_t k = b - 1; k >= 0; --k) {
      acc += th[k];
      tails[k] = acc + rem;
    }
    total_out[l] = total;
    rank_out[l] = -1;
    tail_out[l] = 0.0;
    int64_t r;
    if (forced && forced[l] > 0) {
      r = forced[l];
    } else if (total == 0.0) {
      r = 1;
    } else {
      const double thr = eps * total;
      r = -1;
      for (int64_t k = 0; k < b; ++k)
        if (tails[k] <= thr) {
          r = k;
          break;
        }
      if (r < 0) continue;
      r = std::max<int64_t>(r, 1);
    }
    if (limit > 0) r = std::min(r, limit);
    if (b < n) {
      const double lam_r = (0 < r && r <= b) ? th[r - 1] : 0.0;
      if (r >= b || lam_r <= 0.0 || th[0] <= 0.0 ||
          1e2 * std::pow(th[b - 1] / lam_r, (double)iters) * std::sqrt(lam_r / th[0]) > 1e-11)
        continue;
    }
    rank_out[l] = r;
    tail_out[l] = r < b ? tails[r] : 0.0;
  }
  return RS_OK;
}
}  // extern "C"
