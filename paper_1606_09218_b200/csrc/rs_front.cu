// Front of the RS build in one host call: snap -> node sort -> bucket-ordered
// copies -> shift histograms -> short-range bucket table, all enqueued on one
// stream from C++ (the Python driver's per-call overhead was the critical
// path of a C2 step).  Buffers live in one caller-owned region whose layout
// rs_front_offsets describes.  Reference: particles.py:302-329 (snap),
// assembly.py:139-184 / formats.py:179-244 (CCT buckets), rankred.py:82-126
// (the shift regrouping behind the histograms).
#include <cub/device/device_radix_sort.cuh>

#include "rs_common.cuh"

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
             int64_t work_bytes, void *side, int oz_slices) {
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
  if (cudaEventRecord(ev[dev & 63], s) != cudaSuccess ||
      cudaStreamWaitEvent(as_stream(side), ev[dev & 63], 0) != cudaSuccess)
    return fail(RS_ERR_CUDA, "rs_front: stream dependency");
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(n, count));
  const int flags = RS_ASM_SHORT | RS_ASM_OZ(oz_slices);
  const int64_t one = rs_assemble_workspace_bytes(n, 1, 1, nb_max, Rs, flags);
  const int64_t per = rs_assemble_workspace_bytes(n, 2, 1, nb_max, Rs, flags) - one;
  const int64_t chunk = std::max<int64_t>(
      1, std::min<int64_t>(x1_hi - x1_lo, (work_bytes - (one - per)) / std::max<int64_t>(per, 1)));
  for (int64_t p0 = x1_lo; p0 < x1_hi; p0 += chunk) {
    const int64_t p1 = std::min<int64_t>(x1_hi, p0 + chunk);
    if ((st = rs_assemble_planes(nullptr, 1, 1, 1, nullptr, nullptr, nullptr, n, ul, wl, Rs, gamma,
                                 (const int32_t *)P(F_C1), (const int32_t *)P(F_C2),
                                 (const double *)P(F_ZQ), (const int32_t *)P(F_BSTART),
                                 (const int32_t *)P(F_BC3), (const int32_t *)P(F_NB), nb_max, p0,
                                 p1, flags, out + (p0 - x1_lo) * n * n, work, work_bytes,
                                 side)))
      return st;
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
}  // namespace

extern "C" {
int rs_shift_project3(const double *Z1, const double *Z2, const double *Z3, int64_t r1, int64_t r2,
                      int64_t r3, int64_t n, const double *table, int64_t ld_table, int64_t R,
                      int64_t n_shift, double *TT1, double *TT2, double *TT3, void *stream);
int64_t rs_core_workspace_bytes(int64_t r1, int64_t r2, int64_t r3, int64_t count, int64_t R);
int rs_core(const double *TT1, const double *TT2, const double *TT3, int64_t r1, int64_t r2,
            int64_t r3, int64_t n_shift, int64_t R, const int64_t *shift, const double *z,
            const double *w, int64_t count, double *core, void *work, int64_t work_bytes,
            void *stream);

int64_t rs_back_workspace_bytes(int64_t n, int64_t r1, int64_t r2, int64_t r3, int64_t count,
                                int64_t R) {
  return round_up((r1 + r2 + r3) * n * R * 8, 256) + rs_core_workspace_bytes(r1, r2, r3, count, R);
}

/* U: (3, b, n) Ritz rows (descending); Z_l (n, r_l) = U[l, :r_l]^T; core
 * (r1, r2, r3) of the shift-structured long part. */
int rs_back(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
            const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
            const double *z, const double *w, int64_t count, double *Z1, double *Z2, double *Z3,
            double *core, void *work, int64_t work_bytes, void *stream) {
  RS_REQUIRE(r1 >= 1 && r2 >= 1 && r3 >= 1 && r1 <= b && r2 <= b && r3 <= b && n >= 2,
             "rs_back: bad ranks");
  if (work_bytes < rs_back_workspace_bytes(n, r1, r2, r3, count, R))
    return fail(RS_ERR_CAPACITY, "rs_back: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t tot = n * (r1 + r2 + r3);
  k_ritz_to_factors<<<(unsigned)std::min<int64_t>(ceil_div(tot, 256), 1024), 256, 0, s>>>(
      U, b, n, (int)r1, (int)r2, (int)r3, Z1, Z2, Z3);
  int st;
  if ((st = check_launch("rs_back factors"))) return st;
  double *TT1 = (double *)work, *TT2 = TT1 + r1 * n * R, *TT3 = TT2 + r2 * n * R;
  if ((st = rs_shift_project3(Z1, Z2, Z3, r1, r2, r3, n, table, ld_table, R, n, TT1, TT2, TT3,
                              stream)))
    return st;
  char *cw = (char *)work + round_up((r1 + r2 + r3) * n * R * 8, 256);
  return rs_core(TT1, TT2, TT3, r1, r2, r3, n, R, starts, z, w, count, core, cw,
                 rs_core_workspace_bytes(r1, r2, r3, count, R), stream);
}
}  // extern "C"
