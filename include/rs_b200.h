/*
 * rs_b200.h -- C ABI of the B200 range-separated (RS) tensor assembly path.
 *
 * The reference (rstensor 0.1.0, pure numpy/scipy) has no FFI layer: its
 * boundary is the public Python API in pkg/src/rstensor/__init__.py:4-94.
 * Every entry point below replaces the numerical core of one reference
 * function; the Python package paper_1606_09218_b200 binds them with ctypes
 * (paper_1606_09218_b200/_native.py) and keeps the reference's names,
 * argument meanings and exception classes on top.
 *
 * Conventions
 *   - All arrays are device pointers (cudaMalloc / torch CUDA storage),
 *     row-major, fp64 unless the name says i64/i32.  "ld" = leading dimension
 *     in elements.  No pointer is retained after a call returns.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call
 *     only enqueues work; nothing synchronises the host.
 *   - Return value: RS_OK or one of the RS_ERR_* codes; rs_last_error()
 *     returns the message of the last failure on the calling thread.
 *   - Results are deterministic: no floating-point atomics, fixed-order
 *     split-K reductions.
 */
#ifndef RS_B200_H
#define RS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_OK 0
#define RS_ERR_DOMAIN 1      /* -> DomainError      */
#define RS_ERR_CAPACITY 2    /* -> CapacityError    */
#define RS_ERR_NUMERICAL 3   /* -> NumericalError   */
#define RS_ERR_CUDA 4        /* -> RsTensorError    */
#define RS_ERR_UNSUPPORTED 5 /* -> CapabilityError  */

int rs_abi_version(void);
const char *rs_last_error(void);

/* Instrumentation: number of kernels this library has launched, and optional
 * CUDA-event timing of the hot launches ("gemm_plane", "short_rows", "syrk",
 * "core", "shift_project").  rs_prof_query synchronises on the recorded events. */
int64_t rs_launch_count(void);
int rs_prof_enable(int on);
int rs_prof_query(const char *name, double *total_ms, int64_t *count);

/* (a2) snap_to_grid, particles.py:302-329.
 * idx[3p+l] = clip(ceil(pos[3p+l]/h + n/2 - 0.5), 1, n-1);
 * disp[p] = |pos_p - (idx_p - n/2) h|_2 (IEEE-exact, no FMA contraction);
 * optional: key[p] = (x3 n + x2) n + x1 (node key, x3-major) and
 * snapped[3p+l] = (idx - n/2) h (grid.position, particles.py:89-91). */
int rs_snap(const double *pos, int64_t count, double h, int64_t n,
            int64_t *idx, double *disp, int64_t *key, double *snapped, void *stream);

/* After sorting the node keys (ks ascending, order = permutation): copies in
 * bucket order c1s/c2s/zqs, window starts starts = n - idx (assembly.py:131),
 * *dup_pos = the first duplicated node key (int64; -1 if none: the
 * ResolutionError of particles.py:319-325) and the max displacement as the
 * bits of a non-negative double. */
int rs_prep(const int64_t *ks, const int64_t *order, const int64_t *idx,
            const double *z, const double *disp, int64_t count, int64_t n,
            int32_t *c1s, int32_t *c2s, double *zqs, int64_t *starts,
            uint64_t *dup_pos, uint64_t *dmax_bits, void *stream);

/* (a7) window gather, assembly.py:111-136 (assemble_long) and the
 * shift-merged Gram operand of rankred.py:90-96.
 * out[i*ld_out + g*n_terms + k] = gscale[g] * tscale[k] *
 *                                 table[(starts[g]+i)*ld_table + term0 + k]
 * for i < n_rows, g < n_groups, k < n_terms.  gscale/tscale may be NULL (=1). */
int rs_gather_windows(const double *table, int64_t ld_table, int64_t n_rows,
                      const int64_t *starts, int64_t n_groups, int64_t n_terms,
                      int64_t term0, const double *gscale, const double *tscale,
                      double *out, int64_t ld_out, void *stream);

/* (a8) Gram of a side matrix, rankred.py:91 (gram = a @ a.T).
 * G (n x n, ld n) = A A^T with A n x K (ld lda, lda even, A 16-byte aligned).
 * FP64 tensor cores (DMMA), lower-triangle tiles, fixed-order split-K into
 * `work` (rs_syrk_workspace_bytes), mirrored to a full symmetric matrix. */
int64_t rs_syrk_workspace_bytes(int64_t n, int64_t K);
int rs_syrk(const double *A, int64_t lda, int64_t n, int64_t K, double *G,
            void *work, int64_t work_bytes, void *stream);

/* Plain NT GEMM on DMMA: C (M x N, ldc) = A (M x K, lda) * B^T (B: N x K, ldb).
 * Used for projections Z^T U (rankred.py:175) on explicit side matrices. */
int rs_gemm_nt(const double *A, int64_t lda, const double *B, int64_t ldb,
               double *C, int64_t ldc, int64_t M, int64_t N, int64_t K, void *stream);

/* (a10) shift projection: for the doubled table T (ld_table) and an orthonormal
 * basis Z (n x r, ld ldz): TT[(a*n_shift + s)*R + k] = sum_i Z[i*ldz+a] *
 * T[(s+i)*ld_table + k], s < n_shift, k < R.  This is Z^T U restricted to one
 * particle shift -- rankred.py:175 without materialising U. */
int rs_shift_project(const double *Z, int64_t ldz, int64_t n, int64_t r,
                     const double *table, int64_t ld_table, int64_t R,
                     int64_t n_shift, double *TT, void *stream);

/* (a8) shift histograms of the long side matrices: c[l*n + s] = sum of z_p^2
 * over particles p whose mode-l window starts at s = n - idx[3p+l] (l = 0,1,2),
 * summed in particle order; cnt3[x] = number of particles with idx[3p+2] == x.
 * With them G_l = sum_s c[l][s] sum_k w_k^2 u_k[s:s+n] u_k[s:s+n]^T equals
 * the reference Gram A A^T of rankred.py:91 (A = side matrix * |weights|). */
int rs_shift_hist(const int64_t *idx, const double *z, int64_t count, int64_t n,
                  double *c, int32_t *cnt3, void *stream);

/* The three per-mode Grams of the shift-structured long part in one call
 * (G: 3 x n x n): operands X_l[:, (s,k)] = sqrt(c[l][s]) |w_k| T[s:s+n, k]
 * (c from rs_shift_hist, wabs = |w_k|, k < R) and X_l X_l^T on DMMA. */
int64_t rs_gram_shifted_workspace_bytes(int64_t n, int64_t R);
int rs_gram_shifted(const double *table, int64_t ld_table, int64_t n, int64_t R,
                    const double *c, const double *wabs, double *G, void *work,
                    int64_t work_bytes, void *stream);

/* Top-b eigenpairs of nmat symmetric PSD n x n matrices G (contiguous), for
 * the eigen-truncation of rankred.py:90-96/129-148: block subspace iteration
 * (iters steps, CGS2), Rayleigh-Ritz, cyclic Jacobi.  evals (nmat x b,
 * descending), U (nmat x b x n, rows = Ritz vectors, largest-|entry|
 * positive), trace (nmat).  b even, b <= min(n, 96). */
/* (a8) full spectra of m symmetric n x n matrices (cuSOLVER syevd, one forked
 * stream per matrix, no host sync): G is overwritten with the eigenvectors as
 * the ROWS of each row-major block, evals (m x n) ascending.  Reference:
 * rankred.py:92 (eigh of the side Gram). */
int64_t rs_eigh_workspace_bytes(int64_t m, int64_t n);
int rs_eigh(double *G, int64_t m, int64_t n, double *evals, void *work, int64_t work_bytes,
            void *stream);
int64_t rs_topeig_workspace_bytes(int64_t nmat, int64_t n, int64_t b);
int rs_topeig(const double *G, int64_t nmat, int64_t n, int64_t b, int64_t iters,
              double *evals, double *U, double *trace, void *work, int64_t work_bytes,
              void *stream);

/* The long-range chain up to the host's rank decision in ONE call, enqueued
 * right behind rs_front on the same stream: rs_gram_shifted (hist = the
 * front's shift histograms) -> rs_topeig (3 modes, block b) -> packed
 * [evals (3b) | trace (3) | dmax | duplicate-node key | occupied x3 count]
 * (3b + 6 doubles) into packed_dev and then into pinned packed_host, and the
 * cudaEvent_t `done` recorded; the host waits on `done` only.  nb may be NULL.
 * Reference: rankred.py:82-148 (side Gram, eigh, eps-rank inputs). */
int rs_chain_eig(const double *table, int64_t ld_table, int64_t n, int64_t R,
                 const double *hist, const double *wabs, double *G, void *gram_work,
                 int64_t gram_work_bytes, int64_t b, int64_t iters, double *evals,
                 double *U, double *trace, void *eig_work, int64_t eig_work_bytes,
                 const double *dmax, const int64_t *dup_key, const int32_t *nb,
                 double *packed_dev, double *packed_host, void *done, void *stream);

/* The three modes of rs_shift_project in one launch (Z_l contiguous n x r_l). */
int rs_shift_project3(const double *Z1, const double *Z2, const double *Z3,
                      int64_t r1, int64_t r2, int64_t r3, int64_t n,
                      const double *table, int64_t ld_table, int64_t R, int64_t n_shift,
                      double *TT1, double *TT2, double *TT3, void *stream);

/* (a10) RHOSVD core, rankred.py:151-161 (_core_from_projections) on the
 * particle-major term order of assembly.py:127-135:
 * core[(a*r2+b)*r3+c] = sum_p z[p] sum_k w[k] P1(a,p,k) P2(b,p,k) P3(c,p,k)
 * with Pl(a,p,k) = TTl[(a*n_shift + shift[3p+l])*R + k].  Computed as a DMMA
 * GEMM (Khatri-Rao rows generated on the fly) with fixed-order split-K;
 * `work` (rs_core_workspace_bytes) holds the gathered P_l and the partials. */
int64_t rs_core_workspace_bytes(int64_t r1, int64_t r2, int64_t r3, int64_t count, int64_t R);
int rs_core(const double *TT1, const double *TT2, const double *TT3,
            int64_t r1, int64_t r2, int64_t r3, int64_t n_shift, int64_t R,
            const int64_t *shift, const double *z, const double *w, int64_t count,
            double *core, void *work, int64_t work_bytes, void *stream);

/* (a12-a14) RS grid assembly of x1-planes [x1_lo, x1_hi):
 * out[((x1-x1_lo)*n + x2)*n + x3] (=, or += with RS_ASM_ACCUMULATE)
 *     [RS_ASM_LONG]  Tucker(core,V1,V2,V3)[x1,x2,x3]
 *   + [RS_ASM_SHORT] sum_p z_p L0[x - c_p + gamma]
 * with L0 = sum_k wl[k] ul[.,k] (x) ul[.,k] (x) ul[.,k] (the normalised CCT
 * local tensor, formats.py:103-118, 432-445), windows clipped to the grid.
 * Computed as one plane GEMM on FP64 tensor cores: rows (x1,x2), columns x3,
 * K = [Tucker ranks | copies merged by x3 index x R_s].
 * Copies are bucketed by their x3 index: bucket b holds the x3-sorted entries
 * [bstart[b], bstart[b+1]) with x3 index bc3[b] (ascending), x1/x2 indices
 * c1/c2 and charges zq; *nb_dev buckets (device), nb_max >= *nb_dev sizes
 * the launch (rs_short_layout produces all of these on the device).
 * Workspace: rs_assemble_workspace_bytes(n, planes, max rank, nb_max, Rs, flags). */
#define RS_ASM_LONG 1
#define RS_ASM_SHORT 2
#define RS_ASM_ACCUMULATE 4
/* long part only, split in two calls on the same workspace: RS_ASM_F_ONLY
 * computes the per-plane Tucker operands A = V2 (core x1 V1[x1]) and returns;
 * RS_ASM_F_READY skips that stage (A already in the workspace) */
#define RS_ASM_F_ONLY 16
#define RS_ASM_F_READY 32
/* the per-distance term table (first (n+1) ints of the workspace) is already
 * filled for this plan (ul, wl, Rs, gamma) */
#define RS_ASM_KOFD_READY 64
/* plane GEMM as Ozaki-split FP64 with s int8 slices (tcgen05 kind::i8), s in 6..8 */
#define RS_ASM_OZ(s) ((s) << 8)
int64_t rs_assemble_workspace_bytes(int64_t n, int64_t planes, int64_t rmax,
                                    int64_t nb_max, int64_t Rs, int flags);
int rs_assemble_planes(const double *core, int64_t r1, int64_t r2, int64_t r3,
                       const double *V1, const double *V2, const double *V3,
                       int64_t n, const double *ul, const double *wl, int64_t Rs,
                       int64_t gamma, const int32_t *c1, const int32_t *c2,
                       const double *zq, const int32_t *bstart, const int32_t *bc3,
                       const int32_t *nb_dev, int64_t nb_max, int64_t x1_lo,
                       int64_t x1_hi, int flags, double *out, void *work,
                       int64_t work_bytes, void *stream);

/* Short-range part by dense-L0 gather (low window overlap):
 * out[((x1-x1_lo)*n + x2)*n + x3] (= or +=) sum_p zq_p L0[x - c_p + gamma]
 * over the same bucket layout as rs_assemble_planes; L0 (W^3, W = 2 gamma+1)
 * from rs_short_l0_table.  rs_short_method picks RS_SHORT_GEMM (plane GEMM)
 * or RS_SHORT_L0 from the mean window overlap (env RSB200_SHORT=gemm|l0
 * forces one).  Reference: formats.py:423-445 (dense_cct). */
#define RS_SHORT_GEMM 0
#define RS_SHORT_L0 1
#define RS_SHORT_MMA 2
int rs_short_method(int64_t n, int64_t count, int64_t gamma, int64_t Rs);
int64_t rs_short_l0_bytes(int64_t gamma);
int rs_short_l0_table(const double *ul, const double *wl, int64_t Rs, int64_t gamma,
                      double *L0, void *stream);
/* (a13) dense_cct, formats.py:423-445, as ONE fused FP64 tensor-core kernel
 * (RS_SHORT_MMA): per 8 x 16 x 64 output tile a GEMM over (x3 bucket, term)
 * columns whose A fragments are formed in registers from shared-memory staged
 * 1-D factors (outer products summed over the bucket's copies near the tile)
 * and whose B fragments are gathered from the same table; nothing but the
 * grid goes to HBM.  work: rs_short_mma_workspace_bytes(n, gamma).  flags:
 * RS_ASM_ACCUMULATE adds to `out`; RS_ASM_KOFD_READY: the per-distance term
 * table at offset 0 of `work` is already filled. */
int rs_short_mma_supported(int64_t n, int64_t gamma, int64_t Rs);
int64_t rs_short_mma_workspace_bytes(int64_t n, int64_t gamma);
int rs_assemble_short_mma(const double *ul, const double *wl, int64_t Rs, int64_t gamma,
                          int64_t n, int64_t count /* copies: sizes the CTAs' tile batches */,
                          const int32_t *c1, const int32_t *c2, const double *zq,
                          const int32_t *bstart, const int32_t *bc3, const int32_t *nb_dev,
                          int64_t x1_lo, int64_t x1_hi, int flags, double *out, void *work,
                          int64_t work_bytes, void *stream);
int rs_assemble_short_l0(const double *L0, int64_t gamma, int64_t n, const int32_t *c1,
                         const int32_t *c2, const double *zq, const int32_t *bstart,
                         const int32_t *bc3, const int32_t *nb_dev, int64_t x1_lo,
                         int64_t x1_hi, int accumulate, double *out, void *stream);

/* Single-pass grid store of the low-overlap regime (formats.py:448-453,
 * dense_rs = TuckerTensor.dense + dense_cct, the short part by the dense-L0
 * gather): out[((x1-x1_lo)*n + x2)*n + x3] = Tucker[x] + sum_p zq_p L0[x - c_p + gamma]
 * for x1 in [x1_lo, x1_hi), every grid value stored once.  The per-plane
 * Tucker operands must have been formed on `work` by
 * rs_assemble_planes(RS_ASM_LONG | RS_ASM_F_ONLY) for planes [a_lo, a_hi)
 * containing [x1_lo, x1_hi) (same ranks, same workspace).  Bitwise equal to
 * rs_assemble_short_l0 followed by the accumulating Tucker pass.
 * rs_fused_l0_supported: 1 when the kernel handles (n, r3, gamma). */
int rs_assemble_fused_l0(int64_t r1, int64_t r2, int64_t r3, const double *V3, int64_t n,
                         const double *L0, int64_t gamma, const int32_t *c1, const int32_t *c2,
                         const double *zq, const int32_t *bstart, const int32_t *bc3,
                         const int32_t *nb_dev, int64_t a_lo, int64_t a_hi, int64_t x1_lo,
                         int64_t x1_hi, double *out, void *work, int64_t work_bytes,
                         void *stream);
int rs_fused_l0_supported(int64_t n, int64_t r3, int64_t gamma);

/* L2 read bandwidth probe: every CTA streams the first `bytes` of buf (sized
 * to fit in L2) `iters` times with L1-bypassing loads (the roofline of
 * rs_assemble_short_l0; time it with events on `stream`). */
int rs_l2_probe(const double *buf, int64_t bytes, int64_t iters, double *out, void *stream);

/* Bucket layout of the short-range copies from the x3 occupancy counts
 * cnt3 (n): bc3 (capacity n), bstart (capacity n+1), *nb (device int). */
int rs_short_layout(const int32_t *cnt3, int64_t n, int32_t *bstart, int32_t *bc3,
                    int32_t *nb, void *stream);

/* (a15) Tucker point values, formats.py:347-352 (eval_tucker_many). */
int rs_eval_tucker(const double *core, int64_t r1, int64_t r2, int64_t r3,
                   const double *V1, const double *V2, const double *V3,
                   const int64_t *idx, int64_t m, double *out, void *stream);

/* (a15) CCT point values, formats.py:380-398 (eval_cct) for m points; also
 * returns the number of covering copies per point (hits) so the caller can
 * apply the soft-overlap cap (CapacityError).  centers i64 (count x 3). */
int rs_eval_cct(const double *ul, const double *wl, int64_t Rs, int64_t gamma,
                const int64_t *centers, const double *zq, int64_t count,
                const int64_t *idx, int64_t m, double *out, int32_t *hits,
                void *stream);

/* (a16-a18) windowed long-range pair sums, observables.py:175-259.
 * For every target j in [0, m): with offsets o = idx[tgt[j]] - idx[p] (+ shift):
 *   base[j]      = sum_{p != excl} z[p] * pl(o)            (double-double)
 *   dshift[3j+a] = sum_{p != tgt} z[p] * (pl(o - e_a) - pl(o))
 * where pl(o) = sum_{k<R_l} w[k] T[n0+o0,k] T[n0+o1,k] T[n0+o2,k] / h3.
 * mode 0: energy terms (all p, incl. self), mode 1: forces (p != j),
 * mode 2: dshift[3j+a] = sum_{p != tgt} |z[p]| (|pl(o - e_a)| + |pl(o)|), the
 * magnitude the mode-1 differences cancel from (their rounding-error scale). */
int rs_pair_sums(const double *table, int64_t ld_table, int64_t n0,
                 const double *w, int64_t Rl, double h3,
                 const int64_t *idx, const double *z, int64_t count,
                 const int64_t *tgt, int64_t m, int mode,
                 double *base, double *dshift, void *stream);

/* Compensated (double-double, fixed order) sum of v[0..m), result in out[0]. */
int rs_sum_dd(const double *v, int64_t m, double *out, void *work,
              int64_t work_bytes, void *stream);
int64_t rs_sum_workspace_bytes(int64_t m);

/* ---- build front ---------------------------------------------------------
 * snap + node sort (CUB radix) + bucket-ordered copies + shift histograms +
 * short-range bucket table in ONE call (replaces rs_snap, a torch sort,
 * rs_prep, rs_shift_hist, rs_short_layout issued one by one from Python).
 * Buffers: one region, byte offsets from rs_front_offsets (18 slots + total):
 * idx | disp | key | snapped | sorted keys | order | c1 | c2 | zq | starts |
 * scal (dup key, dmax) | hist (3,n) | cnt3 | bstart | bc3 | nb | iota | scratch.
 * Reference: particles.py:302-329, assembly.py:139-184, rankred.py:82-126. */
int rs_front_offsets(int64_t count, int64_t n, int64_t *offsets);
int rs_front(const double *pos, const double *z, int64_t count, double h, int64_t n,
             void *buf, int64_t buf_bytes, void *stream,
             /* optional: short-range planes [x1_lo, x1_hi) into `out` on `side`
              * (after the bucket table; NULL side = none) */
             const double *ul, const double *wl, int64_t Rs, int64_t gamma,
             int64_t x1_lo, int64_t x1_hi, double *out, void *work,
             int64_t work_bytes, void *side, int oz_slices,
             /* planes in groups of `group` (<= 0: one group); events[g]
              * (caller-created cudaEvent_t, or NULL) recorded on `side` when
              * group g is complete */
             int64_t group, void **events);

/* ---- build back: Ritz rows -> Tucker factors + shift projections + core in
 * one call (rs_shift_project3 + rs_core behind a transpose).  Reference:
 * rankred.py:151-177. */
int64_t rs_back_workspace_bytes(int64_t n, int64_t r1, int64_t r2, int64_t r3,
                                int64_t count, int64_t R, int64_t nq);
int rs_back(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
            const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
            const double *z, const double *w, int64_t count, double *Z1, double *Z2,
            double *Z3, double *core, void *work, int64_t work_bytes, void *stream,
            /* optional (NULL: particle-K core): the x3-bucket layout of the
             * short part (rs_front) -> the core GEMM runs over occupied x3
             * values x terms instead of particles x terms */
            const int32_t *c1, const int32_t *c2, const double *zq,
            const int32_t *bstart, const int32_t *bc3, const int32_t *nb,
            int64_t nq /* occupied x3 values if known on the host, else 0 */);

/* rs_back for one rank of a sharded run: the factors and shift
 * projections as in rs_back (replicated), but `core` receives only this
 * rank's partial of rankred.py:151-161's sum over the K = N (R_l+1) columns --
 * the x3 buckets [q_lo, q_hi) of the nq occupied ones on the bucket-K path,
 * the particles [p_lo, p_hi) on the particle-K path (the path is chosen from
 * sizes all ranks share).  The caller all-reduces `core` (r1 r2 r3 doubles). */
int rs_back_shard(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
                  const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
                  const double *z, const double *w, int64_t count, double *Z1, double *Z2,
                  double *Z3, double *core, void *work, int64_t work_bytes, void *stream,
                  const int32_t *c1, const int32_t *c2, const double *zq,
                  const int32_t *bstart, const int32_t *bc3, const int32_t *nb,
                  int64_t nq, int64_t q_lo, int64_t q_hi, int64_t p_lo, int64_t p_hi);

/* rs_back, then (after `wait_event`, a cudaEvent_t, when not NULL) the
 * Tucker part of planes [x1_lo, x1_hi) accumulated into `out` (the
 * prefetched short-range slab, (x1_hi - x1_lo) x n x n) by rs_assemble_planes
 * in chunks of `chunk` planes with `asm_work`: build_rs's post-rank device
 * work in one call.  Reference: rankred.py:151-177, formats.py:173-176. */
int rs_back_tucker(const double *U, int64_t b, int64_t n, int64_t r1, int64_t r2, int64_t r3,
                   const double *table, int64_t ld_table, int64_t R, const int64_t *starts,
                   const double *z, const double *w, int64_t count, double *Z1, double *Z2,
                   double *Z3, double *core, void *work, int64_t work_bytes, void *stream,
                   const int32_t *c1, const int32_t *c2, const double *zq,
                   const int32_t *bstart, const int32_t *bc3, const int32_t *nb,
                   int64_t nq_host, double *out, int64_t x1_lo, int64_t x1_hi,
                   int64_t chunk, void *asm_work, int64_t asm_work_bytes,
                   void *wait_event);

/* eps-rank rule on top-b Ritz values (host function, no device work), for m
 * modes: thetas (m x b, descending), traces (m); forced = NULL or m ranks
 * (> 0 forces); limit > 0 caps the rank.  rank_out[l] = -1 when the block is
 * too small / not converged to decide (convergence test
 * 1e2 (theta_{b-1}/theta_{r-1})^iters sqrt(theta_{r-1}/theta_0) <= 1e-11).
 * tail_out = sum of the eigenvalues beyond the rank (+ the uncaptured trace),
 * total_out = the captured sum + the uncaptured trace.  Reference:
 * rankred.py:129-148 (_eps_rank: smallest r with tail <= eps * total). */
int rs_rank_rule(const double *thetas, const double *traces, int64_t m, int64_t b, int64_t n,
                 double eps, const int64_t *forced, int64_t limit, int64_t iters,
                 int64_t *rank_out, double *tail_out, double *total_out);

/* ---- SM partitions ------------------------------------------------------
 * A non-blocking stream whose kernels run on a fixed subset of >= `sms` SMs
 * (green context, created once per (device, sms)); *sms_out = its SM count.
 * Used to keep SMs free for the latency-bound long-range chain while the
 * short-range planes are assembled concurrently.  No reference counterpart. */
int rs_partition_stream(int sms, int priority, void **stream_out, int *sms_out);

/* ---- tcgen05 int8 engine (building block of the Ozaki-split FP64 GEMM) --
 * C (M x N int32, ldc) = A (M x K int8, lda) * B (N x K int8, ldb)^T,
 * tcgen05.mma kind::i8 with the accumulator in TMEM.  K, lda, ldb multiples
 * of 16; 16-byte aligned bases.  No reference counterpart (kernel level). */
int rs_tc8_gemm_s8(const int8_t *A, int64_t lda, const int8_t *B, int64_t ldb,
                   int32_t *C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                   void *stream);

/* ---- Ozaki-split FP64 GEMM on the int8 tensor cores -----------------------
 * C (=, or += with accumulate) = A (M x K) B (N x K)^T in FP64: per-row
 * power-of-two scaling, `slices` (6..8) signed 7-bit int8 slices per operand,
 * the slice products with p + q < slices exact in int32 TMEM accumulators
 * (tcgen05.mma kind::i8), recombined in fp64.  Relative error per entry
 * ~ K 2^(-7 slices) of max|A_i.| max|B_j.|.  ranges: NULL or nr fp64 column
 * ranges per 64-column tile of C (columns outside them must hold zero B
 * entries for that tile).  No reference counterpart (kernel level). */
int64_t rs_oz_workspace_bytes(int64_t M, int64_t N, int64_t K, int slices);
int rs_oz_gemm(const double *A, int64_t lda, const double *B, int64_t ldb,
               double *C, int64_t ldc, int64_t M, int64_t N, int64_t K,
               const int64_t *ranges, int nr, int slices, int accumulate,
               void *work, int64_t work_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* RS_B200_H */
