// Internal launcher of the fused Tucker + dense-L0 grid kernel (rs_fused.cu).
#pragma once

#include "rs_common.cuh"

namespace rsb {
int fused_l0_smem_bytes(int64_t K);
bool fused_l0_supported(int64_t n, int64_t K, int64_t gamma);
// out[((x1 - x1_lo) n + x2) n + x3] = sum_c A[g, c] Bt[x3, c] + sum_p zq_p L0[x - c_p + gamma]
// (g = (x1 - x1_lo) n + x2: A's rows start at plane x1_lo)
int launch_fused_l0(const double *A, int64_t lda, const double *Bt, int64_t ldb, int64_t K,
                    const double *L0, int64_t gamma, int64_t n, const int32_t *c1,
                    const int32_t *c2, const double *zq, const int32_t *bstart,
                    const int32_t *bc3, const int32_t *nb_dev, int64_t x1_lo, int64_t x1_hi,
                    double *out, cudaStream_t s);
}  // namespace rsb
