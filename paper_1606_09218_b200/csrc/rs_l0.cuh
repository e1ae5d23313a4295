// Layout of the dense local tensor L0 for the gathers (rs_short_l0.cu,
// rs_fused.cu): "pair table" P[par][da][b][j], par in {0, 1}, da in [0, gamma],
// b in [0, W), j in [0, pitch), W = 2 gamma + 1:
//
//   P[par][da][b][j] = L0[gamma + da][b][j - 2 + par]   (0 outside [0, W))
//
// * folded in x1: the local factors of assemble_short's window are symmetric
//   about gamma (the doubled table's erf cell integrals are even in the
//   offset; checked on the host), so L0[a][b][c] = L0[g + |a - g|][b][c];
//   x2 stays unfolded so the rows of consecutive x2 are one pitch apart;
// * a fixed pitch of 256 doubles (W + 3 <= 256, i.e. gamma <= 126): the
//   rows a warp reads for consecutive x2 are compile-time immediates off one
//   address (the gather is integer-issue bound, not L2 bound, without this);
// * two copies shifted by one element, so the two consecutive x3 values
//   (cA, cA + 1) a lane needs are ONE aligned 16-byte load at any cA: parity
//   par = cA & 1 picks the copy, j = cA + 2 - par is even.  16-byte L2 loads
//   stream ~1.5x the bandwidth of 8-byte ones on B200 (tools/probe_l2.cu:
//   17.8 vs 11.9 TB/s);
// * the zero margins make a pair that straddles the window edge read zeros
//   for its outside half: a lane loads iff cA in [-1, W - 1].
// Values are the same sums as the unfolded W^3 table in the same order.
#pragma once

#include <stdint.h>

namespace rsb {

constexpr int L0_PITCH = 256;
__host__ __device__ inline bool l0_gamma_ok(int64_t gamma) { return 2 * gamma + 1 + 3 <= L0_PITCH; }
__host__ __device__ inline int64_t l0_rows(int64_t gamma) { return 2 * (gamma + 1) * (2 * gamma + 1); }
__host__ __device__ inline int64_t l0_pair_doubles(int64_t gamma) { return l0_rows(gamma) * L0_PITCH; }

// element offset of row (par, da, b), column j = cA + 2 - par
__device__ __forceinline__ int l0_off(int par, int da, int b, int cA, int gamma) {
  return ((par * (gamma + 1) + da) * (2 * gamma + 1) + b) * L0_PITCH + cA + 2 - par;
}

__device__ __forceinline__ uint64_t l0_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// predicated 16-byte L2 load (zeros, and no memory access, when !ok)
__device__ __forceinline__ double2 l0_ld2(const double *p, bool ok, uint64_t pol) {
  double2 v = make_double2(0.0, 0.0);
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n"
      " @q ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %4;\n}"
      : "+d"(v.x), "+d"(v.y)
      : "l"(p), "r"((int)ok), "l"(pol));
  return v;
}

// acc.{x,y} += z * (16-byte L2 load at p) when ok; nothing (no load, no FMA) otherwise
__device__ __forceinline__ void l0_fma2(double2 &acc, double z, const double *p, bool ok,
                                        uint64_t pol) {
  asm("{\n .reg .pred q;\n .reg .f64 t0, t1;\n setp.ne.b32 q, %4, 0;\n"
      " @q ld.global.nc.L2::cache_hint.v2.f64 {t0, t1}, [%3], %5;\n"
      " @q fma.rn.f64 %0, %2, t0, %0;\n @q fma.rn.f64 %1, %2, t1, %1;\n}"
      : "+d"(acc.x), "+d"(acc.y)
      : "d"(z), "l"(p), "r"((int)ok), "l"(pol));
}

}  // namespace rsb
