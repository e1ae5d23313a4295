/* CPU ORACLE (test infrastructure only): C restatement of the reference's
 * dense_cct accumulation loop, rstensor formats.py:432-445.
 *
 *   for nu in range(N):
 *       out[clipped window of centre c_nu] += z_nu * L0[matching local window]
 *
 * Restated per x1 plane so planes can run in parallel (pthreads); inside a
 * plane every output element still receives its contributions in ascending
 * particle order, each as a rounded product z*L0 added to the running value,
 * exactly like the numpy loop -- compiled with -ffp-contract=off the result is
 * bit-identical to the reference.  L0 is the dense (W,W,W) local tensor. */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef struct {
  const double *L0;
  int64_t gamma;
  const int64_t *centers;
  const double *z;
  int64_t count, n, x1_lo, x1_hi, stride, first;
  double *out;
} job_t;

static void *plane_worker(void *arg) {
  const job_t *j = (const job_t *)arg;
  const double *L0 = j->L0;
  const int64_t gamma = j->gamma, count = j->count, n = j->n;
  const int64_t *centers = j->centers;
  const double *z = j->z;
  const int64_t W = 2 * gamma + 1;
  for (int64_t x1 = j->x1_lo + j->first; x1 < j->x1_hi; x1 += j->stride) {
    double *plane = j->out + (x1 - j->x1_lo) * n * n;
    for (int64_t nu = 0; nu < count; ++nu) {
      const int64_t c0 = centers[3 * nu], c1 = centers[3 * nu + 1], c2 = centers[3 * nu + 2];
      const int64_t d0 = x1 - c0;
      if (d0 < -gamma || d0 > gamma) continue;
      const int64_t lo1 = c1 - gamma < 0 ? 0 : c1 - gamma;
      const int64_t hi1 = c1 + gamma > n - 1 ? n - 1 : c1 + gamma;
      const int64_t lo2 = c2 - gamma < 0 ? 0 : c2 - gamma;
      const int64_t hi2 = c2 + gamma > n - 1 ? n - 1 : c2 + gamma;
      const double zz = z[nu];
      const double *Lp = L0 + (d0 + gamma) * W * W;
      for (int64_t x2 = lo1; x2 <= hi1; ++x2) {
        const double *Lr = Lp + (x2 - c1 + gamma) * W + (lo2 - c2 + gamma);
        double *o = plane + x2 * n + lo2;
        for (int64_t x3 = 0; x3 <= hi2 - lo2; ++x3) {
          double t = zz * Lr[x3];
          o[x3] = o[x3] + t;
        }
      }
    }
  }
  return NULL;
}

void oracle_dense_cct(const double *L0, int64_t gamma, const int64_t *centers, const double *z,
                      int64_t count, int64_t n, int64_t x1_lo, int64_t x1_hi, double *out) {
  const int64_t planes = x1_hi - x1_lo;
  memset(out, 0, sizeof(double) * (size_t)(planes * n * n));
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  const char *env = getenv("ORACLE_THREADS");
  if (env) nt = atol(env);
  if (nt < 1) nt = 1;
  if (nt > planes) nt = planes;
  pthread_t th[256];
  job_t jobs[256];
  if (nt > 256) nt = 256;
  for (long t = 0; t < nt; ++t) {
    jobs[t] = (job_t){L0, gamma, centers, z, count, n, x1_lo, x1_hi, nt, t, out};
    pthread_create(&th[t], NULL, plane_worker, &jobs[t]);
  }
  for (long t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}
