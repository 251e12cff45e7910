/* masked_normaliser.c -- TEST INFRASTRUCTURE (never linked into the product).
 *
 * The reference's masked-grid normaliser for an OT plan on coordinates, in the
 * reference's exact order, for problems whose dense K cannot be held (config 4:
 * n = 1e6, 1e12 terms). It restates
 *   ot_probabilities     proj/src/sparsify.cpp:71-91  (ra_i = sqrt(a_i)/sa, cb_j = sqrt(b_j)/sb,
 *                                                      sa, sb sequential sums; grid = ra_i*cb_j)
 *   masked_grid_plan     proj/src/sparsify.cpp:49-67  (grid zeroed where K == 0; total = sequential
 *                                                      row-major sum; inv = 1/total)
 *   pairwise_cost        proj/src/geometry.cpp:16-59  (sequential d2, no FMA)
 *   kernel_from_cost     proj/src/geometry.cpp:83-102 (K = exp(-C/eps), C = d2/scale done by the caller)
 * Support test: d2 far from the underflow edge is decided by a bound with a
 * wide margin; every d2 within [740, 750]*eps*scale is decided by evaluating
 * the reference's expression exp(-(d2/scale)/eps) itself (glibc exp).
 *
 * Phase 1 (threads): per row, the ascending list of columns with K == 0.
 * Phase 2 (one thread): total += ra[i]*cb[j] over every supported (i, j) in
 * row-major order -- the reference's dependent chain of 1e12 fp64 adds.
 *
 * Usage: masked_normaliser x.bin y.bin n dim scale eps a.bin b.bin
 *   (fp64 row-major coords; fp64 weights) -> prints one JSON line.
 * Build: gcc -std=c11 -O2 -ffp-contract=off -pthread masked_normaliser.c -lm
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double *X, *Y;
static int64_t N;
static int DIM;
static double SCALE, EPS, LO, HI;
static uint32_t **masked;  /* per row: columns with K == 0 */
static int64_t *nmasked;
static int64_t next_row;
static pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;

static double *read_f64(const char *path, int64_t count) {
  FILE *f = fopen(path, "rb");
  if (!f) { perror(path); exit(2); }
  double *p = malloc(sizeof(double) * count);
  if (fread(p, sizeof(double), count, f) != (size_t)count) { fprintf(stderr, "short read %s\n", path); exit(2); }
  fclose(f);
  return p;
}

static void *worker(void *arg) {
  (void)arg;
  double *d2 = malloc(sizeof(double) * N);
  uint32_t *tmp = malloc(sizeof(uint32_t) * N);
  for (;;) {
    pthread_mutex_lock(&mu);
    int64_t r0 = next_row;
    next_row += 64;
    pthread_mutex_unlock(&mu);
    if (r0 >= N) break;
    int64_t r1 = r0 + 64 < N ? r0 + 64 : N;
    for (int64_t i = r0; i < r1; ++i) {
      const double *p = X + i * DIM;
      for (int64_t j = 0; j < N; ++j) {  /* sq_dist, geometry.cpp:16-24 */
        const double *q = Y + j * DIM;
        double s = 0.0;
        for (int k = 0; k < DIM; ++k) {
          const double diff = p[k] - q[k];
          s += diff * diff;
        }
        d2[j] = s;
      }
      int64_t m = 0;
      for (int64_t j = 0; j < N; ++j) {
        if (d2[j] < LO) continue;
        int zero;
        if (d2[j] > HI) zero = 1;
        else {
          const double c = d2[j] / SCALE;    /* caller's max/percentile normalisation */
          zero = exp(-c / EPS) == 0.0;       /* kernel_from_cost */
        }
        if (zero) tmp[m++] = (uint32_t)j;
      }
      nmasked[i] = m;
      masked[i] = m ? malloc(sizeof(uint32_t) * m) : NULL;
      if (m) memcpy(masked[i], tmp, sizeof(uint32_t) * m);
    }
  }
  free(d2);
  free(tmp);
  return NULL;
}

int main(int argc, char **argv) {
  if (argc != 9) {
    fprintf(stderr, "usage: %s x.bin y.bin n dim scale eps a.bin b.bin\n", argv[0]);
    return 2;
  }
  N = atoll(argv[3]);
  DIM = atoi(argv[4]);
  SCALE = atof(argv[5]);
  EPS = atof(argv[6]);
  X = read_f64(argv[1], N * DIM);
  Y = read_f64(argv[2], N * DIM);
  double *a = read_f64(argv[7], N), *b = read_f64(argv[8], N);
  /* exp(-t) == 0 exactly for t > ~745.13: decide outside [740, 750] by bound */
  LO = 740.0 * EPS * SCALE;
  HI = 750.0 * EPS * SCALE;
  masked = calloc(N, sizeof(uint32_t *));
  nmasked = calloc(N, sizeof(int64_t));
  int nt = 8;
  const char *e = getenv("NTHREADS");
  if (e) nt = atoi(e);
  pthread_t th[256];
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, worker, NULL);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  int64_t total_masked = 0;
  for (int64_t i = 0; i < N; ++i) total_masked += nmasked[i];
  fprintf(stderr, "phase 1 done: %lld masked pairs\n", (long long)total_masked);

  /* ot_probabilities (sparsify.cpp:76-82) */
  double *ra = malloc(sizeof(double) * N), *cb = malloc(sizeof(double) * N);
  double sa = 0.0, sb = 0.0;
  for (int64_t i = 0; i < N; ++i) sa += (ra[i] = sqrt(a[i]));
  for (int64_t j = 0; j < N; ++j) sb += (cb[j] = sqrt(b[j]));
  for (int64_t i = 0; i < N; ++i) ra[i] /= sa;
  for (int64_t j = 0; j < N; ++j) cb[j] /= sb;

  /* masked_grid_plan (sparsify.cpp:53-63): sequential row-major sum */
  double total = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const double r = ra[i];
    int64_t j = 0;
    for (int64_t k = 0; k <= nmasked[i]; ++k) {
      const int64_t stop = k < nmasked[i] ? (int64_t)masked[i][k] : N;
      for (; j < stop; ++j) total += r * cb[j];
      j = stop + 1;  /* masked entry: prow[j] = 0, total += 0.0 leaves total unchanged */
    }
    if ((i & 0xffff) == 0) fprintf(stderr, "row %lld total %.17g\n", (long long)i, total);
  }
  const double inv = 1.0 / total;
  const int64_t kernel_nnz = N * N - total_masked;
  printf("{\"n\": %lld, \"kernel_nnz\": %lld, \"masked_pairs\": %lld, \"total\": \"%a\", \"inv\": \"%a\", "
         "\"total_dec\": %.17g, \"inv_dec\": %.17g, \"sa\": \"%a\", \"sb\": \"%a\"}\n",
         (long long)N, (long long)kernel_nnz, (long long)total_masked, total, inv, total, inv, sa, sb);
  return 0;
}
