/* ORACLE — test infrastructure only (see oracle/__init__.py).
 *
 * Reference SpMV  y = alpha*A*x + beta*y  in long double (x87 80-bit on x86-64),
 * the plain definition of what every operator graph computes ("y=Ax"; P:237 and
 * formats are re-layouts of the same matrix; alpha/beta per north_star and
 * reading A1).  For each row i, entries in canonical order (col ascending):
 *
 *   s_i     = sum_j (long double)a_ij * (long double)x_j
 *   abs_i   = sum_j |(long double)a_ij * (long double)x_j|
 *   yref_i  = alpha*s_i + (beta != 0 ? beta*y0_i : 0)          (beta = 0: y0 not read)
 *   bound_i = |alpha|*abs_i + (beta != 0 ? |beta*y0_i| : 0)
 *
 * Acceptance (north_star): |y_i - yref_i| <= tol * bound_i.
 * Rows are independent, so the result does not depend on the number of threads.
 * Inputs are double (fp32 data is widened exactly by the caller).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  int64_t r0, r1;
  const int64_t *row_ptr, *col;
  const double *val, *x, *y0;
  double alpha, beta;
  long double *y, *bound;
} job_t;

static void *run(void *p) {
  job_t *j = (job_t *)p;
  for (int64_t i = j->r0; i < j->r1; ++i) {
    long double s = 0.0L, a = 0.0L;
    for (int64_t e = j->row_ptr[i]; e < j->row_ptr[i + 1]; ++e) {
      long double t = (long double)j->val[e] * (long double)j->x[j->col[e]];
      s += t;
      a += fabsl(t);
    }
    long double yi = (long double)j->alpha * s;
    long double bi = fabsl((long double)j->alpha) * a;
    if (j->beta != 0.0) {
      long double by = (long double)j->beta * (long double)j->y0[i];
      yi += by;
      bi += fabsl(by);
    }
    j->y[i] = yi;
    j->bound[i] = bi;
  }
  return NULL;
}

/* row_ptr[m+1], col[nnz], val[nnz], x[n], y0[m] (may be NULL if beta == 0);
 * outputs y[m], bound[m] in long double.  nthreads >= 1 splits rows into
 * nnz-balanced contiguous ranges.  Returns 0. */
int oracle_spmv_csr(int64_t m, const int64_t *row_ptr, const int64_t *col, const double *val,
                    const double *x, double alpha, double beta, const double *y0,
                    long double *y, long double *bound, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 1024) nthreads = 1024;
  job_t jobs[1024];
  pthread_t th[1024];
  int64_t nnz = row_ptr[m];
  int64_t r = 0;
  for (int t = 0; t < nthreads; ++t) {
    int64_t target = (nnz * (int64_t)(t + 1)) / nthreads;
    int64_t r1 = r;
    if (t == nthreads - 1) r1 = m;
    else while (r1 < m && row_ptr[r1] < target) ++r1;
    jobs[t] = (job_t){r, r1, row_ptr, col, val, x, y0, alpha, beta, y, bound};
    r = r1;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, run, &jobs[t]);
  run(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}
